#!/bin/bash
# ncu DRAM bytes of the draft-attention launch that bench.py times (the 4th attn_kernel launch of
# `bench.py --profile-kernels`), recorded with the md5 of the CUDA sources it measured (bench.lib_digest); bench.py
# reports roofline.traffic only when the md5 matches the sources it runs.   usage (under gpurun):
#   bash profiles/collect_traffic.sh [extra bench args]
set -e
mkdir -p gpurun_out
QS_BENCH_ISOLATED=1 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:attn_kernel -s 3 -c 1 --csv python bench.py --profile-kernels "$@" > gpurun_out/traffic_ncu.csv 2> gpurun_out/traffic_ncu.err
python - <<'PY'
import csv, hashlib, json, time
rows = list(csv.reader(open("gpurun_out/traffic_ncu.csv")))
hdr = next(r for r in rows if r and r[0] == "ID")
rows = [hdr] + [r for r in rows if len(r) == len(hdr) and r[0].isdigit()]
iN, iV = hdr.index("Metric Name"), hdr.index("Metric Value")
m = {r[iN]: float(r[iV].replace(",", "")) for r in rows[1:]}
unit = {r[iN]: r[hdr.index("Metric Unit")] for r in rows[1:]}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
b = sum(m[k] * scale[unit[k]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
import sys; sys.path.insert(0, "."); import bench; md5 = bench.lib_digest()
out = {"attn_draft_bytes_per_launch": b, "lib_md5": md5, "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
       "kernel_us": m.get("gpu__time_duration.sum", 0) * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(unit.get("gpu__time_duration.sum"), 1.0), "how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum, 4th attn_kernel launch of bench.py --profile-kernels"}
json.dump(out, open("profiles/traffic.json", "w"), indent=1)
json.dump(out, open("gpurun_out/traffic.json", "w"), indent=1)
print(out)
PY
