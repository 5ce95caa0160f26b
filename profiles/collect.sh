#!/bin/bash
# One GPU-box pass that refreshes the committed evidence for a round:
#   1. the default bench line            -> gpurun_out/${TAG}_bench.json (+ log)
#   2. ncu launch list of one steady-state speculative cycle (our kernels only,
#      cold-cache serialised times: compare SHARES)  -> gpurun_out/${TAG}_launches.csv
#   3. ncu --set full summaries of the hot kernels -> gpurun_out/${TAG}_summary.txt
# Usage (under gpurun): bash profiles/collect.sh r01
TAG=${1:-r01}
mkdir -p gpurun_out
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
    -k 'regex:attn_kernel|linear_|prep_act|embed_kernel|argmax|accept|add_int|kv_quant|fp_rotate' \
    -s 400 -c 1400 --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 3 --modes both > /tmp/${TAG}_ll.log 2>&1
python profiles/launch_shares.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launch_shares.txt 2>&1
bash profiles/profile_kernels.sh ${TAG} full attn_draft
# per-launch DRAM traffic of the roofline kernel (draft attention) for bench.py's roofline.traffic
python - "$TAG" <<'PY'
import json, re, sys
tag = sys.argv[1]
txt = open(f"gpurun_out/{tag}_summary.txt").read().split("# ")
unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
for blk in txt:
    if "attn_kernel<128, 1, 0" in blk:
        tot = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            m = re.search(k + r" = ([0-9.]+) (\w+)", blk)
            tot += float(m.group(1)) * unit[m.group(2)]
        json.dump({"attn_draft_bytes_per_launch": tot, "source": f"ncu --set full, {tag}_summary.txt"},
                  open(f"gpurun_out/{tag}_traffic.json", "w"))
        break
PY
