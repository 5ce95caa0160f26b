#!/usr/bin/env python
"""Per-kernel share of device time from an ncu `--metrics gpu__time_duration.sum` launch list.

    python profiles/launch_shares.py launches.csv

ncu serialises launches and runs them cold-cache, so the absolute times are not
bench numbers; the SHARE of each kernel family is what should agree with the
bench's own breakdown.
"""
import collections
import csv
import re
import sys


def family(name: str) -> str:
    m = re.search(r"(attn_kernel|linear_i4_kernel|linear_f16p_kernel|prep_act_kernel|embed_kernel|argmax_kernel|accept_kernel|add_int_kernel|"
                  r"kv_quant_kernel|fp_rotate_kernel)(<[^>]*>)?", name)
    return (m.group(1) + (m.group(2) or "")) if m else name[:60]


def main(path: str) -> None:
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rd = csv.DictReader(lines)
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
        rows.append((family(r["Kernel Name"]), v * scale))
    tot = sum(t for _, t in rows)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for k, t in rows:
        agg[k][0] += 1
        agg[k][1] += t
    print(f"# {len(rows)} launches, {tot:.1f} us total (ncu-serialised, cold cache)")
    print(f"{'kernel':60s} {'launches':>8s} {'total_us':>10s} {'avg_us':>8s} {'share':>7s}")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:60s} {n:8d} {t:10.1f} {t / n:8.2f} {t / tot:7.1%}")


if __name__ == "__main__":
    main(sys.argv[1])
