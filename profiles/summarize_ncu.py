#!/usr/bin/env python
"""Summarise ncu reports into small text files (runs where the .ncu-rep is).

For each report: key raw metrics (time, DRAM bytes/throughput, issue, warps,
stall reasons, tensor pipe) and a per-opcode breakdown of executed SASS
instructions and stall samples from the source page.
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
STALLS = ["barrier", "long_scoreboard", "short_scoreboard", "mio_throttle", "wait", "math_pipe_throttle",
          "lg_throttle", "no_instruction", "not_selected", "selected", "dispatch_stall", "membar", "branch_resolving",
          "drain", "sleeping", "tex_throttle", "misc"]


def ncu(args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def summarize(rep):
    out = [f"# {rep}"]
    rows = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "raw", "--csv"]))))
    if len(rows) >= 3:
        h, u, v = rows[0], rows[1], rows[2]
        idx = {k: i for i, k in enumerate(h)}
        for k in KEYS:
            if k in idx:
                out.append(f"{k} = {v[idx[k]]} {u[idx[k]]}")
        for s in STALLS:
            k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if k in idx:
                out.append(f"stall_{s} = {v[idx[k]]}")
    src = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "source", "--csv", "--print-source=sass"]))))
    if len(src) > 2:
        h = src[1]
        try:
            ii = h.index("Instructions Executed")
            ss = h.index("Warp Stall Sampling (All Samples)")
        except ValueError:
            return "\n".join(out)
        ops, st = collections.Counter(), collections.Counter()
        tot = stot = 0
        for x in src[2:]:
            try:
                n, s_ = int(x[ii]), int(x[ss])
            except (ValueError, IndexError):
                continue
            o = x[1].split()
            if not o:
                continue
            op = o[1] if o[0].startswith("@") and len(o) > 1 else o[0]
            op = op.split(".")[0]
            ops[op] += n
            st[op] += s_
            tot += n
            stot += s_
        out.append(f"sass_total_inst = {tot}  stall_samples = {stot}")
        for op, n in ops.most_common(25):
            out.append(f"  {op:10s} inst {100.0 * n / max(1, tot):5.1f}%  stall {100.0 * st[op] / max(1, stot):5.1f}%")
    return "\n".join(out)


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print(summarize(rep))
        print()
