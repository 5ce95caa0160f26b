"""Micro-benchmark of the stream-K linear kernel (qs_linear) on synthetic weights.

    python profiles/gemv_micro.py [--shapes K,N ...] [--ncols 1] [--groups 32,128] [--nctas 0]

Prints device time, algorithmic bytes and GB/s per (mode, shape).  Weights
are several hundred MB in total, so each launch streams from HBM (> L2).
"""

import argparse
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2502_10424_b200 import _lib  # noqa: E402
from paper_2502_10424_b200.runtime import PackedLinear  # noqa: E402


def timeit(fn, iters=40):
    """Device time per launch of fn() replayed from a CUDA graph (no host launch overhead)."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(iters):
            fn()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / (5 * iters) * 1e3  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="4096,12288;4096,4096;4096,22016;11008,4096;4096,32000")
    ap.add_argument("--ncols", type=int, default=1)
    ap.add_argument("--groups", default="32,128")
    ap.add_argument("--modes", default="f16,int4")
    ap.add_argument("--copies", type=int, default=4, help="distinct weight copies rotated (defeats L2)")
    ap.add_argument("--dbg", type=int, default=0, help="diagnostic bits (1: consumers skip the MMA work)")
    a = ap.parse_args()
    peak = 6542.1
    for mode in a.modes.split(","):
        for grp in ([16] if mode == "f16" else [int(g) for g in a.groups.split(",")]):
            for shp in a.shapes.split(";"):
                K, N = (int(v) for v in shp.split(","))
                pls = []
                for c in range(a.copies):
                    w = torch.randn(K, N, device="cuda") / math.sqrt(K)
                    pls.append(PackedLinear.f16(w) if mode == "f16" else PackedLinear.int4(w, grp))
                    del w
                x = torch.randn(a.ncols, K, device="cuda")
                xh = torch.zeros(a.ncols, K + 64, dtype=torch.float16, device="cuda")
                xs = torch.zeros(a.ncols, K // 16 + 8, device="cuda")
                _lib.check(_lib.load().qs_prep_act(x.data_ptr(), None, 0.0, xh.data_ptr(), xh.shape[1], xs.data_ptr(),
                                                   xs.shape[1], a.ncols, K, _lib.stream_ptr()))
                y = torch.zeros(a.ncols, N, device="cuda")
                args = []
                for pl in pls:
                    ar = _lib.LinearArgs()
                    ar.wmode, ar.epi, ar.N, ar.K, ar.ncols = pl.wmode, _lib.EPI_STORE, N, K, a.ncols
                    ar.wgroup = pl.group if pl.wmode == _lib.W_INT4 else 16
                    ar.w = pl.w.data_ptr()
                    ar.wparams = pl.params.data_ptr() if pl.params is not None else None
                    ar.xh, ar.ldxh, ar.xs, ar.ldxs = xh.data_ptr(), xh.shape[1], xs.data_ptr(), xs.shape[1]
                    ar.y, ar.ldy = y.data_ptr(), N
                    ar.dbg = a.dbg
                    args.append(ar)
                lib = _lib.load()
                it = [0]

                def run():
                    _lib.check(lib.qs_linear(args[it[0] % len(args)], _lib.stream_ptr()))
                    it[0] += 1

                us = timeit(run)
                algo = pls[0].algorithmic_bytes() + 2.0 * K * a.ncols + 4.0 * N * a.ncols
                gbs = algo / us / 1e3
                print(f"{mode:5s} g={grp:4d} K={K:6d} N={N:6d} ncols={a.ncols:2d}  "
                      f"{us:8.2f} us  {algo / 1e6:8.2f} MB  {gbs:7.1f} GB/s  {gbs / peak:5.1%}", flush=True)
                del pls, args
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
