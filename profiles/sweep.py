#!/usr/bin/env python
"""Config-5 kernel microbenchmark: hierarchical-KV flash-decode attention over
context 4K-256K for the draft view (T=1) and the verify view (T = gamma+1,
gamma 1..8), plus the flush-quantise kernel (K1) per flush, on a synthetic
Llama-2-7B-shaped store (32 KV heads, hd 128, G 128; one layer).

    python profiles/sweep.py [--contexts 4096,16384,32768,65536,131072,262144] [--gammas 1,2,4,8]

Times are CUDA-event medians of back-to-back launches (each launch preceded by
its own event pair, queued behind a GPU sleep), and "in-stream": 8 launches replayed
from one CUDA graph (PDL overlap between them, as in a decode forward); GB/s counts algorithmic bytes
(planes + (S, Z) params + fp tails + q/o).
"""

import argparse
import math
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, iters=11):
    import torch

    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    torch.cuda._sleep(int(1e8))
    for s, e in ev:
        s.record()
        fn()
        e.record()
    torch.cuda.synchronize()
    return statistics.median(s.elapsed_time(e) for s, e in ev) * 1e3  # us


def timed_stream(fn, n=8, reps=5):
    """Per-launch device time of n back-to-back launches replayed from one CUDA graph (PDL overlaps
    each launch's prologue with the previous one's tail, as inside a decode forward)."""
    import torch

    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            fn()
    g.replay()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        g.replay()
        e.record()
        torch.cuda.synchronize()
        out.append(s.elapsed_time(e) * 1e3 / n)
    return statistics.median(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--contexts", default="4096,16384,32768,65536,131072,262144")
    ap.add_argument("--gammas", default="1,2,4,8")
    a = ap.parse_args()
    import torch

    import __graft_entry__

    __graft_entry__.build()
    from paper_2502_10424_b200 import _lib
    from paper_2502_10424_b200.cache import CacheLayout, HierarchicalKVCache
    from paper_2502_10424_b200.runtime import Geometry, Runner

    import json

    try:
        peak = float(json.load(open(os.path.join(ROOT, 'MEASURED_PEAKS.json')))['hbm_gbs'])
    except Exception:
        peak = 6459.6
    G, H, hd = 128, 32, 128
    kv = H * hd
    gammas = [int(g) for g in a.gammas.split(",")]
    print(f"# attention (one layer, {H} KV heads x {hd}, G={G}); peak {peak} GB/s (measured copy)")
    for ctx in (int(c) for c in a.contexts.split(",")):
        lay = CacheLayout(1, H, hd, G)
        c = HierarchicalKVCache(lay, max_tokens=ctx + 2 * G)
        nb = ctx // G - 1
        for t in (c.ku, c.kl, c.vu, c.vl):
            t.random_(0, 256)
        c.kp[..., 0].uniform_(0.01, 0.1)
        c.kp[..., 1].uniform_(-1.0, 0.0)
        c.vp[..., 0].uniform_(0.01, 0.1)
        c.vp[..., 1].uniform_(-1.0, 0.0)
        c.fp_k.normal_()
        c.fp_v.normal_()
        c.d_n_blocks.fill_(nb)
        c.d_fp1_len.fill_(G)
        c.d_fp2_len.fill_(3)
        geo = Geometry(1, kv, H, H, hd, 16, 16, 1 << 20)
        s = _lib.stream_ptr()
        for view, T in [(_lib.VIEW_DRAFT, 1)] + [(_lib.VIEW_TARGET, g + 1) for g in gammas]:
            run = Runner(geo, c, max_cols=max(T, 5))
            run.q.normal_()
            per_tok = kv * (1.0 if view == _lib.VIEW_DRAFT else 2.0) + 8.0 * kv / G + 8.0 * math.ceil(kv / G)
            nbytes = nb * G * per_tok + (G + 3 + T) * kv * 4.0 + T * kv * 8.0
            us = timed(lambda: run._attention(0, view, T, 0, s))
            # in-stream replays the same layer: only meaningful when it does not fit the 126 MB L2 twice
            uss = timed_stream(lambda: run._attention(0, view, T, 0, _lib.stream_ptr())) if nbytes > 2.5e8 else float("nan")
            name = "draft " if view == _lib.VIEW_DRAFT else f"verify g={T - 1}"
            print(f"ctx={ctx:7d} {name:11s} T={T}  {us:8.1f} us  {nbytes / us / 1e3:7.0f} GB/s  "
                  f"{nbytes / us / 1e3 / peak:6.1%}   in-stream {uss:8.1f} us {nbytes / uss / 1e3 / peak:6.1%}", flush=True)
            del run
        del c
        torch.cuda.empty_cache()

    # ---- K1 flush-quantise: one flush of all 32 layers (fp1 -> one quantised block per layer) ----
    L = 32
    lay = CacheLayout(L, H, hd, G)
    c = HierarchicalKVCache(lay, max_tokens=(L + 8) * G)
    c.fp_k.normal_()
    c.fp_v.normal_()
    st = c.store_struct()
    rd = L * 2 * G * kv * 2.0
    wr = L * (G * kv * 2 * 1.0 + 16.0 * kv)
    # the K1 kernel alone on the same work (32 blocks x H heads, one launch)
    src_k = torch.randn(H, L * G, hd, device="cuda").half()
    src_v = torch.randn(H, L * G, hd, device="cuda").half()
    us_q = timed(lambda: _lib.call("qs_kv_quantize_blocks", st, 0, 0, src_k.data_ptr(), src_v.data_ptr(), L * G * hd, L,
                                   0, c.d_flags.data_ptr(), _lib.stream_ptr()))
    print(f"# K1 quantise kernel, {L} blocks x {H} heads: {us_q:.1f} us ({(rd + wr) / us_q / 1e3:.0f} GB/s)")

    def flush():  # the decode-time flush (device-conditioned: quantise + rotate + lengths), lengths re-armed
        c.d_fp1_len.fill_(G)
        c.d_fp2_len.fill_(G)
        c.d_n_blocks.zero_()
        c.launch_device_flush()

    us = timed(flush)
    print(f"# flush-quantise, {L} layers x {H} heads, one block each (incl. 3 length re-arm fills): {us:.1f} us "
          f"({(rd + wr) / us / 1e3:.0f} GB/s; reads {rd / 1e6:.1f} MB fp16, writes {wr / 1e6:.1f} MB planes+params)")


if __name__ == "__main__":
    main()
