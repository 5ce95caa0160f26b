#!/usr/bin/env python
"""Attention kernel microbenchmark on a synthetic hierarchical store (no prefill).

    python profiles/attn_micro.py --context 131072 --splits 9,18 --dbg 0,1,2,3

dbg bits (diagnostics only): 1 = consumers skip the math, 2 = producer skips
the query-scale fold.  Prints one line per (view, splits, dbg) with the
device time (CUDA events, mean of --iters launches) and algorithmic GB/s.
"""

import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--context", type=int, default=131072)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--hd", type=int, default=128)
    ap.add_argument("--splits", default="0")
    ap.add_argument("--dbg", default="0")
    ap.add_argument("--T", default="1,5")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--r", type=int, default=1, help="query heads per KV head (GQA: 4)")
    ap.add_argument("--batch", type=int, default=1, help="sequences per launch")
    ap.add_argument("--graph", type=int, default=0, help="1: replay the launches from a CUDA graph")
    a = ap.parse_args()
    import torch

    import __graft_entry__

    __graft_entry__.build()
    from paper_2502_10424_b200 import _lib
    from paper_2502_10424_b200.cache import CacheLayout, HierarchicalKVCache
    from paper_2502_10424_b200.runtime import Geometry, Runner

    G, H, hd = 128, a.heads, a.hd
    lay = CacheLayout(1, H * a.r, hd, G, num_kv_heads=H)
    c = HierarchicalKVCache(lay, max_tokens=a.context + 2 * G, batch=a.batch)
    nb = a.context // G - 1
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
    kv = H * hd
    geo = Geometry(1, kv * a.r, H * a.r, H, hd, 16, 16, 1 << 20)
    s = _lib.stream_ptr()
    for T in [int(x) for x in a.T.split(",")]:
        view = _lib.VIEW_DRAFT if T == 1 else _lib.VIEW_TARGET
        per_tok = (kv * (1.0 if T == 1 else 2.0)) + 8.0 * kv / G + 8.0 * math.ceil(kv / G)
        nbytes = a.batch * (nb * G * per_tok + (G + 3 + T) * kv * 4.0)
        for sp in [int(x) for x in a.splits.split(",")]:
            run = Runner(geo, c, max_cols=max(T, 5) * a.batch, attn_splits=sp or None)
            run.q.normal_()
            for dbg in [int(x) for x in a.dbg.split(",")]:
                run._attention(0, view, T, 0, s)  # build args
                key = [k for k in run._lin_cache if k[0] == "attn" and k[3] == T][0]
                args, mode = run._lin_cache[key]
                args.dbg = dbg
                for _ in range(3):
                    _lib.check(_lib.load().qs_attn_decode(args, mode, s))
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                if a.graph:
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g):
                        for _ in range(a.iters):
                            _lib.check(_lib.load().qs_attn_decode(args, mode, _lib.stream_ptr()))
                    g.replay()
                    torch.cuda.synchronize()
                e0.record()
                if a.graph:
                    g.replay()
                else:
                    for _ in range(a.iters):
                        _lib.check(_lib.load().qs_attn_decode(args, mode, s))
                e1.record()
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) / a.iters * 1e3
                print(f"T={T} view={'draft' if view == 0 else 'target'} splits={args.n_main} dbg={dbg} "
                      f"{us:8.1f} us  {nbytes / us / 1e3:7.0f} GB/s", flush=True)
                args.dbg = 0


if __name__ == "__main__":
    main()
