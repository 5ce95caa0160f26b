#!/usr/bin/env python
"""Benchmark of the QuantSpec decode hot path on B200 (BASELINE.json config 3).

Workload (default): Llama-2-7B-shaped random-init model (32 layers, 32 heads,
hd 128, d 4096, mlp 11008, vocab 32000), a 128K-token synthetic prompt,
batch 1, gamma = 4, greedy.  A "step" is one draft/verify cycle of
self-speculative decoding (INT4 hierarchical KV + INT4 draft weights, the
config-3 mode); the same kernels also run the kv_only mode (fp16 draft
weights) and the FP16 autoregressive baseline (fp16 weights + fp16 KV) for
the speed-up.  Prefill is setup, outside every timed region.

Prints ONE JSON line (rank 0).  ``--impl reference`` times the CPU oracle
(oracle/qs_oracle.py, the NumPy restatement of the reference) on a bounded
sample of the same workload instead.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

LLAMA2_7B = dict(num_layers=32, num_heads=32, num_kv_heads=32, head_dim=128, hidden=4096, mlp_hidden=11008, vocab=32000)
LLAMA31_8B = dict(num_layers=32, num_heads=32, num_kv_heads=8, head_dim=128, hidden=4096, mlp_hidden=14336, vocab=128256)
METRIC = "decode tokens/sec @128K ctx + speedup vs FP16 AR; attn HBM GB/s vs peak"
# BASELINE.json configs; config 3 is the headline (the default), the others are extra profile lines
WORKLOADS = {
    "config3": dict(model=LLAMA2_7B, shape="llama2_7b", context=131072, batch=1,
                    name="config3: LWM-Text-Chat-128k shape (Llama-2-7B arch) random init, 128K ctx, batch 1 per GPU, "
                         "gamma 4, greedy, mode=both (INT4 KV + INT4 draft weights)"),
    "config2": dict(model=LLAMA2_7B, shape="llama2_7b", context=32768, batch=1,
                    name="config2: Llama-2-7B shape random init, 32K ctx, batch 1 per GPU, gamma 4, greedy, mode=both"),
    "config5": dict(model=LLAMA2_7B, shape="llama2_7b", context=131072, batch=1, shard_heads=True,
                    name="config5: Llama-2-7B shape random init, ONE 128K sequence with its KV heads sharded over the "
                         "GPUs (fused all-gather of the attention rows), gamma 4, greedy, mode=both"),
    "config4": dict(model=LLAMA31_8B, shape="llama31_8b", context=131072, batch=8,
                    name="config4: Llama-3.1-8B shape (GQA, 8 KV heads) random init, 128K ctx, batch 8 partitioned "
                         "batch-wise over the GPUs, gamma 4, greedy, mode=both"),
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=48)
    p.add_argument("--warmup", type=int, default=4)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--workload", default="config3", choices=sorted(WORKLOADS))
    p.add_argument("--context", type=int, default=0, help="override the workload's context")
    p.add_argument("--batch", type=int, default=0, help="override the workload's total batch (all ranks)")
    p.add_argument("--weights", default="reference", choices=["reference", "device"],
                   help="reference: the reference init_weights stream replayed bit-exactly (initstream); "
                        "device: torch.randn on the GPU (same recipe, not the reference's draws)")
    p.add_argument("--gamma", type=int, default=4)
    p.add_argument("--layers", type=int, default=32)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--no-graphs", action="store_true")
    p.add_argument("--modes", default="both,kv_only,fp16_ar")
    p.add_argument("--profile-kernels", action="store_true", help="only run the isolated kernel timings (for ncu)")
    return p.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sms, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sms.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sms)}


# ---------------------------------------------------------------------------
# model + caches (setup, untimed)
# ---------------------------------------------------------------------------


def resolve(args):
    """Workload dict with the command-line overrides applied (context, total batch, depth)."""
    wl = dict(WORKLOADS[args.workload])
    wl["model"] = dict(wl["model"], num_layers=args.layers)
    if args.context:
        wl["context"] = args.context
    if args.batch:
        wl["batch"] = args.batch
    return wl


def weight_source(args, wl, geo):
    """Yields ("layers.i.<mat>" | "embedding" | "lm_head", f32 CUDA tensor) in the reference's
    init_weights draw order (Q/model.py:89-117).  ``reference``: the numpy PCG64 stream replayed
    bit-exactly on host threads from recorded per-matrix states (paper_2502_10424_b200/initstream);
    ``device``: the same recipe (N(0,1)/sqrt(fan_in), unscaled embedding) drawn by torch on the GPU."""
    import torch

    from paper_2502_10424_b200 import initstream

    m = wl["model"]
    plan = initstream.draw_plan(m["num_layers"], m["hidden"], m["num_kv_heads"] * m["head_dim"], m["mlp_hidden"],
                                m["vocab"])
    if args.weights == "reference":
        full = initstream.draw_plan(32, m["hidden"], m["num_kv_heads"] * m["head_dim"], m["mlp_hidden"], m["vocab"])
        states = initstream.load_states(32, m["hidden"], m["num_kv_heads"] * m["head_dim"], m["mlp_hidden"],
                                        m["vocab"], args.seed)
        if states is None:
            raise SystemExit(f"no recorded init stream for {wl['shape']} seed {args.seed}: "
                             f"run tools/make_init_states.py {wl['shape']} {args.seed} (or --weights device)")
        # a shallower bench (--layers) keeps the first layers' draws and the embedding / lm_head of the full model
        idx = {name: i for i, (name, *_) in enumerate(full)}
        sel = [full[idx[name]] for name, *_ in plan]
        st = [states[idx[name]] for name, *_ in plan]
        for name, arr in initstream.stream_matrices(sel, st):
            yield name, torch.from_numpy(arr).cuda(non_blocking=False)
    else:
        gen = torch.Generator(device="cuda").manual_seed(args.seed)
        for name, rows, cols, scaled in plan:
            t = torch.randn(rows, cols, device="cuda", generator=gen)
            yield name, (t / math.sqrt(rows) if scaled else t)


def build_weights(args, wl, geo, head_shard=None):
    """Packed fp16 (target) and INT4 g32 (draft) DeviceWeights + f32 embedding / lm_head, streamed one
    layer at a time so only packed copies stay resident.  Returns (fw, qw, emb, head)."""
    import torch

    from paper_2502_10424_b200 import _lib
    from paper_2502_10424_b200.runtime import DeviceWeights, PackedLinear, rope_table

    f_layers, q_layers = [], []
    cur = {}
    emb = head = None
    for name, t in weight_source(args, wl, geo):
        if name == "embedding":
            emb = t
            continue
        if name == "lm_head":
            head = t
            continue
        cur[name.split(".")[-1]] = t
        if len(cur) == 7:
            wq, wk, wv = cur["wq"], cur["wk"], cur["wv"]
            if head_shard is not None:  # this rank's query / KV head columns (KV-head sharding)
                r, n = head_shard
                qn, kn = geo.nq // n, geo.nk // n
                wq, wk, wv = wq[:, r * qn:(r + 1) * qn], wk[:, r * kn:(r + 1) * kn], wv[:, r * kn:(r + 1) * kn]
            qkv = torch.cat([wq, wk, wv], dim=1)
            f_layers.append(dict(qkv=PackedLinear.f16(qkv), o=PackedLinear.f16(cur["wo"]),
                                 gu=PackedLinear.f16_pair(cur["w_gate"], cur["w_up"]),
                                 down=PackedLinear.f16(cur["w_down"])))
            q_layers.append(dict(qkv=PackedLinear.int4(qkv, 32), o=PackedLinear.int4(cur["wo"], 32),
                                 gu=PackedLinear.int4_pair(cur["w_gate"], cur["w_up"], 32),
                                 down=PackedLinear.int4(cur["w_down"], 32)))
            del qkv
            cur = {}
    ones = torch.ones(geo.hidden, device="cuda")
    rope = rope_table(geo.head_dim, geo.rope_base, geo.max_positions)
    common = dict(embedding=emb, attn_norms=[ones] * geo.num_layers, mlp_norms=[ones] * geo.num_layers,
                  final_norm=ones, rope=rope)
    fw = DeviceWeights(geo, f_layers, PackedLinear.f16(head), wmode=_lib.W_F16, **common)
    qw = DeviceWeights(geo, q_layers, PackedLinear.int4(head, 32), wmode=_lib.W_INT4, **common)
    torch.cuda.synchronize()
    return fw, qw, emb, head


def prompts_for(args, wl, seqs):
    """Uniform random prompt tokens; sequence b of the job uses seed + 1 + b (b = 0: the reference
    CLI's seed + 1, Q/cli.py:137), so a sequence's prompt does not depend on the GPU count."""
    import numpy as np

    V = wl["model"]["vocab"]
    return [np.random.default_rng(args.seed + 1 + b).integers(0, V, size=wl["context"]).astype(np.int32) for b in seqs]


def prefill_into(args, wl, geo, fw, head, prompts, sinks):
    """Prompt prefill (setup, untimed) with torch/cuBLAS/SDPA, layer-outer over all of this rank's
    prompts; ``sinks[b](layer, k, v)`` receive sequence b's K/V.  The f32 weight matrices are
    re-streamed for the pass (they are not kept)."""
    import torch
    from torch.nn.attention import SDPBackend, sdpa_kernel

    from paper_2502_10424_b200._prefill import run_prefill_batch

    def layers():
        cur = {}
        for name, t in weight_source(args, wl, geo):
            if not name.startswith("layers."):
                continue
            cur[name.split(".")[-1]] = t
            if len(cur) == 7:
                cur["attn_norm"] = cur["mlp_norm"] = fw.final_norm
                yield cur
                cur = {}

    # prompts per pass: the f32 residual streams of a group must fit next to the caches
    S = max(int(p.size) for p in prompts)
    free, _ = torch.cuda.mem_get_info()
    per_seq = S * geo.hidden * 4 * 2 + S * (geo.nq + 2 * geo.nk) * 2 * 3
    group = max(1, min(len(prompts), int(0.6 * free) // per_seq))
    firsts = []
    for g0 in range(0, len(prompts), group):
        ids = [torch.from_numpy(p).cuda() for p in prompts[g0:g0 + group]]
        with sdpa_kernel([SDPBackend.FLASH_ATTENTION, SDPBackend.EFFICIENT_ATTENTION, SDPBackend.CUDNN_ATTENTION]):
            logits = run_prefill_batch(geo, ids, fw.embedding, layers(), fw.final_norm, head, fw.rope,
                                       sinks[g0:g0 + group], dtype=torch.float16)
        torch.cuda.synchronize()
        firsts += [int(torch.argmax(lg).item()) for lg in logits]
        del ids, logits
    return firsts


def build_workload(args, wl, seqs):
    """Weights, the hierarchical store of this rank's sequences (prefilled), the fp16 baseline cache
    when both fit (else None: built later by ``fp16_cache``) and the first decode tokens."""
    import torch

    from paper_2502_10424_b200.cache import CacheLayout, FpKVCache, HierarchicalKVCache
    from paper_2502_10424_b200.runtime import Geometry

    m = wl["model"]
    S = wl["context"]
    margin = 4096
    geo = Geometry(m["num_layers"], m["hidden"], m["num_heads"], m["num_kv_heads"], m["head_dim"], m["mlp_hidden"],
                   m["vocab"], S + margin)
    t0 = time.time()
    shard = wl.get("shard")  # (rank, world) of a KV-head-sharded single sequence
    fw, qw, emb, head = build_weights(args, wl, geo, head_shard=shard)
    t_w = time.time() - t0
    B = len(seqs)
    nh, nkv = geo.num_heads, geo.num_kv_heads
    if shard is not None:
        nh, nkv = nh // shard[1], nkv // shard[1]
    lay = CacheLayout(geo.num_layers, nh, geo.head_dim, 128, num_kv_heads=nkv)
    hcache = HierarchicalKVCache(lay, max_tokens=S + margin, batch=B)
    # fp16 baseline cache alongside when it fits (config 3: 64 GiB + 34 GiB store), else after the spec modes
    kvd = nkv * geo.head_dim
    fp_bytes = 2 * 2 * B * geo.num_layers * kvd * (S + margin)
    free, _ = torch.cuda.mem_get_info()
    fcache = None
    if fp_bytes < free - (24 << 30):
        fcache = FpKVCache(geo.num_layers, kvd, capacity=S + margin, head_dim=geo.head_dim, batch=B)
    prompts = prompts_for(args, wl, seqs)
    loc = slice(shard[0] * kvd, (shard[0] + 1) * kvd) if shard is not None else slice(None)

    def sink(b):
        def f(l, k, v):
            k, v = k[:, loc], v[:, loc]
            hcache.load_prefill_layer(l, k, v, seq=b)
            if fcache is not None:
                fcache.load_prefill_layer(l, k, v, seq=b)
        return f

    firsts = prefill_into(args, wl, geo, fw, head, prompts, [sink(b) for b in range(B)])
    for b in range(B):
        hcache.finish_prefill(S, seq=b)
        if fcache is not None:
            fcache.finish_prefill(S, seq=b)
    setup = {"weights_s": t_w, "prefill_s": time.time() - t0 - t_w, "weights": args.weights}
    return geo, fw, qw, head, hcache, fcache, firsts, prompts, setup


def fp16_cache(args, wl, geo, fw, head, prompts):
    """The FP16-AR baseline cache of this rank's sequences, prefilled in its own pass (config 4:
    the quantised store and the fp16 cache of 8 x 128K sequences do not fit one GPU together)."""
    import torch

    from paper_2502_10424_b200.cache import FpKVCache

    S = wl["context"]
    B = len(prompts)
    fcache = FpKVCache(geo.num_layers, geo.nk, capacity=S + 4096, head_dim=geo.head_dim, batch=B)
    firsts = prefill_into(args, wl, geo, fw, head, prompts,
                          [lambda l, k, v, b=b: fcache.load_prefill_layer(l, k, v, seq=b) for b in range(B)])
    for b in range(B):
        fcache.finish_prefill(S, seq=b)
    torch.cuda.synchronize()
    return fcache, firsts


def time_kernel(fn, iters: int = 21):
    """Median device time of fn() (CUDA events around each launch on the launching stream;
    the event between launches also keeps consecutive launches from overlapping via PDL)."""
    import statistics

    import torch

    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    # hold the GPU while the host enqueues every launch, so no event pair brackets host launch latency
    torch.cuda._sleep(int(2e8))
    for s, e in ev:
        s.record()
        fn()
        e.record()
    torch.cuda.synchronize()
    return statistics.median(s.elapsed_time(e) for s, e in ev) / 1e3


# QS_BENCH_ISOLATED=1: isolated launches only (the ncu captures of profiles/profile_kernels.sh count
# launches; graph replays would shift their -s offsets)
ISO_ONLY = bool(os.environ.get("QS_BENCH_ISOLATED"))


def time_graph(fns, reps: int = 5):
    """Mean device time per call of the launches ``fns`` captured back to back in one CUDA graph
    (the decode loop's own launch mode, PDL included): the steady-state duration of a kernel inside
    a forward, where its prologue overlaps the previous launch."""
    import torch

    for f in fns:
        f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for f in fns:
            f()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / 1e3 / (reps * len(fns))


def kernel_roofline(geo, fw, qw, hcache, peak, shard=None):
    """Per-launch timings of the hot kernels at the bench context over this rank's sequences.
    Attention: isolated launches (each streams 0.1-9 GB >> the 126 MB L2).  Linear layers: the 32
    layers' matrices launched back to back from a graph (distinct weights, > L2), i.e. the in-forward
    steady state; the isolated single-launch time is reported next to it."""
    import torch

    from paper_2502_10424_b200 import _lib
    from paper_2502_10424_b200.runtime import Runner

    out = {}
    B = hcache.batch
    G = hcache.layout.group_size
    kv = hcache.layout.kv_dim  # this rank's KV heads (all of them unless KV-head sharded)
    nq_tok = hcache.quantized_token_count
    nfp = hcache.fp1_len + hcache.fp2_len + 1
    run = Runner(geo, hcache, max_cols=5 * B, shard=(shard[0], shard[1], None) if shard else None)
    run._rope = fw.rope  # the QKV epilogue's RoPE table (set by forward() in the decode loop)
    run.q.normal_()
    s = _lib.stream_ptr()
    per_tok = {"draft": kv * 1.0 + 8.0 * kv / G + 8.0 * math.ceil(kv / G),
               "target": kv * 2.0 + 8.0 * kv / G + 8.0 * math.ceil(kv / G)}
    L = geo.num_layers
    for name, view, T in (("attn_draft", _lib.VIEW_DRAFT, 1), ("attn_verify", _lib.VIEW_TARGET, 5)):
        dt_iso = time_kernel(lambda: run._attention(0, view, T, 0, s))
        # in-forward steady state: the L layers' launches back to back from one graph (PDL lets each
        # launch's barrier setup and first plane copies overlap its predecessor, as in the decode loop)
        dt = dt_iso if ISO_ONLY else time_graph(
            [(lambda li=li: run._attention(li, view, T, 0, _lib.stream_ptr())) for li in range(L)])
        algo = B * (nq_tok * per_tok["draft" if view == _lib.VIEW_DRAFT else "target"] + (nfp + T) * kv * 4.0
                    + T * run.lgeo.nq * 8.0)
        out[name] = {"us": dt * 1e6, "us_isolated": dt_iso * 1e6, "bytes": algo, "gbs": algo / dt / 1e9,
                     "frac": algo / dt / 1e9 / peak, "frac_isolated": algo / dt_iso / 1e9 / peak, "sequences": B,
                     "timing": f"graph of {L} launches (layers' own stores)"}
    L = len(fw.layers)
    for name, ws in (("gemv_f16_down", [lw["down"] for lw in fw.layers]),
                     ("gemv_int4_down", [lw["down"] for lw in qw.layers]),
                     ("gemv_int4_qkv", [lw["qkv"] for lw in qw.layers]),
                     ("gemv_int4_gate_up", [lw["gu"] for lw in qw.layers]),
                     ("gemv_int4_o", [lw["o"] for lw in qw.layers]),
                     ("gemv_draft_lm_head", [qw.lm_head]),
                     ("gemv_f16_lm_head", [fw.lm_head])):  # lm_head: one matrix, isolated
        w = ws[0]
        src = (run.hh, run.hs) if w.K == geo.mlp_hidden else (run.xh, run.xs)
        src[0].normal_()
        src[1].normal_()
        y = run.x if w.N == geo.hidden else (run.logits if w.N == geo.vocab else None)
        epi = _lib.EPI_STORE if y is not None else _lib.EPI_SILU_MUL if "gate" in name else _lib.EPI_QKV
        kw = dict(yh=(run.hh, run.hs)) if epi == _lib.EPI_SILU_MUL else {}
        if epi == _lib.EPI_SILU_MUL:
            src = (run.xh, run.xs)
        # the stream is resolved per call: inside graph capture it is the capture stream
        fns = [(lambda w_=w_, li=li: run._linear(w_, src, y, 1, epi, layer=li, stream=_lib.stream_ptr(), **kw))
               for li, w_ in enumerate(ws)]
        dt_iso = time_kernel(fns[0])
        dt = time_graph(fns) if len(fns) > 1 and not ISO_ONLY else dt_iso
        algo = w.algorithmic_bytes() + 2.0 * w.K + 4.0 * w.N
        out[name] = {"us": dt * 1e6, "us_isolated": dt_iso * 1e6, "bytes": algo, "gbs": algo / dt / 1e9,
                     "frac": algo / dt / 1e9 / peak, "frac_isolated": algo / dt_iso / 1e9 / peak,
                     "timing": f"graph of {len(fns)} launches (layers' own matrices)" if len(fns) > 1 else "isolated"}
    if not shard and not ISO_ONLY:
        # one whole draft forward (INT4 weights, T = 1 per sequence) replayed from a graph, against the
        # sum of its kernels' in-forward times: what the kernel boundaries cost inside a forward
        fwd = time_graph([lambda: run.forward(qw, 1, _lib.VIEW_DRAFT)])
        ksum = L * sum(out[k]["us"] for k in ("attn_draft", "gemv_int4_qkv", "gemv_int4_o", "gemv_int4_gate_up",
                                              "gemv_int4_down")) + out["gemv_draft_lm_head"]["us"]
        launches = 1 + 5 * L + 1  # embed, per layer QKV / attention / O / gate-up / down, lm_head
        out["forward_draft"] = {"us": fwd * 1e6, "kernels_in_forward_us": ksum, "launches": launches,
                                "boundary_us_per_launch": (fwd * 1e6 - ksum) / launches,
                                "timing": "graph of one draft forward vs the sum of the kernels' in-forward times"}
        # the other forwards of the cycles, whole (the cycle time minus gamma draft forwards and one verify
        # forward is what accept / flush / argmax / the per-cycle host round trip cost)
        out["forward_draft_f16"] = {"us": time_graph([lambda: run.forward(fw, 1, _lib.VIEW_DRAFT)]) * 1e6,
                                    "timing": "graph of one kv_only draft forward (fp16 weights, T = 1)"}
        out["forward_verify"] = {"us": time_graph([lambda: run.forward(fw, 5, _lib.VIEW_TARGET)]) * 1e6,
                                 "timing": "graph of one verify forward (fp16 weights, T = 5 per sequence)"}
        # the cycle's five forwards back to back in one graph, without argmax / accept / flush / copies
        five = [(lambda i=i: run.forward(qw, 1, _lib.VIEW_DRAFT, row_offset=i, tok_col=i)) for i in range(4)]
        five.append(lambda: run.forward(fw, 5, _lib.VIEW_TARGET))
        out["forwards_of_a_cycle"] = {"us": time_graph(five) * 5 * 1e6,
                                      "timing": "graph of 4 INT4 draft forwards + 1 verify forward (no argmax/accept/copies)"}
    torch.cuda.synchronize()
    return out


def kernel_fp16(geo, fcache, peak):
    import torch

    from paper_2502_10424_b200 import _lib
    from paper_2502_10424_b200.runtime import Runner

    B = fcache.batch
    frun = Runner(geo, fcache, max_cols=B)
    frun.q.normal_()
    s = _lib.stream_ptr()
    n = fcache.seq_len + 1
    dt = time_kernel(lambda: frun._attention(0, _lib.VIEW_FP16, 1, 0, s))
    algo = B * (n * geo.nk * 4.0 + geo.nq * 8.0)
    torch.cuda.synchronize()
    return {"us": dt * 1e6, "bytes": algo, "gbs": algo / dt / 1e9, "frac": algo / dt / 1e9 / peak, "sequences": B}


def _binom_ci(acc: int, n: int) -> list:
    """95% Wilson interval of an acceptance rate."""
    if n == 0:
        return [None, None]
    z, p = 1.96, acc / n
    den = 1 + z * z / n
    c = (p + z * z / (2 * n)) / den
    h = z * math.sqrt(p * (1 - p) / n + z * z / (4 * n * n)) / den
    return [c - h, c + h]


def measure_spec(geo, fw, dw, cache, first, gamma, steps, warmup, use_graphs, *, weight_mode, int4_bytes=0.0,
                 long_drafted=1000, runner=None):
    """Device time (CUDA events) and wall time of the SAME ``steps`` cycles of the public decode loop
    (SpeculativeDecoder.decode over a SpecEngine): per cycle the loop uploads the gamma_steps
    (pinned H2D), replays the captured cycle, and reads back (v, next, drafts, status); so the
    event-timed value and the wall-clock e2e cover identical work."""
    import torch

    from paper_2502_10424_b200.engine import SpecEngine
    from paper_2502_10424_b200.model import ModelConfig
    from paper_2502_10424_b200.specdec import SpecConfig, SpeculativeDecoder

    cfg = ModelConfig(geo.num_layers, geo.num_heads, geo.head_dim, geo.hidden, geo.mlp_hidden, geo.vocab,
                      geo.max_positions, num_kv_heads=geo.num_kv_heads)
    dec = SpeculativeDecoder.for_device(cfg, SpecConfig(gamma=gamma, decode_len=1 << 30, weight_mode=weight_mode),
                                        fw, dw, int4_weight_bytes=int4_bytes, use_graphs=use_graphs)
    eng = SpecEngine(fw, dw, cache, gamma, use_graphs=use_graphs, runner=runner)
    B = cache.batch
    pending = list(first) if isinstance(first, (list, tuple)) else [first] * B
    res = dec.decode(eng, pending, max_cycles=warmup, costs=False)
    pending = [r.tokens[-1] for r in res]
    torch.cuda.synchronize()
    l0 = eng.launches
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    s.record()
    res = dec.decode(eng, pending, max_cycles=steps, costs=False)
    e.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    dt = s.elapsed_time(e) / 1e3
    launches = eng.launches - l0
    emitted = sum(len(r.tokens) - 1 for r in res)
    drafted = sum(r.metrics.drafted_tokens for r in res)
    accepted = sum(r.metrics.accepted_tokens for r in res)
    out = {"tok_s": emitted / dt, "ms_per_step": dt * 1e3 / steps, "acceptance": accepted / max(1, drafted),
           "drafted": drafted, "tokens_per_cycle": emitted / steps / B, "e2e_tok_s": emitted / wall,
           "launches": launches, "h2d_bytes_per_step": eng.h2d_bytes, "d2h_bytes_per_step": eng.d2h_bytes,
           "context_after": int(cache.seq_lens().max()), "batch": B}
    # acceptance over >= long_drafted drafted tokens (untimed continuation of the same trajectory)
    if long_drafted:
        pending = [r.tokens[-1] for r in res]
        d_all, a_all, cyc = drafted, accepted, 0
        while d_all < long_drafted and cyc < 4000:
            r2 = dec.decode(eng, pending, max_cycles=16, costs=False)
            pending = [r.tokens[-1] for r in r2]
            d_all += sum(r.metrics.drafted_tokens for r in r2)
            a_all += sum(r.metrics.accepted_tokens for r in r2)
            cyc += 16
        out["acceptance_long"] = {"rate": a_all / max(1, d_all), "drafted": d_all, "ci95": _binom_ci(a_all, d_all)}
        # the same cycle time at the long-run acceptance: every cycle emits its accepted drafts + one
        # target token per sequence, so tokens per cycle per sequence = 1 + accepted / (cycles * B)
        tpc = 1.0 + a_all / max(1, (steps + cyc) * B)
        out["tokens_per_cycle_long"] = tpc
        out["tok_s_at_long_acceptance"] = B * tpc / (dt / steps)
    # device span of the cycle graph alone (events right around the replay, untimed continuation):
    # ms_per_step minus this is the GPU's idle time per cycle while the host turns the cycle around
    spans = []
    for _ in range(8):
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record()
        eng.cycle(sync=False)
        eb.record()
        eng.finish()
        spans.append(ea.elapsed_time(eb))
    out["cycle_graph_ms"] = sorted(spans)[len(spans) // 2]
    return out


def measure_ar(fw, cache, first, steps, warmup, use_graphs, runner=None):
    import torch

    from paper_2502_10424_b200.engine import ARAutoEngine

    eng = ARAutoEngine(fw, cache, use_graphs=use_graphs, runner=runner)
    B = cache.batch
    eng.set_pending(list(first) if isinstance(first, (list, tuple)) else [first] * B)
    for _ in range(warmup):
        eng.step(sync=False)
    torch.cuda.synchronize()
    l0 = eng.launches
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    s.record()
    for _ in range(steps):
        eng.step(sync=True)  # the public step: one token per sequence read back every step
    e.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    dt = s.elapsed_time(e) / 1e3
    return {"tok_s": B * steps / dt, "ms_per_step": dt * 1e3 / steps, "e2e_tok_s": B * steps / wall,
            "launches": eng.launches - l0, "batch": B}


# ---------------------------------------------------------------------------
# CPU baseline: the oracle (NumPy restatement of the reference) on a bounded sample
# ---------------------------------------------------------------------------


def cpu_sample(geo: dict, context: int, nlayers: int, seg_tokens: int = 16384):
    """Wall time of ``nlayers`` full decoder layers of ONE target-view decode token of the
    reference algorithm (the oracle port, oracle/qs_oracle.py) at ``context`` tokens:
    merged_attention (the reference's running f64 merge, Q/model.py:176-195) over the dequantised
    f32 target view, fed as ``seg_tokens``-token segments (GQA: each KV head repeated r times, as
    the oracle restates it), plus the layer's f32 projections.  Returns (seconds, lm_head seconds)."""
    import numpy as np

    from oracle import qs_oracle as O

    H, Hk, hd, d, m, V, G = (geo["num_heads"], geo["num_kv_heads"], geo["head_dim"], geo["hidden"], geo["mlp_hidden"],
                             geo["vocab"], 128)
    kv = Hk * hd
    rng = np.random.default_rng(0)
    blk = O.quantize_kv_block(O.Layout(1, Hk, hd, G), rng.standard_normal((G, kv)).astype(np.float32),
                              rng.standard_normal((G, kv)).astype(np.float32))
    kb, vb = O.dequant_kv_block(O.Layout(1, Hk, hd, G), blk, "target")
    seg_tokens = min(seg_tokens, context)
    ks = np.tile(kb, (seg_tokens // G, 1)).reshape(-1, Hk, hd)
    vs = np.tile(vb, (seg_tokens // G, 1)).reshape(-1, Hk, hd)
    if Hk != H:
        ks, vs = np.repeat(ks, H // Hk, axis=1), np.repeat(vs, H // Hk, axis=1)
    segs = [(ks, vs)] * max(1, context // seg_tokens)  # the context as segments (bounded memory)
    q = rng.standard_normal((H, hd)).astype(np.float32)
    mats = [rng.standard_normal((d, H * hd + 2 * kv), dtype=np.float32), rng.standard_normal((d, d), dtype=np.float32),
            rng.standard_normal((d, 2 * m), dtype=np.float32), rng.standard_normal((m, d), dtype=np.float32)]
    head = rng.standard_normal((d, V), dtype=np.float32)
    x = rng.standard_normal(d).astype(np.float32)
    xm = rng.standard_normal(m).astype(np.float32)
    t0 = time.perf_counter()
    for _ in range(nlayers):
        O.merged_attention(q, segs, 1.0 / np.sqrt(hd))
        _ = x @ mats[0]
        _ = x @ mats[1]
        _ = x @ mats[2]
        _ = xm @ mats[3]
    t_layers = time.perf_counter() - t0
    t0 = time.perf_counter()
    _ = x @ head
    return t_layers, time.perf_counter() - t0


def cpu_baseline(context: int, layers: int, geo: dict, sample_layers: int = 2):
    """The reference algorithm's target-view decode rate on this host: ``sample_layers`` of the
    ``layers`` decoder layers timed at the full context, extrapolated to one whole token."""
    cores = os.cpu_count() or 1
    t_l, t_h = cpu_sample(geo, context, sample_layers)
    per_tok = t_l * layers / sample_layers + t_h
    return {"value": 1.0 / per_tok, "unit": "tokens/s", "cores": cores, "kind": "port",
            "sample": (f"oracle (NumPy restatement of the reference) target-view decode of one token at {context} "
                       f"tokens: {sample_layers} of {layers} decoder layers timed ({t_l:.1f} s) and scaled "
                       f"x{layers / sample_layers:g}, + lm_head; extrapolated per-token time {per_tok:.1f} s"),
            "per_token_s": per_tok, "extrapolated": True}


def reference_arm(args):
    """--impl reference: the reference's CPU algorithm (the oracle port; the pure-Python reference
    package does not travel to the GPU box) on this box's host cores, on the b200 arm's config.
    Each step times ONE full decoder layer of one decode token at the full context (a bounded
    sample: ms_per_step is that measured time, so ms_per_step x steps is the run's wall time);
    value = the per-token rate those layer times extrapolate to (x layers, + lm_head)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    wl = resolve(args)
    t0 = time.time()
    for _ in range(min(args.warmup, 1)):
        cpu_sample(wl["model"], wl["context"], 1)
    per_layer, heads = [], []
    for _ in range(args.steps):
        t_l, t_h = cpu_sample(wl["model"], wl["context"], 1)
        per_layer.append(t_l)
        heads.append(t_h)
    t_layer = statistics.median(per_layer)
    per_tok = t_layer * args.layers + statistics.median(heads)
    v = 1.0 / per_tok
    cores = os.cpu_count() or 1
    cb = {"value": v, "unit": "tokens/s", "cores": cores, "kind": "port",
          "sample": (f"per step: one decoder layer of one target-view decode token at {wl['context']} tokens "
                     f"(median {t_layer:.2f} s over {args.steps} steps), extrapolated x{args.layers} layers + lm_head "
                     f"= {per_tok:.1f} s per token"),
          "extrapolated": True}
    line = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": min(args.warmup, 1), "ms_per_step": 1e3 * statistics.mean(per_layer), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64 attention / f32 projections", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": wl["name"], "context": wl["context"], "layers": args.layers, "gamma": args.gamma,
                       "batch_total": wl["batch"]},
            "cpu_baseline": cb, "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": time.time() - t0}
    print(json.dumps(line))


# ---------------------------------------------------------------------------


def lib_digest() -> str:
    """md5 over the CUDA sources and build flags of libqsb200.so (stable across rebuilds of the same
    sources, unlike the .so's own bytes), so a traffic capture is tied to the code it measured."""
    import glob
    import hashlib

    h = hashlib.md5()
    pkg = os.path.join(ROOT, "paper_2502_10424_b200")
    for p in sorted(glob.glob(os.path.join(pkg, "csrc", "*"))) + [os.path.join(pkg, "_build.py")]:
        with open(p, "rb") as f:
            h.update(os.path.basename(p).encode() + b"\0" + f.read())
    return h.hexdigest()


def measured_traffic():
    """ncu DRAM bytes (read + write) per draft-attention launch, recorded by profiles/collect_traffic.sh
    for a specific build of libqsb200.so; null when it was measured on a different build."""
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        t = json.load(open(tpath))
    except Exception:
        return None, "no ncu capture (profiles/traffic.json)"
    if t.get("lib_md5") != lib_digest():
        return None, f"ncu capture is of build {t.get('lib_md5')}, not this build"
    return t.get("attn_draft_bytes_per_launch"), f"ncu DRAM-bytes capture of these CUDA sources ({t.get('when', '')})"


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
        return
    import torch
    import torch.distributed as dist

    from paper_2502_10424_b200.parallel import partition

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import __graft_entry__

    __graft_entry__.build()
    peak, peak_kind = load_peaks()
    wl = resolve(args)
    # config 4: the job's sequences partitioned batch-wise over the ranks (no data-path collective);
    # configs 2/3: one sequence per GPU (replicas); config 5: ONE sequence, its KV heads over the ranks
    sharded = bool(wl.get("shard_heads"))
    if sharded:
        wl["shard"] = (rank, world)
        seqs = [0]
    else:
        seqs = list(partition(wl["batch"], world, rank)) if wl["batch"] > 1 else [rank]
    geo, fw, qw, head_w, hcache, fcache, firsts, prompts, setup = build_workload(args, wl, seqs)
    use_graphs = not args.no_graphs
    modes = args.modes.split(",")
    shard = wl.get("shard")
    kv_heads_local = hcache.layout.kv_heads

    def spec_runner():
        # KV-head sharding: the fused all-gather, buffers exchanged as CUDA IPC handles (collective)
        from paper_2502_10424_b200.runtime import Runner

        if not sharded:
            return None
        return Runner(geo, hcache, max_cols=args.gamma + 1, shard=(rank, world, None), gather="ipc")

    # QS_BENCH_NO_KERNELS=1: skip the per-kernel timings (ncu launch-list runs count only the decode loop)
    kr = {} if os.environ.get("QS_BENCH_NO_KERNELS") else kernel_roofline(geo, fw, qw, hcache, peak, shard)
    if fcache is not None and kr:
        kr["attn_fp16"] = kernel_fp16(geo, fcache, peak)
    if args.profile_kernels:
        print(json.dumps({"kernels": kr}))
        return

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    res = {}
    clocks = ClockSampler(local)
    t_timed = 0.0
    with clocks:
        barrier()
        t0 = time.time()
        if "both" in modes:
            res["both"] = measure_spec(geo, fw, qw, hcache, firsts, args.gamma, args.steps, args.warmup, use_graphs,
                                       weight_mode="int4", int4_bytes=qw.algorithmic_bytes(), runner=spec_runner())
        if "kv_only" in modes:
            res["kv_only"] = measure_spec(geo, fw, fw, hcache, firsts, args.gamma, args.steps, args.warmup, use_graphs,
                                          weight_mode="fp", runner=spec_runner())
        barrier()
        t_timed += time.time() - t0
    if "fp16_ar" in modes:
        ffirst = firsts
        if fcache is None:
            import gc

            del hcache, qw  # the spec engines' graphs / runners die with them
            gc.collect()
            torch.cuda.empty_cache()
            fcache, ffirst = fp16_cache(args, wl, geo, fw, head_w, prompts)
            if kr:
                kr["attn_fp16"] = kernel_fp16(geo, fcache, peak)
        with clocks:
            barrier()
            t0 = time.time()
            ar_runner = None
            if sharded:
                from paper_2502_10424_b200.runtime import Runner

                ar_runner = Runner(geo, fcache, max_cols=1, shard=(rank, world, None), gather="ipc")
            res["fp16_ar"] = measure_ar(fw, fcache, ffirst, args.steps, args.warmup, use_graphs, runner=ar_runner)
            barrier()
            t_timed += time.time() - t0
    head = res.get("both") or res.get("kv_only")
    # whole-job throughput: tokens emitted on all ranks / the slowest rank's device time
    emitted = head["tok_s"] * head["ms_per_step"] * args.steps / 1e3
    e2e_s = emitted / head["e2e_tok_s"]
    ar = res.get("fp16_ar")
    ar_tok = ar["tok_s"] * ar["ms_per_step"] * args.steps / 1e3 if ar else 0.0
    vals = torch.tensor([head["ms_per_step"], e2e_s, ar["ms_per_step"] if ar else 0.0, emitted, ar_tok],
                        dtype=torch.float64, device="cuda")
    if world > 1:
        t = vals.clone()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        s2 = vals.clone()
        dist.all_reduce(s2, op=dist.ReduceOp.SUM)
        if sharded:  # one sequence decoded by all ranks together: its tokens count once
            s2 = s2 / world
        ms = float(t[0])
        value = float(s2[3]) / (ms * args.steps / 1e3)
        e2e = float(s2[3]) / float(t[1])
        ar_job = float(s2[4]) / (float(t[2]) * args.steps / 1e3) if ar else None
    else:
        ms, value, e2e = head["ms_per_step"], head["tok_s"], head["e2e_tok_s"]
        ar_job = ar["tok_s"] if ar else None
    if rank != 0:
        dist.destroy_process_group() if world > 1 else None
        return
    dom = kr.get("attn_draft", {"gbs": 0.0, "bytes": 0.0})
    traffic, traffic_src = measured_traffic()
    cb = cpu_baseline(wl["context"], args.layers, geo=wl["model"])
    B = wl["batch"]
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f16 (KV int4/int8 planes, INT4 draft weights), f32 accumulate",
        "data": (f"synthetic: random-init weights ({'the reference init_weights stream, seed %d, replayed bit-exactly' % args.seed if args.weights == 'reference' else 'torch.randn on device, the reference recipe'}), "
                 f"uniform random prompt tokens (seed {args.seed}+1+b)"),
        "config": {"workload": wl["name"], "context": wl["context"], "layers": args.layers, "gamma": args.gamma,
                   "batch_total": B, "batch_per_gpu": len(seqs), "kv_heads_per_gpu": kv_heads_local,
                   "l2": "working set per forward (GBs) >> 126 MB L2; no flush needed",
                   "parallelism": (f"KV-head sharding x{world} (fused all-gather in the attention merge)" if sharded
                                   else f"batch partition x{world} (no data-path collective)" if B > 1
                                   else f"replicas x{world} (one sequence per GPU)"),
                   "cuda_graphs": use_graphs},
        "speedup_vs_fp16_ar": value / ar_job if ar_job else None,
        "fp16_ar_tok_s_job": ar_job,
        "modes": res,
        "kernels": kr,
        "roofline": {"bound": "hbm", "kernel": "attn_draft (K2, upper INT4 plane, split-K)", "achieved": dom["gbs"],
                     "peak": peak, "peak_kind": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs, burst copy)", "unit": "GB/s",
                     "frac": dom["gbs"] / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "algorithmic_bytes_per_launch": dom["bytes"]},
        "cpu_baseline": cb,
        "e2e": {"value": e2e, "unit": "tokens/s", "h2d_bytes_per_step": head["h2d_bytes_per_step"],
                "d2h_bytes_per_step": head["d2h_bytes_per_step"],
                "path": "SpeculativeDecoder.decode (public API) over the same cycles as value"},
        "gpu_launches": head["launches"],
        "clocks": clocks.summary(),
        "setup": setup,
        "timed_wall_s": t_timed,
        "lib_md5": lib_digest(),
    }
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
