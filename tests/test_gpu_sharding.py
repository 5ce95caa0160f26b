"""KV-head sharding (one sequence whose context exceeds one GPU) on a
single B200: two ranks (gloo; both on cuda:0) each hold half of the KV heads -- their
own store, QKV head columns and attention launches -- and all-gather the attention
rows before the replicated output projection / MLP.  The sharded forwards must equal
the unsharded forward (draft view T=1 and target view T=3) within the attention
tolerance; the only difference is the split-K plan of the smaller head set."""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _device_weights(w, head_shard=None):
    from paper_2502_10424_b200.model import _MATS
    from paper_2502_10424_b200.runtime import build_device_weights, rope_table

    cfg = w.config
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()  # noqa: E731
    mats = ({n: dev(getattr(lw, n)) for n in _MATS} for lw in w.layers)
    fw, _ = build_device_weights(cfg.geometry(), mats, dev(w.embedding), dev(w.final_norm), dev(w.lm_head),
                                 [dev(lw.attn_norm) for lw in w.layers], [dev(lw.mlp_norm) for lw in w.layers],
                                 rope=rope_table(cfg.head_dim, cfg.rope_base, cfg.max_positions),
                                 head_shard=head_shard)
    return fw


def _worker(rank: int, world: int, port: int, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    try:
        import paper_2502_10424_b200 as qs
        from paper_2502_10424_b200 import _lib
        from paper_2502_10424_b200.runtime import Runner

        cfg = qs.ModelConfig(num_layers=2, num_heads=4, head_dim=32, hidden=128, mlp_hidden=256, vocab=96,
                             max_positions=512, num_kv_heads=2)
        geo = cfg.geometry()
        w = qs.init_weights(cfg, seed=5)
        rng = np.random.default_rng(3)
        S, G, L = 200, 32, cfg.num_layers
        ks = [rng.standard_normal((S, geo.nk)).astype(np.float16).astype(np.float32) for _ in range(L)]
        vs = [rng.standard_normal((S, geo.nk)).astype(np.float16).astype(np.float32) for _ in range(L)]
        full_cache = qs.HierarchicalKVCache.from_prefill(qs.CacheLayout(L, 4, 32, G, num_kv_heads=2), ks, vs)
        kn = geo.nk // world
        loc = slice(rank * kn, (rank + 1) * kn)
        shard_cache = qs.HierarchicalKVCache.from_prefill(
            qs.CacheLayout(L, 4 // world, 32, G, num_kv_heads=2 // world), [k[:, loc] for k in ks], [v[:, loc] for v in vs])
        full = Runner(geo, full_cache, max_cols=8)
        part = Runner(geo, shard_cache, max_cols=8, shard=(rank, world, None))
        fw, fw_l = _device_weights(w), _device_weights(w, head_shard=(rank, world))
        errs = []
        for view, T, toks in ((_lib.VIEW_DRAFT, 1, [7]), (_lib.VIEW_TARGET, 3, [11, 40, 2])):
            for run, weights in ((full, fw), (part, fw_l)):
                run.tok[0, :T] = torch.tensor(toks, dtype=torch.int32, device="cuda")
                run.forward(weights, T, view)
            torch.cuda.synchronize()
            a, b = full.logits[:T].cpu().numpy(), part.logits[:T].cpu().numpy()
            errs.append(float(np.abs(a - b).max() / max(1e-6, np.abs(a).max())))
        out[rank] = errs
    finally:
        dist.destroy_process_group()


def test_kv_head_sharded_forward_matches_unsharded():
    import torch.multiprocessing as mp

    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        assert all(e <= 2e-3 for e in out[r]), (r, list(out[r]))


def test_shard_rejects_indivisible_heads():
    import paper_2502_10424_b200 as qs
    from paper_2502_10424_b200.errors import ConfigError
    from paper_2502_10424_b200.runtime import Runner

    cfg = qs.ModelConfig(num_layers=1, num_heads=4, head_dim=32, hidden=128, mlp_hidden=256, vocab=96,
                         max_positions=256, num_kv_heads=2)
    cache = qs.HierarchicalKVCache(qs.CacheLayout(1, 4, 32, 32, num_kv_heads=2), max_tokens=128)
    with pytest.raises(ConfigError):
        Runner(cfg.geometry(), cache, max_cols=4, shard=(0, 3, None))


# ---------------------------------------------------------------------------------------------
# fused all-gather (qs_gather_args): ranks as threads of one process, one CUDA stream each
# ---------------------------------------------------------------------------------------------

def _shard_setup(world, splits, S=200, G=32, seed=5):
    import paper_2502_10424_b200 as qs
    from paper_2502_10424_b200.parallel import HeadGather
    from paper_2502_10424_b200.runtime import Runner

    cfg = qs.ModelConfig(num_layers=2, num_heads=4, head_dim=32, hidden=128, mlp_hidden=256, vocab=96,
                         max_positions=512, num_kv_heads=2)
    geo = cfg.geometry()
    w = qs.init_weights(cfg, seed=seed)
    rng = np.random.default_rng(3)
    L = cfg.num_layers
    ks = [rng.standard_normal((S, geo.nk)).astype(np.float16).astype(np.float32) for _ in range(L)]
    vs = [rng.standard_normal((S, geo.nk)).astype(np.float16).astype(np.float32) for _ in range(L)]
    full_cache = qs.HierarchicalKVCache.from_prefill(qs.CacheLayout(L, 4, 32, G, num_kv_heads=2), ks, vs)
    kn = geo.nk // world
    caches, weights, gathers = [], [], []
    for r in range(world):
        loc = slice(r * kn, (r + 1) * kn)
        caches.append(qs.HierarchicalKVCache.from_prefill(
            qs.CacheLayout(L, 4 // world, 32, G, num_kv_heads=2 // world), [k[:, loc] for k in ks], [v[:, loc] for v in vs]))
        weights.append(_device_weights(w, head_shard=(r, world)))
    return cfg, geo, w, full_cache, caches, weights


def test_fused_gather_forward_bit_identical_to_unsharded():
    """Same split-K plan per head on both sides -> every head's row is computed identically, and
    the fused gather only moves bits: sharded logits (on every rank) == unsharded logits, exactly."""
    import threading

    from paper_2502_10424_b200 import _lib
    from paper_2502_10424_b200.parallel import HeadGather
    from paper_2502_10424_b200.runtime import Runner

    world, splits = 2, 3
    cfg, geo, w, full_cache, caches, weights = _shard_setup(world, splits)
    full = Runner(geo, full_cache, max_cols=8, attn_splits=splits)
    fw = _device_weights(w)
    probe = Runner(geo, caches[0], max_cols=8, attn_splits=splits, shard=(0, world, None))
    gathers = [HeadGather(world, r, 8, probe.xh.shape[1], probe.xs.shape[1]) for r in range(world)]
    HeadGather.link_local(gathers)
    parts = [Runner(geo, caches[r], max_cols=8, attn_splits=splits, shard=(r, world, None), gather=gathers[r])
             for r in range(world)]
    streams = [torch.cuda.Stream() for _ in range(world)]
    for view, T, toks in ((_lib.VIEW_DRAFT, 1, [7]), (_lib.VIEW_TARGET, 3, [11, 40, 2]), (_lib.VIEW_DRAFT, 1, [9])):
        full.tok[0, :T] = torch.tensor(toks, dtype=torch.int32, device="cuda")
        full.forward(fw, T, view)
        for p in parts:
            p.tok[0, :T] = torch.tensor(toks, dtype=torch.int32, device="cuda")
        torch.cuda.synchronize()

        def run(r):
            with torch.cuda.stream(streams[r]):
                parts[r].forward(weights[r], T, view)
            streams[r].synchronize()

        ths = [threading.Thread(target=run, args=(r,)) for r in range(world)]
        for t in ths:
            t.start()
        for t in ths:
            t.join(60)
        assert not any(t.is_alive() for t in ths), "fused gather deadlocked"
        ref = full.logits[:T].cpu().numpy()
        for p in parts:
            assert np.array_equal(p.logits[:T].cpu().numpy(), ref), (view, T)
    for g in gathers:
        g.close()


def test_sharded_spec_cycles_token_exact():
    """A full speculative loop (draft / verify / accept / flush, fp2 wrap-around included) with the
    KV heads split over two ranks (fused gather, one stream and engine per rank) emits exactly the
    unsharded engine's tokens, and both ranks agree."""
    import threading

    import paper_2502_10424_b200 as qs
    from paper_2502_10424_b200.engine import SpecEngine
    from paper_2502_10424_b200.parallel import HeadGather
    from paper_2502_10424_b200.runtime import Runner

    world, splits, gamma, cycles = 2, 3, 4, 14
    cfg, geo, w, full_cache, caches, weights = _shard_setup(world, splits, S=230)
    fw = _device_weights(w)
    ref_eng = SpecEngine(fw, fw, full_cache, gamma, use_graphs=False,
                         runner=Runner(geo, full_cache, max_cols=gamma + 1, attn_splits=splits))
    probe = Runner(geo, caches[0], max_cols=gamma + 1, attn_splits=splits, shard=(0, world, None))
    gathers = [HeadGather(world, r, gamma + 1, probe.xh.shape[1], probe.xs.shape[1]) for r in range(world)]
    HeadGather.link_local(gathers)
    engs = [SpecEngine(weights[r], weights[r], caches[r], gamma, use_graphs=False,
                       runner=Runner(geo, caches[r], max_cols=gamma + 1, attn_splits=splits, shard=(r, world, None),
                                     gather=gathers[r])) for r in range(world)]
    first = 5
    ref_eng.set_pending([first])
    ref = []
    for _ in range(cycles):
        gs, drafts, v, nxt, _ = ref_eng.cycle()
        ref.append((int(gs[0]), drafts[0], int(v[0]), int(nxt[0])))
    out = [[] for _ in range(world)]
    streams = [torch.cuda.Stream() for _ in range(world)]

    def run(r):
        with torch.cuda.stream(streams[r]):
            engs[r].set_pending([first])
            for _ in range(cycles):
                gs, drafts, v, nxt, _ = engs[r].cycle()
                out[r].append((int(gs[0]), drafts[0], int(v[0]), int(nxt[0])))

    ths = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(120)
    assert not any(t.is_alive() for t in ths), "sharded engines deadlocked"
    assert out[0] == out[1] == ref
    assert int(caches[0].quantized_token_count) > 192  # the prompt quantised 192 tokens: a decode-time flush ran
    for g in gathers:
        g.close()


def _worker_ipc(rank: int, world: int, port: int, out):
    """One process per rank (both on cuda:0 here; one GPU each on a multi-GPU box): the gather
    buffers are exchanged as CUDA IPC handles over the process group, as bench/engine do."""
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    try:
        from paper_2502_10424_b200 import _lib
        from paper_2502_10424_b200.runtime import Runner

        splits = 3
        cfg, geo, w, full_cache, caches, weights = _shard_setup(world, splits)
        full = Runner(geo, full_cache, max_cols=8, attn_splits=splits)
        fw = _device_weights(w)
        part = Runner(geo, caches[rank], max_cols=8, attn_splits=splits, shard=(rank, world, None), gather="ipc")
        res = []
        for view, T, toks in ((_lib.VIEW_DRAFT, 1, [7]), (_lib.VIEW_TARGET, 3, [11, 40, 2])):
            for run, wts in ((full, fw), (part, weights[rank])):
                run.tok[0, :T] = torch.tensor(toks, dtype=torch.int32, device="cuda")
                run.forward(wts, T, view)
            torch.cuda.synchronize()
            res.append(bool(np.array_equal(full.logits[:T].cpu().numpy(), part.logits[:T].cpu().numpy())))
        dist.barrier()
        part.gather.close()
        out[rank] = res
    finally:
        dist.destroy_process_group()


def test_fused_gather_across_processes_ipc():
    import torch.multiprocessing as mp

    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_ipc, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        assert all(out[r]), (r, list(out[r]))
