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
