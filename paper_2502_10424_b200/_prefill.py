"""Prompt prefill on the device (outside the measured decode path).

Restates the causal prompt forward of /root/reference/pkg/src/quantspec/model.py:268-321
with library GEMMs (cuBLAS via torch.matmul) and PyTorch SDPA flash attention,
chunked over tokens so a 128K prompt fits, then hands the per-layer K/V to
the cache builders (HierarchicalKVCache.load_prefill_layer quantises the
oldest floor((S-G)/G)*G tokens with the sm_100a flush kernel, Q/cache.py:139-182).

Small prompts run in f32 (closest to the reference's f32/f64 math); long
prompts run fp16 with f32 residuals.
"""

from __future__ import annotations

import numpy as np

from .cache import CacheLayout, FpKVCache, HierarchicalKVCache


def _torch():
    import torch

    return torch


def _rmsnorm(x, gain, eps):
    torch = _torch()
    ms = torch.mean(x * x, dim=-1, keepdim=True)
    return x / torch.sqrt(ms + eps) * gain


def _rope(x, cs):
    """x [S, H, hd]; cs [S, hd/2, 2] (cos, sin) -> adjacent-pair rotation (Q/tensor.py:65-82)."""
    torch = _torch()
    c = cs[:, None, :, 0]
    s = cs[:, None, :, 1]
    e, o = x[..., 0::2], x[..., 1::2]
    out = torch.empty_like(x)
    out[..., 0::2] = e * c - o * s
    out[..., 1::2] = e * s + o * c
    return out


def run_prefill(geo, ids_dev, embedding, layer_iter, final_norm, lm_head, rope, sink, *, dtype=None,
                chunk: int = 8192):
    """Generic prefill.  ``layer_iter`` yields dicts of CUDA tensors
    (wq, wk, wv, wo, w_gate, w_up, w_down as [d_in, d_out], attn_norm, mlp_norm);
    ``sink(layer, k, v)`` receives K/V [S, kv_dim].  Returns f32 logits of the last row."""
    return run_prefill_batch(geo, [ids_dev], embedding, layer_iter, final_norm, lm_head, rope,
                             [sink], dtype=dtype, chunk=chunk)[0]


def run_prefill_batch(geo, ids_list, embedding, layer_iter, final_norm, lm_head, rope, sinks, *, dtype=None,
                      chunk: int = 8192):
    """Prefill of several independent prompts, layer-outer: each layer's weights are produced once
    (``layer_iter``) and applied to every prompt; ``sinks[b](layer, k, v)`` receives prompt b's
    K/V [S_b, kv_dim].  Returns the f32 last-row logits of every prompt."""
    torch = _torch()
    import torch.nn.functional as F

    H, Hk, hd = geo.num_heads, geo.num_kv_heads, geo.head_dim
    if dtype is None:
        dtype = torch.float32 if max(int(i.numel()) for i in ids_list) * geo.hidden <= (1 << 23) else torch.float16
    xs = [embedding[ids.long()].float() for ids in ids_list]  # residual streams stay f32
    for li, lw in enumerate(layer_iter):
        W = {k: (v.to(dtype) if v.dim() == 2 else v.float()) for k, v in lw.items()}
        for b, x in enumerate(xs):
            S = int(x.shape[0])
            cs = rope[:S]
            q = torch.empty((S, H, hd), dtype=dtype, device=x.device)
            k = torch.empty((S, Hk, hd), dtype=dtype, device=x.device)
            v = torch.empty((S, Hk, hd), dtype=dtype, device=x.device)
            for c0 in range(0, S, chunk):
                c1 = min(S, c0 + chunk)
                h = _rmsnorm(x[c0:c1], W["attn_norm"], geo.norm_eps).to(dtype)
                q[c0:c1] = _rope((h @ W["wq"]).float().view(c1 - c0, H, hd), cs[c0:c1]).to(dtype)
                k[c0:c1] = _rope((h @ W["wk"]).float().view(c1 - c0, Hk, hd), cs[c0:c1]).to(dtype)
                v[c0:c1] = (h @ W["wv"]).view(c1 - c0, Hk, hd)
            sinks[b](li, k.reshape(S, Hk * hd), v.reshape(S, Hk * hd))
            kq = k if Hk == H else k.repeat_interleave(H // Hk, dim=1)
            vq = v if Hk == H else v.repeat_interleave(H // Hk, dim=1)
            ctx = F.scaled_dot_product_attention(q.transpose(0, 1)[None], kq.transpose(0, 1)[None],
                                                 vq.transpose(0, 1)[None], is_causal=True)[0].transpose(0, 1)
            del kq, vq, q, k, v
            ctx = ctx.reshape(S, H * hd)
            for c0 in range(0, S, chunk):
                c1 = min(S, c0 + chunk)
                x[c0:c1] += (ctx[c0:c1].to(dtype) @ W["wo"]).float()
                hm = _rmsnorm(x[c0:c1], W["mlp_norm"], geo.norm_eps).to(dtype)
                g = (hm @ W["w_gate"]).float()
                u = (hm @ W["w_up"]).float()
                act = (g / (1.0 + torch.exp(-g)) * u).to(dtype)
                x[c0:c1] += (act @ W["w_down"]).float()
            del ctx
        del W
    out = []
    for x in xs:
        last = _rmsnorm(x[-1:], final_norm, geo.norm_eps)
        out.append((last.to(dtype) @ lm_head.to(dtype)).float()[0])
    return out


def prefill_device(weights, ids: np.ndarray, cache_mode: str, *, group_size=None, sensitive_layers=frozenset(),
                   max_tokens=None):
    torch = _torch()
    cfg = weights.config
    fw, _ = weights.device()
    geo = fw.geo
    S = int(ids.size)
    ids_dev = torch.from_numpy(ids.astype(np.int32)).cuda()
    cap = max_tokens or max(S + 256, 2 * S)
    if cache_mode == "hierarchical":
        g = group_size if group_size is not None else 128
        lay = CacheLayout(cfg.num_layers, cfg.num_heads, cfg.head_dim, g, frozenset(sensitive_layers), cfg.num_kv_heads)
        cache = HierarchicalKVCache(lay, max_tokens=max(cap, S + 2 * g))
    else:
        cache = FpKVCache(cfg.num_layers, cfg.kv_dim, capacity=max(64, cap), head_dim=cfg.head_dim)

    def layers():
        for lw in weights.layers:
            d = {n: torch.from_numpy(np.ascontiguousarray(getattr(lw, n), dtype=np.float32)).cuda()
                 for n in ("wq", "wk", "wv", "wo", "w_gate", "w_up", "w_down")}
            d["attn_norm"] = torch.from_numpy(np.asarray(lw.attn_norm, np.float32)).cuda()
            d["mlp_norm"] = torch.from_numpy(np.asarray(lw.mlp_norm, np.float32)).cuda()
            yield d

    head = torch.from_numpy(np.ascontiguousarray(weights.lm_head, dtype=np.float32)).cuda()
    logits = run_prefill(geo, ids_dev, fw.embedding, layers(), fw.final_norm, head, fw.rope,
                         lambda l, k, v: cache.load_prefill_layer(l, k, v))
    cache.finish_prefill(S)
    return logits.cpu().numpy().astype(np.float32), cache


def prefill_batch_device(weights, prompts, *, group_size=None, sensitive_layers=frozenset(), max_tokens=None):
    """Prefill several independent prompts (ragged lengths) into ONE batched HierarchicalKVCache
    (sequence b <- prompts[b]); returns (per-sequence last-row logits, cache)."""
    torch = _torch()
    cfg = weights.config
    fw, _ = weights.device()
    g = group_size if group_size is not None else 128
    lens = [int(np.asarray(p).size) for p in prompts]
    cap = max_tokens or (max(lens) + 2 * g + 256)
    lay = CacheLayout(cfg.num_layers, cfg.num_heads, cfg.head_dim, g, frozenset(sensitive_layers), cfg.num_kv_heads)
    cache = HierarchicalKVCache(lay, max_tokens=max(cap, max(lens) + 2 * g), batch=len(prompts))

    def layers():
        for lw in weights.layers:
            d = {n: torch.from_numpy(np.ascontiguousarray(getattr(lw, n), dtype=np.float32)).cuda()
                 for n in ("wq", "wk", "wv", "wo", "w_gate", "w_up", "w_down")}
            d["attn_norm"] = torch.from_numpy(np.asarray(lw.attn_norm, np.float32)).cuda()
            d["mlp_norm"] = torch.from_numpy(np.asarray(lw.mlp_norm, np.float32)).cuda()
            yield d

    head = torch.from_numpy(np.ascontiguousarray(weights.lm_head, dtype=np.float32)).cuda()
    out = []
    for b, p in enumerate(prompts):
        ids = torch.from_numpy(np.asarray(p, dtype=np.int32).ravel()).cuda()
        lg = run_prefill(fw.geo, ids, fw.embedding, layers(), fw.final_norm, head, fw.rope,
                         lambda l, k, v, b=b: cache.load_prefill_layer(l, k, v, seq=b))
        cache.finish_prefill(lens[b], seq=b)
        out.append(lg.cpu().numpy().astype(np.float32))
    return out, cache
