"""Full-size attention parity (BASELINE config 3's shape: 32 KV heads x 128, G = 128, a
131072-token prompt, one layer).  The oracle cannot run this size in seconds, so the
reference here is a plain fp32 torch attention on the GPU over the store's own
dequantised view (qs_kv_dequant_view, f64 math -- pinned bit-exact against the oracle's
decode_plane_draft / decode_plane_target at small sizes in test_gpu_parity.py) plus the
fp16 fp1 / fp2 buffers.  Tolerance: 2e-3 x max|V| per element, as at small sizes.

This covers the full-size split plan (9-18 splits per head over 1023 blocks), the
last-CTA merge across them, and the verify kernel's causal mask for T = gamma + 1 rows."""

import math

import pytest
import torch

pytestmark = pytest.mark.gpu

H, HD, G = 32, 128, 128
S_P = 131072 + 40  # 1023 quantised blocks + fp1 (128) + fp2 (40)


@pytest.fixture(scope="module")
def store():
    import paper_2502_10424_b200 as qs

    g = torch.Generator(device="cuda").manual_seed(2025)
    kv = H * HD
    k = torch.randn(S_P, kv, device="cuda", generator=g) * (torch.rand(kv, device="cuda", generator=g) * 1.8 + 0.2)
    v = torch.randn(S_P, kv, device="cuda", generator=g)
    k16, v16 = k.half(), v.half()
    del k, v
    cache = qs.HierarchicalKVCache.from_prefill(qs.CacheLayout(1, H, HD, G), [k16], [v16], max_tokens=S_P + 2 * G)
    cache.prompt = (k16, v16)  # kept for the block checks below
    return cache


def _dequant(cache, target: bool):
    from paper_2502_10424_b200 import _lib

    nb = cache.quantized_token_count // G
    ok = torch.empty((nb * G, H * HD), dtype=torch.float32, device="cuda")
    ov = torch.empty_like(ok)
    _lib.call("qs_kv_dequant_view", cache.store_struct(), 0, 0, nb, 1 if target else 0, ok.data_ptr(),
              ov.data_ptr(), _lib.stream_ptr())
    return ok, ov


def _fp(cache, which: int, n: int):
    k = cache.fp_k[0, 0, which, :, :n].permute(1, 0, 2).reshape(n, H * HD).float()
    v = cache.fp_v[0, 0, which, :, :n].permute(1, 0, 2).reshape(n, H * HD).float()
    return k, v


def _reference(q, ks, vs):
    """fp32 softmax attention of q [H, hd] over the concatenated segments."""
    k = torch.cat(ks).view(-1, H, HD)
    v = torch.cat(vs).view(-1, H, HD)
    s = torch.einsum("shd,hd->hs", k, q) / math.sqrt(HD)
    p = torch.softmax(s, dim=1)
    return torch.einsum("hs,shd->hd", p, v)


@pytest.mark.parametrize("view,T", [("draft", 1), ("target", 1), ("target", 5), ("target", 9)])
def test_attention_full_size_vs_fp32_reference(store, view, T):
    from paper_2502_10424_b200 import _lib
    from paper_2502_10424_b200.runtime import Geometry, Runner

    cache = store
    g = torch.Generator(device="cuda").manual_seed(7 + T)
    base = cache.fp2_len
    assert cache.quantized_token_count == 1023 * G and base == 40
    new_k = torch.randn(T, H, HD, device="cuda", generator=g).half()
    new_v = torch.randn(T, H, HD, device="cuda", generator=g).half()
    for t in range(T):  # the verify forward's rows (QKV epilogue writes them the same way)
        cache.fp_k[0, 0, 1, :, base + t] = new_k[t]
        cache.fp_v[0, 0, 1, :, base + t] = new_v[t]
    geo = Geometry(1, H * HD, H, H, HD, 16, 16, 1 << 20)
    run = Runner(geo, cache, max_cols=16)
    q = torch.randn(T, H * HD, device="cuda", generator=g) * 2.0
    run.q[:T] = q
    run._attention(0, _lib.VIEW_DRAFT if view == "draft" else _lib.VIEW_TARGET, T, 0, _lib.stream_ptr())
    torch.cuda.synchronize()
    got = run.attn[:T].view(T, H, HD)

    qk, qv = _dequant(cache, view == "target")
    f1k, f1v = _fp(cache, 0, cache.fp1_len)
    f2k, f2v = _fp(cache, 1, base + T)
    vmax = max(qv.abs().max().item(), f1v.abs().max().item(), f2v.abs().max().item())
    for t in range(T):
        n2 = base + t + 1  # causal: row t sees the fp2 rows up to its own
        want = _reference(q[t].view(H, HD), [qk, f1k, f2k[:n2]], [qv, f1v, f2v[:n2]])
        err = (got[t] - want).abs().max().item()
        assert err <= 2e-3 * vmax, (view, t, err, vmax)


def _check_block(cache, block, k_rows, v_rows):
    import numpy as np

    from oracle import qs_oracle as O

    want = O.quantize_kv_block(O.Layout(1, H, HD, G), k_rows, v_rows)
    got = cache.export_block_planes(0, block)
    for gp, wp in zip(got, (want.ku, want.kl, want.vu, want.vl)):
        assert np.array_equal(gp.codes, wp.codes), block
        assert np.array_equal(gp.scales.view(np.uint32), wp.scales.view(np.uint32)), block
        assert np.array_equal(gp.zeros.view(np.uint32), wp.zeros.view(np.uint32)), block


def test_full_size_blocks_and_flush_bit_exact(store):
    """Prefill blocks at the start, middle and end of the 1023-block arena, then a decode-time
    flush into block 1023 (fp1 -> planes, fp2 -> fp1), bit-exact against the oracle's
    quantize_kv_block (Q/cache.py:249-303) on the same fp16 rows.  Runs last: it mutates the store."""
    cache = store
    k16, v16 = cache.prompt
    f = lambda t: t.float().cpu().numpy()  # noqa: E731
    for b in (0, 511, 1022):
        _check_block(cache, b, f(k16[b * G : (b + 1) * G]), f(v16[b * G : (b + 1) * G]))
    fp1_k, fp1_v = (f(x) for x in _fp(cache, 0, G))
    g = torch.Generator(device="cuda").manual_seed(99)
    base = cache.fp2_len
    rows_k = torch.randn(G - base, H * HD, device="cuda", generator=g).half()
    rows_v = torch.randn(G - base, H * HD, device="cuda", generator=g).half()
    for t in range(G - base):
        cache.append_decode_token(0, rows_k[t], rows_v[t])
    assert cache.fp2_len == G and cache.flush_if_full()
    assert cache.quantized_token_count == 1024 * G and cache.fp2_len == 0 and cache.fp1_len == G
    _check_block(cache, 1023, fp1_k, fp1_v)
