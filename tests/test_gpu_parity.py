"""Parity of the CUDA path (through the C ABI) against the CPU oracle and the
reference golden vectors.  Needs a B200: run with ``-m gpu``.

Bars (stated per test):
  * codes, scales, zero points, buffer state, accept decisions: bit-exact;
  * attention outputs: max |err| <= 2e-3 * max|V| against the oracle's f64
    _merged_attention over the oracle's views of the SAME fp16 K/V inputs;
  * linear layers: <= 2e-3 relative (f16 weights/activations, f32 accumulate);
  * logits: toy model vs the oracle decode_step on identical cache contents.
"""

import copy
import json
import math
import os

import numpy as np
import pytest

from oracle import qs_oracle as O

from .conftest import GOLDEN

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2502_10424_b200 as qs  # noqa: E402
from paper_2502_10424_b200 import _lib  # noqa: E402
from paper_2502_10424_b200.runtime import Geometry, Runner  # noqa: E402


def f16(a):
    return np.asarray(a, np.float32).astype(np.float16).astype(np.float32)


# ---------------------------------------------------------------------------
# L0: quantisation entry points vs the reference's own golden vectors
# ---------------------------------------------------------------------------


def test_plane_encode_decode_golden_bit_exact():
    z = np.load(os.path.join(GOLDEN, "quant_golden.npz"))
    for i in range(int(z["n_cases"])):
        g, rl = (int(x) for x in z[f"c{i}_group"])
        up, lo = qs.encode_plane_hierarchical(z[f"c{i}_values"], g, "channel", rl or None)
        for tag, p in (("up", up), ("lo", lo)):
            assert np.array_equal(p.codes, z[f"c{i}_{tag}_codes"]), (i, tag)
            assert np.array_equal(p.scales.view(np.uint32), z[f"c{i}_{tag}_scales"].view(np.uint32)), (i, tag)
            assert np.array_equal(p.zeros.view(np.uint32), z[f"c{i}_{tag}_zeros"].view(np.uint32)), (i, tag)
        assert np.array_equal(qs.decode_plane_draft(up), z[f"c{i}_draft"]), i
        assert np.array_equal(qs.decode_plane_target(up, lo), z[f"c{i}_target"]), i


def test_group_kats_and_errors():
    with open(os.path.join(GOLDEN, "group_kat.json")) as f:
        kats = json.load(f)
    for k in kats:
        (uc, up), (lc, lp) = qs.hierarchical_encode(k["values"])
        assert uc.tolist() == k["cu"] and lc.tolist() == k["cl"]
        assert up.scale == k["S"] and up.zero_point == k["Z"] and lp.scale == k["Sl"]
    codes, p = qs.quantize_group_asym_u4([0.0, 1.0, 2.0, 3.0])
    assert codes.tolist() == [0, 5, 10, 15] and p.zero_point == 0.0
    codes, _ = qs.quantize_group_sym_s4([0.07], scale=0.0125)
    assert codes.tolist() == [6]
    codes, _ = qs.quantize_group_sym_s4([0.0125 * 12.0, -0.0125 * 12.0, 0.0125 * 7.49], scale=0.0125)
    assert codes.tolist() == [7, -8, 7]
    with pytest.raises(qs.DataError):
        qs.quantize_group_asym_u4([])
    with pytest.raises(qs.DataError):
        qs.quantize_group_asym_u4([1.0, np.nan])
    with pytest.raises(qs.ConfigError):
        qs.quantize_group_sym_s4([0.1], scale=0.0)
    with pytest.raises(qs.CacheIntegrityError):
        qs.encode_plane_hierarchical(np.arange(10.0), 4, "token", 3)


def test_weight_quant_golden_bit_exact():
    z = np.load(os.path.join(GOLDEN, "quant_golden.npz"))
    w = z["w_in"]
    for g in (32, 16, 7):
        q = qs.quantize_weights(w, g)
        assert np.array_equal(q.plane.codes, z[f"w{g}_codes"])
        assert np.array_equal(q.plane.scales, z[f"w{g}_scales"])
        assert np.array_equal(q.plane.zeros, z[f"w{g}_zeros"])
        assert np.array_equal(qs.dequantize_weights(q), z[f"w{g}_deq"])


# ---------------------------------------------------------------------------
# L1: the flush kernel (K1) and the store state machine
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("H,hd,G", [(2, 128, 128), (4, 16, 16), (4, 16, 128), (2, 64, 64), (8, 32, 32)])
def test_flush_quantize_bit_exact_vs_oracle(H, hd, G):
    rng = np.random.default_rng(H * 1000 + hd + G)
    kv = H * hd
    n = 4 * G + 7
    k = f16(rng.standard_normal((n, kv)) * rng.uniform(0.1, 4.0, kv) + rng.uniform(-2, 2, kv))
    v = f16(rng.standard_normal((n, kv)) * 3.0)
    lay = qs.CacheLayout(1, H, hd, G)
    cache = qs.HierarchicalKVCache.from_prefill(lay, [k], [v])
    olay = O.Layout(1, H, hd, G)
    assert cache.quantized_token_count == ((n - G) // G) * G
    for b in range(cache.quantized_token_count // G):
        want = O.quantize_kv_block(olay, k[b * G : (b + 1) * G], v[b * G : (b + 1) * G])
        got = cache.export_block_planes(0, b)
        for gp, wp in zip(got, (want.ku, want.kl, want.vu, want.vl)):
            assert np.array_equal(gp.codes, wp.codes), b
            assert np.array_equal(gp.scales.view(np.uint32), wp.scales.view(np.uint32)), b
            assert np.array_equal(gp.zeros.view(np.uint32), wp.zeros.view(np.uint32)), b
    # device f32 views == oracle views (same fp16 inputs), bit for bit
    oc = O.OracleKVCache.from_prefill(olay, [k], [v])
    for kind in ("draft", "target"):
        vw = getattr(cache, f"{kind}_view")(0)
        ov = oc.view(0, kind)
        gk, gv = vw.concat()
        assert np.array_equal(gk, ov.k) and np.array_equal(gv, ov.v), kind
        assert (vw.quantized_bytes, vw.param_bytes, vw.fp_bytes, vw.quantized_elements) == (
            ov.quantized_bytes, ov.param_bytes, ov.fp_bytes, ov.quantized_elements)


def test_scripted_session_matches_oracle_state_machine():
    """Replay the reference cache script (tests/golden/cache_script.json) on the
    device store and on the oracle fed the same fp16-rounded rows."""
    z = np.load(os.path.join(GOLDEN, "cache_golden.npz"))
    with open(os.path.join(GOLDEN, "cache_script.json")) as f:
        script = json.load(f)
    keys = [f16(z["keys0"]), f16(z["keys1"])]
    vals = [f16(z["vals0"]), f16(z["vals1"])]
    lay = qs.CacheLayout(2, 2, 16, 16)
    dev = qs.HierarchicalKVCache.from_prefill(lay, keys, vals, max_tokens=4096)
    orc = O.OracleKVCache.from_prefill(O.Layout(2, 2, 16, 16), keys, vals)
    ak, av = f16(z["appended_k"]), f16(z["appended_v"])
    for op, arg in script:
        if op == "append":
            for layer in range(2):
                dev.append_decode_token(layer, ak[arg][layer], av[arg][layer])
                orc.append_decode_token(layer, ak[arg][layer], av[arg][layer])
        elif op == "rollback":
            dev.rollback(arg)
            orc.rollback(arg)
        elif op == "flush":
            assert int(dev.flush_if_full()) == arg == int(orc.flush_if_full())
        else:
            assert [dev.quantized_token_count, dev.fp1_len, dev.fp2_len] == arg
    for layer in range(2):
        for kind in ("draft", "target"):
            gk, gv = getattr(dev, f"{kind}_view")(layer).concat()
            ov = orc.view(layer, kind)
            assert np.array_equal(gk, ov.k) and np.array_equal(gv, ov.v)
    rep = dev.memory_report()
    assert [rep.upper_bytes, rep.lower_bytes, rep.param_bytes, rep.fp_buffer_bytes, rep.archived_fp_bytes] == z["mem"].tolist()


def test_rollback_overflow_and_errors():
    lay = qs.CacheLayout(2, 2, 16, 16)
    rng = np.random.default_rng(1)
    kv = 32
    c = qs.HierarchicalKVCache.from_prefill(lay, [rng.standard_normal((32, kv))] * 2, [rng.standard_normal((32, kv))] * 2)
    for _ in range(16):
        for layer in range(2):
            c.append_decode_token(layer, np.zeros(kv), np.zeros(kv))
    with pytest.raises(qs.BufferOverflowError):
        c.append_decode_token(0, np.zeros(kv), np.zeros(kv))
    c.rollback(3)
    assert c.fp2_len == 13
    with pytest.raises(qs.CacheIntegrityError):
        c.rollback(14)
    with pytest.raises(qs.EmptyPromptError):
        qs.HierarchicalKVCache.from_prefill(lay, [np.zeros((0, kv))] * 2, [np.zeros((0, kv))] * 2)
    bad = np.ones((40, kv), np.float32)
    bad[3, 5] = np.nan
    with pytest.raises(qs.DataError):
        qs.HierarchicalKVCache.from_prefill(lay, [bad] * 2, [bad] * 2)


def test_sensitive_layers_and_snapshot_round_trip(tmp_path):
    lay = qs.CacheLayout(2, 2, 16, 16, sensitive_layers=frozenset({0}))
    rng = np.random.default_rng(2)
    keys = [f16(rng.standard_normal((3 * 16 + 5, 32))) for _ in range(2)]
    vals = [f16(rng.standard_normal((3 * 16 + 5, 32))) for _ in range(2)]
    c = qs.HierarchicalKVCache.from_prefill(lay, keys, vals)
    k0, v0 = c.draft_view(0).concat()
    assert np.array_equal(k0, keys[0]) and np.array_equal(v0, vals[0])
    assert c.draft_view(0).quantized_bytes == 0
    p = tmp_path / "c.qskv"
    c.save_snapshot(p)
    d = qs.HierarchicalKVCache.load_snapshot(p)
    for layer in range(2):
        a = c.target_view(layer).concat()
        b = d.target_view(layer).concat()
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    p2 = tmp_path / "d.qskv"
    d.save_snapshot(p2)
    assert p.read_bytes() == p2.read_bytes()


def test_snapshot_interoperates_with_oracle_planes(tmp_path):
    """Planes exported from the device store decode (oracle) to the device view."""
    lay = qs.CacheLayout(1, 4, 16, 16)
    rng = np.random.default_rng(4)
    k = f16(rng.standard_normal((5 * 16, 64)))
    v = f16(rng.standard_normal((5 * 16, 64)))
    c = qs.HierarchicalKVCache.from_prefill(lay, [k], [v])
    ku, kl, vu, vl = c.export_block_planes(0, 1)
    blk = O.Block(*(O.Plane(p.codes, p.count, p.group_size, p.scales, p.zeros, p.mode, p.axis, p.row_len) for p in (ku, kl, vu, vl)))
    ok, ov = O.dequant_kv_block(O.Layout(1, 4, 16, 16), blk, "target")
    gk, gv = c.target_view(0).concat()
    assert np.array_equal(gk[16:32], ok) and np.array_equal(gv[16:32], ov)


# ---------------------------------------------------------------------------
# L2: attention kernels (K2 draft, K3 verify, K4 fp16) vs oracle _merged_attention
# ---------------------------------------------------------------------------


def _attn_setup(H, hd, G, n_prompt, extra, seed=0, r=1):
    rng = np.random.default_rng(seed)
    kv = H * hd
    k = f16(rng.standard_normal((n_prompt, kv)) * rng.uniform(0.2, 2.0, kv))
    v = f16(rng.standard_normal((n_prompt, kv)))
    lay = qs.CacheLayout(1, H * r, hd, G, num_kv_heads=H)
    cache = qs.HierarchicalKVCache.from_prefill(lay, [k], [v], max_tokens=n_prompt + 4 * G)
    olay = O.Layout(1, H, hd, G)
    orc = O.OracleKVCache.from_prefill(olay, [k], [v])
    rows_k = f16(rng.standard_normal((extra, kv)))
    rows_v = f16(rng.standard_normal((extra, kv)))
    return cache, orc, rows_k, rows_v, rng


def _run_attention(cache, q, view, T, row_offset=0, r=1, splits=None):
    lay = cache.layout
    geo = Geometry(1, lay.num_heads * lay.head_dim, lay.num_heads, lay.kv_heads, lay.head_dim, 16, 16, 1 << 20)
    run = Runner(geo, cache, max_cols=32, attn_splits=splits)
    run.q[:T] = torch.from_numpy(q.reshape(T, -1)).cuda()
    run._attention(0, view, T, row_offset, _lib.stream_ptr())
    torch.cuda.synchronize()
    return run.attn[:T].cpu().numpy()


@pytest.mark.parametrize("H,hd,G,n_prompt", [(4, 128, 128, 5 * 128 + 40), (4, 16, 16, 291), (4, 16, 128, 700),
                                             (2, 64, 64, 64 * 9 + 3)])
@pytest.mark.parametrize("view", ["draft", "target"])
@pytest.mark.parametrize("T", [1, 5, 9])
def test_attention_vs_oracle(H, hd, G, n_prompt, view, T):
    cache, orc, rk, rv, rng = _attn_setup(H, hd, G, n_prompt, T, seed=H + hd + G + T)
    # append T new rows (as a verify forward would) then attend causally
    room = G - cache.fp2_len
    if room < T:
        pytest.skip("fp2 too full for this T")
    base = cache.fp2_len
    for t in range(T):
        for_oracle = (rk[t], rv[t])
        cache.fp_k[0, 0, 1, :, base + t] = torch.from_numpy(rk[t]).cuda().half().reshape(H, hd)
        cache.fp_v[0, 0, 1, :, base + t] = torch.from_numpy(rv[t]).cuda().half().reshape(H, hd)
    q = (rng.standard_normal((T, H, hd)) * 2.0).astype(np.float32)
    got = _run_attention(cache, q, _lib.VIEW_DRAFT if view == "draft" else _lib.VIEW_TARGET, T)
    vmax = 0.0
    for t in range(T):
        orc.append_decode_token(0, rk[t], rv[t])
        vw = orc.view(0, view)
        want = O.attend_view(q[t], vw, H, hd)
        vmax = max(vmax, float(np.abs(vw.v).max()))
        err = np.abs(got[t].reshape(H, hd) - want).max()
        assert err <= 2e-3 * vmax, (t, err)


@pytest.mark.parametrize("view", ["draft", "target"])
@pytest.mark.parametrize("T", [1, 2, 5])
def test_attention_gqa_vs_oracle(view, T):
    """GQA (config 4 shape class): r query heads share one KV head.  The oracle has no GQA
    model; it is restated by repeating each KV head r times.  Covers the
    query-row variants of the target kernel (1-8 rows per CTA and two query tiles) and
    the draft's 1-3 column tiles."""
    H, hd, G, r = 2, 128, 128, 4
    cache, orc, rk, rv, rng = _attn_setup(H, hd, G, 3 * 128 + 70, T, seed=40 + T, r=r)
    base = cache.fp2_len
    for t in range(T):
        cache.fp_k[0, 0, 1, :, base + t] = torch.from_numpy(rk[t]).cuda().half().reshape(H, hd)
        cache.fp_v[0, 0, 1, :, base + t] = torch.from_numpy(rv[t]).cuda().half().reshape(H, hd)
    q = (rng.standard_normal((T, H * r, hd)) * 2.0).astype(np.float32)
    got = _run_attention(cache, q, _lib.VIEW_DRAFT if view == "draft" else _lib.VIEW_TARGET, T)
    for t in range(T):
        orc.append_decode_token(0, rk[t], rv[t])
        vw = orc.view(0, view)
        segs = [(np.repeat(k.reshape(-1, H, hd), r, axis=1), np.repeat(v.reshape(-1, H, hd), r, axis=1))
                for k, v in vw.segments]
        want = O.merged_attention(q[t], segs, 1.0 / np.sqrt(hd))
        vmax = float(np.abs(vw.v).max())
        err = np.abs(got[t].reshape(H * r, hd) - want).max()
        assert err <= 2e-3 * vmax, (t, err)


@pytest.mark.parametrize("r,splits", [(1, None), (1, 1), (4, None), (4, 1)])
def test_attention_batch_invariance_bit_exact(r, splits):
    """Row t of a T-row launch == the same row launched alone at its position -- also when one CTA
    streams many chunks (splits=1: the lazy softmax reference must be decided per query, not per
    warp) and for GQA, where the T-row verify parks its accumulators in TMEM (r*T = 20 queries)
    while a single row keeps them in registers."""
    H, hd, G = 4, 128, 128
    cache, orc, rk, rv, rng = _attn_setup(H, hd, G, 9 * 128 + 17, 5, seed=11, r=r)
    base = cache.fp2_len
    for t in range(5):
        cache.fp_k[0, 0, 1, :, base + t] = torch.from_numpy(rk[t]).cuda().half().reshape(H, hd)
        cache.fp_v[0, 0, 1, :, base + t] = torch.from_numpy(rv[t]).cuda().half().reshape(H, hd)
    q = (rng.standard_normal((5, H * r, hd)) * 2.0).astype(np.float32)
    for view in (_lib.VIEW_DRAFT, _lib.VIEW_TARGET):
        full = _run_attention(cache, q, view, 5, r=r, splits=splits)
        for t in range(5):
            one = _run_attention(cache, q[t : t + 1], view, 1, row_offset=t, r=r, splits=splits)
            assert np.array_equal(one[0], full[t]), (view, t)


def test_fp16_cache_attention_vs_oracle():
    rng = np.random.default_rng(5)
    H, hd, n = 4, 128, 1000
    k = f16(rng.standard_normal((n, H * hd)))
    v = f16(rng.standard_normal((n, H * hd)))
    c = qs.FpKVCache.from_prefill([k[:-3]], [v[:-3]], head_dim=hd)
    for t in range(3):
        c.k[0, 0, :, n - 3 + t] = torch.from_numpy(k[n - 3 + t]).cuda().half().reshape(H, hd)
        c.v[0, 0, :, n - 3 + t] = torch.from_numpy(v[n - 3 + t]).cuda().half().reshape(H, hd)
    geo = Geometry(1, H * hd, H, H, hd, 16, 16, 1 << 20)
    run = Runner(geo, c, max_cols=3)
    q = rng.standard_normal((3, H, hd)).astype(np.float32)
    run.q[:3] = torch.from_numpy(q.reshape(3, -1)).cuda()
    run._attention(0, _lib.VIEW_FP16, 3, 0, _lib.stream_ptr())
    got = run.attn[:3].cpu().numpy()
    for t in range(3):
        m = n - 3 + t + 1
        want = O.merged_attention(q[t], [(k[:m].reshape(m, H, hd), v[:m].reshape(m, H, hd))], 1 / math.sqrt(hd))
        assert np.abs(got[t].reshape(H, hd) - want).max() <= 2e-3 * np.abs(v).max()


def test_chunked_attention_matches_monolithic():
    rng = np.random.default_rng(6)
    q = rng.standard_normal(16).astype(np.float32)
    chunks = [(f16(rng.standard_normal((n, 16))), f16(rng.standard_normal((n, 16)))) for n in (7, 33, 1, 64)]
    got = qs.chunked_attention(q, chunks)
    k = np.concatenate([c[0] for c in chunks])
    v = np.concatenate([c[1] for c in chunks])
    want = O.merged_attention(q.reshape(1, 16), [(k.reshape(-1, 1, 16), v.reshape(-1, 1, 16))], 0.25).ravel()
    assert np.abs(got - want).max() <= 2e-3 * np.abs(v).max()


# ---------------------------------------------------------------------------
# L2: linear layers (K5 W4A16, K6 fp16) vs an f32 torch reference
# ---------------------------------------------------------------------------


def _act_buffers(x):
    """f16 rows + 16-sums of ``x`` through qs_prep_act (the layout qs_linear reads)."""
    n, K = x.shape
    xh = torch.zeros(n, K + 64, dtype=torch.float16, device="cuda")
    xs = torch.zeros(n, (K // 16 + 4 + 3) // 4 * 4, device="cuda")
    _lib.check(_lib.load().qs_prep_act(x.data_ptr(), None, 0.0, xh.data_ptr(), xh.shape[1], xs.data_ptr(),
                                       xs.shape[1], n, K, _lib.stream_ptr()))
    return xh, xs


def _run_linear(pl, x, ncols, *, epi=None, y=None, yh=None, xf=None, gain=None, eps=1e-5):
    xh, xs = _act_buffers(x)
    a = _lib.LinearArgs()
    a.wmode, a.epi, a.N, a.K, a.ncols = pl.wmode, _lib.EPI_STORE if epi is None else epi, pl.N, pl.K, ncols
    a.wgroup = pl.group if pl.wmode == _lib.W_INT4 else 16
    a.w = pl.w.data_ptr()
    a.wparams = pl.params.data_ptr() if pl.params is not None else None
    a.xh, a.ldxh, a.xs, a.ldxs = xh.data_ptr(), xh.shape[1], xs.data_ptr(), xs.shape[1]
    if y is None and yh is None:
        y = torch.zeros(ncols, pl.N, device="cuda")
    if y is not None:
        a.y, a.ldy = y.data_ptr(), y.shape[1]
    if yh is not None:
        a.yh, a.ldyh, a.ys, a.ldys = yh[0].data_ptr(), yh[0].shape[1], yh[1].data_ptr(), yh[1].shape[1]
    if xf is not None:  # INT4 in-kernel activation prep (xh / xs are then not read)
        a.xf, a.ldxf, a.eps = xf.data_ptr(), xf.shape[1], eps
        a.gain = gain.data_ptr() if gain is not None else None
    _lib.check(_lib.load().qs_linear(a, _lib.stream_ptr()))
    torch.cuda.synchronize()
    return y


_LIN_SHAPES = [(64, 48 * 4, 1), (4096, 4096, 1), (176, 64, 5), (4096, 11008 * 2, 9), (11008, 4096, 5),
               (4096, 32000, 16), (1024, 576, 2), (176, 64, 3), (11008, 128, 4), (272, 4096, 1), (4096, 6144, 24),
               (1024, 512, 40), (4096, 4096, 48), (4096, 1024, 33)]


# INT4 weights are draft-only: one row per sequence, at most 16 sequences per launch
@pytest.mark.parametrize("K,N,ncols,mode", [(*s, m) for m in ("f16", "int4") for s in _LIN_SHAPES
                                            if m == "f16" or s[2] <= 16])
def test_linear_vs_torch(K, N, ncols, mode):
    from paper_2502_10424_b200.runtime import PackedLinear

    g = torch.Generator(device="cuda").manual_seed(K + N)
    w = torch.randn(K, N, device="cuda", generator=g) / math.sqrt(K)
    x = torch.randn(ncols, K, device="cuda", generator=g)
    if mode == "f16":
        pl = PackedLinear.f16(w)
        wref = w.half().float()
    else:
        pl = PackedLinear.int4(w, 32)
        q = qs.quantize_weights(w.cpu().numpy(), 32)
        wref = torch.from_numpy(qs.dequantize_weights(q)).cuda()
    y = _run_linear(pl, x, ncols)
    ref = x.half().float() @ wref
    err = (y - ref).abs().max().item()
    assert err <= 2e-3 * ref.abs().max().item() + 1e-4, err


@pytest.mark.parametrize("mode", ["f16", "int4"])
@pytest.mark.parametrize("K,N", [(1024, 576), (272, 48), (4112, 80), (64, 16), (4096, 4112)])
@pytest.mark.parametrize("ncols", [1, 3])
def test_linear_ragged_shapes(mode, K, N, ncols):
    """Odd tile counts (a zero padding tile in the last pair), K ranges ending inside a
    stage, a single tile, more pairs than SMs."""
    from paper_2502_10424_b200.runtime import PackedLinear

    g = torch.Generator(device="cuda").manual_seed(K + N + ncols)
    w = torch.randn(K, N, device="cuda", generator=g) / math.sqrt(K)
    x = torch.randn(ncols, K, device="cuda", generator=g)
    pl = PackedLinear.f16(w) if mode == "f16" else PackedLinear.int4(w, 16)
    wref = w.half().float() if mode == "f16" else torch.from_numpy(
        qs.dequantize_weights(qs.quantize_weights(w.cpu().numpy(), 16))).cuda()
    y = _run_linear(pl, x, ncols)
    ref = x.half().float() @ wref
    assert (y - ref).abs().max().item() <= 2e-3 * ref.abs().max().item() + 1e-4


@pytest.mark.parametrize("K,N,epi", [(4096, 4096, 0), (4096, 22016, 0), (128, 4112, 0), (4096, 4096, 1)])
@pytest.mark.parametrize("with_gain", [False, True])
@pytest.mark.parametrize("mode", ["int4", "f16"])
def test_in_kernel_prep_matches_prep_act(K, N, epi, with_gain, mode):
    """A linear kernel building its f16 input (+ RMS norm) from an f32 row is bit-identical
    to qs_prep_act + the same kernel reading xh / xs: both run the same device function
    (act_prep_row), which keeps the f16 target's single-row steps equal to a verify."""
    from paper_2502_10424_b200.runtime import PackedLinear

    g = torch.Generator(device="cuda").manual_seed(K + N)
    w = torch.randn(K, N, device="cuda", generator=g) / math.sqrt(K)
    x = torch.randn(1, K, device="cuda", generator=g) * 3.0
    gain = (torch.rand(K, device="cuda", generator=g) + 0.5) if with_gain else None
    pl = PackedLinear.int4(w, 32) if mode == "int4" else PackedLinear.f16(w)
    # reference: qs_prep_act (rmsnorm when gain) -> f16 + 16-sums -> the kernel
    xh = torch.zeros(1, K + 64, dtype=torch.float16, device="cuda")
    xs = torch.zeros(1, (K // 16 + 4 + 3) // 4 * 4, device="cuda")
    _lib.check(_lib.load().qs_prep_act(x.data_ptr(), gain.data_ptr() if gain is not None else None, 1e-5,
                                       xh.data_ptr(), xh.shape[1], xs.data_ptr(), xs.shape[1], 1, K,
                                       _lib.stream_ptr()))
    base = torch.randn(1, N, device="cuda", generator=g)
    y0, y1 = base.clone(), base.clone()
    want = _run_linear(pl, xh[:, :K].float(), 1, epi=epi, y=y0)  # the (normed) f16 rows as input
    got = _run_linear(pl, x, 1, epi=epi, y=y1, xf=x, gain=gain)
    assert torch.equal(got, want)


@pytest.mark.parametrize("mode", ["f16", "int4"])
def test_linear_batch_invariant(mode):
    """f16 (target) weights: column c of a 9-column launch is bit-identical to a
    1-column launch of the same row (what makes a (gamma+1)-row verify equal
    gamma+1 AR steps).  INT4 (draft-only) weights pack weight groups into the
    free MMA columns when few rows are active, so there the check is numeric."""
    from paper_2502_10424_b200.runtime import PackedLinear

    K, N = 4096, 4096
    g = torch.Generator(device="cuda").manual_seed(3)
    w = torch.randn(K, N, device="cuda", generator=g) / math.sqrt(K)
    big = 40 if mode == "f16" else 9  # f16: up to the 8-sequence x 5-row verify of config 4
    x = torch.randn(big, K, device="cuda", generator=g)
    pl = PackedLinear.f16(w) if mode == "f16" else PackedLinear.int4(w, 64)
    yb = _run_linear(pl, x, big)
    for c in (0, 4, 8, big - 1):
        for n in (1, 2, 3, 6, 17):
            n = min(n, big - c)
            yn = _run_linear(pl, x[c:c + n].contiguous(), n)
            if mode == "f16":
                assert torch.equal(yn[0], yb[c])
            else:
                assert (yn[0] - yb[c]).abs().max().item() <= 1e-4 * yb[c].abs().max().item()


@pytest.mark.parametrize("mode", ["f16", "int4"])
def test_linear_silu_epilogue(mode):
    """Fused gate/up -> SiLU(gate)*up -> f16 + 16-sums (the down projection's input)."""
    from paper_2502_10424_b200.runtime import PackedLinear

    K, M, ncols = 256, 352, 5
    g = torch.Generator(device="cuda").manual_seed(11)
    wg = torch.randn(K, M, device="cuda", generator=g) / math.sqrt(K)
    wu = torch.randn(K, M, device="cuda", generator=g) / math.sqrt(K)
    x = torch.randn(ncols, K, device="cuda", generator=g)
    if mode == "f16":
        pl = PackedLinear.f16_pair(wg, wu)
        rg, ru = wg.half().float(), wu.half().float()
    else:
        pl = PackedLinear.int4_pair(wg, wu, 64)
        rg, ru = (torch.from_numpy(qs.dequantize_weights(qs.quantize_weights(m.cpu().numpy(), 64))).cuda()
                  for m in (wg, wu))
    hh = torch.zeros(ncols, M + 64, dtype=torch.float16, device="cuda")
    hs = torch.zeros(ncols, M // 16 + 8, device="cuda")
    y = torch.zeros(ncols, M, device="cuda")
    _run_linear(pl, x, ncols, epi=_lib.EPI_SILU_MUL, y=y, yh=(hh, hs))
    xf = x.half().float()
    a, b = xf @ rg, xf @ ru
    ref = a / (1 + torch.exp(-a)) * b
    assert (y - ref).abs().max().item() <= 3e-3 * ref.abs().max().item() + 1e-4
    assert torch.equal(hh[:, :M], y.half())
    sums = hh[:, :M].float().view(ncols, M // 16, 16).sum(-1)
    assert torch.allclose(hs[:, :M // 16], sums, rtol=1e-5, atol=1e-4)


def test_prep_act_rmsnorm():
    d, n = 4096, 3
    x = torch.randn(n, d, device="cuda")
    gain = torch.rand(d, device="cuda") + 0.5
    xh = torch.zeros(n, d + 64, dtype=torch.float16, device="cuda")
    xs = torch.zeros(n, d // 16 + 4, device="cuda")
    _lib.check(_lib.load().qs_prep_act(x.data_ptr(), gain.data_ptr(), 1e-5, xh.data_ptr(), xh.shape[1],
                                       xs.data_ptr(), xs.shape[1], n, d, _lib.stream_ptr()))
    ref = (x / torch.sqrt((x * x).mean(-1, keepdim=True) + 1e-5) * gain)
    assert (xh[:, :d].float() - ref).abs().max().item() <= 2e-3 * ref.abs().max().item()
    assert torch.allclose(xs[:, :d // 16], xh[:, :d].float().view(n, -1, 16).sum(-1), rtol=1e-5, atol=1e-4)


# ---------------------------------------------------------------------------
# L2/L3: model forward, accept rule, greedy losslessness
# ---------------------------------------------------------------------------

TOY = qs.ModelConfig(num_layers=2, num_heads=4, head_dim=16, hidden=64, mlp_hidden=176, vocab=64, max_positions=4096 + 256)
OTOY = O.Config(2, 4, 16, 64, 176, 64, 4096 + 256)


@pytest.fixture(scope="module")
def toy():
    return qs.init_weights(TOY, seed=7), O.init_weights(OTOY, seed=7)


def _oracle_cache_like(dev_cache):
    """Oracle cache holding exactly the device cache's contents (fp16 values; sensitive
    layers' archived fp16 rows)."""
    lay = dev_cache.layout
    olay = O.Layout(lay.num_layers, lay.kv_heads, lay.head_dim, lay.group_size, frozenset(lay.sensitive_layers))
    oc = O.OracleKVCache(olay)
    G = lay.group_size
    nb = dev_cache.quantized_token_count // G
    for layer in range(lay.num_layers):
        if layer in lay.sensitive_layers:
            slot = sorted(lay.sensitive_layers).index(layer)
            for b in range(nb):
                rows = slice(b * G, (b + 1) * G)
                k = dev_cache.arch_k[0, slot, :, rows].permute(1, 0, 2).reshape(G, lay.kv_dim).float().cpu().numpy()
                v = dev_cache.arch_v[0, slot, :, rows].permute(1, 0, 2).reshape(G, lay.kv_dim).float().cpu().numpy()
                oc.archived[layer].append((k, v))
        for b in range(nb if layer not in lay.sensitive_layers else 0):
            ku, kl, vu, vl = dev_cache.export_block_planes(layer, b)
            oc.blocks[layer].append(O.Block(*(O.Plane(p.codes, p.count, p.group_size, p.scales, p.zeros, p.mode, p.axis, p.row_len) for p in (ku, kl, vu, vl))))
        for which, n in ((0, dev_cache.fp1_len), (1, dev_cache.fp2_len)):
            if n:
                k, v = dev_cache._fp_rows(which, layer, n)
                buf = oc.fp1 if which == 0 else oc.fp2
                buf[layer, 0, :n] = k
                buf[layer, 1, :n] = v
    oc.fp1_len = dev_cache.fp1_len
    oc.fp2_lens[:] = dev_cache.fp2_len
    oc.quantized_token_count = dev_cache.quantized_token_count
    return oc


def test_weights_bit_exact_with_oracle(toy):
    w, ow = toy
    assert np.array_equal(w.embedding, ow["embedding"]) and np.array_equal(w.lm_head, ow["lm_head"])
    for lw, olw in zip(w.layers, ow["layers"]):
        for n in O.MATS:
            assert np.array_equal(getattr(lw, n), olw[n])


@pytest.mark.parametrize("view", ["draft", "target"])
def test_decode_step_logits_vs_oracle(toy, view):
    """Same cache contents, same token: logits agree to fp16-weight tolerance."""
    w, ow = toy
    prompt = np.random.default_rng(31).integers(0, 64, size=300)
    _, cache = qs.prefill(w, prompt, "hierarchical", group_size=16)
    oc = _oracle_cache_like(cache)
    # oracle uses the fp16-rounded weights the device holds
    ow16 = copy.deepcopy(ow)
    for olw in ow16["layers"]:
        for n in O.MATS:
            olw[n] = f16(olw[n])
    ow16["lm_head"] = f16(ow16["lm_head"])
    lg, cost = qs.decode_step(w, 11, cache, view=view)
    olg, ocost = O.decode_step(ow16, 11, oc, view)
    scale = max(1.0, float(np.abs(olg).max()))
    assert np.abs(lg - olg).max() <= 2e-2 * scale, np.abs(lg - olg).max()
    assert [cost.flops, cost.weight_bytes, cost.kv_quantized_bytes, cost.kv_param_bytes, cost.kv_fp_bytes,
            cost.kv_quantized_elements] == [ocost.flops, ocost.weight_bytes, ocost.kv_quantized_bytes,
                                            ocost.kv_param_bytes, ocost.kv_fp_bytes, ocost.kv_quantized_elements]


def _f16_weights(ow):
    ow16 = copy.deepcopy(ow)
    for olw in ow16["layers"]:
        for n in O.MATS:
            olw[n] = f16(olw[n])
    ow16["lm_head"] = f16(ow16["lm_head"])
    return ow16


def test_int4_decode_step_vs_oracle(toy):
    """INT4-weight draft forward (W4A16 GEMV, f16 activations) vs O.decode_step(..., "int4") with
    the oracle's dequantised INT4 weights (Q/model.py:141-168) on the same cache contents; the
    codes and (S, Z) are bit-exact on both sides, so the bar is the f16-activation tolerance:
    max |err| <= 1e-2 * max |logit|."""
    w, ow = toy
    prompt = np.random.default_rng(33).integers(0, 64, size=300)
    _, cache = qs.prefill(w, prompt, "hierarchical", group_size=16)
    oc = _oracle_cache_like(cache)
    q = qs.quantize_model_weights(w, 32)
    draft = O.quantize_model(ow, 32)
    for tok in (11, 40):
        lg, cost = qs.decode_step(w, tok, cache, view="draft", weight_mode="int4", draft_weights=q)
        olg, ocost = O.decode_step(ow, tok, oc, "draft", "int4", draft)
        scale = max(1.0, float(np.abs(olg).max()))
        assert np.abs(lg - olg).max() <= 1e-2 * scale, np.abs(lg - olg).max()
        assert cost.weight_bytes == ocost.weight_bytes == draft["int4_weight_bytes"]


@pytest.mark.parametrize("view", ["draft", "target"])
def test_sensitive_layer_decode_vs_oracle(toy, view):
    """Sensitive layers (Q/cache.py:286-289, :351-356) keep fp history: the device archives fp16
    rows and routes the layer to the fp16 attention kernel (K4) over the archive + fp1/fp2; the
    other layer reads the planes.  Logits vs the oracle on identical contents (2e-2 bar as above)."""
    w, ow = toy
    prompt = np.random.default_rng(34).integers(0, 64, size=150)
    _, cache = qs.prefill(w, prompt, "hierarchical", group_size=16, sensitive_layers=frozenset({0}))
    assert cache.quantized_token_count > 0
    oc = _oracle_cache_like(cache)
    ow16 = _f16_weights(ow)
    for tok in (3, 17, 60):
        lg, cost = qs.decode_step(w, tok, cache, view=view)
        olg, ocost = O.decode_step(ow16, tok, oc, view)
        scale = max(1.0, float(np.abs(olg).max()))
        assert np.abs(lg - olg).max() <= 2e-2 * scale, np.abs(lg - olg).max()
        assert cost.kv_fp_bytes == ocost.kv_fp_bytes and cost.kv_quantized_bytes == ocost.kv_quantized_bytes
        cache.flush_if_full()
        oc.flush_if_full()


@pytest.mark.parametrize("V", [32000, 32003, 128256])
def test_argmax_first_max_wide_rows(V):
    """qs_argmax == np.argmax (first maximum; first NaN) on vocabulary-sized rows: the
    16-byte-load path (V % 4 == 0) and its scalar tail (V % 4 != 0), planted exact ties."""
    rng = np.random.default_rng(V)
    rows = rng.standard_normal((6, V)).astype(np.float32)
    rows[1, [7, 9000, V - 1]] = rows[1].max() + 1.0            # tie across the row -> 7
    rows[2, [V - 2, V - 1]] = rows[2].max() + 1.0              # tie in the tail
    rows[3, 4 * (V // 8) + 3] = rows[3].max() + 2.0            # max on a float4 lane 3
    rows[4, [11, 5000]] = np.nan                               # np.argmax returns the first NaN
    rows[5, :] = 0.0                                           # all equal -> 0
    lg = torch.from_numpy(rows).cuda()
    am = torch.zeros(6, dtype=torch.int32, device="cuda")
    _lib.check(_lib.load().qs_argmax(lg.data_ptr(), 6, V, am.data_ptr(), 1, _lib.stream_ptr()))
    assert am.cpu().tolist() == np.argmax(rows, axis=1).tolist()


def test_greedy_accept_kernel_matches_oracle_rule():
    """Batched accept kernel vs the reference rule (Q/specdec.py:276-298), one ragged batch of B
    sequences per trial: each sequence has its own gamma_step (padding rows past it ignored)."""
    rng = np.random.default_rng(9)
    dev = torch.device("cuda")
    for trial in range(100):
        B = int(rng.integers(1, 6))
        T = int(rng.integers(1, 10))
        gs = rng.integers(0, T, size=B)
        V = 37
        logits = rng.standard_normal((B, T, V)).astype(np.float32)
        if trial % 3 == 0:
            logits[:, :, 5] = logits.max(axis=2) + 0.0  # exact ties -> lowest index wins
        tgt = logits.argmax(axis=2)
        TS = T + 1
        toks = np.zeros((B, TS), np.int32)
        want = []
        for b in range(B):
            drafts = [int(tgt[b, i]) if rng.random() < 0.7 else int(rng.integers(0, V)) for i in range(T - 1)]
            toks[b, 1:T] = drafts
            want.append(O.greedy_accept(drafts[: gs[b]], list(logits[b, : gs[b] + 1])))
        lg = torch.from_numpy(logits.reshape(B * T, V)).to(dev)
        am = torch.zeros(B * T, dtype=torch.int32, device=dev)
        _lib.check(_lib.load().qs_argmax(lg.data_ptr(), B * T, V, am.data_ptr(), 1, _lib.stream_ptr()))
        dtok = torch.from_numpy(toks).to(dev)
        dgs = torch.from_numpy(gs.astype(np.int32)).to(dev)
        res = torch.zeros(2 * B, dtype=torch.int32, device=dev)
        f2 = torch.full((B,), 3, dtype=torch.int32, device=dev)
        _lib.check(_lib.load().qs_greedy_accept(dtok.data_ptr(), TS, am.data_ptr(), T, dgs.data_ptr(), B,
                                                res.data_ptr(), f2.data_ptr(), None, _lib.stream_ptr()))
        r = res.cpu().numpy().reshape(B, 2)
        assert am.cpu().numpy().reshape(B, T).tolist() == tgt.tolist()
        for b, (v, corr, bonus) in enumerate(want):
            assert r[b, 0] == v and r[b, 1] == (corr if corr is not None else bonus), (trial, b)
            assert int(f2[b]) == 3 + v + 1 and int(dtok[b, 0]) == r[b, 1]


@pytest.mark.parametrize("gamma", [1, 2, 4, 6])
def test_greedy_spec_equals_gpu_target_ar(toy, gamma):
    """Internal exactness: spec decode == target-view AR on the same kernels (token for token)."""
    w, _ = toy
    for seed in (2, 5):
        prompt = np.random.default_rng(seed).integers(0, 64, size=80)
        res = qs.SpeculativeDecoder(w, qs.SpecConfig(gamma=gamma, decode_len=60), group_size=16).run(prompt)
        ar = qs.autoregressive_decode(w, prompt, 60, group_size=16)
        assert res.tokens == ar
        assert len(res.tokens) == 60


def test_int4_draft_still_lossless_and_fp2_edge(toy):
    w, _ = toy
    prompt = np.random.default_rng(3).integers(0, 64, size=80)
    res = qs.SpeculativeDecoder(w, qs.SpecConfig(gamma=4, decode_len=60, weight_mode="int4"), group_size=16).run(prompt)
    assert res.tokens == qs.autoregressive_decode(w, prompt, 60, group_size=16)
    prompt = np.random.default_rng(4).integers(0, 64, size=3 * 16 - 1)
    res = qs.SpeculativeDecoder(w, qs.SpecConfig(gamma=6, decode_len=60), group_size=16).run(prompt)
    assert res.tokens == qs.autoregressive_decode(w, prompt, 60, group_size=16)
    assert any(len(s.drafted) < 6 for s in res.trace.steps)


def test_lossless_config_accepts_everything(toy):
    w, _ = toy
    prompt = np.random.default_rng(1).integers(0, 64, size=40)
    res = qs.SpeculativeDecoder(w, qs.SpecConfig(gamma=4, decode_len=40), kv_quant=False).run(prompt)
    assert res.metrics.acceptance_rate == 1.0
    assert res.tokens == qs.autoregressive_decode(w, prompt, 40, kv_quant=False)


def test_graph_replay_equals_eager(toy):
    w, _ = toy
    prompt = np.random.default_rng(8).integers(0, 64, size=120)
    a = qs.SpeculativeDecoder(w, qs.SpecConfig(gamma=4, decode_len=50), group_size=16, use_graphs=True).run(prompt)
    b = qs.SpeculativeDecoder(w, qs.SpecConfig(gamma=4, decode_len=50), group_size=16, use_graphs=False).run(prompt)
    assert a.tokens == b.tokens
    assert a.trace.to_ndjson() == b.trace.to_ndjson()


def test_trace_matches_reference_structure(toy):
    """Emission budget, trace reconciliation and buffer invariants (pkg/tests/test_specdec.py:136-216)."""
    w, _ = toy
    for decode_len in (1, 2, 7, 77):
        prompt = np.random.default_rng(10).integers(0, 64, size=80)
        res = qs.SpeculativeDecoder(w, qs.SpecConfig(gamma=4, decode_len=decode_len), group_size=16).run(prompt)
        assert len(res.tokens) == decode_len
        rebuilt = [res.tokens[0]]
        for s in res.trace.steps:
            rebuilt.extend(s.emitted)
        assert rebuilt == res.tokens
        for line in res.trace.to_ndjson().strip().splitlines() if res.trace.steps else []:
            rec = json.loads(line)
            assert set(rec) == {"step", "drafted", "accepted", "corrected", "bonus", "flushed", "draft_bytes", "target_bytes"}


def test_reference_written_qskv_round_trips_through_the_device_store(tmp_path):
    """A QSKV file written by the REFERENCE (tests/golden/make_qskv_golden.py: prefill, decode appends,
    a full-fp1 flush, a sensitive layer) loads into the device store with the reference's views, and
    the device writes it back byte for byte (Q/cache.py:405-553)."""
    src = os.path.join(GOLDEN, "ref_cache.qskv")
    z = np.load(os.path.join(GOLDEN, "ref_cache_views.npz"))
    c = qs.HierarchicalKVCache.load_snapshot(src)
    assert c.seq_len == int(z["seq_len"]) and c.quantized_token_count == int(z["quantized"])
    for layer in range(2):
        for kind in ("draft", "target"):
            view = c.draft_view(layer) if kind == "draft" else c.target_view(layer)
            k, v = view.concat()
            assert np.array_equal(k, z[f"{kind}_k{layer}"]) and np.array_equal(v, z[f"{kind}_v{layer}"]), (layer, kind)
    out = tmp_path / "dev.qskv"
    c.save_snapshot(out)
    with open(src, "rb") as f:
        assert out.read_bytes() == f.read()


def test_stochastic_decode_on_device_logits(toy):
    """Stochastic verification end to end (host decisions, Q/specdec.py:148-170, over device logits):
    the lossless configuration (fp cache, fp draft: p == q bit for bit) accepts every draft, and the
    hierarchical one keeps the emission budget with a valid trace; a fixed seed reproduces the run."""
    w, _ = toy
    prompt = np.random.default_rng(6).integers(0, 64, size=150)
    spec = qs.SpecConfig(gamma=4, decode_len=40, sampling="stochastic", temperature=0.8, seed=3)
    res = qs.SpeculativeDecoder(w, spec, kv_quant=False).run(prompt)
    assert res.metrics.acceptance_rate == 1.0 and len(res.tokens) == 40
    sd = qs.SpeculativeDecoder(w, spec, group_size=16)
    a, b = sd.run(prompt), qs.SpeculativeDecoder(w, spec, group_size=16).run(prompt)
    assert len(a.tokens) == 40 and all(0 <= t < 64 for t in a.tokens)
    assert 0.0 < a.metrics.acceptance_rate <= 1.0
    assert a.tokens == b.tokens
    assert len(a.trace.to_ndjson().splitlines()) == len(a.trace.steps)


def test_cli_run_and_ablate_measure_on_device(tmp_path):
    """The harness (cli.py, Q/cli.py:233-284) runs on the device and reports measured tok/s; greedy
    kv_quant tokens equal target-view AR tokens (losslessness through the CLI path too)."""
    from paper_2502_10424_b200 import cli

    assert cli.main(["run", "--out", str(tmp_path / "r"), "--decode-len", "40", "--gamma", "4"]) == 0
    hdr, row = (tmp_path / "r" / "metrics.csv").read_text().strip().split("\n")
    m = dict(zip(hdr.split(","), row.split(",")))
    assert float(m["measured_tok_s"]) > 0 and float(m["measured_ar_tok_s"]) > 0
    assert int(m["emitted_tokens"]) == 40
    toks = [int(t) for t in (tmp_path / "r" / "tokens.txt").read_text().split()]
    cfg = cli.resolve_config(cli.build_parser().parse_args(["run"]))
    w = cli._weights(cfg)
    assert toks == qs.autoregressive_decode(w, cli._prompt(cfg, w.config.vocab), 40, group_size=128)
    assert cli.main(["ablate", "--out", str(tmp_path / "a"), "--decode-len", "20"]) == 0
    lines = (tmp_path / "a" / "ablate.csv").read_text().strip().split("\n")
    assert [l.split(",")[0] for l in lines[1:]] == ["neither", "kv_only", "weight_only", "both"]


@pytest.mark.parametrize("mode", ["draft", "target", "int4"])
def test_gqa_forward_vs_oracle(mode):
    """GQA model path (configs 4/5: the oracle repeats each KV head r times into the
    reference's merged attention): bit-exact weights, prefill logits, and the draft / target /
    INT4-weight decode logits on the same cache contents, at the fp16-weight tolerance."""
    cfg = qs.ModelConfig(num_layers=2, num_heads=8, head_dim=16, hidden=128, mlp_hidden=176, vocab=96,
                         max_positions=1024, num_kv_heads=2)
    ocfg = O.Config(2, 8, 16, 128, 176, 96, 1024, num_kv_heads=2)
    w, ow = qs.init_weights(cfg, seed=13), O.init_weights(ocfg, seed=13)
    assert np.array_equal(w.layers[1].wk, ow["layers"][1]["wk"]) and w.layers[1].wk.shape == (128, 32)
    prompt = np.random.default_rng(5).integers(0, 96, size=230)
    lg0, cache = qs.prefill(w, prompt, "hierarchical", group_size=16)
    olg0, _ = O.prefill(ow, prompt, "hierarchical", 16)
    assert np.abs(lg0 - olg0).max() <= 2e-3 * max(1.0, float(np.abs(olg0).max()))
    oc = _oracle_cache_like(cache)
    ow16 = _f16_weights(ow)
    if mode == "int4":
        q = qs.quantize_model_weights(w, 32)
        lg, _ = qs.decode_step(w, 17, cache, view="draft", weight_mode="int4", draft_weights=q)
        olg, _ = O.decode_step(ow, 17, oc, "draft", "int4", O.quantize_model(ow, 32))
        tol = 2e-3
    else:
        lg, _ = qs.decode_step(w, 17, cache, view=mode)
        olg, _ = O.decode_step(ow16, 17, oc, mode)
        tol = 2e-2
    scale = max(1.0, float(np.abs(olg).max()))
    assert np.abs(lg - olg).max() <= tol * scale, (mode, float(np.abs(lg - olg).max()))


def test_decode_time_flush_of_non_finite_kv_raises(toy):
    """A non-finite K/V row reaching the decode-time flush (K1 inside the captured step) sets the
    device status word; the per-step readback raises the reference's DataError (Q/quant.py:60-64,
    reached from Q/cache.py:261-262) -- one step later than the reference, which raises before mutating."""
    from paper_2502_10424_b200.engine import ARAutoEngine

    w, _ = toy
    prompt = np.random.default_rng(12).integers(0, 64, size=63)  # 32 quantised + fp1 16 + fp2 15 (G = 16)
    _, cache = qs.prefill(w, prompt, "hierarchical", group_size=16)
    assert (cache.fp1_len, cache.fp2_len) == (16, 15)
    cache.fp_k[0, 1, 0, 0, 3, 5] = float("nan")  # layer 1, fp1, head 0, row 3
    fw, _ = w.device()
    eng = ARAutoEngine(fw, cache, use_graphs=False)
    eng.set_pending([7])
    with pytest.raises(qs.DataError):
        eng.step()  # fp2 fills -> the flush quantises fp1 (with the NaN) -> status word -> DataError
