"""CPU oracle for the QuantSpec decode hot path -- TEST INFRASTRUCTURE ONLY.

This module is a from-scratch NumPy restatement of the reference algorithm
(arXiv 2502.10424, package ``quantspec`` under ``/root/reference/pkg/src``).
It exists so that the B200 product path can be checked against the reference
semantics on the GPU box, where ``/root/reference`` does not exist.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import it, and only as the checker / the timed
CPU baseline.  The product package (``paper_2502_10424_b200``) never imports
it: there is no CPU fallback.

Parity is pinned: ``tests/test_oracle_golden.py`` checks every function here
against golden vectors produced by the *reference itself*
(``tests/golden/make_golden.py`` imports ``/root/reference/pkg/src``).

Every function cites the reference ``file:line`` whose arithmetic it restates
(``Q/`` = ``pkg/src/quantspec/``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

F32 = np.float32
F64 = np.float64

# reference constants: Q/quant.py:24-31, Q/cache.py:34-36, Q/model.py:31-32
SCALE_FLOOR = 1e-8
ASYM_MAX = 15
SYM_LO, SYM_HI = -8, 7
LOWER_DIV = 16.0
CODE_BYTES = 0.5
PARAM_PAIR_BYTES = 8.0
FP_ELEM_BYTES = 4.0
DRAFT_CODE_BYTES = 0.5
TARGET_CODE_BYTES = 1.0
F32_BYTES = 4.0


class OracleError(Exception):
    """Raised where the reference raises one of its typed errors."""


# ---------------------------------------------------------------------------
# L0 quantisation (Q/quant.py)
# ---------------------------------------------------------------------------


def round_half_away(x: np.ndarray) -> np.ndarray:
    """RTN with ties away from zero: Q/quant.py:55-57 (x + copysign(.5) then trunc)."""
    return np.trunc(x + np.copysign(0.5, x))


def group_starts(count: int, group: int, row_len: int | None) -> np.ndarray:
    """Start offsets of the quantisation groups, Q/quant.py:210-217."""
    if row_len is None or row_len >= count:
        return np.arange(0, count, group, dtype=np.int64)
    if count % row_len:
        raise OracleError("count is not a whole number of rows")
    inner = np.arange(0, row_len, group, dtype=np.int64)
    return (np.arange(0, count, row_len, dtype=np.int64)[:, None] + inner[None, :]).reshape(-1)


def group_lengths(count: int, starts: np.ndarray) -> np.ndarray:
    return np.diff(np.concatenate([starts, [count]]))


def asym_params(mins_f64: np.ndarray, maxs_f64: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """(S, Z) per group, Q/quant.py:234-235: Z=f32(min); S=f32(max((max-Z)/15, 1e-8))."""
    z = mins_f64.astype(F32)
    s = np.maximum((maxs_f64 - z.astype(F64)) / ASYM_MAX, SCALE_FLOOR).astype(F32)
    return s, z


def encode_upper(v: np.ndarray, s: np.ndarray, z: np.ndarray, lens: np.ndarray) -> np.ndarray:
    """Upper codes clip(rha((v-Z)/S), 0, 15) in f64, Q/quant.py:236-238."""
    se = np.repeat(s.astype(F64), lens)
    ze = np.repeat(z.astype(F64), lens)
    return np.clip(round_half_away((v - ze) / se), 0, ASYM_MAX).astype(np.int64)


def encode_lower(v: np.ndarray, cu: np.ndarray, s: np.ndarray, z: np.ndarray, lens: np.ndarray):
    """Lower plane on the upper residual at step S/16, Q/quant.py:257-265.

    Returns (codes int64 in [-8,7], lower scales f32 = S/16 exactly).
    """
    se = np.repeat(s.astype(F64), lens)
    ze = np.repeat(z.astype(F64), lens)
    resid = v - (cu.astype(F64) * se + ze)
    ls = (s / F32(LOWER_DIV)).astype(F32)
    lse = np.repeat(ls.astype(F64), lens)
    return np.clip(round_half_away(resid / lse), SYM_LO, SYM_HI).astype(np.int64), ls


def pack4(codes: np.ndarray) -> np.ndarray:
    """Two 4-bit codes per byte, even index in the low nibble, Q/quant.py:137-145."""
    c = (np.asarray(codes).astype(np.int64) & 0xF).reshape(-1)
    if c.size & 1:
        c = np.concatenate([c, [0]])
    return (c[0::2] | (c[1::2] << 4)).astype(np.uint8)


def unpack4(packed: np.ndarray, count: int, signed: bool) -> np.ndarray:
    """Inverse of pack4, Q/quant.py:148-158."""
    p = np.asarray(packed, dtype=np.uint8).reshape(-1).astype(np.int16)
    out = np.stack([p & 0xF, p >> 4], axis=1).reshape(-1)[:count]
    if signed:
        return np.where(out >= 8, out - 16, out).astype(np.int8)
    return out.astype(np.uint8)


@dataclass
class Plane:
    """Field-for-field twin of the reference QuantPlane (Q/quant.py:166-207)."""

    codes: np.ndarray
    count: int
    group_size: int
    scales: np.ndarray
    zeros: np.ndarray
    mode: str
    axis: str
    row_len: int | None = None

    def lens(self) -> np.ndarray:
        return group_lengths(self.count, group_starts(self.count, self.group_size, self.row_len))

    def unpacked(self) -> np.ndarray:
        return unpack4(self.codes, self.count, self.mode == "symmetric_s4")


def encode_plane_hier(values, group: int, axis: str, row_len: int | None = None) -> tuple[Plane, Plane]:
    """Q/quant.py:220-276 (encode_plane_asym + encode_plane_hierarchical)."""
    v = np.asarray(values, dtype=F64).reshape(-1)
    if v.size == 0 or not np.all(np.isfinite(v)):
        raise OracleError("empty or non-finite plane")
    if group < 1:
        raise OracleError("group size must be >= 1")
    st = group_starts(v.size, group, row_len)
    lens = group_lengths(v.size, st)
    s, z = asym_params(np.minimum.reduceat(v, st), np.maximum.reduceat(v, st))
    cu = encode_upper(v, s, z, lens)
    cl, ls = encode_lower(v, cu, s, z, lens)
    up = Plane(pack4(cu), v.size, group, s, z, "asymmetric_u4", axis, row_len)
    lo = Plane(pack4(cl), v.size, group, ls, np.zeros_like(ls), "symmetric_s4", axis, row_len)
    return up, lo


def decode_draft(p: Plane) -> np.ndarray:
    """c_u*S + Z in f64, Q/quant.py:293-298."""
    lens = p.lens()
    return p.unpacked().astype(F64) * np.repeat(p.scales.astype(F64), lens) + np.repeat(
        p.zeros.astype(F64), lens
    )


def decode_target(u: Plane, l: Plane) -> np.ndarray:
    """c_u*S + c_l*(S/16) + Z in f64 (left-to-right), Q/quant.py:301-309."""
    lens = u.lens()
    se = np.repeat(u.scales.astype(F64), lens)
    ze = np.repeat(u.zeros.astype(F64), lens)
    return u.unpacked().astype(F64) * se + l.unpacked().astype(F64) * (se / LOWER_DIV) + ze


def group_encode(values):
    """Single-group hierarchical encode, Q/quant.py:67-104.

    Returns ((cu uint8, S, Z), (cl int8, S_l)).
    """
    v = np.asarray(values, dtype=F64).reshape(-1)
    if v.size == 0 or not np.all(np.isfinite(v)):
        raise OracleError("empty or non-finite group")
    z = float(F32(v.min()))
    s = float(F32(max((float(v.max()) - z) / ASYM_MAX, SCALE_FLOOR)))
    cu = np.clip(round_half_away((v - z) / s), 0, ASYM_MAX).astype(np.uint8)
    resid = v - (cu.astype(F64) * s + z)
    sl = float(F32(s / LOWER_DIV))
    cl = np.clip(round_half_away(resid / sl), SYM_LO, SYM_HI).astype(np.int8)
    return (cu, s, z), (cl, sl)


def quantize_matrix(w: np.ndarray, group: int) -> Plane:
    """INT4 weights, groups along d_in of W^T rows, Q/quant.py:335-349."""
    w = np.asarray(w, dtype=F32)
    d_in, _ = w.shape
    flat = np.ascontiguousarray(w.T).reshape(-1).astype(F64)
    g = min(group, d_in)
    st = group_starts(flat.size, g, d_in)
    lens = group_lengths(flat.size, st)
    s, z = asym_params(np.minimum.reduceat(flat, st), np.maximum.reduceat(flat, st))
    cu = encode_upper(flat, s, z, lens)
    return Plane(pack4(cu), flat.size, g, s, z, "asymmetric_u4", "channel", d_in)


def dequantize_matrix(p: Plane, shape: tuple[int, int]) -> np.ndarray:
    """f32 [d_in, d_out] reconstruction, Q/quant.py:352-356."""
    d_in, d_out = shape
    return np.ascontiguousarray(decode_draft(p).reshape(d_out, d_in).T.astype(F32))


# ---------------------------------------------------------------------------
# L1 hierarchical KV cache (Q/cache.py)
# ---------------------------------------------------------------------------


@dataclass
class Layout:
    """Q/cache.py:42-63 (kv_dim = heads * head_dim)."""

    num_layers: int
    num_heads: int
    head_dim: int
    group_size: int
    sensitive_layers: frozenset = frozenset()

    @property
    def kv_dim(self) -> int:
        return self.num_heads * self.head_dim


@dataclass
class Block:
    """One flushed block of one layer: the K/V plane quartet (Q/cache.py:107-116)."""

    ku: Plane
    kl: Plane
    vu: Plane
    vl: Plane


@dataclass
class View:
    """Q/cache.py:66-83 plus the byte fields filled by Q/cache.py:345-378."""

    k: np.ndarray
    v: np.ndarray
    quantized_bytes: float = 0.0
    param_bytes: float = 0.0
    fp_bytes: float = 0.0
    quantized_elements: int = 0
    segments: list = field(default_factory=list)


def quantize_kv_block(layout: Layout, k_block: np.ndarray, v_block: np.ndarray) -> Block:
    """Q/cache.py:283-301: keys channel-major (one group per channel), values
    token-major with groups confined to a token (row_len = kv_dim)."""
    ku, kl = encode_plane_hier(np.ascontiguousarray(np.asarray(k_block, F32).T).reshape(-1), layout.group_size, "channel")
    vu, vl = encode_plane_hier(np.asarray(v_block, F32).reshape(-1), layout.group_size, "token", layout.kv_dim)
    return Block(ku, kl, vu, vl)


def dequant_kv_block(layout: Layout, b: Block, kind: str) -> tuple[np.ndarray, np.ndarray]:
    """Q/cache.py:317-329: f64 reconstruction cast to f32, keys transposed back."""
    g, kv = layout.group_size, layout.kv_dim
    if kind == "draft":
        kf, vf = decode_draft(b.ku), decode_draft(b.vu)
    else:
        kf, vf = decode_target(b.ku, b.kl), decode_target(b.vu, b.vl)
    return np.ascontiguousarray(kf.reshape(kv, g).T).astype(F32), vf.reshape(g, kv).astype(F32)


class OracleKVCache:
    """State machine of HierarchicalKVCache, Q/cache.py:119-403."""

    def __init__(self, layout: Layout):
        self.layout = layout
        g, kv, n = layout.group_size, layout.kv_dim, layout.num_layers
        self.blocks: list[list[Block]] = [[] for _ in range(n)]
        self.archived: list[list[tuple[np.ndarray, np.ndarray]]] = [[] for _ in range(n)]
        self.fp1 = np.zeros((n, 2, g, kv), F32)  # [layer, k|v, token, channel]
        self.fp2 = np.zeros((n, 2, g, kv), F32)
        self.fp1_len = 0
        self.fp2_lens = np.zeros(n, np.int64)
        self.quantized_token_count = 0

    # Q/cache.py:139-182
    @classmethod
    def from_prefill(cls, layout: Layout, keys, values) -> "OracleKVCache":
        c = cls(layout)
        s_p = int(np.asarray(keys[0]).shape[0])
        if s_p == 0:
            raise OracleError("empty prompt")
        g = layout.group_size
        n_quant = ((s_p - g) // g) * g if s_p >= g else 0
        fp1_n = min(g, s_p - n_quant)
        fp2_n = s_p - n_quant - fp1_n
        for layer in range(layout.num_layers):
            k = np.asarray(keys[layer], F32)
            v = np.asarray(values[layer], F32)
            for b0 in range(0, n_quant, g):
                c._archive_or_quantize(layer, k[b0 : b0 + g], v[b0 : b0 + g])
            c.fp1[layer, 0, :fp1_n] = k[n_quant : n_quant + fp1_n]
            c.fp1[layer, 1, :fp1_n] = v[n_quant : n_quant + fp1_n]
            c.fp2[layer, 0, :fp2_n] = k[n_quant + fp1_n :]
            c.fp2[layer, 1, :fp2_n] = v[n_quant + fp1_n :]
        c.fp1_len, c.quantized_token_count = fp1_n, n_quant
        c.fp2_lens[:] = fp2_n
        return c

    @property
    def fp2_len(self) -> int:
        return int(self.fp2_lens[0])

    @property
    def seq_len(self) -> int:
        return self.quantized_token_count + self.fp1_len + self.fp2_len

    def fp2_space(self) -> int:
        return self.layout.group_size - self.fp2_len

    def _archive_or_quantize(self, layer: int, kb: np.ndarray, vb: np.ndarray) -> None:
        """Q/cache.py:283-289: sensitive layers archive f32 rows instead."""
        if layer in self.layout.sensitive_layers:
            self.archived[layer].append((np.array(kb, F32), np.array(vb, F32)))
        else:
            self.blocks[layer].append(quantize_kv_block(self.layout, kb, vb))

    # Q/cache.py:216-234
    def append_decode_token(self, layer: int, k, v) -> None:
        pos = int(self.fp2_lens[layer])
        if pos >= self.layout.group_size:
            raise OracleError("fp2 overflow")
        self.fp2[layer, 0, pos] = np.asarray(k, F32).reshape(-1)
        self.fp2[layer, 1, pos] = np.asarray(v, F32).reshape(-1)
        self.fp2_lens[layer] = pos + 1

    # Q/cache.py:236-247
    def rollback(self, n: int) -> None:
        if n < 0 or n > self.fp2_len or not np.all(self.fp2_lens == self.fp2_lens[0]):
            raise OracleError("bad rollback")
        self.fp2_lens -= n

    # Q/cache.py:249-281
    def flush_if_full(self) -> bool:
        g = self.layout.group_size
        if self.fp2_len != g:
            return False
        if self.fp1_len == g:
            for layer in range(self.layout.num_layers):
                self._archive_or_quantize(layer, self.fp1[layer, 0], self.fp1[layer, 1])
            self.fp1[:] = self.fp2
            self.quantized_token_count += g
            self.fp2_lens[:] = 0
        else:
            short = self.fp1_len
            take = g - short
            self.fp1[:, :, short:] = self.fp2[:, :, :take]
            self.fp2[:, :, :short] = self.fp2[:, :, take:].copy()
            self.fp2_lens[:] = short
        self.fp1_len = g
        return True

    # Q/cache.py:345-378
    def view(self, layer: int, kind: str) -> View:
        lay = self.layout
        segs = []
        qb = pb = fb = 0.0
        qe = 0
        if layer in lay.sensitive_layers:
            if self.archived[layer]:
                k = np.concatenate([a for a, _ in self.archived[layer]])
                v = np.concatenate([b for _, b in self.archived[layer]])
                segs.append((k, v))
                fb += FP_ELEM_BYTES * (k.size + v.size)
        elif self.blocks[layer]:
            parts = [dequant_kv_block(lay, b, kind) for b in self.blocks[layer]]
            k = np.concatenate([p[0] for p in parts])
            v = np.concatenate([p[1] for p in parts])
            segs.append((k, v))
            qe = k.size + v.size
            qb = (DRAFT_CODE_BYTES if kind == "draft" else TARGET_CODE_BYTES) * qe
            ngroups = sum(b.ku.scales.size + b.vu.scales.size for b in self.blocks[layer])
            pb = PARAM_PAIR_BYTES * ngroups * (2 if kind == "target" else 1)
        for buf, n in ((self.fp1[layer], self.fp1_len), (self.fp2[layer], int(self.fp2_lens[layer]))):
            if n:
                segs.append((buf[0, :n], buf[1, :n]))
                fb += FP_ELEM_BYTES * 2 * n * lay.kv_dim
        k = np.concatenate([s[0] for s in segs]) if segs else np.zeros((0, lay.kv_dim), F32)
        v = np.concatenate([s[1] for s in segs]) if segs else np.zeros((0, lay.kv_dim), F32)
        return View(k, v, qb, pb, fb, qe, segs)

    # Q/cache.py:384-403
    def memory_report(self) -> dict:
        up = lo = par = arch = 0.0
        for layer in range(self.layout.num_layers):
            for b in self.blocks[layer]:
                up += CODE_BYTES * (b.ku.count + b.vu.count)
                lo += CODE_BYTES * (b.kl.count + b.vl.count)
                par += PARAM_PAIR_BYTES * (b.ku.scales.size + b.vu.scales.size + b.kl.scales.size + b.vl.scales.size)
            for a, b2 in self.archived[layer]:
                arch += FP_ELEM_BYTES * (a.size + b2.size)
        lay = self.layout
        buffers = FP_ELEM_BYTES * lay.num_layers * 2 * 2 * lay.group_size * lay.kv_dim
        return {"upper_bytes": up, "lower_bytes": lo, "param_bytes": par,
                "fp_buffer_bytes": buffers, "archived_fp_bytes": arch,
                "total": up + lo + par + buffers + arch}


class OracleFpCache:
    """Lossless twin (FpKVCache), Q/cache.py:561-656: every view is plain f32."""

    def __init__(self, keys, values):
        self.k = [np.asarray(k, F32).copy() for k in keys]
        self.v = [np.asarray(v, F32).copy() for v in values]
        if self.k[0].shape[0] == 0:
            raise OracleError("empty prompt")

    @property
    def seq_len(self) -> int:
        return self.k[0].shape[0]

    quantized_token_count = 0

    def fp2_space(self) -> int:
        return 1 << 30

    def append_decode_token(self, layer, k, v):
        self.k[layer] = np.concatenate([self.k[layer], np.asarray(k, F32).reshape(1, -1)])
        self.v[layer] = np.concatenate([self.v[layer], np.asarray(v, F32).reshape(1, -1)])

    def rollback(self, n):
        if n:
            self.k = [a[:-n] for a in self.k]
            self.v = [a[:-n] for a in self.v]

    def flush_if_full(self):
        return False

    def view(self, layer, kind):
        k, v = self.k[layer], self.v[layer]
        return View(k, v, fp_bytes=FP_ELEM_BYTES * 2 * k.size, segments=[(k, v)])


# ---------------------------------------------------------------------------
# L2 model (Q/model.py, Q/tensor.py)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Config:
    """Q/model.py:35-56."""

    num_layers: int
    num_heads: int
    head_dim: int
    hidden: int
    mlp_hidden: int
    vocab: int
    max_positions: int
    rope_base: float = 10000.0
    norm_eps: float = 1e-5
    # GQA (configs 4/5) has no reference model: SURVEY 8(c) restates it by repeating each KV head
    # num_heads / num_kv_heads times into the reference's _merged_attention (None = MHA)
    num_kv_heads: int | None = None

    @property
    def kv_heads(self) -> int:
        return self.num_kv_heads or self.num_heads

    @property
    def kv_dim(self) -> int:
        return self.kv_heads * self.head_dim


MATS = ("wq", "wk", "wv", "wo", "w_gate", "w_up", "w_down")


def init_weights(cfg: Config, seed: int = 0) -> dict:
    """Seeded weights in the reference's draw order, Q/model.py:89-117.

    Per layer wq, wk, wv, wo, w_gate, w_up, w_down, then embedding, then
    lm_head; matrices are N(0,1)/sqrt(rows) divided in f64 then cast to f32.
    """
    rng = np.random.default_rng(seed)
    d, m, vocab = cfg.hidden, cfg.mlp_hidden, cfg.vocab
    kvd = cfg.kv_dim
    shapes = {"wq": (d, d), "wk": (d, kvd), "wv": (d, kvd), "wo": (d, d),
              "w_gate": (d, m), "w_up": (d, m), "w_down": (m, d)}

    def draw(r, c):
        return (rng.standard_normal((r, c)) / np.sqrt(r)).astype(F32)

    layers = []
    for _ in range(cfg.num_layers):
        lw = {name: draw(*shapes[name]) for name in MATS}
        lw["attn_norm"] = np.ones(d, F32)
        lw["mlp_norm"] = np.ones(d, F32)
        layers.append(lw)
    emb = rng.standard_normal((vocab, d)).astype(F32)
    head = draw(d, vocab)
    return {"config": cfg, "embedding": emb, "layers": layers, "final_norm": np.ones(d, F32), "lm_head": head}


def quantize_model(weights: dict, group: int) -> dict:
    """Draft weight set as dequantised f32 copies, Q/model.py:141-168."""
    out_layers = []
    nbytes = 0.0
    for lw in weights["layers"]:
        q = {}
        for name in MATS:
            p = quantize_matrix(lw[name], group)
            nbytes += CODE_BYTES * p.count
            q[name] = dequantize_matrix(p, lw[name].shape)
        q["attn_norm"], q["mlp_norm"] = lw["attn_norm"], lw["mlp_norm"]
        out_layers.append(q)
    p = quantize_matrix(weights["lm_head"], group)
    nbytes += CODE_BYTES * p.count
    return {"layers": out_layers, "lm_head": dequantize_matrix(p, weights["lm_head"].shape), "int4_weight_bytes": nbytes}


def rmsnorm(x: np.ndarray, gain: np.ndarray, eps: float) -> np.ndarray:
    """Q/tensor.py:35-42 (f32 throughout)."""
    x = np.asarray(x, F32)
    ms = np.mean(np.square(x), axis=-1, keepdims=True)
    return (x / np.sqrt(ms + F32(eps)) * np.asarray(gain, F32)).astype(F32)


def rope_tables(dim: int, base: float, position: int) -> tuple[np.ndarray, np.ndarray]:
    """cos/sin of theta_j = pos * base^(-2j/dim) in f64 cast to f32, Q/tensor.py:50-62."""
    ex = np.arange(dim // 2, dtype=F64) * (2.0 / dim)
    th = position * base ** -ex
    return np.cos(th).astype(F32), np.sin(th).astype(F32)


def rope(x: np.ndarray, position: int, base: float) -> np.ndarray:
    """Adjacent-pair rotation, Q/tensor.py:65-82."""
    x = np.asarray(x, F32)
    c, s = rope_tables(x.shape[-1], base, position)
    a, b = x[..., 0::2], x[..., 1::2]
    out = np.empty_like(x)
    out[..., 0::2] = a * c - b * s
    out[..., 1::2] = a * s + b * c
    return out


def silu(x: np.ndarray) -> np.ndarray:
    """Q/tensor.py:85-89."""
    x = np.asarray(x, F32)
    return (x / (1.0 + np.exp(-x))).astype(F32)


def merged_attention(q: np.ndarray, segments, scale: float) -> np.ndarray:
    """Running (max, denom, acc) merge across segments in f64, Q/model.py:176-195."""
    nh, hd = q.shape
    m = np.full(nh, -np.inf)
    den = np.zeros(nh)
    acc = np.zeros((nh, hd))
    for ks, vs in segments:
        sc = np.einsum("thd,hd->ht", ks, q, dtype=F64) * scale
        mn = np.maximum(m, sc.max(axis=1))
        a = np.exp(m - mn)
        p = np.exp(sc - mn[:, None])
        den = den * a + p.sum(axis=1)
        acc = acc * a[:, None] + np.einsum("ht,thd->hd", p, vs, dtype=F64)
        m = mn
    return (acc / den[:, None]).astype(F32)


def attend_view(q: np.ndarray, view: View, nh: int, hd: int, nkv: int | None = None) -> np.ndarray:
    nkv = nkv or nh
    r = nh // nkv
    segs = [(k.reshape(-1, nkv, hd), v.reshape(-1, nkv, hd)) for k, v in view.segments]
    if r > 1:  # GQA: each KV head serves r consecutive query heads
        segs = [(np.repeat(k, r, axis=1), np.repeat(v, r, axis=1)) for k, v in segs]
    return merged_attention(q, segs, 1.0 / np.sqrt(hd))


@dataclass
class Cost:
    """StepCost, Q/model.py:230-251."""

    flops: float = 0.0
    weight_bytes: float = 0.0
    kv_quantized_bytes: float = 0.0
    kv_param_bytes: float = 0.0
    kv_fp_bytes: float = 0.0
    kv_quantized_elements: int = 0

    @property
    def total_bytes(self) -> float:
        return self.weight_bytes + self.kv_quantized_bytes + self.kv_param_bytes + self.kv_fp_bytes


# Q/roofline.py constants used by decode_step's flop model
SOFTMAX_FLOPS_PER_SCORE = 5.0
NORM_FLOPS_PER_ELEM = 4.0
ACT_FLOPS_PER_ELEM = 4.0


def decode_step(weights: dict, token: int, cache, view: str = "fp", weight_mode: str = "fp", draft: dict | None = None):
    """One token through every layer, Q/model.py:324-407.  Returns (f32 logits, Cost)."""
    cfg: Config = weights["config"]
    nh, hd, d, m = cfg.num_heads, cfg.head_dim, cfg.hidden, cfg.mlp_hidden
    pos = cache.seq_len
    layers = draft["layers"] if weight_mode == "int4" else weights["layers"]
    head = draft["lm_head"] if weight_mode == "int4" else weights["lm_head"]
    cost = Cost()
    cost.weight_bytes = draft["int4_weight_bytes"] if weight_mode == "int4" else F32_BYTES * (
        cfg.num_layers * (4 * d * d + 3 * d * m) + d * cfg.vocab)
    x = weights["embedding"][token].copy()
    for li, lw in enumerate(layers):
        h = rmsnorm(x, lw["attn_norm"], cfg.norm_eps)
        nkv = cfg.kv_heads
        q = rope((h @ lw["wq"]).reshape(nh, hd), pos, cfg.rope_base)
        k = rope((h @ lw["wk"]).reshape(nkv, hd), pos, cfg.rope_base)
        v = (h @ lw["wv"]).reshape(nkv, hd)
        cache.append_decode_token(li, k.reshape(nkv * hd), v.reshape(nkv * hd))
        vw = cache.view(li, view)
        cost.kv_quantized_bytes += vw.quantized_bytes
        cost.kv_param_bytes += vw.param_bytes
        cost.kv_fp_bytes += vw.fp_bytes
        cost.kv_quantized_elements += vw.quantized_elements
        ctx = attend_view(q, vw, nh, hd, nkv)
        x = x + ctx.reshape(d) @ lw["wo"]
        hm = rmsnorm(x, lw["mlp_norm"], cfg.norm_eps)
        x = x + (silu(hm @ lw["w_gate"]) * (hm @ lw["w_up"])) @ lw["w_down"]
        t = vw.k.shape[0]
        cost.flops += 2.0 * (4 * d * d + 3 * d * m) + 4.0 * t * d + SOFTMAX_FLOPS_PER_SCORE * t * nh
        cost.flops += NORM_FLOPS_PER_ELEM * 2 * d + ACT_FLOPS_PER_ELEM * m
    logits = rmsnorm(x, weights["final_norm"], cfg.norm_eps) @ head
    cost.flops += 2.0 * d * cfg.vocab + NORM_FLOPS_PER_ELEM * d
    return logits.astype(F32), cost


def prefill_kv(weights: dict, tokens) -> tuple[np.ndarray, list, list]:
    """Causal f32/f64 prompt forward, Q/model.py:268-314; returns (logits, keys, values)."""
    cfg: Config = weights["config"]
    ids = np.asarray(tokens, np.int64).reshape(-1)
    s, nh, hd = ids.size, cfg.num_heads, cfg.head_dim
    x = weights["embedding"][ids]
    mask = np.triu(np.full((s, s), -np.inf, F32), k=1)
    keys, vals = [], []
    for lw in weights["layers"]:
        h = rmsnorm(x, lw["attn_norm"], cfg.norm_eps)
        nkv = cfg.kv_heads
        q = np.stack([rope(r, p, cfg.rope_base) for p, r in enumerate((h @ lw["wq"]).reshape(s, nh, hd))])
        k = np.stack([rope(r, p, cfg.rope_base) for p, r in enumerate((h @ lw["wk"]).reshape(s, nkv, hd))])
        v = (h @ lw["wv"]).reshape(s, nkv, hd)
        kr, vr = (k, v) if nkv == nh else (np.repeat(k, nh // nkv, axis=1), np.repeat(v, nh // nkv, axis=1))
        sc = np.einsum("shd,thd->hst", q, kr, dtype=F64) * (1.0 / np.sqrt(hd)) + mask
        sc -= sc.max(axis=2, keepdims=True)
        p = np.exp(sc)
        p /= p.sum(axis=2, keepdims=True)
        ctx = np.einsum("hst,thd->shd", p, vr, dtype=F64).astype(F32)
        x = x + ctx.reshape(s, cfg.hidden) @ lw["wo"]
        hm = rmsnorm(x, lw["mlp_norm"], cfg.norm_eps)
        x = x + (silu(hm @ lw["w_gate"]) * (hm @ lw["w_up"])) @ lw["w_down"]
        keys.append(np.ascontiguousarray(k.reshape(s, cfg.kv_dim)))
        vals.append(np.ascontiguousarray(v.reshape(s, cfg.kv_dim)))
    logits = rmsnorm(x[-1], weights["final_norm"], cfg.norm_eps) @ weights["lm_head"]
    return logits.astype(F32), keys, vals


def prefill(weights: dict, tokens, mode: str = "fp", group_size: int = 128, sensitive=frozenset()):
    """Q/model.py:268-321: prompt forward then cache construction."""
    logits, keys, vals = prefill_kv(weights, tokens)
    cfg = weights["config"]
    if mode == "hierarchical":
        lay = Layout(cfg.num_layers, cfg.kv_heads, cfg.head_dim, group_size, frozenset(sensitive))
        return logits, OracleKVCache.from_prefill(lay, keys, vals)
    return logits, OracleFpCache(keys, vals)


# ---------------------------------------------------------------------------
# L3 greedy draft/verify loop (Q/specdec.py)
# ---------------------------------------------------------------------------


def greedy_accept(drafts: list[int], target_logits: list[np.ndarray]) -> tuple[int, int | None, int | None]:
    """Greedy verification rule, Q/specdec.py:276-298.

    Accept while draft == argmax (first max index); the first mismatch emits
    the corrected argmax, otherwise the bonus argmax of the last row.
    Returns (v, corrected, bonus).
    """
    for i, g in enumerate(drafts):
        best = int(np.argmax(target_logits[i]))
        if g != best:
            return i, best, None
    return len(drafts), None, int(np.argmax(target_logits[len(drafts)]))


def spec_decode_greedy(weights, prompt, gamma, decode_len, kv_quant=True, group_size=128,
                       weight_mode="fp", draft=None, sensitive=frozenset()):
    """Q/specdec.py:314-397 restricted to greedy selection.

    Returns (tokens, steps) with one dict per cycle (drafted, v, corrected,
    bonus, flushed, emitted, draft_bytes, target_bytes).
    """
    logits, cache = prefill(weights, prompt, "hierarchical" if kv_quant else "fp", group_size, sensitive)
    out = [int(np.argmax(logits))]
    pending = out[0]
    steps = []
    while len(out) < decode_len:
        remaining = decode_len - len(out)
        gs = max(0, min(gamma, cache.fp2_space() - 1, remaining))
        if gs == 0:
            lg, c = decode_step(weights, pending, cache, "target")
            tok = int(np.argmax(lg))
            steps.append({"drafted": [], "v": 0, "corrected": tok, "bonus": None,
                          "flushed": cache.flush_if_full(), "emitted": [tok],
                          "draft_bytes": 0.0, "target_bytes": c.total_bytes})
            out.append(tok)
            pending = tok
            continue
        dc, tc = Cost(), Cost()
        drafts = []
        tok = pending
        for _ in range(gs):
            lg, c = decode_step(weights, tok, cache, "draft", weight_mode, draft)
            dc.weight_bytes += c.weight_bytes
            dc.kv_quantized_bytes += c.kv_quantized_bytes
            dc.kv_param_bytes += c.kv_param_bytes
            dc.kv_fp_bytes += c.kv_fp_bytes
            tok = int(np.argmax(lg))
            drafts.append(tok)
        cache.rollback(gs)
        tl = []
        for t in [pending, *drafts]:
            lg, c = decode_step(weights, t, cache, "target")
            tc.weight_bytes += c.weight_bytes
            tc.kv_quantized_bytes += c.kv_quantized_bytes
            tc.kv_param_bytes += c.kv_param_bytes
            tc.kv_fp_bytes += c.kv_fp_bytes
            tl.append(lg)
        v, corr, bonus = greedy_accept(drafts, tl)
        cache.rollback(gs - v)
        emitted = (drafts[:v] + [corr if corr is not None else bonus])[:remaining]
        steps.append({"drafted": drafts, "v": v, "corrected": corr, "bonus": bonus,
                      "flushed": cache.flush_if_full(), "emitted": emitted,
                      "draft_bytes": dc.total_bytes, "target_bytes": tc.total_bytes})
        out.extend(emitted)
        pending = corr if corr is not None else bonus
    return out, steps


def ar_decode_greedy(weights, prompt, decode_len, kv_quant=True, group_size=128, sensitive=frozenset()):
    """Q/specdec.py:400-434 (greedy): target-view AR, the losslessness oracle."""
    logits, cache = prefill(weights, prompt, "hierarchical" if kv_quant else "fp", group_size, sensitive)
    out = [int(np.argmax(logits))]
    view = "target" if kv_quant else "fp"
    while len(out) < decode_len:
        lg, _ = decode_step(weights, out[-1], cache, view)
        cache.flush_if_full()
        out.append(int(np.argmax(lg)))
    return out


def modeled_speedup(a: float, gamma: int) -> float:
    """E = (1 - a^(gamma+1)) / (1 - a), Q/roofline.py speedup_model's expected tokens."""
    if a >= 1.0:
        return float(gamma + 1)
    return (1.0 - a ** (gamma + 1)) / (1.0 - a)


def softmax_f64(logits, temperature: float = 1.0) -> np.ndarray:
    """Q/specdec.py:133-138."""
    z = np.asarray(logits, F64) / float(temperature)
    z = z - z.max()
    e = np.exp(z)
    return e / e.sum()


__all__ = [n for n in dir() if not n.startswith("_")]
