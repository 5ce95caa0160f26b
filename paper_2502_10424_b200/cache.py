"""Device-resident hierarchical KV cache (B200).

Drop-in for the reference object protocol of
/root/reference/pkg/src/quantspec/cache.py:119-403 (HierarchicalKVCache) and
:561-656 (FpKVCache): same constructors, counters, append/rollback/flush
semantics, views, byte accounting and QSKV snapshots.  The storage lives in
HBM in the layout of csrc/qs_layout.h:

  * quantised blocks: frag4 code planes (K/V x upper/lower) + f32 (S, Z) per
    group, in per-(sequence, layer, head) arenas of ``max_blocks`` blocks
    (no per-block Python objects, no f32 view memo);
  * fp1/fp2 recent-token buffers in fp16 (the paper's "FP16 buffer");
  * sensitive layers archive fp16 rows instead of quantising.

Lengths live twice: a host mirror (for the reference's counters and the
modeled byte accounting, computed with the reference formulas) and int32
device arrays read by the kernels (so CUDA graphs stay valid across steps).

Differences from the reference, by design: the fp buffers hold fp16, so a
view returns fp16-rounded values for the unquantised rows; quantisation of a
block sees those fp16 values upcast exactly (codes/params are bit-exact for
that input).
"""

from __future__ import annotations

import io
import math
import struct
from dataclasses import dataclass, field

import numpy as np

from . import _lib, layout, quant
from .errors import (
    BufferOverflowError,
    CacheIntegrityError,
    ConfigError,
    DataError,
    DimensionError,
    EmptyPromptError,
    FormatError,
)

FP_ELEM_BYTES = 4.0
DRAFT_CODE_BYTES = 0.5
TARGET_CODE_BYTES = 1.0

SNAPSHOT_MAGIC = b"QSKV"
SNAPSHOT_VERSION = 1


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise ConfigError("the B200 KV cache needs a CUDA device (no CPU fallback)")
    return torch


@dataclass(frozen=True)
class CacheLayout:
    """Static shape of one cache instance (Q/cache.py:42-63).

    ``num_kv_heads`` extends the reference (MHA only) to GQA; it defaults to
    ``num_heads``.
    """

    num_layers: int
    num_heads: int
    head_dim: int
    group_size: int
    sensitive_layers: frozenset = frozenset()
    num_kv_heads: int | None = None

    def __post_init__(self) -> None:
        if self.num_layers < 1 or self.num_heads < 1 or self.head_dim < 1:
            raise ConfigError("cache layout dimensions must be positive")
        if self.group_size < 1:
            raise ConfigError(f"group size must be >= 1, got {self.group_size}")
        bad = [l for l in self.sensitive_layers if not 0 <= l < self.num_layers]
        if bad:
            raise ConfigError(f"sensitive layer indices out of range: {bad}")

    @property
    def kv_heads(self) -> int:
        return self.num_kv_heads or self.num_heads

    @property
    def kv_dim(self) -> int:
        return self.kv_heads * self.head_dim


@dataclass
class CacheView:
    """Token-ordered dequantised segments plus byte-load accounting (Q/cache.py:66-83)."""

    segments: list = field(default_factory=list)
    quantized_bytes: float = 0.0
    param_bytes: float = 0.0
    fp_bytes: float = 0.0
    quantized_elements: int = 0

    @property
    def seq_len(self) -> int:
        return sum(k.shape[0] for k, _ in self.segments)

    def concat(self):
        return np.concatenate([k for k, _ in self.segments], axis=0), np.concatenate([v for _, v in self.segments], axis=0)


@dataclass
class MemoryReport:
    upper_bytes: float
    lower_bytes: float
    param_bytes: float
    fp_buffer_bytes: float
    archived_fp_bytes: float

    @property
    def total(self) -> float:
        return self.upper_bytes + self.lower_bytes + self.param_bytes + self.fp_buffer_bytes + self.archived_fp_bytes


def _check_device_geometry(layout: CacheLayout) -> None:
    hd, G = layout.head_dim, layout.group_size
    if hd not in (16, 32, 64, 128):
        raise ConfigError(f"head_dim {hd} not supported by the B200 store (16/32/64/128)")
    if G not in (16, 32, 64, 128):
        raise ConfigError(f"group size {G} not supported by the B200 store (16/32/64/128)")
    if not (G % hd == 0 or layout.kv_dim <= G):
        raise ConfigError(f"value groups of {G} channels would split a {hd}-channel head")


class HierarchicalKVCache:
    """Mutable per-session device cache; one logical owner mutates it at a time."""

    def __init__(self, layout: CacheLayout, *, max_tokens: int | None = None, batch: int = 1):
        _check_device_geometry(layout)
        torch = _torch()
        self.layout = layout
        self.batch = batch
        L, H, hd, G = layout.num_layers, layout.kv_heads, layout.head_dim, layout.group_size
        self.max_blocks = max(1, math.ceil((max_tokens or 8 * G) / G))
        dev = torch.device("cuda")
        self._dev = dev
        self._alloc_arena(self.max_blocks)
        self.fp_k = torch.zeros((batch, L, 2, H, G, hd), dtype=torch.float16, device=dev)
        self.fp_v = torch.zeros_like(self.fp_k)
        self._sens = sorted(layout.sensitive_layers)
        self._alloc_archive(self.max_blocks)
        # device lengths (kernels read these)
        self.d_n_blocks = torch.zeros(batch, dtype=torch.int32, device=dev)
        self.d_fp1_len = torch.zeros(batch, dtype=torch.int32, device=dev)
        self.d_fp2_len = torch.zeros(batch, dtype=torch.int32, device=dev)
        self.d_pos = torch.zeros(batch, dtype=torch.int32, device=dev)
        self.d_flags = torch.zeros(1, dtype=torch.int32, device=dev)
        # host mirror (sequence 0 for the reference protocol)
        self._fp1_len = 0
        self._fp2_len = np.zeros(L, dtype=np.int64)
        self.quantized_token_count = 0
        self.generation = 0  # bumps when arenas are reallocated (CUDA graphs re-capture)

    # ------------------------------------------------------------------ storage
    def _alloc_arena(self, max_blocks: int) -> None:
        torch = _torch()
        B, lay = self.batch, self.layout
        L, H, hd, G = lay.num_layers, lay.kv_heads, lay.head_dim, lay.group_size
        pb = G * hd // 2
        shp = (B, L, H, max_blocks, pb)
        self.ku = torch.zeros(shp, dtype=torch.uint8, device=self._dev)
        self.kl = torch.zeros(shp, dtype=torch.uint8, device=self._dev)
        self.vu = torch.zeros(shp, dtype=torch.uint8, device=self._dev)
        self.vl = torch.zeros(shp, dtype=torch.uint8, device=self._dev)
        self.kp = torch.zeros((B, L, H, max_blocks, hd, 2), dtype=torch.float32, device=self._dev)
        self.vp = torch.zeros((B, L, H, max_blocks, G, 2), dtype=torch.float32, device=self._dev)

    def _alloc_archive(self, max_blocks: int) -> None:
        torch = _torch()
        lay = self.layout
        if self._sens:
            shp = (self.batch, len(self._sens), lay.kv_heads, max_blocks * lay.group_size, lay.head_dim)
            self.arch_k = torch.zeros(shp, dtype=torch.float16, device=self._dev)
            self.arch_v = torch.zeros_like(self.arch_k)
        else:
            self.arch_k = self.arch_v = None

    def _grow(self, need_blocks: int) -> None:
        if need_blocks <= self.max_blocks:
            return
        torch = _torch()
        new = max(need_blocks, 2 * self.max_blocks)
        old = (self.ku, self.kl, self.vu, self.vl, self.kp, self.vp, self.arch_k, self.arch_v)
        nb = self.max_blocks
        self._alloc_arena(new)
        self._alloc_archive(new)
        for dst, src in zip((self.ku, self.kl, self.vu, self.vl, self.kp, self.vp), old[:6]):
            dst[:, :, :, :nb].copy_(src)
        if self.arch_k is not None:
            rows = nb * self.layout.group_size
            self.arch_k[:, :, :, :rows].copy_(old[6])
            self.arch_v[:, :, :, :rows].copy_(old[7])
        self.max_blocks = new
        self.generation += 1

    def store_struct(self) -> _lib.KVStore:
        lay = self.layout
        s = _lib.KVStore()
        s.B, s.L, s.Hkv, s.hd, s.G, s.max_blocks = (self.batch, lay.num_layers, lay.kv_heads, lay.head_dim,
                                                   lay.group_size, self.max_blocks)
        s.ku, s.kl, s.vu, s.vl = (self.ku.data_ptr(), self.kl.data_ptr(), self.vu.data_ptr(), self.vl.data_ptr())
        s.kp, s.vp = self.kp.data_ptr(), self.vp.data_ptr()
        s.fp_k, s.fp_v = self.fp_k.data_ptr(), self.fp_v.data_ptr()
        s.arch_k = self.arch_k.data_ptr() if self.arch_k is not None else None
        s.arch_v = self.arch_v.data_ptr() if self.arch_v is not None else None
        m0 = m1 = 0
        for l in self._sens:
            if l < 64:
                m0 |= 1 << l
            else:
                m1 |= 1 << (l - 64)
        s.sens_mask[0], s.sens_mask[1] = m0, m1
        return s

    def _check_flags(self, what: str) -> None:
        f = int(self.d_flags.item())
        if f:
            self.d_flags.zero_()
            raise DataError(f"{what}: non-finite K/V values")

    # ------------------------------------------------------------ construction
    @classmethod
    def from_prefill(cls, layout: CacheLayout, keys, values, *, max_tokens: int | None = None) -> "HierarchicalKVCache":
        """Build a cache from per-layer prompt K/V of shape [S_P, kv_dim] (Q/cache.py:139-182).

        ``keys``/``values`` may be NumPy arrays or CUDA tensors.
        """
        if len(keys) != layout.num_layers or len(values) != layout.num_layers:
            raise DimensionError("prefill K/V must supply one tensor per layer")
        s_p = int(keys[0].shape[0])
        if s_p == 0:
            raise EmptyPromptError("cannot prefill an empty prompt")
        for k, v in zip(keys, values):
            if tuple(k.shape) != (s_p, layout.kv_dim) or tuple(v.shape) != (s_p, layout.kv_dim):
                raise DimensionError(f"prefill tensors must be [S_P, {layout.kv_dim}], got {tuple(k.shape)} / {tuple(v.shape)}")
        g = layout.group_size
        cache = cls(layout, max_tokens=max(max_tokens or 0, s_p + 2 * g))
        for layer in range(layout.num_layers):
            cache.load_prefill_layer(layer, keys[layer], values[layer])
        cache.finish_prefill(s_p)
        return cache

    def load_prefill_layer(self, layer: int, k, v, seq: int = 0) -> None:
        """Quantise / buffer one layer's prompt K/V (rows [S_P, kv_dim])."""
        torch = _torch()
        lay = self.layout
        g, H, hd = lay.group_size, lay.kv_heads, lay.head_dim
        s_p = int(k.shape[0])
        n_quant = ((s_p - g) // g) * g if s_p >= g else 0
        fp1_n = min(g, s_p - n_quant)
        fp2_n = s_p - n_quant - fp1_n
        self._grow(n_quant // g + 1)

        def head_major(x):
            t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
            t = t.to(self._dev).to(torch.float16)
            return t.reshape(s_p, H, hd).permute(1, 0, 2).contiguous()  # [H][S][hd]

        hk, hv = head_major(k), head_major(v)
        if n_quant:
            st = self.store_struct()
            _lib.call("qs_kv_quantize_blocks", st, seq, layer, hk.data_ptr(), hv.data_ptr(), s_p * hd, n_quant // g, 0,
                      self.d_flags.data_ptr(), _lib.stream_ptr())
        self.fp_k[seq, layer, 0, :, :fp1_n] = hk[:, n_quant : n_quant + fp1_n]
        self.fp_v[seq, layer, 0, :, :fp1_n] = hv[:, n_quant : n_quant + fp1_n]
        if fp2_n:
            self.fp_k[seq, layer, 1, :, :fp2_n] = hk[:, n_quant + fp1_n :]
            self.fp_v[seq, layer, 1, :, :fp2_n] = hv[:, n_quant + fp1_n :]

    def finish_prefill(self, s_p: int, seq: int = 0) -> None:
        g = self.layout.group_size
        n_quant = ((s_p - g) // g) * g if s_p >= g else 0
        fp1_n = min(g, s_p - n_quant)
        fp2_n = s_p - n_quant - fp1_n
        self._check_flags("prefill")
        if seq == 0:
            self._fp1_len = fp1_n
            self._fp2_len[:] = fp2_n
            self.quantized_token_count = n_quant
        self.d_n_blocks[seq] = n_quant // g
        self.d_fp1_len[seq] = fp1_n
        self.d_fp2_len[seq] = fp2_n
        self.d_pos[seq] = s_p

    # ----------------------------------------------------------------- counters
    @property
    def fp1_len(self) -> int:
        return self._fp1_len

    @property
    def fp2_len(self) -> int:
        return int(self._fp2_len[0])

    @property
    def fp_token_count(self) -> int:
        return self._fp1_len + self.fp2_len

    @property
    def seq_len(self) -> int:
        return self.quantized_token_count + self.fp_token_count

    def fp2_space(self) -> int:
        return self.layout.group_size - self.fp2_len

    def check_layer_consistency(self) -> None:
        if not np.all(self._fp2_len == self._fp2_len[0]):
            raise CacheIntegrityError(f"per-layer append counts diverged: {self._fp2_len.tolist()}")

    # ----------------------------------------------------------------- mutation
    def append_decode_token(self, layer: int, k, v) -> None:
        """Store one token's K/V row in fp2 for ``layer`` (Q/cache.py:216-234)."""
        torch = _torch()
        lay = self.layout
        kv = lay.kv_dim
        kt = k if isinstance(k, torch.Tensor) else torch.from_numpy(np.asarray(k, dtype=np.float32).ravel())
        vt = v if isinstance(v, torch.Tensor) else torch.from_numpy(np.asarray(v, dtype=np.float32).ravel())
        if kt.numel() != kv or vt.numel() != kv:
            raise DimensionError(f"expected kv rows of width {kv}, got {kt.numel()}/{vt.numel()}")
        pos = int(self._fp2_len[layer])
        if pos >= lay.group_size:
            raise BufferOverflowError(f"fp2 is full (layer {layer}); the engine must flush before appending")
        self.fp_k[0, layer, 1, :, pos] = kt.to(self._dev, torch.float16).reshape(lay.kv_heads, lay.head_dim)
        self.fp_v[0, layer, 1, :, pos] = vt.to(self._dev, torch.float16).reshape(lay.kv_heads, lay.head_dim)
        self._fp2_len[layer] = pos + 1
        if np.all(self._fp2_len == self._fp2_len[0]):
            self.d_fp2_len[0] = int(self._fp2_len[0])
            self.d_pos[0] = self.seq_len

    def _advance(self, n: int) -> None:
        """Account for n rows the device forward appended to every layer."""
        if self.fp2_len + n > self.layout.group_size:
            raise BufferOverflowError("fp2 overflow")
        self._fp2_len += n
        _lib.call("qs_add_int", self.d_fp2_len.data_ptr(), self.batch, n, _lib.stream_ptr())
        _lib.call("qs_add_int", self.d_pos.data_ptr(), self.batch, n, _lib.stream_ptr())

    def rollback(self, n_reject: int) -> None:
        """Drop the last ``n_reject`` fp2 tokens in every layer (Q/cache.py:236-247)."""
        if n_reject < 0:
            raise ConfigError(f"rollback count must be nonnegative, got {n_reject}")
        if n_reject == 0:
            return
        self.check_layer_consistency()
        if n_reject > self.fp2_len:
            raise CacheIntegrityError(f"cannot roll back {n_reject} tokens; fp2 holds only {self.fp2_len}")
        self._fp2_len -= n_reject
        _lib.call("qs_add_int", self.d_fp2_len.data_ptr(), self.batch, -n_reject, _lib.stream_ptr())
        _lib.call("qs_add_int", self.d_pos.data_ptr(), self.batch, -n_reject, _lib.stream_ptr())

    def flush_if_full(self) -> bool:
        """Quantise fp1 and rotate fp2 into it once fp2 is full (Q/cache.py:249-281)."""
        self.check_layer_consistency()
        g = self.layout.group_size
        if self.fp2_len != g:
            return False
        if self._fp1_len == g:
            nb = self.quantized_token_count // g
            self._grow(nb + 1)
            st = self.store_struct()
            _lib.call("qs_kv_flush", st, 0, nb, self.d_flags.data_ptr(), _lib.stream_ptr())
            _lib.call("qs_add_int", self.d_n_blocks.data_ptr(), self.batch, 1, _lib.stream_ptr())
            _lib.call("qs_add_int", self.d_fp2_len.data_ptr(), self.batch, -g, _lib.stream_ptr())
            self.quantized_token_count += g
            self._fp1_len = g
            self._fp2_len[:] = 0
            return True
        short = self._fp1_len
        take = g - short
        self.fp_k[:, :, 0, :, short:] = self.fp_k[:, :, 1, :, :take]
        self.fp_v[:, :, 0, :, short:] = self.fp_v[:, :, 1, :, :take]
        keep_k = self.fp_k[:, :, 1, :, take:].clone()
        keep_v = self.fp_v[:, :, 1, :, take:].clone()
        self.fp_k[:, :, 1, :, :short] = keep_k
        self.fp_v[:, :, 1, :, :short] = keep_v
        self._fp2_len[:] = short
        self._fp1_len = g
        self.d_fp1_len.fill_(g)
        self.d_fp2_len.fill_(short)
        return True

    def _quantize_block_for_test(self, layer: int, k_block, v_block) -> None:  # pragma: no cover - debug aid
        raise NotImplementedError

    # ------------------------------------------------------------------- views
    def draft_view(self, layer: int) -> CacheView:
        return self._view(layer, "draft")

    def target_view(self, layer: int) -> CacheView:
        return self._view(layer, "target")

    def _fp_rows(self, which: int, layer: int, n: int, seq: int = 0) -> tuple[np.ndarray, np.ndarray]:
        lay = self.layout
        k = self.fp_k[seq, layer, which, :, :n].permute(1, 0, 2).reshape(n, lay.kv_dim)
        v = self.fp_v[seq, layer, which, :, :n].permute(1, 0, 2).reshape(n, lay.kv_dim)
        return k.float().cpu().numpy(), v.float().cpu().numpy()

    def quantized_region(self, layer: int, kind: str, seq: int = 0):
        """f32 dequantised quantised history [n_q, kv_dim] (device kernel, f64 math)."""
        torch = _torch()
        lay = self.layout
        nb = self.quantized_token_count // lay.group_size
        if nb == 0:
            return None
        ok = torch.empty((nb * lay.group_size, lay.kv_dim), dtype=torch.float32, device=self._dev)
        ov = torch.empty_like(ok)
        st = self.store_struct()
        _lib.call("qs_kv_dequant_view", st, seq, layer, nb, 1 if kind == "target" else 0, ok.data_ptr(), ov.data_ptr(),
                  _lib.stream_ptr())
        return ok.cpu().numpy(), ov.cpu().numpy()

    def _view(self, layer: int, kind: str) -> CacheView:
        lay = self.layout
        if not 0 <= layer < lay.num_layers:
            raise ConfigError(f"layer index {layer} out of range")
        view = CacheView(segments=[])
        code_bytes = DRAFT_CODE_BYTES if kind == "draft" else TARGET_CODE_BYTES
        nq = self.quantized_token_count
        if layer in lay.sensitive_layers:
            if nq:
                slot = self._sens.index(layer)
                k = self.arch_k[0, slot, :, :nq].permute(1, 0, 2).reshape(nq, lay.kv_dim).float().cpu().numpy()
                v = self.arch_v[0, slot, :, :nq].permute(1, 0, 2).reshape(nq, lay.kv_dim).float().cpu().numpy()
                view.segments.append((k, v))
                view.fp_bytes += FP_ELEM_BYTES * (k.size + v.size)
        elif nq:
            k, v = self.quantized_region(layer, kind)
            view.segments.append((k, v))
            elems = k.size + v.size
            view.quantized_elements += elems
            view.quantized_bytes += code_bytes * elems
            groups = self._groups_per_block() * (nq // lay.group_size)
            if kind == "target":
                groups *= 2
            view.param_bytes += quant.PARAM_PAIR_BYTES * groups
        for which, n in ((0, self._fp1_len), (1, int(self._fp2_len[layer]))):
            if n:
                view.segments.append(self._fp_rows(which, layer, n))
                view.fp_bytes += FP_ELEM_BYTES * 2 * n * lay.kv_dim
        return view

    def _groups_per_block(self) -> int:
        """Key groups (one per channel) + value groups (ceil(kv/G) per token) of one block."""
        lay = self.layout
        return lay.kv_dim + lay.group_size * (-(-lay.kv_dim // lay.group_size))

    # ------------------------------------------------------- accounting / export
    def memory_report(self) -> MemoryReport:
        """Exact modeled byte totals (Q/cache.py:384-403)."""
        lay = self.layout
        nb = self.quantized_token_count // lay.group_size
        nq_layers = lay.num_layers - len(self._sens)
        elems = lay.group_size * lay.kv_dim  # per tensor per block
        upper = nq_layers * nb * 2 * elems * quant.CODE_BYTES
        lower = upper
        params = nq_layers * nb * 2 * self._groups_per_block() * quant.PARAM_PAIR_BYTES
        archived = len(self._sens) * nb * 2 * FP_ELEM_BYTES * elems
        buffers = FP_ELEM_BYTES * lay.num_layers * 2 * 2 * lay.group_size * lay.kv_dim
        return MemoryReport(float(upper), float(lower), float(params), float(buffers), float(archived))

    def device_bytes(self) -> int:
        ts = [self.ku, self.kl, self.vu, self.vl, self.kp, self.vp, self.fp_k, self.fp_v]
        if self.arch_k is not None:
            ts += [self.arch_k, self.arch_v]
        return int(sum(t.numel() * t.element_size() for t in ts))

    def export_block_planes(self, layer: int, block: int, seq: int = 0):
        """Reference-packed QuantPlane quartet (K_u, K_l, V_u, V_l) of one flushed block."""
        lay = self.layout
        G, hd, H, kv = lay.group_size, lay.head_dim, lay.kv_heads, lay.kv_dim
        kw, kn, vw, vn = layout.block_maps(G, hd)

        def words(t):
            return t[seq, layer, :, block].contiguous().cpu().numpy().view(np.uint32)  # [H][nwords]

        wku, wkl, wvu, wvl = words(self.ku), words(self.kl), words(self.vu), words(self.vl)
        kp = self.kp[seq, layer, :, block].cpu().numpy()  # [H][hd][2]
        vpp = self.vp[seq, layer, :, block].cpu().numpy()  # [H][G][2]
        cku = np.concatenate([layout.unpack_block(wku[h], kw, kn) for h in range(H)], axis=1)  # [G][kv]
        ckl = np.concatenate([layout.unpack_block(wkl[h], kw, kn) for h in range(H)], axis=1) - 8
        cvu = np.concatenate([layout.unpack_block(wvu[h], vw, vn) for h in range(H)], axis=1)
        cvl = np.concatenate([layout.unpack_block(wvl[h], vw, vn) for h in range(H)], axis=1) - 8
        ks = kp[:, :, 0].reshape(kv).astype(np.float32)
        kz = kp[:, :, 1].reshape(kv).astype(np.float32)
        ngv = -(-kv // G)
        first_head = [(j * G) // hd for j in range(ngv)]
        vs = np.stack([vpp[h, :, 0] for h in first_head], axis=1).reshape(-1).astype(np.float32)  # [G*ngv]
        vz = np.stack([vpp[h, :, 1] for h in first_head], axis=1).reshape(-1).astype(np.float32)
        count = G * kv
        mk = lambda codes, s, z, mode, axis, rl: quant.QuantPlane(quant.pack_nibbles(codes), count, G, s, z, mode, axis, rl)
        ku = mk(cku.T.reshape(-1), ks, kz, quant.MODE_ASYM_U4, quant.AXIS_CHANNEL, None)
        kl = mk(ckl.T.reshape(-1), (ks / np.float32(16)).astype(np.float32), np.zeros_like(ks), quant.MODE_SYM_S4, quant.AXIS_CHANNEL, None)
        vu = mk(cvu.reshape(-1), vs, vz, quant.MODE_ASYM_U4, quant.AXIS_TOKEN, kv)
        vl = mk(cvl.reshape(-1), (vs / np.float32(16)).astype(np.float32), np.zeros_like(vs), quant.MODE_SYM_S4, quant.AXIS_TOKEN, kv)
        return ku, kl, vu, vl

    def import_block_planes(self, layer: int, block: int, planes, seq: int = 0) -> None:
        """Inverse of export_block_planes (snapshot load)."""
        torch = _torch()
        lay = self.layout
        G, hd, H, kv = lay.group_size, lay.head_dim, lay.kv_heads, lay.kv_dim
        kw, kn, vw, vn = layout.block_maps(G, hd)
        ku, kl, vu, vl = planes
        nwords = G * hd // 8
        cku = ku.unpacked().astype(np.int64).reshape(kv, G).T
        ckl = kl.unpacked().astype(np.int64).reshape(kv, G).T + 8
        cvu = vu.unpacked().astype(np.int64).reshape(G, kv)
        cvl = vl.unpacked().astype(np.int64).reshape(G, kv) + 8
        for h in range(H):
            sl = slice(h * hd, (h + 1) * hd)
            for dst, codes, wi, ni in ((self.ku, cku, kw, kn), (self.kl, ckl, kw, kn), (self.vu, cvu, vw, vn), (self.vl, cvl, vw, vn)):
                w = layout.pack_block(codes[:, sl], wi, ni, nwords)
                dst[seq, layer, h, block] = torch.from_numpy(w.view(np.uint8)).to(self._dev)
        kp = np.stack([ku.scales, ku.zeros], axis=-1).reshape(H, hd, 2)
        self.kp[seq, layer, :, block] = torch.from_numpy(np.ascontiguousarray(kp, dtype=np.float32)).to(self._dev)
        ngv = -(-kv // G)
        s = vu.scales.reshape(G, ngv)
        z = vu.zeros.reshape(G, ngv)
        for h in range(H):
            j = (h * hd) // G
            self.vp[seq, layer, h, block] = torch.from_numpy(np.stack([s[:, j], z[:, j]], axis=-1).astype(np.float32)).to(self._dev)

    # --------------------------------------------------------------- snapshots
    def save_snapshot(self, path) -> None:
        with open(path, "wb") as f:
            self._write_snapshot(f)

    def _write_snapshot(self, f) -> None:
        """QSKV format of Q/cache.py:405-447 (fp rows written as f32)."""
        self.check_layer_consistency()
        lay = self.layout
        f.write(SNAPSHOT_MAGIC)
        f.write(struct.pack("<B", SNAPSHOT_VERSION))
        sens = sorted(lay.sensitive_layers)
        f.write(struct.pack("<IIIII", lay.num_layers, lay.num_heads, lay.head_dim, lay.group_size, len(sens)))
        for s in sens:
            f.write(struct.pack("<I", s))
        f.write(struct.pack("<QII", self.quantized_token_count, self._fp1_len, self.fp2_len))
        nb = self.quantized_token_count // lay.group_size
        for layer in range(lay.num_layers):
            if layer in lay.sensitive_layers:
                f.write(struct.pack("<I", nb))
                slot = self._sens.index(layer)
                for b in range(nb):
                    rows = slice(b * lay.group_size, (b + 1) * lay.group_size)
                    ak = self.arch_k[0, slot, :, rows].permute(1, 0, 2).reshape(lay.group_size, lay.kv_dim)
                    av = self.arch_v[0, slot, :, rows].permute(1, 0, 2).reshape(lay.group_size, lay.kv_dim)
                    f.write(struct.pack("<I", lay.group_size))
                    f.write(ak.float().cpu().numpy().astype("<f4").tobytes())
                    f.write(av.float().cpu().numpy().astype("<f4").tobytes())
            else:
                f.write(struct.pack("<I", nb))
                for b in range(nb):
                    for plane in self.export_block_planes(layer, b):
                        _write_plane(f, plane)
            k1, v1 = self._fp_rows(0, layer, self._fp1_len) if self._fp1_len else (np.zeros((0, lay.kv_dim), np.float32),) * 2
            k2, v2 = self._fp_rows(1, layer, self.fp2_len) if self.fp2_len else (np.zeros((0, lay.kv_dim), np.float32),) * 2
            for arr in (k1, v1, k2, v2):
                f.write(np.asarray(arr, dtype="<f4").tobytes())

    @classmethod
    def load_snapshot(cls, path) -> "HierarchicalKVCache":
        with open(path, "rb") as f:
            data = f.read()
        return cls._read_snapshot(io.BytesIO(data))

    @classmethod
    def _read_snapshot(cls, f) -> "HierarchicalKVCache":
        torch = _torch()
        if f.read(4) != SNAPSHOT_MAGIC:
            raise FormatError("bad snapshot magic")
        (version,) = _unpack(f, "<B")
        if version != SNAPSHOT_VERSION:
            raise FormatError(f"unsupported snapshot version {version}")
        L, H, hd, G, n_sens = _unpack(f, "<IIIII")
        sens = frozenset(_unpack(f, "<I")[0] for _ in range(n_sens))
        lay = CacheLayout(L, H, hd, G, sens)
        quantized, fp1_len, fp2_len = _unpack(f, "<QII")
        cache = cls(lay, max_tokens=quantized + 2 * G)
        kv = lay.kv_dim
        for layer in range(L):
            (nblk,) = _unpack(f, "<I")
            if layer in sens:
                slot = cache._sens.index(layer)
                for b in range(nblk):
                    (rows,) = _unpack(f, "<I")
                    ak = _read_f32(f, (rows, kv))
                    av = _read_f32(f, (rows, kv))
                    r0 = b * G
                    cache.arch_k[0, slot, :, r0 : r0 + rows] = torch.from_numpy(ak).reshape(rows, H, hd).permute(1, 0, 2).to(cache._dev, torch.float16)
                    cache.arch_v[0, slot, :, r0 : r0 + rows] = torch.from_numpy(av).reshape(rows, H, hd).permute(1, 0, 2).to(cache._dev, torch.float16)
            else:
                for b in range(nblk):
                    planes = tuple(_read_plane(f) for _ in range(4))
                    cache.import_block_planes(layer, b, planes)
            for which, n in ((0, fp1_len), (1, fp2_len)):
                k = _read_f32(f, (n, kv))
                v = _read_f32(f, (n, kv))
                if n:
                    cache.fp_k[0, layer, which, :, :n] = torch.from_numpy(k).reshape(n, H, hd).permute(1, 0, 2).to(cache._dev, torch.float16)
                    cache.fp_v[0, layer, which, :, :n] = torch.from_numpy(v).reshape(n, H, hd).permute(1, 0, 2).to(cache._dev, torch.float16)
        cache._fp1_len = fp1_len
        cache._fp2_len[:] = fp2_len
        cache.quantized_token_count = quantized
        cache.d_n_blocks.fill_(quantized // G)
        cache.d_fp1_len.fill_(fp1_len)
        cache.d_fp2_len.fill_(fp2_len)
        cache.d_pos.fill_(quantized + fp1_len + fp2_len)
        return cache


_AXIS_CODES = {quant.AXIS_CHANNEL: 0, quant.AXIS_TOKEN: 1}
_MODE_CODES = {quant.MODE_ASYM_U4: 0, quant.MODE_SYM_S4: 1}
_AXIS_NAMES = {v: k for k, v in _AXIS_CODES.items()}
_MODE_NAMES = {v: k for k, v in _MODE_CODES.items()}


def _unpack(f, fmt: str):
    size = struct.calcsize(fmt)
    raw = f.read(size)
    if len(raw) != size:
        raise FormatError("snapshot truncated")
    return struct.unpack(fmt, raw)


def _read_f32(f, shape) -> np.ndarray:
    count = int(np.prod(shape)) if shape else 0
    raw = f.read(count * 4)
    if len(raw) != count * 4:
        raise FormatError("snapshot truncated")
    return np.frombuffer(raw, dtype="<f4").reshape(shape).astype(np.float32)


def _write_plane(f, plane: quant.QuantPlane) -> None:
    f.write(struct.pack("<QIIBBI", plane.count, plane.group_size, plane.row_len or 0, _AXIS_CODES[plane.axis],
                        _MODE_CODES[plane.mode], plane.num_groups))
    f.write(plane.codes.tobytes())
    f.write(plane.scales.astype("<f4").tobytes())
    f.write(plane.zeros.astype("<f4").tobytes())


def _read_plane(f) -> quant.QuantPlane:
    count, group_size, row_len, axis_code, mode_code, ngroups = _unpack(f, "<QIIBBI")
    n = (count + 1) // 2
    raw = f.read(n)
    if len(raw) != n:
        raise FormatError("snapshot truncated")
    return quant.QuantPlane(np.frombuffer(raw, dtype=np.uint8).copy(), count, group_size, _read_f32(f, (ngroups,)),
                            _read_f32(f, (ngroups,)), _MODE_NAMES[mode_code], _AXIS_NAMES[axis_code], row_len or None)


# -----------------------------------------------------------------------------
# fp16 cache (lossless runs and the FP16 autoregressive baseline)
# -----------------------------------------------------------------------------


class FpKVCache:
    """Device fp16 cache with the same append/rollback/view surface (Q/cache.py:561-656).

    Rows live head-major ``[B][L][Hkv][cap][hd]`` so the attention kernel
    streams one head's history contiguously.
    """

    def __init__(self, num_layers: int, kv_dim: int, capacity: int = 64, *, head_dim: int | None = None,
                 batch: int = 1):
        if num_layers < 1 or kv_dim < 1:
            raise ConfigError("cache dimensions must be positive")
        torch = _torch()
        self.num_layers = num_layers
        self.kv_dim = kv_dim
        self.head_dim = head_dim or (128 if kv_dim % 128 == 0 else 16)
        self.kv_heads = kv_dim // self.head_dim
        self.batch = batch
        self._cap = max(int(capacity), 1)
        self._dev = torch.device("cuda")
        self.k = torch.zeros((batch, num_layers, self.kv_heads, self._cap, self.head_dim), dtype=torch.float16, device=self._dev)
        self.v = torch.zeros_like(self.k)
        self._len = np.zeros(num_layers, dtype=np.int64)
        self.d_len = torch.zeros(batch, dtype=torch.int32, device=self._dev)
        self.generation = 0

    @classmethod
    def from_prefill(cls, keys, values, *, head_dim: int | None = None, capacity: int | None = None) -> "FpKVCache":
        s_p = int(keys[0].shape[0])
        if s_p == 0:
            raise EmptyPromptError("cannot prefill an empty prompt")
        cache = cls(len(keys), int(keys[0].shape[1]), capacity=max(64, 2 * s_p, capacity or 0), head_dim=head_dim)
        for layer in range(len(keys)):
            cache.load_prefill_layer(layer, keys[layer], values[layer])
        cache.finish_prefill(s_p)
        return cache

    def load_prefill_layer(self, layer: int, k, v, seq: int = 0) -> None:
        torch = _torch()
        s_p = int(k.shape[0])
        self._ensure(s_p + 1)
        for dst, x in ((self.k, k), (self.v, v)):
            t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
            t = t.to(self._dev).to(torch.float16).reshape(s_p, self.kv_heads, self.head_dim).permute(1, 0, 2)
            dst[seq, layer, :, :s_p] = t

    def finish_prefill(self, s_p: int, seq: int = 0) -> None:
        if seq == 0:
            self._len[:] = s_p
        self.d_len[seq] = s_p

    @property
    def seq_len(self) -> int:
        return int(self._len[0])

    @property
    def quantized_token_count(self) -> int:
        return 0

    @property
    def capacity(self) -> int:
        return self._cap

    def fp2_space(self) -> int:
        return 1 << 30

    def check_layer_consistency(self) -> None:
        if not np.all(self._len == self._len[0]):
            raise CacheIntegrityError(f"per-layer append counts diverged: {self._len.tolist()}")

    def _ensure(self, need: int) -> None:
        if need <= self._cap:
            return
        torch = _torch()
        new = max(need, 2 * self._cap)
        k = torch.zeros((self.batch, self.num_layers, self.kv_heads, new, self.head_dim), dtype=torch.float16, device=self._dev)
        v = torch.zeros_like(k)
        k[:, :, :, : self._cap] = self.k
        v[:, :, :, : self._cap] = self.v
        self.k, self.v, self._cap = k, v, new
        self.generation += 1

    def append_decode_token(self, layer: int, k, v) -> None:
        torch = _torch()
        kt = k if isinstance(k, torch.Tensor) else torch.from_numpy(np.asarray(k, dtype=np.float32).ravel())
        vt = v if isinstance(v, torch.Tensor) else torch.from_numpy(np.asarray(v, dtype=np.float32).ravel())
        if kt.numel() != self.kv_dim or vt.numel() != self.kv_dim:
            raise DimensionError(f"expected kv rows of width {self.kv_dim}")
        pos = int(self._len[layer])
        self._ensure(pos + 1)
        self.k[0, layer, :, pos] = kt.to(self._dev, torch.float16).reshape(self.kv_heads, self.head_dim)
        self.v[0, layer, :, pos] = vt.to(self._dev, torch.float16).reshape(self.kv_heads, self.head_dim)
        self._len[layer] = pos + 1
        if np.all(self._len == self._len[0]):
            self.d_len[0] = int(self._len[0])

    def _advance(self, n: int) -> None:
        self._len += n
        _lib.call("qs_add_int", self.d_len.data_ptr(), self.batch, n, _lib.stream_ptr())

    def rollback(self, n_reject: int) -> None:
        if n_reject < 0:
            raise ConfigError(f"rollback count must be nonnegative, got {n_reject}")
        if n_reject == 0:
            return
        self.check_layer_consistency()
        if n_reject > self.seq_len:
            raise CacheIntegrityError("rollback past the sequence start")
        self._len -= n_reject
        _lib.call("qs_add_int", self.d_len.data_ptr(), self.batch, -n_reject, _lib.stream_ptr())

    def flush_if_full(self) -> bool:
        return False

    def _view(self, layer: int) -> CacheView:
        n = int(self._len[layer])
        k = self.k[0, layer, :, :n].permute(1, 0, 2).reshape(n, self.kv_dim).float().cpu().numpy()
        v = self.v[0, layer, :, :n].permute(1, 0, 2).reshape(n, self.kv_dim).float().cpu().numpy()
        view = CacheView(segments=[(k, v)])
        view.fp_bytes = FP_ELEM_BYTES * 2 * n * self.kv_dim
        return view

    def fp_view(self, layer: int) -> CacheView:
        return self._view(layer)

    def draft_view(self, layer: int) -> CacheView:
        return self._view(layer)

    def target_view(self, layer: int) -> CacheView:
        return self._view(layer)

    def memory_report(self) -> MemoryReport:
        used = FP_ELEM_BYTES * 2 * self.seq_len * self.kv_dim * self.num_layers
        return MemoryReport(0.0, 0.0, 0.0, used, 0.0)

    def device_bytes(self) -> int:
        return int(2 * self.k.numel() * self.k.element_size())
