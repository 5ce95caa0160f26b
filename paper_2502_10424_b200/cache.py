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

import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib, layout, qskv, quant
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

# fp2 rows past G: a ragged batch pads every sequence's draft / verify rows to the longest
# gamma_step of the cycle; the padding rows' K/V land here and are never committed
FP_SLACK = 16


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
    """Mutable device cache of ``batch`` independent sequences; one logical owner mutates it at a time.

    The reference protocol (append_decode_token / rollback / flush_if_full / views / snapshots)
    acts on sequence 0; the batched decode engine (engine.SpecEngine) drives every sequence
    through the device length arrays and keeps the per-sequence host mirror in step with
    ``commit_cycle``.
    """

    def __init__(self, layout: CacheLayout, *, max_tokens: int | None = None, batch: int = 1):
        _check_device_geometry(layout)
        torch = _torch()
        if batch < 1:
            raise ConfigError(f"batch must be >= 1, got {batch}")
        self.layout = layout
        self.batch = batch
        L, H, hd, G = layout.num_layers, layout.kv_heads, layout.head_dim, layout.group_size
        self.max_blocks = max(1, math.ceil((max_tokens or 8 * G) / G))
        self.fp_rows = G + FP_SLACK
        dev = torch.device("cuda")
        self._dev = dev
        self._alloc_arena(self.max_blocks)
        self.fp_k = torch.zeros((batch, L, 2, H, self.fp_rows, hd), dtype=torch.float16, device=dev)
        self.fp_v = torch.zeros_like(self.fp_k)
        self._sens = sorted(layout.sensitive_layers)
        self._alloc_archive(self.max_blocks)
        # device lengths (kernels read these)
        self.d_n_blocks = torch.zeros(batch, dtype=torch.int32, device=dev)
        self.d_fp1_len = torch.zeros(batch, dtype=torch.int32, device=dev)
        self.d_fp2_len = torch.zeros(batch, dtype=torch.int32, device=dev)
        self.d_pos = torch.zeros(batch, dtype=torch.int32, device=dev)
        self.d_flags = torch.zeros(1, dtype=torch.int32, device=dev)
        # host mirror: per sequence quantised tokens and fp1 rows, per (sequence, layer) fp2 rows
        self._nq = np.zeros(batch, dtype=np.int64)
        self._fp1 = np.zeros(batch, dtype=np.int64)
        self._fp2 = np.zeros((batch, L), dtype=np.int64)
        self.generation = 0  # bumps when arenas are reallocated (CUDA graphs re-capture)

    # ------------------------------------------------------------------ storage
    def _alloc_arena(self, max_blocks: int) -> None:
        torch = _torch()
        B, lay = self.batch, self.layout
        L, H, hd, G = lay.num_layers, lay.kv_heads, lay.head_dim, lay.group_size
        shp = (B, L, H, max_blocks, G * hd // 2)
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

    def ensure_blocks(self, need_blocks: int) -> None:
        """Grow the quantised arenas to hold ``need_blocks`` blocks per (sequence, layer, head)."""
        if need_blocks <= self.max_blocks:
            return
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

    _grow = ensure_blocks

    def store_struct(self) -> _lib.KVStore:
        lay = self.layout
        s = _lib.KVStore()
        s.B, s.L, s.Hkv, s.hd, s.G, s.max_blocks = (self.batch, lay.num_layers, lay.kv_heads, lay.head_dim,
                                                   lay.group_size, self.max_blocks)
        s.fp_rows = self.fp_rows
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

    def raise_device_flags(self, what: str, flags: int | None = None) -> None:
        """Map the device status word to the reference exceptions (read it when ``flags`` is None)."""
        f = int(self.d_flags.item()) if flags is None else int(flags)
        if not f:
            return
        self.d_flags.zero_()
        if f & _lib.FLAG_NONFINITE:
            raise DataError(f"{what}: cannot quantize non-finite K/V values")
        if f & _lib.FLAG_OVERFLOW:
            raise BufferOverflowError(f"{what}: quantised arena full ({self.max_blocks} blocks)")
        raise DataError(f"{what}: device status {f:#x}")

    _check_flags = raise_device_flags

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

    @staticmethod
    def _fill_rule(s_p: int, g: int) -> tuple[int, int, int]:
        """(quantised, fp1, fp2) token counts of a prompt (Q/cache.py:165-171)."""
        n_quant = ((s_p - g) // g) * g if s_p >= g else 0
        fp1_n = min(g, s_p - n_quant)
        return n_quant, fp1_n, s_p - n_quant - fp1_n

    def load_prefill_layer(self, layer: int, k, v, seq: int = 0) -> None:
        """Quantise / buffer one layer's prompt K/V (rows [S_P, kv_dim]) of sequence ``seq``."""
        torch = _torch()
        lay = self.layout
        g, H, hd = lay.group_size, lay.kv_heads, lay.head_dim
        s_p = int(k.shape[0])
        n_quant, fp1_n, fp2_n = self._fill_rule(s_p, g)
        self.ensure_blocks(n_quant // g + 1)

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
        n_quant, fp1_n, fp2_n = self._fill_rule(s_p, self.layout.group_size)
        self.raise_device_flags("prefill")
        self._nq[seq], self._fp1[seq] = n_quant, fp1_n
        self._fp2[seq, :] = fp2_n
        self.d_n_blocks[seq] = n_quant // self.layout.group_size
        self.d_fp1_len[seq] = fp1_n
        self.d_fp2_len[seq] = fp2_n
        self.d_pos[seq] = s_p

    # ----------------------------------------------------------------- counters
    @property
    def quantized_token_count(self) -> int:
        return int(self._nq[0])

    @property
    def fp1_len(self) -> int:
        return int(self._fp1[0])

    @property
    def fp2_len(self) -> int:
        return int(self._fp2[0, 0])

    @property
    def fp_token_count(self) -> int:
        return self.fp1_len + self.fp2_len

    @property
    def seq_len(self) -> int:
        return self.quantized_token_count + self.fp_token_count

    def seq_lens(self) -> np.ndarray:
        """Tokens held per sequence."""
        return self._nq + self._fp1 + self._fp2[:, 0]

    def fp2_space(self, seq: int = 0) -> int:
        return self.layout.group_size - int(self._fp2[seq, 0])

    def check_layer_consistency(self) -> None:
        if not np.all(self._fp2 == self._fp2[:, :1]):
            raise CacheIntegrityError(f"per-layer append counts diverged: {self._fp2.tolist()}")

    def _single(self, what: str) -> None:
        if self.batch != 1:
            raise ConfigError(f"{what} is the single-sequence protocol; a batch of {self.batch} runs through SpecEngine")

    # ----------------------------------------------------------------- mutation
    def append_decode_token(self, layer: int, k, v) -> None:
        """Store one token's K/V row in fp2 for ``layer`` (Q/cache.py:216-234)."""
        self._single("append_decode_token")
        torch = _torch()
        lay = self.layout
        kv = lay.kv_dim
        kt = k if isinstance(k, torch.Tensor) else torch.from_numpy(np.asarray(k, dtype=np.float32).ravel())
        vt = v if isinstance(v, torch.Tensor) else torch.from_numpy(np.asarray(v, dtype=np.float32).ravel())
        if kt.numel() != kv or vt.numel() != kv:
            raise DimensionError(f"expected kv rows of width {kv}, got {kt.numel()}/{vt.numel()}")
        pos = int(self._fp2[0, layer])
        if pos >= lay.group_size:
            raise BufferOverflowError(f"fp2 is full (layer {layer}); the engine must flush before appending")
        self.fp_k[0, layer, 1, :, pos] = kt.to(self._dev, torch.float16).reshape(lay.kv_heads, lay.head_dim)
        self.fp_v[0, layer, 1, :, pos] = vt.to(self._dev, torch.float16).reshape(lay.kv_heads, lay.head_dim)
        self._fp2[0, layer] = pos + 1
        if np.all(self._fp2[0] == self._fp2[0, 0]):
            self.d_fp2_len[0] = int(self._fp2[0, 0])
            self.d_pos[0] = self.seq_len

    def _advance(self, n: int) -> None:
        """Account for n rows the device forward appended to every layer (single sequence)."""
        if self.fp2_len + n > self.layout.group_size:
            raise BufferOverflowError("fp2 overflow")
        self._fp2 += n
        _lib.call("qs_add_int", self.d_fp2_len.data_ptr(), self.batch, n, _lib.stream_ptr())
        _lib.call("qs_add_int", self.d_pos.data_ptr(), self.batch, n, _lib.stream_ptr())

    def rollback(self, n_reject: int) -> None:
        """Drop the last ``n_reject`` fp2 tokens in every layer (Q/cache.py:236-247)."""
        self._single("rollback")
        if n_reject < 0:
            raise ConfigError(f"rollback count must be nonnegative, got {n_reject}")
        if n_reject == 0:
            return
        self.check_layer_consistency()
        if n_reject > self.fp2_len:
            raise CacheIntegrityError(f"cannot roll back {n_reject} tokens; fp2 holds only {self.fp2_len}")
        self._fp2 -= n_reject
        _lib.call("qs_add_int", self.d_fp2_len.data_ptr(), self.batch, -n_reject, _lib.stream_ptr())
        _lib.call("qs_add_int", self.d_pos.data_ptr(), self.batch, -n_reject, _lib.stream_ptr())

    # -- flush (Q/cache.py:249-281) ------------------------------------------------
    def flush_due(self) -> np.ndarray:
        """Per sequence: 0 = no flush, 1 = quantise fp1 (device kernel), 2 = short-fp1 top-up."""
        g = self.layout.group_size
        full = self._fp2[:, 0] == g
        return np.where(full, np.where(self._fp1 == g, 1, 2), 0)

    def launch_device_flush(self, stream=None) -> None:
        """Enqueue the device-conditioned flush of every sequence whose lengths say so (K1 + rotate);
        stream ordered, no host sync -- the engine captures it into the decode cycle graph."""
        _lib.call("qs_kv_flush", self.store_struct(), self.d_n_blocks.data_ptr(), self.d_fp1_len.data_ptr(),
                  self.d_fp2_len.data_ptr(), self.d_flags.data_ptr(), _lib.stream_ptr(stream))

    def commit_flush(self, due: np.ndarray) -> None:
        """Host-mirror side of a flush: the full-fp1 sequences were flushed on the device; the
        short-fp1 ones are topped up here (rare: only after a prompt shorter than 2G)."""
        g = self.layout.group_size
        for b in np.nonzero(due == 1)[0]:
            self._nq[b] += g
            self._fp2[b, :] = 0
        for b in np.nonzero(due == 2)[0]:
            self._short_topup(int(b))

    def _short_topup(self, b: int) -> None:
        g = self.layout.group_size
        short = int(self._fp1[b])
        take = g - short
        self.fp_k[b, :, 0, :, short:g] = self.fp_k[b, :, 1, :, :take]
        self.fp_v[b, :, 0, :, short:g] = self.fp_v[b, :, 1, :, :take]
        keep_k = self.fp_k[b, :, 1, :, take:g].clone()
        keep_v = self.fp_v[b, :, 1, :, take:g].clone()
        self.fp_k[b, :, 1, :, :short] = keep_k
        self.fp_v[b, :, 1, :, :short] = keep_v
        self._fp2[b, :] = short
        self._fp1[b] = g
        self.d_fp1_len[b] = g
        self.d_fp2_len[b] = short

    def flush_if_full(self) -> bool:
        """Quantise fp1 and rotate fp2 into it once fp2 is full (Q/cache.py:249-281); sequence 0's
        answer is returned (every due sequence of a batch is flushed).  Non-finite K/V raise
        DataError here, as the reference's quantiser does (Q/quant.py:60-64)."""
        self.check_layer_consistency()
        due = self.flush_due()
        if not due.any():
            return False
        if (due == 1).any():
            self.ensure_blocks(int(self._nq.max()) // self.layout.group_size + 1)
            self.launch_device_flush()
            self.raise_device_flags("flush_if_full")
        self.commit_flush(due)
        return bool(due[0])

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

    def _arch_rows(self, layer: int, r0: int, r1: int, seq: int = 0) -> tuple[np.ndarray, np.ndarray]:
        lay = self.layout
        slot = self._sens.index(layer)
        n = r1 - r0
        k = self.arch_k[seq, slot, :, r0:r1].permute(1, 0, 2).reshape(n, lay.kv_dim)
        v = self.arch_v[seq, slot, :, r0:r1].permute(1, 0, 2).reshape(n, lay.kv_dim)
        return k.float().cpu().numpy(), v.float().cpu().numpy()

    def quantized_region(self, layer: int, kind: str, seq: int = 0):
        """f32 dequantised quantised history [n_q, kv_dim] (device kernel, f64 math)."""
        torch = _torch()
        lay = self.layout
        nb = int(self._nq[seq]) // lay.group_size
        if nb == 0:
            return None
        ok = torch.empty((nb * lay.group_size, lay.kv_dim), dtype=torch.float32, device=self._dev)
        ov = torch.empty_like(ok)
        _lib.call("qs_kv_dequant_view", self.store_struct(), seq, layer, nb, 1 if kind == "target" else 0,
                  ok.data_ptr(), ov.data_ptr(), _lib.stream_ptr())
        return ok.cpu().numpy(), ov.cpu().numpy()

    def _view(self, layer: int, kind: str, seq: int = 0) -> CacheView:
        lay = self.layout
        if not 0 <= layer < lay.num_layers:
            raise ConfigError(f"layer index {layer} out of range")
        view = CacheView(segments=[])
        code_bytes = DRAFT_CODE_BYTES if kind == "draft" else TARGET_CODE_BYTES
        nq = int(self._nq[seq])
        if layer in lay.sensitive_layers:
            if nq:
                k, v = self._arch_rows(layer, 0, nq, seq)
                view.segments.append((k, v))
                view.fp_bytes += FP_ELEM_BYTES * (k.size + v.size)
        elif nq:
            k, v = self.quantized_region(layer, kind, seq)
            view.segments.append((k, v))
            elems = k.size + v.size
            view.quantized_elements += elems
            view.quantized_bytes += code_bytes * elems
            groups = self._groups_per_block() * (nq // lay.group_size)
            if kind == "target":
                groups *= 2
            view.param_bytes += quant.PARAM_PAIR_BYTES * groups
        for which, n in ((0, int(self._fp1[seq])), (1, int(self._fp2[seq, layer]))):
            if n:
                view.segments.append(self._fp_rows(which, layer, n, seq))
                view.fp_bytes += FP_ELEM_BYTES * 2 * n * lay.kv_dim
        return view

    def _groups_per_block(self) -> int:
        """Key groups (one per channel) + value groups (ceil(kv/G) per token) of one block."""
        lay = self.layout
        return lay.kv_dim + lay.group_size * (-(-lay.kv_dim // lay.group_size))

    # ------------------------------------------------------- accounting / export
    def memory_report(self) -> MemoryReport:
        """Exact modeled byte totals (Q/cache.py:384-403) of sequence 0."""
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

        def codes(t, word_idx, nib):  # [G][kv] nibble values of every head
            words = t[seq, layer, :, block].contiguous().cpu().numpy().view(np.uint32)
            return np.concatenate([layout.unpack_block(words[h], word_idx, nib) for h in range(H)], axis=1)

        cku, ckl = codes(self.ku, kw, kn), codes(self.kl, kw, kn) - 8
        cvu, cvl = codes(self.vu, vw, vn), codes(self.vl, vw, vn) - 8
        kp = self.kp[seq, layer, :, block].cpu().numpy().reshape(kv, 2)          # channel-major (S, Z)
        vpp = self.vp[seq, layer, :, block].cpu().numpy()                         # [H][G][2]
        ngv = -(-kv // G)
        heads = [(j * G) // hd for j in range(ngv)]                               # first head of value group j
        vsz = np.stack([vpp[h] for h in heads], axis=1).reshape(G * ngv, 2)       # token-major groups
        count = G * kv

        def plane(c, s, z, mode, axis, rl):
            return quant.QuantPlane(quant.pack_nibbles(c), count, G, np.ascontiguousarray(s, np.float32),
                                    np.ascontiguousarray(z, np.float32), mode, axis, rl)

        sixteenth = np.float32(1.0 / 16.0)
        return (plane(cku.T.reshape(-1), kp[:, 0], kp[:, 1], quant.MODE_ASYM_U4, quant.AXIS_CHANNEL, None),
                plane(ckl.T.reshape(-1), kp[:, 0] * sixteenth, np.zeros(kv), quant.MODE_SYM_S4, quant.AXIS_CHANNEL, None),
                plane(cvu.reshape(-1), vsz[:, 0], vsz[:, 1], quant.MODE_ASYM_U4, quant.AXIS_TOKEN, kv),
                plane(cvl.reshape(-1), vsz[:, 0] * sixteenth, np.zeros(G * ngv), quant.MODE_SYM_S4, quant.AXIS_TOKEN, kv))

    def import_block_planes(self, layer: int, block: int, planes, seq: int = 0) -> None:
        """Inverse of export_block_planes (snapshot load)."""
        torch = _torch()
        lay = self.layout
        G, hd, H, kv = lay.group_size, lay.head_dim, lay.kv_heads, lay.kv_dim
        kw, kn, vw, vn = layout.block_maps(G, hd)
        ku, kl, vu, vl = planes
        nwords = G * hd // 8
        per_plane = ((self.ku, ku.unpacked().astype(np.int64).reshape(kv, G).T, kw, kn),
                     (self.kl, kl.unpacked().astype(np.int64).reshape(kv, G).T + 8, kw, kn),
                     (self.vu, vu.unpacked().astype(np.int64).reshape(G, kv), vw, vn),
                     (self.vl, vl.unpacked().astype(np.int64).reshape(G, kv) + 8, vw, vn))
        for dst, c, wi, ni in per_plane:
            words = np.stack([layout.pack_block(c[:, h * hd:(h + 1) * hd], wi, ni, nwords) for h in range(H)])
            dst[seq, layer, :, block] = torch.from_numpy(words.view(np.uint8).reshape(H, -1)).to(self._dev)
        kpar = np.stack([ku.scales, ku.zeros], axis=-1).reshape(H, hd, 2)
        self.kp[seq, layer, :, block] = torch.from_numpy(np.ascontiguousarray(kpar, np.float32)).to(self._dev)
        ngv = -(-kv // G)
        vs, vz = vu.scales.reshape(G, ngv), vu.zeros.reshape(G, ngv)
        vpar = np.stack([np.stack([vs[:, (h * hd) // G], vz[:, (h * hd) // G]], axis=-1) for h in range(H)])
        self.vp[seq, layer, :, block] = torch.from_numpy(np.ascontiguousarray(vpar, np.float32)).to(self._dev)

    # --------------------------------------------------------------- snapshots
    def to_snapshot(self) -> qskv.Snapshot:
        """Sequence 0 as a QSKV snapshot value (fp rows as their exact fp16 values in f32)."""
        self.check_layer_consistency()
        lay = self.layout
        G, nb = lay.group_size, self.quantized_token_count // lay.group_size
        layers = []
        for layer in range(lay.num_layers):
            lc = qskv.LayerContent()
            if layer in lay.sensitive_layers:
                lc.archived = [self._arch_rows(layer, b * G, (b + 1) * G) for b in range(nb)]
            else:
                lc.blocks = [self.export_block_planes(layer, b) for b in range(nb)]
            lc.fp1 = self._fp_rows(0, layer, self.fp1_len)
            lc.fp2 = self._fp_rows(1, layer, self.fp2_len)
            layers.append(lc)
        return qskv.Snapshot(lay.num_layers, lay.kv_heads, lay.head_dim, G, tuple(sorted(lay.sensitive_layers)),
                             self.quantized_token_count, self.fp1_len, self.fp2_len, layers)

    @classmethod
    def from_snapshot(cls, snap: qskv.Snapshot) -> "HierarchicalKVCache":
        torch = _torch()
        lay = CacheLayout(snap.num_layers, snap.num_heads, snap.head_dim, snap.group_size, frozenset(snap.sensitive))
        G, H, hd = snap.group_size, snap.num_heads, snap.head_dim
        cache = cls(lay, max_tokens=snap.quantized + 2 * G)

        def put(dst, rows):  # f32 [n, kv] -> fp16 head-major rows
            n = rows.shape[0]
            if n:
                dst[:, :n] = torch.from_numpy(rows).reshape(n, H, hd).permute(1, 0, 2).to(cache._dev, torch.float16)

        for layer, lc in enumerate(snap.layers):
            if layer in lay.sensitive_layers:
                slot = cache._sens.index(layer)
                r0 = 0
                for k, v in lc.archived:
                    put(cache.arch_k[0, slot, :, r0:], k)
                    put(cache.arch_v[0, slot, :, r0:], v)
                    r0 += k.shape[0]
            else:
                for b, quartet in enumerate(lc.blocks):
                    cache.import_block_planes(layer, b, quartet)
            for which, (k, v) in ((0, lc.fp1), (1, lc.fp2)):
                put(cache.fp_k[0, layer, which], k)
                put(cache.fp_v[0, layer, which], v)
        cache._nq[0], cache._fp1[0] = snap.quantized, snap.fp1_len
        cache._fp2[0, :] = snap.fp2_len
        cache.d_n_blocks.fill_(snap.quantized // G)
        cache.d_fp1_len.fill_(snap.fp1_len)
        cache.d_fp2_len.fill_(snap.fp2_len)
        cache.d_pos.fill_(snap.quantized + snap.fp1_len + snap.fp2_len)
        return cache

    def save_snapshot(self, path) -> None:
        """QSKV file of Q/cache.py:405-447 (readable by the reference)."""
        with open(path, "wb") as f:
            f.write(qskv.encode(self.to_snapshot()))

    @classmethod
    def load_snapshot(cls, path) -> "HierarchicalKVCache":
        with open(path, "rb") as f:
            return cls.from_snapshot(qskv.decode(f.read()))


# -----------------------------------------------------------------------------
# fp16 cache (lossless runs and the FP16 autoregressive baseline)
# -----------------------------------------------------------------------------


class FpKVCache:
    """Device fp16 cache with the same append/rollback/view surface (Q/cache.py:561-656).

    Rows live head-major ``[B][L][Hkv][cap][hd]`` so the attention kernel streams one head's
    history contiguously.  Capacity doubles when it runs out, as the reference's does
    (Q/cache.py:606-612); ``generation`` bumps so runners and graphs rebuild.
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
        self._lens = np.zeros((batch, num_layers), dtype=np.int64)
        self.d_len = torch.zeros(batch, dtype=torch.int32, device=self._dev)
        self.d_flags = torch.zeros(1, dtype=torch.int32, device=self._dev)
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
        self._lens[seq, :] = s_p
        self.d_len[seq] = s_p

    @property
    def _len(self) -> np.ndarray:  # per-layer lengths of sequence 0 (reference protocol)
        return self._lens[0]

    @property
    def seq_len(self) -> int:
        return int(self._lens[0, 0])

    def seq_lens(self) -> np.ndarray:
        return self._lens[:, 0].copy()

    @property
    def quantized_token_count(self) -> int:
        return 0

    @property
    def capacity(self) -> int:
        return self._cap

    def fp2_space(self, seq: int = 0) -> int:
        return 1 << 30

    def check_layer_consistency(self) -> None:
        if not np.all(self._lens == self._lens[:, :1]):
            raise CacheIntegrityError(f"per-layer append counts diverged: {self._lens.tolist()}")

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

    ensure_tokens = _ensure

    def append_decode_token(self, layer: int, k, v) -> None:
        torch = _torch()
        kt = k if isinstance(k, torch.Tensor) else torch.from_numpy(np.asarray(k, dtype=np.float32).ravel())
        vt = v if isinstance(v, torch.Tensor) else torch.from_numpy(np.asarray(v, dtype=np.float32).ravel())
        if kt.numel() != self.kv_dim or vt.numel() != self.kv_dim:
            raise DimensionError(f"expected kv rows of width {self.kv_dim}")
        pos = int(self._lens[0, layer])
        self._ensure(pos + 1)
        self.k[0, layer, :, pos] = kt.to(self._dev, torch.float16).reshape(self.kv_heads, self.head_dim)
        self.v[0, layer, :, pos] = vt.to(self._dev, torch.float16).reshape(self.kv_heads, self.head_dim)
        self._lens[0, layer] = pos + 1
        if np.all(self._lens[0] == self._lens[0, 0]):
            self.d_len[0] = int(self._lens[0, 0])

    def _advance(self, n: int) -> None:
        self._ensure(int(self._lens.max()) + n)
        self._lens += n
        _lib.call("qs_add_int", self.d_len.data_ptr(), self.batch, n, _lib.stream_ptr())

    def rollback(self, n_reject: int) -> None:
        if n_reject < 0:
            raise ConfigError(f"rollback count must be nonnegative, got {n_reject}")
        if n_reject == 0:
            return
        self.check_layer_consistency()
        if n_reject > int(self._lens[:, 0].min()):
            raise CacheIntegrityError("rollback past the sequence start")
        self._lens -= n_reject
        _lib.call("qs_add_int", self.d_len.data_ptr(), self.batch, -n_reject, _lib.stream_ptr())

    def flush_if_full(self) -> bool:
        return False

    def raise_device_flags(self, what: str, flags: int | None = None) -> None:
        f = int(self.d_flags.item()) if flags is None else int(flags)
        if f:
            self.d_flags.zero_()
            if f & _lib.FLAG_OVERFLOW:
                raise BufferOverflowError(f"{what}: fp16 cache capacity {self._cap} exceeded")
            raise DataError(f"{what}: device status {f:#x}")

    def _view(self, layer: int, seq: int = 0) -> CacheView:
        n = int(self._lens[seq, layer])
        k = self.k[seq, layer, :, :n].permute(1, 0, 2).reshape(n, self.kv_dim).float().cpu().numpy()
        v = self.v[seq, layer, :, :n].permute(1, 0, 2).reshape(n, self.kv_dim).float().cpu().numpy()
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
