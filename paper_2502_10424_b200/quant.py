"""Two-plane INT4 quantisation entry points, B200 edition.

Same names, argument meaning and error behaviour as the reference module
/root/reference/pkg/src/quantspec/quant.py; every encode/decode runs in the
sm_100a kernels of csrc/qs_quant.cu (f64 arithmetic, bit-exact codes and
params).  Only nibble packing -- a storage format, not arithmetic -- is done
with NumPy here.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import CacheIntegrityError, ConfigError, DataError

SCALE_FLOOR = 1e-8
LOWER_SCALE_DIV = 16.0
ASYM_LEVELS = 15
SYM_MIN = -8
SYM_MAX = 7

CODE_BYTES = 0.5
PARAM_PAIR_BYTES = 8.0

MODE_ASYM_U4 = "asymmetric_u4"
MODE_SYM_S4 = "symmetric_s4"

AXIS_CHANNEL = "channel"
AXIS_TOKEN = "token"


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise DataError("the B200 quantisation path needs a CUDA device (no CPU fallback)")
    return torch


@dataclass(frozen=True)
class GroupQuantParams:
    """Scale and zero point for one quantization group (Q/quant.py:40-52)."""

    scale: float
    zero_point: float
    mode: str

    def __post_init__(self) -> None:
        if self.scale <= 0.0:
            raise ConfigError(f"group scale must be positive, got {self.scale}")
        if self.mode not in (MODE_ASYM_U4, MODE_SYM_S4):
            raise ConfigError(f"unknown quantization mode {self.mode!r}")


# ---------------------------------------------------------------------------
# nibble packing (format helpers, Q/quant.py:137-158)
# ---------------------------------------------------------------------------


def pack_nibbles(codes: np.ndarray) -> np.ndarray:
    """Two 4-bit codes per byte, the low nibble holding the even index."""
    c = (np.asarray(codes).astype(np.int64) & 0xF).reshape(-1)
    if c.size % 2:
        c = np.concatenate([c, np.zeros(1, np.int64)])
    return (c[0::2] | (c[1::2] << 4)).astype(np.uint8)


def unpack_nibbles(packed: np.ndarray, count: int, *, signed: bool) -> np.ndarray:
    p = np.asarray(packed, dtype=np.uint8).reshape(-1)
    both = np.empty(p.size * 2, dtype=np.int16)
    both[0::2] = p & 0xF
    both[1::2] = p >> 4
    both = both[:count]
    if signed:
        return np.where(both >= 8, both - 16, both).astype(np.int8)
    return both.astype(np.uint8)


def _group_starts(count: int, group_size: int, row_len: int | None) -> np.ndarray:
    if row_len is None or row_len >= count:
        return np.arange(0, count, group_size, dtype=np.int64)
    if count % row_len:
        raise CacheIntegrityError(f"plane of {count} codes is not a whole number of {row_len}-rows")
    per_row = np.arange(0, row_len, group_size, dtype=np.int64)
    return (np.arange(0, count, row_len, dtype=np.int64)[:, None] + per_row[None, :]).reshape(-1)


@dataclass
class QuantPlane:
    """One packed 4-bit plane plus per-group parameters (Q/quant.py:166-207)."""

    codes: np.ndarray
    count: int
    group_size: int
    scales: np.ndarray
    zeros: np.ndarray
    mode: str
    axis: str
    row_len: int | None = None

    @property
    def num_groups(self) -> int:
        return int(self.scales.size)

    def group_params(self, i: int) -> GroupQuantParams:
        return GroupQuantParams(float(self.scales[i]), float(self.zeros[i]), self.mode)

    def unpacked(self) -> np.ndarray:
        return unpack_nibbles(self.codes, self.count, signed=self.mode == MODE_SYM_S4)

    def group_starts(self) -> np.ndarray:
        return _group_starts(self.count, self.group_size, self.row_len)

    def group_counts(self) -> np.ndarray:
        return np.diff(np.append(self.group_starts(), self.count))

    def code_bytes(self) -> float:
        return self.count * CODE_BYTES

    def param_bytes(self) -> float:
        return self.num_groups * PARAM_PAIR_BYTES


# ---------------------------------------------------------------------------
# device plane encode / decode
# ---------------------------------------------------------------------------


def _num_groups(count: int, group: int, row_len: int | None) -> int:
    if row_len is not None and 0 < row_len < count:
        return (count // row_len) * (-(-row_len // group))
    return -(-count // group)


def _encode_device(v: np.ndarray, group: int, row_len: int | None, lower: bool):
    torch = _torch()
    count = int(v.size)
    if count == 0:
        raise DataError("cannot quantize an empty group")
    if group < 1:
        if not bool(torch.isfinite(torch.from_numpy(v)).all()):
            raise DataError("group contains non-finite values")
        raise ConfigError(f"group size must be >= 1, got {group}")
    rl = int(row_len) if row_len else 0
    if rl and rl < count and count % rl:
        raise CacheIntegrityError(f"plane of {count} codes is not a whole number of {rl}-rows")
    dev = torch.device("cuda")
    tv = torch.from_numpy(np.ascontiguousarray(v)).to(dev)
    ng = _num_groups(count, group, row_len)
    nbytes = (count + 1) // 2
    up = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    lo = torch.empty(nbytes, dtype=torch.uint8, device=dev) if lower else None
    s = torch.empty(ng, dtype=torch.float32, device=dev)
    z = torch.empty(ng, dtype=torch.float32, device=dev)
    sl = torch.empty(ng, dtype=torch.float32, device=dev) if lower else None
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.call("qs_encode_plane_hierarchical", _lib.ptr(tv), count, group, rl, _lib.ptr(up), _lib.ptr(lo),
              _lib.ptr(s), _lib.ptr(z), _lib.ptr(sl), _lib.ptr(flags), _lib.stream_ptr())
    if int(flags.item()) & 1:
        raise DataError("group contains non-finite values")
    out = (up.cpu().numpy(), s.cpu().numpy(), z.cpu().numpy())
    if lower:
        out = out + (lo.cpu().numpy(), sl.cpu().numpy())
    return out


def encode_plane_asym(values, group_size: int, axis: str, row_len: int | None = None) -> QuantPlane:
    """Asymmetric upper-plane encoding (Q/quant.py:220-248), on device."""
    v = np.asarray(values, dtype=np.float64).ravel()
    up, s, z = _encode_device(v, group_size, row_len, lower=False)
    return QuantPlane(up, v.size, group_size, s, z, MODE_ASYM_U4, axis, row_len)


def encode_plane_hierarchical(values, group_size: int, axis: str, row_len: int | None = None):
    """Upper + lower plane encoding (Q/quant.py:251-276), on device."""
    v = np.asarray(values, dtype=np.float64).ravel()
    up, s, z, lo, sl = _encode_device(v, group_size, row_len, lower=True)
    upper = QuantPlane(up, v.size, group_size, s, z, MODE_ASYM_U4, axis, row_len)
    lower = QuantPlane(lo, v.size, group_size, sl, np.zeros_like(sl), MODE_SYM_S4, axis, row_len)
    return upper, lower


def _check_plane_pair(upper: QuantPlane, lower: QuantPlane) -> None:
    if upper.count != lower.count or upper.group_size != lower.group_size or upper.row_len != lower.row_len:
        raise CacheIntegrityError(
            "upper/lower planes disagree on group structure: "
            f"count {upper.count}/{lower.count}, group {upper.group_size}/{lower.group_size}"
        )
    if upper.mode != MODE_ASYM_U4 or lower.mode != MODE_SYM_S4:
        raise CacheIntegrityError("plane modes do not match the hierarchy")


def _decode_device(upper: QuantPlane, lower: QuantPlane | None) -> np.ndarray:
    torch = _torch()
    dev = torch.device("cuda")
    up = torch.from_numpy(np.ascontiguousarray(upper.codes)).to(dev)
    lo = torch.from_numpy(np.ascontiguousarray(lower.codes)).to(dev) if lower is not None else None
    s = torch.from_numpy(np.ascontiguousarray(upper.scales, dtype=np.float32)).to(dev)
    z = torch.from_numpy(np.ascontiguousarray(upper.zeros, dtype=np.float32)).to(dev)
    out = torch.empty(upper.count, dtype=torch.float64, device=dev)
    _lib.call("qs_decode_plane", _lib.ptr(up), _lib.ptr(lo), _lib.ptr(s), _lib.ptr(z), upper.count,
              upper.group_size, int(upper.row_len or 0), _lib.ptr(out), _lib.stream_ptr())
    return out.cpu().numpy()


def decode_plane_draft(plane: QuantPlane) -> np.ndarray:
    """Upper-plane reconstruction c_u*S + Z (f64), Q/quant.py:293-298."""
    return _decode_device(plane, None)


def decode_plane_target(upper: QuantPlane, lower: QuantPlane) -> np.ndarray:
    """Two-plane reconstruction c_u*S + c_l*S/16 + Z (f64), Q/quant.py:301-309."""
    _check_plane_pair(upper, lower)
    return _decode_device(upper, lower)


# ---------------------------------------------------------------------------
# single-group entry points (Q/quant.py:67-129): one-group planes on device
# ---------------------------------------------------------------------------


def quantize_group_asym_u4(values) -> tuple[np.ndarray, GroupQuantParams]:
    v = np.asarray(values, dtype=np.float64).ravel()
    if v.size == 0:
        raise DataError("cannot quantize an empty group")
    up, s, z = _encode_device(v, v.size, None, lower=False)
    codes = unpack_nibbles(up, v.size, signed=False)
    return codes, GroupQuantParams(float(s[0]), float(z[0]), MODE_ASYM_U4)


def quantize_group_sym_s4(errors, scale: float) -> tuple[np.ndarray, GroupQuantParams]:
    """Symmetric RTN with a caller-fixed scale (Q/quant.py:83-91), on device."""
    if scale <= 0.0:
        raise ConfigError(f"symmetric quantization needs a positive scale, got {scale}")
    e = np.asarray(errors, dtype=np.float64).ravel()
    if e.size == 0:
        raise DataError("cannot quantize an empty group")
    torch = _torch()
    sc = float(np.float32(scale))
    te = torch.from_numpy(np.ascontiguousarray(e)).cuda()
    out = torch.empty(e.size, dtype=torch.int8, device=te.device)
    flags = torch.zeros(1, dtype=torch.int32, device=te.device)
    _lib.call("qs_quantize_sym_s4", _lib.ptr(te), e.size, sc, _lib.ptr(out), _lib.ptr(flags), _lib.stream_ptr())
    if int(flags.item()) & 1:
        raise DataError("group contains non-finite values")
    return out.cpu().numpy(), GroupQuantParams(sc, 0.0, MODE_SYM_S4)


def hierarchical_encode(values):
    """Encode one group into (upper, lower) code/param pairs (Q/quant.py:94-104)."""
    v = np.asarray(values, dtype=np.float64).ravel()
    if v.size == 0:
        raise DataError("cannot quantize an empty group")
    up, s, z, lo, sl = _encode_device(v, v.size, None, lower=True)
    uc = unpack_nibbles(up, v.size, signed=False)
    lc = unpack_nibbles(lo, v.size, signed=True)
    return (uc, GroupQuantParams(float(s[0]), float(z[0]), MODE_ASYM_U4)), (
        lc,
        GroupQuantParams(float(sl[0]), 0.0, MODE_SYM_S4),
    )


def dequant_group_draft(codes: np.ndarray, params: GroupQuantParams) -> np.ndarray:
    c = np.asarray(codes).ravel()
    p = QuantPlane(pack_nibbles(c), c.size, max(c.size, 1), np.array([params.scale], np.float32),
                   np.array([params.zero_point], np.float32), MODE_ASYM_U4, AXIS_CHANNEL)
    return _decode_device(p, None)


def dequant_group_target(upper_codes, upper: GroupQuantParams, lower_codes, lower: GroupQuantParams) -> np.ndarray:
    uc = np.asarray(upper_codes).ravel()
    lc = np.asarray(lower_codes).ravel()
    if uc.shape != lc.shape:
        raise CacheIntegrityError(f"upper/lower planes disagree on group structure: {uc.shape} vs {lc.shape}")
    if lower.mode != MODE_SYM_S4 or upper.mode != MODE_ASYM_U4:
        raise CacheIntegrityError("plane modes do not match the hierarchy")
    n = max(uc.size, 1)
    pu = QuantPlane(pack_nibbles(uc), uc.size, n, np.array([upper.scale], np.float32),
                    np.array([upper.zero_point], np.float32), MODE_ASYM_U4, AXIS_CHANNEL)
    pl = QuantPlane(pack_nibbles(lc), lc.size, n, np.array([upper.scale / 16.0], np.float32),
                    np.zeros(1, np.float32), MODE_SYM_S4, AXIS_CHANNEL)
    return _decode_device(pu, pl)


# ---------------------------------------------------------------------------
# INT4 weights (Q/quant.py:317-356)
# ---------------------------------------------------------------------------


@dataclass
class QuantizedLinear:
    """A weight matrix stored as a single asymmetric 4-bit plane.

    ``frag``/``frag_params`` (device tensors) hold the same codes and params
    in the mma-fragment order the W4A16 kernel streams.
    """

    plane: QuantPlane
    shape: tuple[int, int]
    frag: object | None = None
    frag_params: object | None = None

    def code_bytes(self) -> float:
        return self.plane.code_bytes()

    def param_bytes(self) -> float:
        return self.plane.param_bytes()


def quantize_weights_device(w_dev, group_size: int, want_plane: bool = True, want_frag: bool = True):
    """Device entry: w_dev is a CUDA f32 tensor [d_in, d_out]."""
    torch = _torch()
    d_in, d_out = (int(x) for x in w_dev.shape)
    g = min(group_size, d_in)
    gpr = -(-d_in // g)
    dev = w_dev.device
    s = torch.empty(d_out * gpr, dtype=torch.float32, device=dev)
    z = torch.empty(d_out * gpr, dtype=torch.float32, device=dev)
    ref = torch.empty((d_in * d_out + 1) // 2, dtype=torch.uint8, device=dev) if want_plane else None
    frag = fparams = None
    if want_frag:
        ks_pad = (d_in // 16 + 3) // 4 * 4
        mt2 = (d_out // 16 + 1) // 2 * 2  # tile-pair-major layout pads to whole pairs
        frag = torch.empty(mt2 * ks_pad * 32, dtype=torch.int32, device=dev)
        fparams = torch.empty(mt2 * gpr * 8 * 4, dtype=torch.float32, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.call("qs_quantize_weights", _lib.ptr(w_dev), d_in, d_out, group_size, _lib.ptr(ref), _lib.ptr(s),
              _lib.ptr(z), _lib.ptr(frag), _lib.ptr(fparams), _lib.ptr(flags), _lib.stream_ptr())
    if int(flags.item()) & 1:
        raise DataError("weight matrix contains non-finite values")
    return ref, s, z, frag, fparams, g


def quantize_weights(w: np.ndarray, group_size: int) -> QuantizedLinear:
    """Quantize a [d_in, d_out] matrix to INT4 with input-dimension groups."""
    torch = _torch()
    w = np.asarray(w, dtype=np.float32)
    if w.ndim != 2 or w.size == 0:
        raise ConfigError(f"weight quantization expects a non-empty 2-D matrix, got shape {w.shape}")
    if not np.isfinite(w).all():
        raise DataError("weight matrix contains non-finite values")
    d_in, d_out = w.shape
    wd = torch.from_numpy(np.ascontiguousarray(w)).cuda()
    want_frag = d_in % 16 == 0 and d_out % 16 == 0 and min(group_size, d_in) % 16 == 0
    ref, s, z, frag, fparams, g = quantize_weights_device(wd, group_size, True, want_frag)
    plane = QuantPlane(ref.cpu().numpy(), d_in * d_out, g, s.cpu().numpy(), z.cpu().numpy(), MODE_ASYM_U4,
                       AXIS_CHANNEL, d_in)
    return QuantizedLinear(plane=plane, shape=(d_in, d_out), frag=frag, frag_params=fparams)


def dequantize_weights(q: QuantizedLinear) -> np.ndarray:
    """Float32 reconstruction with the original [d_in, d_out] shape."""
    d_in, d_out = q.shape
    flat = decode_plane_draft(q.plane)
    return np.ascontiguousarray(flat.reshape(d_out, d_in).T.astype(np.float32))
