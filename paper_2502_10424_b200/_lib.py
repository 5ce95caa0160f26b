"""ctypes binding of the C ABI in include/quantspec_b200.h.

The library is mandatory: importing the compute entry points without a built
``libqsb200.so`` (or without an sm_100 GPU at call time) raises -- there is
no CPU fallback anywhere in this package.
"""

from __future__ import annotations

import ctypes as C
import os

from . import errors

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QS_LIB") or os.path.join(_PKG, "libqsb200.so")  # QS_LIB: A/B builds

VIEW_DRAFT, VIEW_TARGET, VIEW_FP16 = 0, 1, 2
EPI_STORE, EPI_ADD, EPI_QKV, EPI_SILU_MUL = 0, 1, 2, 3
MAX_COLS = 48  # QS_MAX_COLS: activation rows (B * T) of one linear launch
# device status word bits (d_flags / Runner.flags)
FLAG_NONFINITE, FLAG_VOCAB, FLAG_OVERFLOW, FLAG_POSITION = 1, 2, 4, 8
W_F16, W_INT4 = 0, 1

vp = C.c_void_p
i32 = C.c_int
i64 = C.c_int64
f32 = C.c_float


MAX_RANKS = 8  # QS_MAX_RANKS


class GatherArgs(C.Structure):
    """qs_gather_args: fused all-gather of KV-head-sharded attention rows (world = 0: off)."""

    _fields_ = [
        ("world", i32), ("rank", i32), ("q_col_offset", i32), ("arrivals", i32),
        ("par_stride_h", i64), ("par_stride_s", i64),
        ("gh", vp * MAX_RANKS), ("gs", vp * MAX_RANKS), ("flag", vp * MAX_RANKS),
        ("epoch", vp), ("done", vp),
    ]


class AttnArgs(C.Structure):
    _fields_ = [
        ("B", i32), ("Hkv", i32), ("hd", i32), ("G", i32), ("T", i32), ("r", i32),
        ("n_queries", i32), ("n_qgroups", i32), ("n_main", i32), ("row_offset", i32),
        ("main_is_fpcache", i32), ("fpcache_cps", i32), ("sm_scale_log2", f32),
        ("q", vp), ("out", vp), ("q_row_stride", i64),
        ("n_blocks", vp), ("fp1_len", vp), ("fp2_len", vp), ("fp_len", vp),
        ("ku", vp), ("kl", vp), ("vu", vp), ("vl", vp),
        ("plane_seq_stride", i64), ("plane_head_stride", i64),
        ("kp", vp), ("vp", vp),
        ("kp_seq_stride", i64), ("kp_head_stride", i64), ("vp_seq_stride", i64), ("vp_head_stride", i64),
        ("main_k", vp), ("main_v", vp), ("main_seq_stride", i64), ("main_head_stride", i64),
        ("fp1_k", vp), ("fp1_v", vp), ("fp2_k", vp), ("fp2_v", vp), ("fp_seq_stride", i64), ("fp_rows", i32),
        ("partials", vp), ("counters", vp), ("dbg", i32),
        ("out_h", vp), ("ld_out_h", i64), ("out_s", vp), ("ld_out_s", i64),
        ("gather", GatherArgs),
    ]


class LinearArgs(C.Structure):
    _fields_ = [
        ("wmode", i32), ("epi", i32), ("N", i32), ("K", i32), ("ncols", i32), ("wgroup", i32),
        ("w", vp), ("wparams", vp), ("xh", vp), ("ldxh", i64), ("xs", vp), ("ldxs", i64),
        ("y", vp), ("ldy", i64), ("yh", vp), ("ldyh", i64), ("ys", vp), ("ldys", i64),
        ("Nq", i32), ("Nk", i32), ("hd", i32), ("T", i32),
        ("q_out", vp), ("k_dst", vp), ("v_dst", vp), ("kv_seq_stride", i64), ("kv_head_stride", i64),
        ("row_base", vp), ("row_offset", i32), ("row_cap", i32), ("pos_base", vp), ("rope", vp), ("max_pos", i32),
        ("flags", vp), ("dbg", i32),
        ("xf", vp), ("ldxf", i64), ("gain", vp), ("eps", C.c_float),
    ]


class KVStore(C.Structure):
    _fields_ = [
        ("B", i32), ("L", i32), ("Hkv", i32), ("hd", i32), ("G", i32), ("max_blocks", i32), ("fp_rows", i32),
        ("ku", vp), ("kl", vp), ("vu", vp), ("vl", vp), ("kp", vp), ("vp", vp),
        ("fp_k", vp), ("fp_v", vp), ("arch_k", vp), ("arch_v", vp),
        ("sens_mask", C.c_uint64 * 2),
    ]


_SIGS = {
    "qs_version": (C.c_char_p, []),
    "qs_last_error": (i32, [C.c_char_p, C.c_size_t]),
    "qs_device_check": (i32, []),
    "qs_encode_plane_hierarchical": (i32, [vp, i64, i32, i64, vp, vp, vp, vp, vp, vp, vp]),
    "qs_quantize_sym_s4": (i32, [vp, i64, f32, vp, vp, vp]),
    "qs_decode_plane": (i32, [vp, vp, vp, vp, i64, i32, i64, vp, vp]),
    "qs_quantize_weights": (i32, [vp, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp]),
    "qs_pack_weights_f16": (i32, [vp, i32, i32, vp, vp]),
    "qs_kv_quantize_blocks": (i32, [C.POINTER(KVStore), i32, i32, vp, vp, i64, i32, i32, vp, vp]),
    "qs_kv_flush": (i32, [C.POINTER(KVStore), vp, vp, vp, vp, vp]),
    "qs_kv_dequant_view": (i32, [C.POINTER(KVStore), i32, i32, i32, i32, vp, vp, vp]),
    "qs_attn_decode": (i32, [C.POINTER(AttnArgs), i32, vp]),
    "qs_attn_partials_floats": (i32, [C.POINTER(AttnArgs)]),
    "qs_attn_occupancy": (i32, [i32, i32, i32]),
    "qs_linear": (i32, [C.POINTER(LinearArgs), vp]),
    "qs_rmsnorm": (i32, [vp, vp, vp, i32, i32, f32, vp]),
    "qs_prep_act": (i32, [vp, vp, f32, vp, i64, vp, i64, i32, i32, vp]),
    "qs_embed": (i32, [vp, vp, i32, i32, vp, i32, i32, i32, vp, vp]),
    "qs_argmax": (i32, [vp, i32, i32, vp, i32, vp]),
    "qs_greedy_accept": (i32, [vp, i32, vp, i32, vp, i32, vp, vp, vp, vp]),
    "qs_add_int": (i32, [vp, i32, i32, vp]),
    "qs_dev_alloc": (i32, [C.c_size_t, C.POINTER(vp)]),
    "qs_dev_free": (i32, [vp]),
    "qs_ipc_handle": (i32, [vp, C.c_char_p]),
    "qs_ipc_open": (i32, [C.c_char_p, C.POINTER(vp)]),
    "qs_ipc_close": (i32, [vp]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def lib_path() -> str:
    return LIB_PATH


def load() -> C.CDLL:
    """Load libqsb200.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise errors.QuantSpecError(
                f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the B200 path has no CPU fallback)"
            )
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


_STATUS = {
    1: errors.DimensionError,
    2: errors.ConfigError,
    3: errors.DataError,
    4: errors.CacheIntegrityError,
    5: errors.BufferOverflowError,
    6: errors.QuantSpecError,
}


def check(status: int, what: str = "") -> None:
    if status == 0:
        return
    buf = C.create_string_buffer(512)
    load().qs_last_error(buf, 512)
    msg = buf.value.decode(errors="replace")
    raise _STATUS.get(status, errors.QuantSpecError)(f"{what}: {msg}" if what else msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t) -> int | None:
    return None if t is None else int(t.data_ptr())
