"""QSKV snapshot codec: the on-disk format of the reference's HierarchicalKVCache
(/root/reference/pkg/src/quantspec/cache.py:405-553), so a device cache and the reference
read and write each other's files byte for byte.

Layout (little endian): a file header {"QSKV", version u8, L, H, hd, G, n_sensitive u32}, the
sensitive layer ids (u32 each), the counters {quantized u64, fp1_len u32, fp2_len u32}, then per
layer either the archived fp32 blocks {rows u32, K f32[rows, kv], V f32[rows, kv]} (sensitive
layers) or the flushed blocks as four planes each (K upper, K lower, V upper, V lower), every
plane a header {count u64, group u32, row_len u32, axis u8, mode u8, n_groups u32} + packed codes
+ f32 scales + f32 zeros; and finally the layer's fp1 K, fp1 V, fp2 K, fp2 V rows as f32.

This module only converts between bytes and a neutral ``Snapshot`` value; cache.py builds one
from the device store and restores a store from one.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import quant
from .errors import FormatError

MAGIC = b"QSKV"
VERSION = 1

_FILE_HDR = np.dtype([("magic", "S4"), ("version", "u1"), ("L", "<u4"), ("H", "<u4"), ("hd", "<u4"),
                      ("G", "<u4"), ("n_sens", "<u4")])
_COUNTS = np.dtype([("quantized", "<u8"), ("fp1", "<u4"), ("fp2", "<u4")])
_PLANE_HDR = np.dtype([("count", "<u8"), ("group", "<u4"), ("row_len", "<u4"), ("axis", "u1"), ("mode", "u1"),
                       ("ngroups", "<u4")])
_AXES = (quant.AXIS_CHANNEL, quant.AXIS_TOKEN)
_MODES = (quant.MODE_ASYM_U4, quant.MODE_SYM_S4)


@dataclass
class LayerContent:
    blocks: list = field(default_factory=list)    # [(K_u, K_l, V_u, V_l) QuantPlane quartets]
    archived: list = field(default_factory=list)  # [(K f32 [rows, kv], V f32 [rows, kv])]
    fp1: tuple = None                              # (K, V) f32 [fp1_len, kv]
    fp2: tuple = None                              # (K, V) f32 [fp2_len, kv]


@dataclass
class Snapshot:
    num_layers: int
    num_heads: int  # KV heads (the reference format is MHA: heads * head_dim = kv_dim)
    head_dim: int
    group_size: int
    sensitive: tuple
    quantized: int
    fp1_len: int
    fp2_len: int
    layers: list

    @property
    def kv_dim(self) -> int:
        return self.num_heads * self.head_dim


# ----------------------------------------------------------------------------- encode


def encode(snap: Snapshot) -> bytes:
    parts = []
    hdr = np.zeros((), _FILE_HDR)
    hdr["magic"], hdr["version"] = MAGIC, VERSION
    hdr["L"], hdr["H"], hdr["hd"], hdr["G"] = snap.num_layers, snap.num_heads, snap.head_dim, snap.group_size
    hdr["n_sens"] = len(snap.sensitive)
    parts.append(hdr.tobytes())
    parts.append(np.asarray(sorted(snap.sensitive), "<u4").tobytes())
    cnt = np.zeros((), _COUNTS)
    cnt["quantized"], cnt["fp1"], cnt["fp2"] = snap.quantized, snap.fp1_len, snap.fp2_len
    parts.append(cnt.tobytes())
    for layer, lc in enumerate(snap.layers):
        if layer in snap.sensitive:
            parts.append(np.uint32(len(lc.archived)).astype("<u4").tobytes())
            for k, v in lc.archived:
                parts.append(np.uint32(k.shape[0]).astype("<u4").tobytes())
                parts += [np.asarray(k, "<f4").tobytes(), np.asarray(v, "<f4").tobytes()]
        else:
            parts.append(np.uint32(len(lc.blocks)).astype("<u4").tobytes())
            for quartet in lc.blocks:
                parts += [_plane_bytes(p) for p in quartet]
        for k, v in (lc.fp1, lc.fp2):
            parts += [np.asarray(k, "<f4").tobytes(), np.asarray(v, "<f4").tobytes()]
    return b"".join(parts)


def _plane_bytes(p: quant.QuantPlane) -> bytes:
    h = np.zeros((), _PLANE_HDR)
    h["count"], h["group"], h["row_len"] = p.count, p.group_size, p.row_len or 0
    h["axis"], h["mode"], h["ngroups"] = _AXES.index(p.axis), _MODES.index(p.mode), p.num_groups
    return h.tobytes() + np.asarray(p.codes, np.uint8).tobytes() + np.asarray(p.scales, "<f4").tobytes() + \
        np.asarray(p.zeros, "<f4").tobytes()


# ----------------------------------------------------------------------------- decode


class _Cursor:
    def __init__(self, data: bytes):
        self.buf = memoryview(data)
        self.off = 0

    def take(self, n: int) -> memoryview:
        if self.off + n > len(self.buf):
            raise FormatError("snapshot truncated")
        out = self.buf[self.off : self.off + n]
        self.off += n
        return out

    def record(self, dt: np.dtype):
        return np.frombuffer(self.take(dt.itemsize), dt)[0]

    def u32(self, n: int = 1) -> np.ndarray:
        return np.frombuffer(self.take(4 * n), "<u4")

    def f32(self, rows: int, cols: int) -> np.ndarray:
        return np.frombuffer(self.take(4 * rows * cols), "<f4").reshape(rows, cols).astype(np.float32)


def decode(data: bytes) -> Snapshot:
    cur = _Cursor(data)
    if len(data) < 4 or bytes(data[:4]) != MAGIC:
        raise FormatError(f"bad snapshot magic {bytes(data[:4])!r}")
    hdr = cur.record(_FILE_HDR)
    if int(hdr["version"]) != VERSION:
        raise FormatError(f"unsupported snapshot version {int(hdr['version'])}")
    L, H, hd, G = (int(hdr[k]) for k in ("L", "H", "hd", "G"))
    sens = tuple(int(x) for x in cur.u32(int(hdr["n_sens"])))
    cnt = cur.record(_COUNTS)
    fp1_len, fp2_len = int(cnt["fp1"]), int(cnt["fp2"])
    kv = H * hd
    layers = []
    for layer in range(L):
        lc = LayerContent()
        n = int(cur.u32()[0])
        for _ in range(n):
            if layer in sens:
                rows = int(cur.u32()[0])
                lc.archived.append((cur.f32(rows, kv), cur.f32(rows, kv)))
            else:
                lc.blocks.append(tuple(_read_plane(cur) for _ in range(4)))
        lc.fp1 = (cur.f32(fp1_len, kv), cur.f32(fp1_len, kv))
        lc.fp2 = (cur.f32(fp2_len, kv), cur.f32(fp2_len, kv))
        layers.append(lc)
    return Snapshot(L, H, hd, G, sens, int(cnt["quantized"]), fp1_len, fp2_len, layers)


def _read_plane(cur: _Cursor) -> quant.QuantPlane:
    h = cur.record(_PLANE_HDR)
    count, ng = int(h["count"]), int(h["ngroups"])
    if int(h["axis"]) >= len(_AXES) or int(h["mode"]) >= len(_MODES):
        raise FormatError("bad plane header")
    codes = np.frombuffer(cur.take((count + 1) // 2), np.uint8).copy()
    scales = np.frombuffer(cur.take(4 * ng), "<f4").astype(np.float32)
    zeros = np.frombuffer(cur.take(4 * ng), "<f4").astype(np.float32)
    return quant.QuantPlane(codes, count, int(h["group"]), scales, zeros, _MODES[int(h["mode"])], _AXES[int(h["axis"])],
                            int(h["row_len"]) or None)
