"""QSPW weight-file codec: the on-disk format of the reference's save_weights / load_weights
(/root/reference/pkg/src/quantspec/model.py:415-524), so weights written by either side load on
the other byte for byte.

Layout (little endian): header {"QSPW", version u8, L, H, hd, d, mlp, V, max_positions u32,
rope_base f64, norm_eps f64, body_len u64}, the body -- a sequence of tensor records {name_len u16,
name utf-8, rank u8, dims u32[rank], data f32[prod(dims)]} in the model's named_tensors order --
then crc32(body) u32.

This module converts between bytes and (dims, {name: f32 array}); model.py maps those onto
ModelConfig / ModelWeights and validates shapes.
"""

from __future__ import annotations

import zlib

import numpy as np

from .errors import FormatError

MAGIC = b"QSPW"
VERSION = 1

_HDR = np.dtype([("magic", "S4"), ("version", "u1"), ("dims", "<u4", (7,)), ("rope_base", "<f8"),
                 ("norm_eps", "<f8"), ("body_len", "<u8")])
_CRC = np.dtype("<u4")


def encode(dims, rope_base: float, norm_eps: float, tensors) -> bytes:
    """``dims`` = (L, H, hd, d, mlp, V, max_positions); ``tensors`` = iterable of (name, array)."""
    body = []
    for name, arr in tensors:
        a = np.ascontiguousarray(arr, dtype="<f4")
        key = name.encode("utf-8")
        rec = np.zeros((), np.dtype([("n", "<u2"), ("name", f"S{len(key)}"), ("rank", "u1"),
                                     ("shape", "<u4", (a.ndim,))]))
        rec["n"], rec["name"], rec["rank"] = len(key), key, a.ndim
        if a.ndim:
            rec["shape"] = a.shape
        body.append(rec.tobytes())
        body.append(a.tobytes())
    payload = b"".join(body)
    hdr = np.zeros((), _HDR)
    hdr["magic"], hdr["version"], hdr["dims"] = MAGIC, VERSION, dims
    hdr["rope_base"], hdr["norm_eps"], hdr["body_len"] = rope_base, norm_eps, len(payload)
    return hdr.tobytes() + payload + np.asarray(zlib.crc32(payload), _CRC).tobytes()


def decode(raw: bytes):
    """-> (dims tuple, rope_base, norm_eps, {name: f32 ndarray}); FormatError on any damage."""
    if len(raw) < _HDR.itemsize:
        raise FormatError("weight file truncated")
    hdr = np.frombuffer(raw, _HDR, count=1)[0]
    if bytes(hdr["magic"]) != MAGIC:
        raise FormatError("bad weight-file magic")
    if int(hdr["version"]) != VERSION:
        raise FormatError(f"unsupported weight-file version {int(hdr['version'])}")
    start = _HDR.itemsize
    end = start + int(hdr["body_len"])
    if end + _CRC.itemsize > len(raw):
        raise FormatError("weight file truncated")
    body = memoryview(raw)[start:end]
    if zlib.crc32(body) != int(np.frombuffer(raw, _CRC, count=1, offset=end)[0]):
        raise FormatError("weight-file checksum mismatch")
    tensors = {}
    pos = 0
    while pos < len(body):
        if pos + 2 > len(body):
            raise FormatError("weight file truncated inside tensor table")
        n = int(np.frombuffer(body, "<u2", count=1, offset=pos)[0])
        if pos + 3 + n > len(body):
            raise FormatError("weight file truncated inside tensor table")
        name = bytes(body[pos + 2: pos + 2 + n]).decode("utf-8")
        rank = body[pos + 2 + n]
        pos += 3 + n
        if pos + 4 * rank > len(body):
            raise FormatError("weight file truncated inside tensor table")
        shape = tuple(int(x) for x in np.frombuffer(body, "<u4", count=rank, offset=pos))
        pos += 4 * rank
        cnt = int(np.prod(shape)) if rank else 1
        if pos + 4 * cnt > len(body):
            raise FormatError("weight file truncated inside tensor data")
        tensors[name] = np.frombuffer(body, "<f4", count=cnt, offset=pos).reshape(shape).astype(np.float32)
        pos += 4 * cnt
    return tuple(int(x) for x in hdr["dims"]), float(hdr["rope_base"]), float(hdr["norm_eps"]), tensors
