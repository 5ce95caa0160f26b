"""Host mirror of the device layouts in csrc/qs_layout.h.

Used only to *export* device planes into the reference QuantPlane packing
(snapshots, parity checks) and to size buffers; no arithmetic on KV values
happens here.
"""

from __future__ import annotations

from functools import lru_cache

import numpy as np

CHUNK_Q = 128
CHUNK_F = 64


def vec(ni: int) -> int:
    return 4 if ni >= 4 else ni


def frag_index(outer, inner, lane, ni: int):
    v = vec(ni)
    return ((outer * (ni // v) + inner // v) * 32 + lane) * v + inner % v


def frag_pos(row, col):
    """(lane, nibble) of element (row, col) of a 16x16 A tile (frag4)."""
    row = np.asarray(row)
    col = np.asarray(col)
    g, jlo = row & 7, row >> 3
    jhi, rem = col >> 3, col & 7
    t, h = rem >> 1, rem & 1
    return g * 4 + t, (jlo + 2 * jhi) + 4 * h


@lru_cache(maxsize=16)
def block_maps(G: int, hd: int):
    """Word index and nibble of every (token, channel) of one head-block plane.

    Returns (k_word, k_nib, v_word, v_nib), each int64 [G, hd].
    """
    ni = hd // 16
    tok, ch = np.meshgrid(np.arange(G), np.arange(hd), indexing="ij")
    lane, nib = frag_pos(tok & 15, ch & 15)
    kw = frag_index(tok >> 4, ch >> 4, lane, ni)
    lane_v, nib_v = frag_pos(ch & 15, tok & 15)
    vw = frag_index(tok >> 4, ch >> 4, lane_v, ni)
    return kw.astype(np.int64), nib.astype(np.int64), vw.astype(np.int64), nib_v.astype(np.int64)


def unpack_block(words: np.ndarray, word_idx: np.ndarray, nib: np.ndarray) -> np.ndarray:
    """Nibble values [G, hd] of one head-block plane given its u32 words."""
    w = words.astype(np.uint32)[word_idx]
    return ((w >> (4 * nib).astype(np.uint32)) & 0xF).astype(np.int64)


def pack_block(codes: np.ndarray, word_idx: np.ndarray, nib: np.ndarray, nwords: int) -> np.ndarray:
    """Inverse of unpack_block (used when loading reference planes)."""
    out = np.zeros(nwords, dtype=np.uint32)
    np.bitwise_or.at(out, word_idx.reshape(-1), (codes.reshape(-1).astype(np.uint32) & 0xF) << (4 * nib.reshape(-1)).astype(np.uint32))
    return out
