"""QSPW weight files: the codec (paper_2502_10424_b200/qspw.py) reads a file the
REFERENCE wrote (tests/golden/make_qspw_golden.py) into the bit-exact init_weights draw, writes it back
byte for byte, and rejects damaged files with FormatError as the reference does
(pkg/tests/test_model.py:240-262)."""

import os

import numpy as np
import pytest

import paper_2502_10424_b200 as qs
from paper_2502_10424_b200.errors import FormatError

from .conftest import GOLDEN

REF = os.path.join(GOLDEN, "ref_weights.qspw")
CFG = qs.ModelConfig(num_layers=2, num_heads=2, head_dim=8, hidden=16, mlp_hidden=24, vocab=40, max_positions=128)


def test_reference_file_round_trips_byte_for_byte(tmp_path):
    w = qs.load_weights(REF)
    assert w.config == CFG
    want = qs.init_weights(CFG, seed=9)
    for (n, a), (m, b) in zip(w.named_tensors(), want.named_tensors()):
        assert n == m and np.array_equal(a, b), n
    out = tmp_path / "w.qspw"
    qs.save_weights(out, w)
    with open(REF, "rb") as f:
        assert out.read_bytes() == f.read()


def test_gqa_weights_round_trip(tmp_path):
    cfg = qs.ModelConfig(num_layers=1, num_heads=4, head_dim=8, hidden=32, mlp_hidden=40, vocab=24, max_positions=64,
                         num_kv_heads=2)
    w = qs.init_weights(cfg, seed=1)
    qs.save_weights(tmp_path / "g.qspw", w)
    g = qs.load_weights(tmp_path / "g.qspw")
    assert g.config.kv_dim == 16 and np.array_equal(g.layers[0].wk, w.layers[0].wk)


@pytest.mark.parametrize("damage", ["magic", "version", "truncate", "crc", "shape"])
def test_damaged_files_raise_format_error(tmp_path, damage):
    with open(REF, "rb") as f:
        raw = bytearray(f.read())
    if damage == "magic":
        raw[0:4] = b"XXXX"
    elif damage == "version":
        raw[4] = 9
    elif damage == "truncate":
        raw = raw[: len(raw) // 2]
    elif damage == "crc":
        raw[200] ^= 0xFF
    else:  # a tensor with the wrong shape, valid checksum
        from paper_2502_10424_b200 import qspw

        dims, rb, eps, t = qspw.decode(bytes(raw))
        t["layers.1.wo"] = t["layers.1.wo"][:, :8]
        raw = bytearray(qspw.encode(dims, rb, eps, t.items()))
    p = tmp_path / "bad.qspw"
    p.write_bytes(bytes(raw))
    with pytest.raises(FormatError):
        qs.load_weights(p)
