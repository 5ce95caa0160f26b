"""CPU tests of the host-side logic around the kernels: fragment layouts,
launch planning, gate/up interleave, batch partition.
Nothing here launches a kernel (no GPU in the CPU suite)."""

import ctypes

import numpy as np
import pytest

from paper_2502_10424_b200 import layout
from paper_2502_10424_b200.parallel import job_throughput, partition
from paper_2502_10424_b200.runtime import Geometry, interleave_cols, plan_attention_splits


# ---------------------------------------------------------------------------
# frag4 layout == the mma.sync m16n8k16 A-fragment definition
# ---------------------------------------------------------------------------


def _unpack_u4_raw(word: int):
    """Python statement of qs_common.cuh unpack_u4_raw: the four A registers as
    (lo, hi) half pairs of offset codes (1024 + c, or 1024 + 16c for rows g+8)."""
    x, t = word, word >> 8
    regs = [x & 0x000F000F, x & 0x00F000F0, t & 0x000F000F, t & 0x00F000F0]
    out = []
    for j, r in enumerate(regs):
        lo, hi = r & 0xFFFF, r >> 16
        if j & 1:  # high nibble of each byte: value 16c
            lo, hi = lo >> 4, hi >> 4
        out.append((lo, hi))
    return out


def test_frag4_matches_mma_a_fragment():
    """a0=(g, 2t..2t+1), a1=(g+8, 2t..), a2=(g, 2t+8..), a3=(g+8, 2t+8..) (PTX m16n8k16 .f16 A)."""
    rng = np.random.default_rng(0)
    tile = rng.integers(0, 16, size=(16, 16))
    words = np.zeros(32, dtype=np.int64)
    for r in range(16):
        for c in range(16):
            lane, nib = layout.frag_pos(r, c)
            words[lane] |= int(tile[r, c]) << (4 * int(nib))
    for lane in range(32):
        g, t = lane >> 2, lane & 3
        regs = _unpack_u4_raw(int(words[lane]))
        want = [(tile[g, 2 * t], tile[g, 2 * t + 1]), (tile[g + 8, 2 * t], tile[g + 8, 2 * t + 1]),
                (tile[g, 2 * t + 8], tile[g, 2 * t + 9]), (tile[g + 8, 2 * t + 8], tile[g + 8, 2 * t + 9])]
        assert regs == [tuple(int(v) for v in w) for w in want]


@pytest.mark.parametrize("G,hd", [(128, 128), (16, 16), (64, 64), (128, 64), (32, 128)])
def test_block_maps_are_bijections(G, hd):
    kw, kn, vw, vn = layout.block_maps(G, hd)
    nwords = G * hd // 8
    for w, n in ((kw, kn), (vw, vn)):
        slots = w * 8 + n
        assert slots.min() == 0 and slots.max() == nwords * 8 - 1
        assert np.unique(slots).size == G * hd


@pytest.mark.parametrize("G,hd", [(128, 128), (16, 16), (64, 128)])
def test_pack_unpack_block_round_trip(G, hd):
    rng = np.random.default_rng(G + hd)
    codes = rng.integers(0, 16, size=(G, hd))
    kw, kn, _, _ = layout.block_maps(G, hd)
    words = layout.pack_block(codes, kw, kn, G * hd // 8)
    assert np.array_equal(layout.unpack_block(words, kw, kn), codes)


# ---------------------------------------------------------------------------
# launch planning
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("heads", [1, 4, 8, 32, 64, 256])
@pytest.mark.parametrize("occ", [1, 2, 3])
def test_attention_split_plan(heads, occ):
    n = plan_attention_splits(heads, 1024, occ)
    assert 1 <= n <= 1024
    slots = 148 * occ
    # one or two whole waves of main CTAs, never a sliver of a third
    assert n * heads <= 2 * slots or n == 1
    assert plan_attention_splits(heads, 3, occ) <= 3


def test_interleave_cols_gate_up_tiles():
    import torch

    K, N = 32, 48
    a = torch.arange(K * N, dtype=torch.float32).view(K, N)
    b = -a
    w = interleave_cols(a, b)
    assert w.shape == (K, 2 * N)
    for j in range(N // 16):
        assert torch.equal(w[:, 32 * j:32 * j + 16], a[:, 16 * j:16 * j + 16])
        assert torch.equal(w[:, 32 * j + 16:32 * j + 32], b[:, 16 * j:16 * j + 16])


def test_geometry_dims():
    g = Geometry(32, 4096, 32, 8, 128, 14336, 128256, 131072 + 512)
    assert g.nq == 4096 and g.nk == 1024


# ---------------------------------------------------------------------------
# batch partition across ranks (no collective on the data path)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("n,world", [(8, 1), (8, 2), (8, 4), (8, 8), (7, 3), (1, 4), (0, 2)])
def test_partition_covers_batch_once(n, world):
    parts = [partition(n, world, r) for r in range(world)]
    flat = [i for p in parts for i in p]
    assert flat == list(range(n))
    sizes = [len(p) for p in parts]
    assert max(sizes) - min(sizes) <= 1


def test_partition_rejects_bad_rank():
    with pytest.raises(ValueError):
        partition(8, 2, 2)


def test_job_throughput_single_process():
    jt = job_throughput(100, 2.0)
    assert jt.world == 1 and jt.rate == 50.0


def test_cli_config_resolution_and_gen_model(tmp_path):
    """The harness resolves defaults <- JSON file <- flags like the reference CLI (Q/cli.py:81-111) and
    gen-model writes the reference-format weights of the seed + 2 init stream (Q/cli.py:118-133)."""
    import json

    from paper_2502_10424_b200 import cli, model

    cfgf = tmp_path / "c.json"
    cfgf.write_text(json.dumps({"spec": {"gamma": 6}, "model": {"num_layers": 1}}))
    args = cli.build_parser().parse_args(["gen-model", "--config", str(cfgf), "--seed", "5", "--out", str(tmp_path),
                                          "--kv-quant", "false"])
    cfg = cli.resolve_config(args)
    assert cfg["spec"]["gamma"] == 6 and cfg["seed"] == 5 and cfg["quant"]["kv_quant"] is False
    assert cfg["model"]["num_heads"] == 4 and cfg["spec"]["decode_len"] == 90
    assert cli.main(["gen-model", "--config", str(cfgf), "--seed", "5", "--out", str(tmp_path)]) == 0
    w = model.load_weights(tmp_path / "weights.qspw")
    ref = model.init_weights(w.config, seed=7)
    assert all(np.array_equal(a, b) for (_, a), (_, b) in zip(w.named_tensors(), ref.named_tensors()))
    assert json.loads((tmp_path / "manifest.json").read_text())["seed"] == 5
