"""Bit-exact parallel replay of the reference init_weights stream (paper_2502_10424_b200/initstream.py),
used by bench.py to build the 7B/8B bench models from the reference's own draws (Q/model.py:89-117)."""

import numpy as np
import pytest

import paper_2502_10424_b200 as qs
from paper_2502_10424_b200 import initstream as S


def test_replay_equals_init_weights_gqa_toy():
    cfg = qs.ModelConfig(num_layers=3, num_heads=4, head_dim=16, hidden=64, mlp_hidden=176, vocab=96,
                         max_positions=512, num_kv_heads=2)
    w = qs.init_weights(cfg, seed=5)
    plan = S.draw_plan(3, 64, cfg.kv_dim, 176, 96)
    got = dict(S.stream_matrices(plan, S.walk_states(plan, 5, chunk_rows=7), threads=4, ahead=3))
    for i, lw in enumerate(w.layers):
        for n in S.MATS:
            assert np.array_equal(got[f"layers.{i}.{n}"], getattr(lw, n)), (i, n)
    assert np.array_equal(got["embedding"], w.embedding)
    assert np.array_equal(got["lm_head"], w.lm_head)


@pytest.mark.parametrize("shape,kv,mlp,vocab", [("llama2_7b", 4096, 11008, 32000), ("llama31_8b", 1024, 14336, 128256)])
def test_recorded_bench_states_continue_the_stream(shape, kv, mlp, vocab):
    """The committed states of the bench models: state 0 is the seed's initial state, and state 1
    (start of layer 0's wk) is where drawing wq from state 0 leaves the stream."""
    st = S.load_states(32, 4096, kv, mlp, vocab, 0)
    assert st is not None and len(st) == 32 * 7 + 2, shape
    plan = S.draw_plan(32, 4096, kv, mlp, vocab)
    assert S.walk_states(plan[:1], 0) == st[:1]
    rng = S._rng_at(st[0])
    rng.standard_normal((4096, 4096))
    nxt = rng.bit_generator.state
    assert int(nxt["state"]["state"]) == st[1]["state"] and int(nxt["state"]["inc"]) == st[1]["inc"]
    # and a replayed wq equals the direct draw
    full = S.draw(st[0], 4096, 4096, True)
    ref = (np.random.default_rng(0).standard_normal((4096, 4096)) / np.sqrt(4096)).astype(np.float32)
    assert np.array_equal(full, ref)
