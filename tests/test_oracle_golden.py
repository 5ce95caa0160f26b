"""Pin the CPU oracle (oracle/qs_oracle.py) to golden vectors produced by the
reference implementation itself (tests/golden/make_golden.py).  CPU only."""

import copy
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import qs_oracle as O

from .conftest import GOLDEN

TOY = O.Config(num_layers=2, num_heads=4, head_dim=16, hidden=64, mlp_hidden=176, vocab=64, max_positions=4096 + 128)


def load(name):
    return np.load(os.path.join(GOLDEN, name))


def test_plane_encode_bit_exact():
    z = load("quant_golden.npz")
    for i in range(int(z["n_cases"])):
        g, rl = (int(x) for x in z[f"c{i}_group"])
        up, lo = O.encode_plane_hier(z[f"c{i}_values"], g, "channel", rl or None)
        for tag, p in (("up", up), ("lo", lo)):
            assert np.array_equal(p.codes, z[f"c{i}_{tag}_codes"]), (i, tag)
            assert np.array_equal(p.scales.view(np.uint32), z[f"c{i}_{tag}_scales"].view(np.uint32)), (i, tag)
            assert np.array_equal(p.zeros.view(np.uint32), z[f"c{i}_{tag}_zeros"].view(np.uint32)), (i, tag)
        assert np.array_equal(O.decode_draft(up), z[f"c{i}_draft"])
        assert np.array_equal(O.decode_target(up, lo), z[f"c{i}_target"])


def test_group_kats():
    with open(os.path.join(GOLDEN, "group_kat.json")) as f:
        kats = json.load(f)
    for k in kats:
        (cu, s, zp), (cl, sl) = O.group_encode(k["values"])
        assert cu.tolist() == k["cu"] and cl.tolist() == k["cl"]
        assert s == k["S"] and zp == k["Z"] and sl == k["Sl"]
    # reference worked examples (pkg/tests/test_quant.py:36-41, :90-99)
    (cu, s, zp), (cl, sl) = O.group_encode([0.0, 1.07, 2.0, 3.0])
    assert cu.tolist() == [0, 5, 10, 15] and cl[1] == 6 and cl[2] == 0


def test_weight_quant_bit_exact():
    z = load("quant_golden.npz")
    w = z["w_in"]
    for g in (32, 16, 7):
        p = O.quantize_matrix(w, g)
        assert np.array_equal(p.codes, z[f"w{g}_codes"])
        assert np.array_equal(p.scales, z[f"w{g}_scales"])
        assert np.array_equal(p.zeros, z[f"w{g}_zeros"])
        assert np.array_equal(O.dequantize_matrix(p, w.shape), z[f"w{g}_deq"])


def replay_cache_script():
    z = load("cache_golden.npz")
    with open(os.path.join(GOLDEN, "cache_script.json")) as f:
        script = json.load(f)
    lay = O.Layout(2, 2, 16, 16)
    c = O.OracleKVCache.from_prefill(lay, [z["keys0"], z["keys1"]], [z["vals0"], z["vals1"]])
    ak, av = z["appended_k"], z["appended_v"]
    for op, arg in script:
        if op == "append":
            for layer in range(2):
                c.append_decode_token(layer, ak[arg][layer], av[arg][layer])
        elif op == "rollback":
            c.rollback(arg)
        elif op == "flush":
            assert int(c.flush_if_full()) == arg
        else:
            assert [c.quantized_token_count, c.fp1_len, c.fp2_len] == arg
    return c, z


def test_cache_state_machine_and_views():
    c, z = replay_cache_script()
    for layer in range(2):
        for kind in ("draft", "target"):
            vw = c.view(layer, kind)
            assert np.array_equal(vw.k, z[f"view_{kind}_{layer}_k"])
            assert np.array_equal(vw.v, z[f"view_{kind}_{layer}_v"])
            assert [vw.quantized_bytes, vw.param_bytes, vw.fp_bytes, vw.quantized_elements] == z[f"view_{kind}_{layer}_bytes"].tolist()
    rep = c.memory_report()
    assert [rep[k] for k in ("upper_bytes", "lower_bytes", "param_bytes", "fp_buffer_bytes", "archived_fp_bytes")] == z["mem"].tolist()
    b = c.blocks[0][0]
    for tag, p in (("ku", b.ku), ("kl", b.kl), ("vu", b.vu), ("vl", b.vl)):
        assert np.array_equal(p.codes, z[f"blk0_{tag}_codes"])
        assert np.array_equal(p.scales, z[f"blk0_{tag}_scales"])


def _sha(arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.fixture(scope="module")
def toy_w():
    return O.init_weights(TOY, seed=7)


def test_init_weights_bit_exact(toy_w):
    with open(os.path.join(GOLDEN, "model_meta.json")) as f:
        meta = json.load(f)
    arrs = [toy_w["embedding"], toy_w["lm_head"]] + [lw[n] for lw in toy_w["layers"] for n in O.MATS]
    assert _sha(arrs) == meta["weights_sha256"]
    q = O.quantize_model(toy_w, 32)
    assert q["int4_weight_bytes"] == meta["int4_weight_bytes"]
    assert _sha([q["lm_head"]] + [lw[n] for lw in q["layers"] for n in O.MATS]) == meta["int4_sha256"]


def test_prefill_and_decode_logits(toy_w):
    z = load("model_golden.npz")
    logits, cache = O.prefill(toy_w, z["prompt"], "hierarchical", 16)
    assert np.array_equal(logits, z["prefill_logits"])
    vw = cache.view(0, "target")
    assert np.array_equal(vw.k, z["prefill_target_k0"]) and np.array_equal(vw.v, z["prefill_target_v0"])
    for view in ("draft", "target"):
        lg, cost = O.decode_step(toy_w, 11, copy.deepcopy(cache), view)
        assert np.array_equal(lg, z[f"decode_{view}_logits"]), view
        got = [cost.flops, cost.weight_bytes, cost.kv_quantized_bytes, cost.kv_param_bytes, cost.kv_fp_bytes, cost.kv_quantized_elements]
        assert got == z[f"decode_{view}_cost"].tolist()
    q = O.quantize_model(toy_w, 32)
    lg, _ = O.decode_step(toy_w, 11, copy.deepcopy(cache), "draft", "int4", q)
    assert np.array_equal(lg, z["decode_int4_logits"])


def test_greedy_specdec_traces(toy_w):
    with open(os.path.join(GOLDEN, "specdec_golden.json")) as f:
        runs = json.load(f)
    qcache = {}
    for r in runs:
        prompt = np.random.default_rng(r["seed"]).integers(0, TOY.vocab, size=r["prompt_len"])
        draft = None
        if r["weight_mode"] == "int4":
            draft = qcache.setdefault(32, O.quantize_model(toy_w, 32))
        toks, steps = O.spec_decode_greedy(toy_w, prompt, r["gamma"], r["decode_len"], r["kv_quant"], 16, r["weight_mode"], draft)
        assert toks == r["tokens"]
        assert len(steps) == len(r["trace"])
        for s, t in zip(steps, r["trace"]):
            assert s["drafted"] == t["drafted"] and s["v"] == t["accepted"]
            assert s["corrected"] == t["corrected"] and s["bonus"] == t["bonus"] and s["flushed"] == t["flushed"]
            assert s["draft_bytes"] == t["draft_bytes"] and s["target_bytes"] == t["target_bytes"]
        assert O.ar_decode_greedy(toy_w, prompt, r["decode_len"], r["kv_quant"], 16) == r["ar_tokens"]
