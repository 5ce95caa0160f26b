"""Generate the golden fixtures from the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package read-only from /root/reference/pkg/src and
writes small .npz/.json fixtures next to this file.  The fixtures are
committed; nothing at test time (CPU or GPU box) reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from quantspec import quant  # noqa: E402
from quantspec.cache import CacheLayout, HierarchicalKVCache  # noqa: E402
from quantspec.model import (  # noqa: E402
    ModelConfig,
    decode_step,
    init_weights,
    prefill,
    quantize_model_weights,
)
from quantspec.specdec import SpecConfig, SpeculativeDecoder, autoregressive_decode  # noqa: E402

TOY = ModelConfig(num_layers=2, num_heads=4, head_dim=16, hidden=64, mlp_hidden=176, vocab=64, max_positions=4096 + 128)


def sha(arrs) -> str:
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def plane_dict(prefix, p):
    return {
        f"{prefix}_codes": p.codes,
        f"{prefix}_scales": p.scales,
        f"{prefix}_zeros": p.zeros,
        f"{prefix}_meta": np.array([p.count, p.group_size, p.row_len or 0], np.int64),
    }


def gen_quant():
    out = {}
    rng = np.random.default_rng(1234)
    cases = []
    # (values, group, axis, row_len)
    cases.append((rng.standard_normal(128 * 64) * 2.0, 128, "channel", None))
    chan_scale = rng.uniform(0.1, 4.0, size=64)
    blk = (rng.standard_normal((128, 64)) * chan_scale).astype(np.float32)
    cases.append((np.ascontiguousarray(blk.T).ravel(), 128, "channel", None))
    cases.append((blk.ravel(), 16, "token", 64))
    cases.append((rng.standard_normal(55) * 5, 4, "token", 11))
    cases.append((rng.standard_normal(70), 32, "channel", None))  # short trailing group
    ties = np.array([0.0, 0.1, 0.2, 0.30000000000000004, 1.5, 1.5, 0.75, 3.0], np.float64)
    cases.append((ties, 8, "channel", None))
    cases.append((np.full(16, 2.5), 16, "channel", None))  # constant group -> scale floor
    half = (np.arange(64, dtype=np.float64) * (1.0 / 30.0))
    cases.append((half, 32, "channel", None))
    bf = (rng.standard_normal(256) * 1e-3).astype(np.float16).astype(np.float64)
    cases.append((bf, 128, "token", 128))
    big = rng.standard_normal(128) * 1e30
    cases.append((big, 64, "channel", None))
    out["n_cases"] = np.array(len(cases))
    for i, (v, g, axis, rl) in enumerate(cases):
        up, lo = quant.encode_plane_hierarchical(v, g, axis, rl)
        out[f"c{i}_values"] = np.asarray(v, np.float64)
        out[f"c{i}_group"] = np.array([g, rl or 0])
        out.update(plane_dict(f"c{i}_up", up))
        out.update(plane_dict(f"c{i}_lo", lo))
        out[f"c{i}_draft"] = quant.decode_plane_draft(up)
        out[f"c{i}_target"] = quant.decode_plane_target(up, lo)
    # single-group KATs
    grp = []
    for vals in ([0.0, 1.0, 2.0, 3.0], [2.5, 2.5, 2.5, 2.5], [0.0, 1.07, 2.0, 3.0], list(rng.standard_normal(128) * 3.0)):
        (uc, up), (lc, lp) = quant.hierarchical_encode(vals)
        grp.append({"values": [float(x) for x in vals], "cu": uc.tolist(), "S": up.scale, "Z": up.zero_point,
                    "cl": lc.tolist(), "Sl": lp.scale})
    # weight quantisation
    w = (rng.standard_normal((96, 48)) / np.sqrt(96)).astype(np.float32)
    for g in (32, 16, 7):
        ql = quant.quantize_weights(w, g)
        out.update(plane_dict(f"w{g}", ql.plane))
        out[f"w{g}_deq"] = quant.dequantize_weights(ql)
    out["w_in"] = w
    np.savez_compressed(os.path.join(HERE, "quant_golden.npz"), **out)
    with open(os.path.join(HERE, "group_kat.json"), "w") as f:
        json.dump(grp, f, indent=1)


def gen_cache():
    """A scripted cache session: prefill, appends, rollbacks, flushes."""
    g = 16
    layout = CacheLayout(num_layers=2, num_heads=2, head_dim=16, group_size=g, sensitive_layers=frozenset())
    kv = layout.kv_dim
    rng = np.random.default_rng(77)
    s_p = 3 * g + 5
    keys = [(rng.standard_normal((s_p, kv)) * rng.uniform(0.2, 3.0, size=kv)).astype(np.float32) for _ in range(2)]
    vals = [rng.standard_normal((s_p, kv)).astype(np.float32) for _ in range(2)]
    cache = HierarchicalKVCache.from_prefill(layout, keys, vals)
    out = {"keys0": keys[0], "keys1": keys[1], "vals0": vals[0], "vals1": vals[1]}
    script = []
    appended = []
    for step in range(40):
        op = ["append", "append", "append", "rollback", "flush"][step % 5]
        if op == "append":
            n = int(rng.integers(1, 4))
            for _ in range(n):
                if cache.fp2_space() == 0:
                    break
                row_k = rng.standard_normal((2, kv)).astype(np.float32)
                row_v = rng.standard_normal((2, kv)).astype(np.float32)
                for layer in range(2):
                    cache.append_decode_token(layer, row_k[layer], row_v[layer])
                appended.append((row_k, row_v))
                script.append(("append", len(appended) - 1))
        elif op == "rollback":
            n = int(rng.integers(0, min(2, cache.fp2_len) + 1))
            cache.rollback(n)
            script.append(("rollback", n))
        else:
            # force fills so flushes really happen
            while cache.fp2_space() > 0:
                row_k = rng.standard_normal((2, kv)).astype(np.float32)
                row_v = rng.standard_normal((2, kv)).astype(np.float32)
                for layer in range(2):
                    cache.append_decode_token(layer, row_k[layer], row_v[layer])
                appended.append((row_k, row_v))
                script.append(("append", len(appended) - 1))
            flushed = cache.flush_if_full()
            script.append(("flush", int(flushed)))
        state = [cache.quantized_token_count, cache.fp1_len, cache.fp2_len]
        script.append(("state", state))
    for layer in range(2):
        for kind in ("draft", "target"):
            vw = getattr(cache, f"{kind}_view")(layer)
            k, v = vw.concat()
            out[f"view_{kind}_{layer}_k"] = k
            out[f"view_{kind}_{layer}_v"] = v
            out[f"view_{kind}_{layer}_bytes"] = np.array([vw.quantized_bytes, vw.param_bytes, vw.fp_bytes, vw.quantized_elements])
    rep = cache.memory_report()
    out["mem"] = np.array([rep.upper_bytes, rep.lower_bytes, rep.param_bytes, rep.fp_buffer_bytes, rep.archived_fp_bytes])
    out["appended_k"] = np.stack([a for a, _ in appended])
    out["appended_v"] = np.stack([b for _, b in appended])
    st = cache._stores[0]
    out.update(plane_dict("blk0_ku", st.key_upper[0]))
    out.update(plane_dict("blk0_kl", st.key_lower[0]))
    out.update(plane_dict("blk0_vu", st.value_upper[0]))
    out.update(plane_dict("blk0_vl", st.value_lower[0]))
    np.savez_compressed(os.path.join(HERE, "cache_golden.npz"), **out)
    with open(os.path.join(HERE, "cache_script.json"), "w") as f:
        json.dump(script, f)


def gen_model():
    w = init_weights(TOY, seed=7)
    arrs = [w.embedding, w.lm_head] + [getattr(lw, n) for lw in w.layers for n in ("wq", "wk", "wv", "wo", "w_gate", "w_up", "w_down")]
    meta = {"weights_sha256": sha(arrs)}
    rng = np.random.default_rng(2024)
    prompt = rng.integers(0, TOY.vocab, size=70)
    logits, cache = prefill(w, prompt, "hierarchical", group_size=16)
    out = {"prompt": prompt, "prefill_logits": logits}
    import copy

    for view in ("draft", "target"):
        c = copy.deepcopy(cache)
        lg, cost = decode_step(w, 11, c, view=view)
        out[f"decode_{view}_logits"] = lg
        out[f"decode_{view}_cost"] = np.array([cost.flops, cost.weight_bytes, cost.kv_quantized_bytes, cost.kv_param_bytes, cost.kv_fp_bytes, cost.kv_quantized_elements])
    q = quantize_model_weights(w, 32)
    c = copy.deepcopy(cache)
    lg, cost = decode_step(w, 11, c, view="draft", weight_mode="int4", draft_weights=q)
    out["decode_int4_logits"] = lg
    out["decode_int4_cost"] = np.array([cost.flops, cost.weight_bytes, cost.kv_quantized_bytes, cost.kv_param_bytes, cost.kv_fp_bytes, cost.kv_quantized_elements])
    meta["int4_weight_bytes"] = q.int4_weight_bytes
    meta["int4_sha256"] = sha([q.lm_head] + [getattr(lw, n) for lw in q.layers for n in ("wq", "wk", "wv", "wo", "w_gate", "w_up", "w_down")])
    # the cache's K/V after prefill for layer 0 (to pin prefill_kv)
    k0, v0 = cache.target_view(0).concat()
    out["prefill_target_k0"] = k0
    out["prefill_target_v0"] = v0
    np.savez_compressed(os.path.join(HERE, "model_golden.npz"), **out)
    with open(os.path.join(HERE, "model_meta.json"), "w") as f:
        json.dump(meta, f, indent=1)


def gen_specdec():
    w = init_weights(TOY, seed=7)
    runs = []
    for seed, gamma, plen, dlen, wm, kvq in (
        (2, 4, 80, 40, "fp", True),
        (3, 1, 80, 30, "fp", True),
        (4, 6, 47, 40, "fp", True),
        (5, 4, 80, 30, "int4", True),
        (1, 4, 40, 30, "fp", False),
    ):
        prompt = np.random.default_rng(seed).integers(0, TOY.vocab, size=plen)
        spec = SpecConfig(gamma=gamma, decode_len=dlen, weight_mode=wm)
        res = SpeculativeDecoder(w, spec, group_size=16, kv_quant=kvq).run(prompt)
        ar = autoregressive_decode(w, prompt, dlen, group_size=16, kv_quant=kvq)
        runs.append({
            "seed": seed, "gamma": gamma, "prompt_len": plen, "decode_len": dlen, "weight_mode": wm, "kv_quant": kvq,
            "tokens": res.tokens, "ar_tokens": ar,
            "trace": [json.loads(l) for l in res.trace.to_ndjson().splitlines()],
            "acceptance_rate": res.metrics.acceptance_rate,
            "peak_cache_bytes": res.metrics.peak_cache_bytes,
        })
    with open(os.path.join(HERE, "specdec_golden.json"), "w") as f:
        json.dump(runs, f)


if __name__ == "__main__":
    gen_quant()
    gen_cache()
    gen_model()
    gen_specdec()
    print("golden fixtures written to", HERE)
