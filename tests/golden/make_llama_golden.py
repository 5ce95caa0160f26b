"""Llama-2-7B-WIDTH golden fixtures from the REFERENCE itself (SURVEY 8(c) parity contract 2).

Run in the build container (where /root/reference exists; takes ~10-30 min on 8 cores):

    python tests/golden/make_llama_golden.py            # 2-layer logits / K,V rows / spec runs
    python tests/golden/make_llama_golden.py --depth     # acceptance-vs-depth study (L = 2, 4, 8, 16)

The model is ``init_weights`` (Q/model.py:89-117) at Llama-2-7B width (32 x 128 heads, d 4096,
mlp 11008, vocab 32000) with only ``L`` layers, so the GPU box regenerates the identical f32
weights from the seed with this repo's bit-exact ``init_weights`` and no fixture holds weights.
Writes ``llama2w_golden.npz`` / ``llama2w_spec.json`` / ``acceptance_depth.json`` here.
Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import argparse
import copy
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from quantspec.model import ModelConfig, decode_step, init_weights, prefill, quantize_model_weights  # noqa: E402
from quantspec.specdec import SpecConfig, SpeculativeDecoder, autoregressive_decode  # noqa: E402

WSEED = 11
PSEED = 1000
PROMPT_LEN = 1100  # 7 quantised blocks of 128 + fp1 (128) + fp2 (76)
KV_ROWS = (0, 1, 517, 1099)


def cfg(layers: int, max_pos: int = 4096) -> ModelConfig:
    return ModelConfig(num_layers=layers, num_heads=32, head_dim=128, hidden=4096, mlp_hidden=11008, vocab=32000,
                       max_positions=max_pos)


def prompt(n: int = PROMPT_LEN, seed: int = PSEED) -> np.ndarray:
    return np.random.default_rng(seed).integers(0, 32000, size=n, dtype=np.int64)


def run_main() -> None:
    t0 = time.time()
    w = init_weights(cfg(2), seed=WSEED)
    p = prompt()
    out = {"prompt": p}
    logits, cache = prefill(w, p, "hierarchical", group_size=128)
    out["prefill_logits"] = logits
    _, fcache = prefill(w, p, "fp")
    for layer in range(2):
        k, v = fcache.fp_view(layer).concat()
        out[f"kv_rows_k{layer}"] = k[list(KV_ROWS)]
        out[f"kv_rows_v{layer}"] = v[list(KV_ROWS)]
    tok = int(np.argmax(logits))
    out["decode_token"] = np.array(tok)
    q = quantize_model_weights(w, 32)
    for name, kw in (("target", dict(view="target")), ("draft", dict(view="draft")),
                     ("int4", dict(view="draft", weight_mode="int4", draft_weights=q))):
        c = copy.deepcopy(cache)
        lg, _ = decode_step(w, tok, c, **kw)
        out[f"decode_{name}_logits"] = lg
    np.savez_compressed(os.path.join(HERE, "llama2w_golden.npz"), **out)
    print(f"logits fixture written ({time.time() - t0:.0f} s)", flush=True)
    runs = []
    for wm, dlen in (("fp", 60), ("int4", 60)):
        t1 = time.time()
        res = SpeculativeDecoder(w, SpecConfig(gamma=4, decode_len=dlen, weight_mode=wm), group_size=128).run(p)
        runs.append({"weight_mode": wm, "gamma": 4, "decode_len": dlen, "tokens": res.tokens,
                     "acceptance_rate": res.metrics.acceptance_rate, "drafted": res.metrics.drafted_tokens,
                     "accepted": res.metrics.accepted_tokens,
                     "trace": [json.loads(l) for l in res.trace.to_ndjson().splitlines()]})
        print(f"spec {wm}: acceptance {res.metrics.acceptance_rate:.3f} ({time.time() - t1:.0f} s)", flush=True)
    ar = autoregressive_decode(w, p, 60, group_size=128)
    with open(os.path.join(HERE, "llama2w_spec.json"), "w") as f:
        json.dump({"weight_seed": WSEED, "prompt_seed": PSEED, "prompt_len": PROMPT_LEN, "runs": runs,
                   "ar_tokens": ar}, f)
    print(f"done ({time.time() - t0:.0f} s)", flush=True)


def run_depth() -> None:
    """Greedy acceptance of the reference's INT4-weight draft vs model depth (random init)."""
    path = os.path.join(HERE, "acceptance_depth.json")
    res = json.load(open(path)) if os.path.exists(path) else {}
    for layers in (2, 4, 8, 16):
        key = str(layers)
        if key in res:
            continue
        t0 = time.time()
        w = init_weights(cfg(layers), seed=WSEED)
        p = prompt(300, PSEED + 1)
        entry = {}
        for wm in ("int4", "fp"):
            r = SpeculativeDecoder(w, SpecConfig(gamma=4, decode_len=80, weight_mode=wm), group_size=128).run(p)
            entry[wm] = {"acceptance_rate": r.metrics.acceptance_rate, "drafted": r.metrics.drafted_tokens,
                         "accepted": r.metrics.accepted_tokens, "tokens": r.tokens}
        entry["prompt_len"] = 300
        entry["prompt_seed"] = PSEED + 1
        entry["weight_seed"] = WSEED
        entry["seconds"] = time.time() - t0
        res[key] = entry
        with open(path, "w") as f:
            json.dump(res, f)
        print(layers, {k: v["acceptance_rate"] for k, v in entry.items() if isinstance(v, dict)}, flush=True)
        del w


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--depth", action="store_true")
    a = ap.parse_args()
    run_depth() if a.depth else run_main()
