"""QSKV snapshot written by the REFERENCE (Q/cache.py:405-553) for the device-loader interop test.

    python tests/golden/make_qskv_golden.py     (build container only; writes ref_cache.qskv + ref_cache_views.npz)

A 2-layer cache (layer 1 sensitive: archived fp32 history) built with the reference's own
from_prefill / append_decode_token / flush_if_full, fed fp16-representable values so the device
store (fp16 recent-token buffers) holds them exactly.  Nothing at test time reads /root/reference.
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from quantspec.cache import CacheLayout, HierarchicalKVCache  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def f16(a):
    return np.asarray(a, np.float32).astype(np.float16).astype(np.float32)


def main():
    rng = np.random.default_rng(17)
    lay = CacheLayout(num_layers=2, num_heads=2, head_dim=16, group_size=16, sensitive_layers=frozenset({1}))
    kv = 32
    n = 3 * 16 + 7
    keys = [f16(rng.standard_normal((n, kv)) * rng.uniform(0.2, 3.0, kv)) for _ in range(2)]
    vals = [f16(rng.standard_normal((n, kv))) for _ in range(2)]
    c = HierarchicalKVCache.from_prefill(lay, keys, vals)
    for step in range(27):  # crosses a full-fp1 flush
        for layer in range(2):
            c.append_decode_token(layer, f16(rng.standard_normal(kv)), f16(rng.standard_normal(kv)))
        c.flush_if_full()
    c.save_snapshot(os.path.join(HERE, "ref_cache.qskv"))
    out = {"seq_len": np.array(c.seq_len), "quantized": np.array(c.quantized_token_count)}
    for layer in range(2):
        for kind in ("draft", "target"):
            view = c.draft_view(layer) if kind == "draft" else c.target_view(layer)
            k, v = view.concat()
            out[f"{kind}_k{layer}"], out[f"{kind}_v{layer}"] = k, v
    np.savez_compressed(os.path.join(HERE, "ref_cache_views.npz"), **out)
    print("seq_len", c.seq_len, "quantized", c.quantized_token_count, "bytes",
          os.path.getsize(os.path.join(HERE, "ref_cache.qskv")))


if __name__ == "__main__":
    main()
