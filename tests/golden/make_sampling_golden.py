"""Stochastic-verification golden vectors from the REFERENCE (Q/specdec.py:133-170):
softmax_probs / sample_index / speculative_sample_step decisions for seeded RNG streams.

    python tests/golden/make_sampling_golden.py      (build container only; writes sampling_golden.json)
"""

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from quantspec.specdec import sample_index, softmax_probs, speculative_sample_step  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    cases = []
    rng_cases = np.random.default_rng(123)
    for i in range(40):
        V = int(rng_cases.integers(2, 50))
        lt = rng_cases.standard_normal(V) * float(rng_cases.uniform(0.1, 4.0))
        ld = lt + rng_cases.standard_normal(V) * float(rng_cases.uniform(0.0, 2.0))
        if i % 7 == 0:
            ld = lt.copy()  # draft == target: always accepted
        temp = float(rng_cases.choice([0.5, 1.0, 1.7]))
        p = softmax_probs(lt, temp)
        q = softmax_probs(ld, temp)
        rng = np.random.default_rng(1000 + i)
        steps = []
        for _ in range(25):
            g = sample_index(q, rng)
            tok, acc = speculative_sample_step(p, q, g, rng)
            steps.append([int(g), int(tok), bool(acc)])
        cases.append({"target_logits": lt.tolist(), "draft_logits": ld.tolist(), "temperature": temp,
                      "seed": 1000 + i, "p": p.tolist(), "steps": steps})
    with open(os.path.join(HERE, "sampling_golden.json"), "w") as f:
        json.dump(cases, f)
    print(len(cases), "cases")


if __name__ == "__main__":
    main()
