"""Stochastic verification: the host-side sampling of the decode loop
(paper_2502_10424_b200/specdec.py: softmax_probs, sample_index, speculative_sample_step) against
the REFERENCE's decisions on the same seeded RNG streams (tests/golden/make_sampling_golden.py,
Q/specdec.py:133-170) -- bit-exact -- and the reference's own chi-squared property
(pkg/tests/test_specdec.py:225-241, test_acceptance.py:103-115): one draft + verify step over fixed
distributions emits tokens distributed as the target p."""

import json
import os

import numpy as np
import pytest

from paper_2502_10424_b200.errors import DataError
from paper_2502_10424_b200.specdec import sample_index, softmax_probs, speculative_sample_step

from .conftest import GOLDEN


def test_decisions_bit_exact_vs_reference_streams():
    with open(os.path.join(GOLDEN, "sampling_golden.json")) as f:
        cases = json.load(f)
    n_acc = n_rej = 0
    for c in cases:
        p = softmax_probs(np.array(c["target_logits"]), c["temperature"])
        q = softmax_probs(np.array(c["draft_logits"]), c["temperature"])
        assert np.array_equal(p, np.array(c["p"]))
        rng = np.random.default_rng(c["seed"])
        for g_ref, tok_ref, acc_ref in c["steps"]:
            g = sample_index(q, rng)
            tok, acc = speculative_sample_step(p, q, g, rng)
            assert (g, tok, acc) == (g_ref, tok_ref, acc_ref)
            n_acc += acc
            n_rej += not acc
    assert n_acc > 100 and n_rej > 100  # both branches (accept, residual resample) exercised


def test_single_step_distribution_matches_target_chi2():
    from scipy import stats

    rng = np.random.default_rng(42)
    p = np.array([0.22, 0.05, 0.13, 0.02, 0.3, 0.08, 0.12, 0.08])
    q = np.array([0.05, 0.25, 0.05, 0.15, 0.1, 0.2, 0.1, 0.1])
    n = 100_000
    counts = np.zeros(8, dtype=np.int64)
    for _ in range(n):
        g = sample_index(q, rng)
        token, _ = speculative_sample_step(p, q, g, rng)
        counts[token] += 1
    assert stats.chisquare(counts, f_exp=p * n).pvalue > 0.01


def test_identical_distributions_always_accept_and_shape_errors():
    rng = np.random.default_rng(0)
    p = softmax_probs(np.array([0.3, -1.0, 2.0, 0.5]))
    for _ in range(200):
        g = sample_index(p, rng)
        tok, acc = speculative_sample_step(p, p, g, rng)
        assert acc and tok == g
    with pytest.raises(DataError):
        speculative_sample_step(p, p[:3], 0, rng)
