import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN


@pytest.fixture()
def rng():
    return np.random.default_rng(1234)


def make_prompt(length: int, seed: int, vocab: int = 64) -> np.ndarray:
    # same recipe as the reference tests (pkg/tests/conftest.py:27-28)
    return np.random.default_rng(seed).integers(0, vocab, size=length, dtype=np.int64)
