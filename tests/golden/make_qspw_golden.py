"""QSPW weight file written by the REFERENCE (Q/model.py:415-458) for the codec interop test.

    python tests/golden/make_qspw_golden.py      (build container only; writes ref_weights.qspw)
"""

import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
from quantspec.model import ModelConfig, init_weights, save_weights  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

if __name__ == "__main__":
    cfg = ModelConfig(num_layers=2, num_heads=2, head_dim=8, hidden=16, mlp_hidden=24, vocab=40, max_positions=128)
    save_weights(os.path.join(HERE, "ref_weights.qspw"), init_weights(cfg, seed=9))
