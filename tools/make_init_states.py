"""Record the PCG64 state at the start of every matrix of the reference's init_weights stream
(Q/model.py:89-117) for the bench shapes, so paper_2502_10424_b200.initstream can regenerate the
weights bit-exactly in parallel.  Run once per (shape, seed); writes
paper_2502_10424_b200/data/init_states.json.   usage: python tools/make_init_states.py llama2_7b 0"""

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2502_10424_b200 import initstream as S  # noqa: E402

SHAPES = {
    "llama2_7b": dict(num_layers=32, hidden=4096, kv_dim=4096, mlp=11008, vocab=32000),
    "llama31_8b": dict(num_layers=32, hidden=4096, kv_dim=1024, mlp=14336, vocab=128256),
}

if __name__ == "__main__":
    name, seed = sys.argv[1], int(sys.argv[2])
    sh = SHAPES[name]
    t0 = time.time()
    plan = S.draw_plan(sh["num_layers"], sh["hidden"], sh["kv_dim"], sh["mlp"], sh["vocab"])
    states = S.walk_states(plan, seed)
    S.save_states(sh["num_layers"], sh["hidden"], sh["kv_dim"], sh["mlp"], sh["vocab"], seed, states)
    print(f"{name} seed {seed}: {len(states)} states in {time.time() - t0:.0f} s")
