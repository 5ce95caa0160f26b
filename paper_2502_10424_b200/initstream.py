"""Bit-exact, parallel replay of the reference's random weight initialisation at 7B/8B scale.

``init_weights`` (/root/reference/pkg/src/quantspec/model.py:89-117) draws every matrix from ONE
numpy PCG64 stream in a fixed order -- per layer wq, wk, wv, wo, w_gate, w_up, w_down as
``standard_normal((rows, cols)) / sqrt(rows)`` (f64, then cast to f32), then the unscaled
embedding ``standard_normal((V, d))``, then lm_head.  The ziggurat sampler consumes a variable
number of 64-bit words per draw, so the stream cannot be split analytically; instead the PCG64
state at the start of every matrix is recorded once by walking the stream
(``walk_states``, committed per (shape, seed) in ``data/init_states.json``) and the matrices are
then regenerated independently on host threads (numpy's generators release the GIL), each
bit-identical to the sequential draw.  A Llama-2-7B-shaped model (6.7 G draws) takes ~2 min
sequentially; with 16 threads it is bounded by the host->device copy.
"""

from __future__ import annotations

import json
import os
import queue
from concurrent.futures import ThreadPoolExecutor

import numpy as np

MATS = ("wq", "wk", "wv", "wo", "w_gate", "w_up", "w_down")
STATES_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "init_states.json")


def draw_plan(num_layers: int, hidden: int, kv_dim: int, mlp: int, vocab: int):
    """[(name, rows, cols, scaled)] in the reference's draw order (Q/model.py:89-117)."""
    d, m = hidden, mlp
    shapes = {"wq": (d, d), "wk": (d, kv_dim), "wv": (d, kv_dim), "wo": (d, d), "w_gate": (d, m), "w_up": (d, m),
              "w_down": (m, d)}
    plan = [(f"layers.{i}.{n}", *shapes[n], True) for i in range(num_layers) for n in MATS]
    plan.append(("embedding", vocab, d, False))
    plan.append(("lm_head", d, vocab, True))
    return plan


def _key(num_layers, hidden, kv_dim, mlp, vocab, seed) -> str:
    return f"L{num_layers}_d{hidden}_kv{kv_dim}_m{mlp}_V{vocab}_seed{seed}"


def walk_states(plan, seed: int, chunk_rows: int = 4096) -> list:
    """PCG64 state (JSON-able) at the start of every matrix of ``plan``.  Draws are made in row
    chunks: numpy's standard_normal fills in C order, so chunked draws consume the identical stream."""
    rng = np.random.default_rng(seed)
    out = []
    for _, rows, cols, _ in plan:
        st = rng.bit_generator.state
        out.append({"state": int(st["state"]["state"]), "inc": int(st["state"]["inc"]),
                    "has_uint32": int(st["has_uint32"]), "uinteger": int(st["uinteger"])})
        for r0 in range(0, rows, chunk_rows):
            rng.standard_normal((min(chunk_rows, rows - r0), cols))
    return out


def load_states(num_layers, hidden, kv_dim, mlp, vocab, seed):
    try:
        with open(STATES_PATH) as f:
            return json.load(f).get(_key(num_layers, hidden, kv_dim, mlp, vocab, seed))
    except FileNotFoundError:
        return None


def save_states(num_layers, hidden, kv_dim, mlp, vocab, seed, states) -> None:
    os.makedirs(os.path.dirname(STATES_PATH), exist_ok=True)
    try:
        with open(STATES_PATH) as f:
            db = json.load(f)
    except FileNotFoundError:
        db = {}
    db[_key(num_layers, hidden, kv_dim, mlp, vocab, seed)] = states
    with open(STATES_PATH, "w") as f:
        json.dump(db, f, indent=0)


def _rng_at(st: dict) -> np.random.Generator:
    bg = np.random.PCG64()
    bg.state = {"bit_generator": "PCG64", "state": {"state": st["state"], "inc": st["inc"]},
                "has_uint32": st["has_uint32"], "uinteger": st["uinteger"]}
    return np.random.Generator(bg)


def draw(st: dict, rows: int, cols: int, scaled: bool, out: np.ndarray | None = None) -> np.ndarray:
    """One matrix, bit-identical to the sequential reference draw: f64 normals (/ sqrt(rows)) -> f32."""
    rng = _rng_at(st)
    out = np.empty((rows, cols), dtype=np.float32) if out is None else out
    step = max(1, (1 << 24) // cols)  # bounded f64 scratch
    inv = np.sqrt(rows)
    for r0 in range(0, rows, step):
        r1 = min(rows, r0 + step)
        x = rng.standard_normal((r1 - r0, cols))
        if scaled:
            x /= inv
        out[r0:r1] = x
    return out


def stream_matrices(plan, states, *, threads: int | None = None, ahead: int = 6):
    """Yield (name, f32 ndarray) in plan order, generated ``ahead`` matrices in advance on a thread pool."""
    threads = threads or min(16, os.cpu_count() or 1)
    with ThreadPoolExecutor(max_workers=threads) as pool:
        futs = queue.Queue()
        it = iter(zip(plan, states))

        def submit():
            try:
                (name, rows, cols, scaled), st = next(it)
            except StopIteration:
                return False
            futs.put((name, pool.submit(draw, st, rows, cols, scaled)))
            return True

        for _ in range(ahead):
            if not submit():
                break
        while not futs.empty():
            name, f = futs.get()
            arr = f.result()
            submit()
            yield name, arr

