"""Device-resident greedy decode engines with CUDA-graph replay, for a ragged batch of
independent sequences (B = 1 is the plain single-sequence case).

SpecEngine runs the draft -> verify -> accept -> flush cycle of
/root/reference/pkg/src/quantspec/specdec.py:314-397 (greedy) for every sequence of a
HierarchicalKVCache at once.  Each sequence keeps the reference's own schedule:
gamma_step = min(gamma, fp2_space - 1, remaining) (specdec.py:329-333; gamma_step 0 is the
degenerate target-only step), its own accepted count v, and its own flush (cache.py:249-262).
The host computes the per-sequence gamma_steps from its length mirror (the same formula),
uploads them, and replays ONE captured graph per cycle holding

    max(gamma_step) draft forwards (T = 1 row per sequence, draft view)
    -> one verify forward (T = max(gamma_step) + 1 rows per sequence, target view)
    -> batched greedy accept (per-sequence v, next token, fp2 / position bump)
    -> the device-conditioned flush (K1 + fp rotate for the sequences whose fp2 filled)
    -> a copy of (v, next, drafts, status word) into pinned host memory.

Rows past a sequence's gamma_step are padding: their K/V land in the fp2 slack rows and are
never committed.  The host reads back one small buffer per cycle.

ARAutoEngine is the plain autoregressive loop of specdec.py:400-434 on the same kernels
(target view) and, with an FpKVCache, the FP16 autoregressive baseline.

Graphs are keyed by the cycle shape; the first use of a key runs eagerly (which also
configures kernel attributes), the second captures, later uses replay.  They are dropped when
the cache reallocates its arenas.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .errors import ConfigError
from .runtime import DeviceWeights, Runner


def _torch():
    import torch

    return torch


class _GraphCache:
    def __init__(self, enabled: bool):
        self.enabled = enabled
        self.graphs: dict = {}
        self.seen: set = set()
        self.generation = None

    def run(self, key, fn, generation: int) -> None:
        torch = _torch()
        if self.generation != generation:
            self.graphs.clear()
            self.seen.clear()
            self.generation = generation
        if not self.enabled:
            fn()
            return
        g = self.graphs.get(key)
        if g is not None:
            g.replay()
            return
        if key not in self.seen:
            self.seen.add(key)
            fn()
            return
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        self.graphs[key] = g
        g.replay()


class SpecEngine:
    """Greedy self-speculative decoding of every sequence of a HierarchicalKVCache."""

    def __init__(self, target: DeviceWeights, draft: DeviceWeights, cache, gamma: int, *, use_graphs: bool = True,
                 runner: Runner | None = None, max_positions: int | None = None):
        torch = _torch()
        if not hasattr(cache, "d_n_blocks"):
            raise ConfigError("SpecEngine needs a HierarchicalKVCache")
        if gamma + 1 > cache.fp_rows - cache.layout.group_size + 1 or gamma > cache.layout.group_size:
            raise ConfigError(f"gamma {gamma} exceeds the cache's fp2 slack")
        self.target = target
        self.draft = draft
        self.cache = cache
        self.gamma = gamma
        self.B = cache.batch
        self.max_positions = max_positions or target.geo.max_positions
        self.run = runner or Runner(target.geo, cache, max_cols=cache.batch * (gamma + 1))
        if self.run.TS < gamma + 1:
            raise ConfigError("runner token buffer too small for gamma")
        self.graphs = _GraphCache(use_graphs)
        B = self.B
        # pinned host I/O: gamma_steps in; (v, next) per sequence, drafts, status word out
        self.h_gs = torch.zeros(B, dtype=torch.int32).pin_memory()
        self.d_gs = torch.zeros(B, dtype=torch.int32, device="cuda")
        self.h_out = torch.zeros(2 * B + B * self.run.TS + 1, dtype=torch.int32).pin_memory()
        self.launches = 0
        self.h2d_bytes = 4 * B
        self.d2h_bytes = 4 * (2 * B + B * self.run.TS + 1)

    # -- host-side schedule (the reference's per-sequence formula) ------------------
    def gamma_steps(self, remaining=None) -> np.ndarray:
        c = self.cache
        space = c.layout.group_size - c._fp2[:, 0]
        gs = np.minimum(self.gamma, space - 1)
        if remaining is not None:
            gs = np.minimum(gs, np.asarray(remaining))
        return np.maximum(gs, 0).astype(np.int64)

    def set_pending(self, tokens) -> None:
        """Pending (last emitted) token of every sequence."""
        torch = _torch()
        t = torch.as_tensor(np.asarray(tokens, dtype=np.int32).reshape(self.B), device="cuda")
        self.run.tok[:, 0].copy_(t)

    def _cycle_fn(self, nd: int):
        r, c = self.run, self.cache
        lib = _lib.load()
        TS = r.TS

        def fn():
            s = _lib.stream_ptr()
            self.d_gs.copy_(self.h_gs, non_blocking=True)
            for i in range(nd):
                r.forward(self.draft, 1, _lib.VIEW_DRAFT, row_offset=i, tok_col=i,
                          argmax_to=(r.tok.data_ptr() + 4 * (i + 1), TS))
            # the verify forward's tokens are (pending, drafts); keep them before accept replaces tok[:, 0]
            self.h_out[2 * self.B : 2 * self.B + self.B * TS].copy_(r.tok.view(-1), non_blocking=True)
            r.forward(self.target, nd + 1, _lib.VIEW_TARGET, row_offset=0, tok_col=0, argmax_to=(r.amax.data_ptr(), 1))
            _lib.check(lib.qs_greedy_accept(r.tok.data_ptr(), TS, r.amax.data_ptr(), nd + 1, self.d_gs.data_ptr(),
                                            self.B, r.res.data_ptr(), c.d_fp2_len.data_ptr(), c.d_pos.data_ptr(), s),
                       "qs_greedy_accept")
            c.launch_device_flush()
            self.h_out[: 2 * self.B].copy_(r.res, non_blocking=True)
            self.h_out[-1:].copy_(c.d_flags, non_blocking=True)

        return fn

    def launches_per_cycle(self, nd: int) -> int:
        nl = len(self.target.layers)
        fused = self.run._fuse_prep(self.draft.layers[0]["qkv"], self.B)
        return (nd * self.run.kernel_launches_per_forward(nl, fused) + self.run.kernel_launches_per_forward(nl)
                + 1 + 3)  # accept + the three flush launches

    def cycle(self, remaining=None, *, sync: bool = True):
        """One draft/verify/accept/flush cycle of every sequence.

        Returns per-sequence lists (gamma_steps, drafts, v, next_token, flush kinds) after
        committing the host mirror, or None when ``sync`` is False (the caller then calls
        ``finish``)."""
        c = self.cache
        gs = self.gamma_steps(remaining)
        nd = int(gs.max())
        pos_after = c.seq_lens() + gs + 1
        if int(pos_after.max()) > self.max_positions:
            raise ConfigError(f"position {int(pos_after.max()) - 1} exceeds max positions {self.max_positions}")
        # a flush this cycle needs one more block per sequence
        c.ensure_blocks(int(c._nq.max()) // c.layout.group_size + 1)
        self.run.sync_generation()
        self.h_gs.copy_(_torch().from_numpy(gs.astype(np.int32)))
        self.graphs.run(("cycle", nd), self._cycle_fn(nd), c.generation)
        self.launches += self.launches_per_cycle(nd)
        self._pending_gs = gs
        if not sync:
            return None
        return self.finish()

    def finish(self):
        torch = _torch()
        torch.cuda.current_stream().synchronize()
        c = self.cache
        h = self.h_out.numpy()
        B, TS = self.B, self.run.TS
        gs = self._pending_gs
        flags = int(h[-1])
        if flags:
            c.raise_device_flags("decode cycle", flags)
        v = h[0 : 2 * B : 2].astype(np.int64)
        nxt = h[1 : 2 * B : 2].astype(np.int64)
        toks = h[2 * B : 2 * B + B * TS].reshape(B, TS)
        drafts = [toks[b, 1 : 1 + gs[b]].tolist() for b in range(B)]
        # host mirror of the device-side bumps: rows kept after rollback(gamma_step - v), then the flush
        c._fp2 += (v + 1)[:, None]
        due = c.flush_due()
        c.commit_flush(due)
        return gs, drafts, v, nxt, due


class ARAutoEngine:
    """Greedy one-token-at-a-time decoding of every sequence on the same kernels.

    With a HierarchicalKVCache it reads the target view (the losslessness oracle of
    Q/specdec.py:400-434); with an FpKVCache it is the FP16 autoregressive baseline.
    """

    def __init__(self, target: DeviceWeights, cache, *, use_graphs: bool = True, runner: Runner | None = None,
                 max_positions: int | None = None):
        torch = _torch()
        self.target = target
        self.cache = cache
        self.B = cache.batch
        self.max_positions = max_positions or target.geo.max_positions
        self.run = runner or Runner(target.geo, cache, max_cols=cache.batch)
        self.graphs = _GraphCache(use_graphs)
        self.is_fp = not hasattr(cache, "d_n_blocks")
        self.h_out = torch.zeros(self.B + 1, dtype=torch.int32).pin_memory()
        self.launches = 0

    def set_pending(self, tokens) -> None:
        torch = _torch()
        t = torch.as_tensor(np.asarray(tokens, dtype=np.int32).reshape(self.B), device="cuda")
        self.run.tok[:, 0].copy_(t)

    def _step_fn(self):
        r, c = self.run, self.cache
        lib = _lib.load()
        view = _lib.VIEW_FP16 if self.is_fp else _lib.VIEW_TARGET

        def fn():
            s = _lib.stream_ptr()
            r.forward(self.target, 1, view, row_offset=0, tok_col=0, argmax_to=(r.tok.data_ptr() + 4, r.TS))
            r.tok[:, 0].copy_(r.tok[:, 1], non_blocking=True)
            if self.is_fp:
                _lib.check(lib.qs_add_int(c.d_len.data_ptr(), self.B, 1, s), "qs_add_int")
            else:
                _lib.check(lib.qs_add_int(c.d_fp2_len.data_ptr(), self.B, 1, s), "qs_add_int")
                _lib.check(lib.qs_add_int(c.d_pos.data_ptr(), self.B, 1, s), "qs_add_int")
                c.launch_device_flush()
            self.h_out[: self.B].copy_(r.tok[:, 1], non_blocking=True)
            self.h_out[-1:].copy_(c.d_flags, non_blocking=True)

        return fn

    def step(self, *, sync: bool = True):
        """Decode one token per sequence (appends it to the cache); returns them when sync."""
        c = self.cache
        if int(c.seq_lens().max()) + 1 > self.max_positions:
            raise ConfigError(f"position {int(c.seq_lens().max())} exceeds max positions {self.max_positions}")
        if self.is_fp:
            c.ensure_tokens(int(c.seq_lens().max()) + 1)
        else:
            c.ensure_blocks(int(c._nq.max()) // c.layout.group_size + 1)
        self.run.sync_generation()
        self.graphs.run(("ar",), self._step_fn(), c.generation)
        fused = self.run._fuse_prep(self.target.layers[0]["qkv"], self.B)
        self.launches += self.run.kernel_launches_per_forward(len(self.target.layers), fused) + (2 if self.is_fp else 6)
        if self.is_fp:
            c._lens += 1
        else:
            c._fp2 += 1
            c.commit_flush(c.flush_due())  # full-fp1 flushes ran in the graph; short-fp1 top-ups here
        if not sync:
            return None
        _torch().cuda.current_stream().synchronize()
        h = self.h_out.numpy()
        if int(h[-1]):
            c.raise_device_flags("decode step", int(h[-1]))
        out = h[: self.B].astype(np.int64)
        return int(out[0]) if self.B == 1 else out
