"""Device-resident greedy decode engines with CUDA-graph replay.

SpecEngine runs the draft -> verify -> accept cycle of
/root/reference/pkg/src/quantspec/specdec.py:314-397 (greedy) with tokens,
lengths and the accept decision on the device; per cycle the host issues at
most two graph replays and reads back one small buffer (accepted count, next
token, drafted tokens).  ARAutoEngine is the plain autoregressive loop of
specdec.py:400-434 on the same kernels (target view), and with an FpKVCache
it is the FP16 autoregressive baseline.

Graphs are keyed by (phase, gamma_step); the first use of a key runs eagerly
(which also configures kernel attributes), the second captures, later uses
replay.  They are dropped when the cache reallocates its arenas.
"""

from __future__ import annotations

from . import _lib
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
    """Greedy self-speculative decoding for one sequence on a HierarchicalKVCache."""

    def __init__(self, target: DeviceWeights, draft: DeviceWeights, cache, gamma: int, *, use_graphs: bool = True,
                 runner: Runner | None = None):
        torch = _torch()
        self.target = target
        self.draft = draft
        self.cache = cache
        self.gamma = gamma
        self.run = runner or Runner(target.geo, cache, max_cols=cache.batch * (gamma + 1))
        self.graphs = _GraphCache(use_graphs)
        self.host = torch.zeros(4 + gamma + 2, dtype=torch.int32).pin_memory()
        self.launches = 0

    def set_pending(self, token: int) -> None:
        self.run.tok[0] = int(token)

    def _draft_fn(self, gs: int):
        r, w = self.run, self.draft

        def fn():
            for i in range(gs):
                r.forward(w, 1, _lib.VIEW_DRAFT, row_offset=i, tok_offset=i, argmax_to=r.tok.data_ptr() + 4 * (i + 1))

        return fn

    def _verify_fn(self, gs: int):
        r, w, c = self.run, self.target, self.cache
        lib = _lib.load()

        def fn():
            s = _lib.stream_ptr()
            r.forward(w, gs + 1, _lib.VIEW_TARGET, row_offset=0, tok_offset=0, argmax_to=r.amax.data_ptr())
            # drafted tokens are tok[1..gs]; copy them out before tok[0] is replaced
            self.host[4 : 4 + gs + 1].copy_(r.tok[: gs + 1], non_blocking=True)
            _lib.check(lib.qs_greedy_accept(r.tok.data_ptr() + 4, r.amax.data_ptr(), gs, r.res.data_ptr(),
                                            r.tok.data_ptr(), c.d_fp2_len.data_ptr(), c.d_pos.data_ptr(), s),
                       "qs_greedy_accept")
            self.host[:2].copy_(r.res[:2], non_blocking=True)

        return fn

    def cycle(self, gamma_step: int, *, sync: bool = True):
        """One draft/verify cycle; returns (drafts, v, next_token)."""
        torch = _torch()
        gen = self.cache.generation
        if gamma_step > 0:
            self.graphs.run(("draft", gamma_step), self._draft_fn(gamma_step), gen)
        self.graphs.run(("verify", gamma_step), self._verify_fn(gamma_step), gen)
        nl = len(self.target.layers)
        fused = self.run._fuse_prep(self.draft.layers[0]["qkv"], self.cache.batch)
        self.launches += (gamma_step * self.run.kernel_launches_per_forward(nl, fused)
                          + self.run.kernel_launches_per_forward(nl) + 1)
        if not sync:
            return None
        torch.cuda.current_stream().synchronize()
        h = self.host.tolist()
        v, nxt = h[0], h[1]
        drafts = h[5 : 5 + gamma_step]
        # host mirror of the device-side length bump (rows kept after rollback(gamma_step - v))
        self.cache._fp2_len += v + 1
        return drafts, v, nxt


class ARAutoEngine:
    """Greedy one-token-at-a-time decoding on the same kernels.

    With a HierarchicalKVCache it reads the target view (the losslessness
    oracle of Q/specdec.py:400-434); with an FpKVCache it is the FP16
    autoregressive baseline.
    """

    def __init__(self, target: DeviceWeights, cache, *, use_graphs: bool = True, runner: Runner | None = None):
        torch = _torch()
        self.target = target
        self.cache = cache
        self.run = runner or Runner(target.geo, cache, max_cols=cache.batch)
        self.graphs = _GraphCache(use_graphs)
        self.is_fp = not hasattr(cache, "d_n_blocks")
        self.host = torch.zeros(8, dtype=torch.int32).pin_memory()
        self.launches = 0

    def set_pending(self, token: int) -> None:
        self.run.tok[0] = int(token)

    def _step_fn(self):
        r, w, c = self.run, self.target, self.cache
        lib = _lib.load()
        view = _lib.VIEW_FP16 if self.is_fp else _lib.VIEW_TARGET

        def fn():
            s = _lib.stream_ptr()
            r.forward(w, 1, view, row_offset=0, tok_offset=0, argmax_to=r.tok.data_ptr() + 4)
            r.tok[0:1].copy_(r.tok[1:2], non_blocking=True)
            if self.is_fp:
                _lib.check(lib.qs_add_int(c.d_len.data_ptr(), 1, 1, s), "qs_add_int")
            else:
                _lib.check(lib.qs_add_int(c.d_fp2_len.data_ptr(), 1, 1, s), "qs_add_int")
                _lib.check(lib.qs_add_int(c.d_pos.data_ptr(), 1, 1, s), "qs_add_int")
            self.host[:1].copy_(r.tok[1:2], non_blocking=True)

        return fn

    def step(self, *, sync: bool = True):
        """Decode one token (appends it to the cache); returns it when sync."""
        torch = _torch()
        self.graphs.run(("ar",), self._step_fn(), self.cache.generation)
        fused = self.run._fuse_prep(self.target.layers[0]["qkv"], self.cache.batch)
        self.launches += self.run.kernel_launches_per_forward(len(self.target.layers), fused) + 2
        if self.is_fp:
            self.cache._len += 1
        else:
            self.cache._fp2_len += 1
        if not sync:
            return None
        torch.cuda.current_stream().synchronize()
        return int(self.host[0])
