"""Batch partition of independent sequences across GPUs.

Sequences are independent, so one process per GPU runs its own engine and KV
store over a contiguous slice of the batch, with no collective on the data
path.  The only communication is job-level accounting at the end: the total
tokens emitted by all ranks and the maximum elapsed device time over ranks.
Works with any torch.distributed backend (``nccl`` on the GPU box, ``gloo``
in the CPU tests).
"""

from __future__ import annotations

from dataclasses import dataclass


def partition(n_items: int, world: int, rank: int) -> range:
    """Contiguous, balanced slice of ``n_items`` owned by ``rank`` (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


@dataclass
class JobThroughput:
    total_units: float  # units (tokens) processed by all ranks
    max_seconds: float  # slowest rank's timed region
    world: int

    @property
    def rate(self) -> float:
        return self.total_units / self.max_seconds if self.max_seconds > 0 else 0.0


def job_throughput(units: float, seconds: float, device=None) -> JobThroughput:
    """All-reduce (SUM units, MAX seconds) across the default process group.

    Without an initialised process group it is the local value (world 1)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return JobThroughput(float(units), float(seconds), 1)
    dev = device if device is not None else ("cuda" if dist.get_backend() == "nccl" else "cpu")
    u = torch.tensor([float(units)], dtype=torch.float64, device=dev)
    t = torch.tensor([float(seconds)], dtype=torch.float64, device=dev)
    dist.all_reduce(u, op=dist.ReduceOp.SUM)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return JobThroughput(float(u.item()), float(t.item()), dist.get_world_size())


class HeadGather:
    """Gather buffers + arrival counter of one rank for the fused all-gather of KV-head-sharded
    attention rows (qs_gather_args in include/quantspec_b200.h).

    Every buffer is its own cudaMalloc allocation (``qs_dev_alloc``) so it can be exported to the
    other ranks' processes as a CUDA IPC handle; ranks in one process (tests) link directly.
    ``gh`` holds two parity copies of the [rows][ld_h] f16 rows, ``gs`` of the [rows][ld_s] 16-sums.
    """

    def __init__(self, world: int, rank: int, rows: int, ld_h: int, ld_s: int):
        import ctypes as C

        from . import _lib

        if not 1 <= world <= _lib.MAX_RANKS or not 0 <= rank < world:
            raise ValueError(f"bad rank {rank} of world {world}")
        self.world, self.rank, self.rows, self.ld_h, self.ld_s = world, rank, rows, ld_h, ld_s
        self.par_h, self.par_s = rows * ld_h, rows * ld_s
        self._own = []

        def alloc(nbytes):
            p = C.c_void_p()
            _lib.call("qs_dev_alloc", nbytes, C.byref(p))
            self._own.append(p.value)
            return p.value

        self.gh = alloc(2 * self.par_h * 2)
        self.gs = alloc(2 * self.par_s * 4)
        self.flag = alloc(256)
        self.epoch = alloc(256)
        self.done = alloc(256)
        self.peer_gh = [None] * world
        self.peer_gs = [None] * world
        self.peer_flag = [None] * world
        self.peer_gh[rank], self.peer_gs[rank], self.peer_flag[rank] = self.gh, self.gs, self.flag
        self._opened = []

    # -- linking -------------------------------------------------------------------
    def handles(self) -> bytes:
        import ctypes as C

        from . import _lib

        out = b""
        for p in (self.gh, self.gs, self.flag):
            buf = C.create_string_buffer(64)
            _lib.call("qs_ipc_handle", p, buf)
            out += buf.raw
        return out

    def open_peers(self, all_handles) -> None:
        """``all_handles[i]`` = rank i's ``handles()`` (e.g. from dist.all_gather_object)."""
        import ctypes as C

        from . import _lib

        for i, h in enumerate(all_handles):
            if i == self.rank:
                continue
            ptrs = []
            for k in range(3):
                p = C.c_void_p()
                _lib.call("qs_ipc_open", C.create_string_buffer(h[64 * k: 64 * k + 64], 64), C.byref(p))
                self._opened.append(p.value)
                ptrs.append(p.value)
            self.peer_gh[i], self.peer_gs[i], self.peer_flag[i] = ptrs

    @classmethod
    def exchange(cls, world: int, rank: int, rows: int, ld_h: int, ld_s: int, group=None) -> "HeadGather":
        """Collective: every rank of ``group`` allocates its buffers and maps everyone else's."""
        import torch.distributed as dist

        g = cls(world, rank, rows, ld_h, ld_s)
        hs = [None] * world
        dist.all_gather_object(hs, g.handles(), group=group)
        g.open_peers(hs)
        return g

    @staticmethod
    def link_local(gathers) -> None:
        """Ranks living in one process (one stream each): peers are plain device pointers."""
        for g in gathers:
            for o in gathers:
                g.peer_gh[o.rank], g.peer_gs[o.rank], g.peer_flag[o.rank] = o.gh, o.gs, o.flag

    def fill(self, a, *, arrivals: int, q_col_offset: int) -> None:
        ga = a.gather
        ga.world, ga.rank, ga.q_col_offset, ga.arrivals = self.world, self.rank, q_col_offset, arrivals
        ga.par_stride_h, ga.par_stride_s = self.par_h, self.par_s
        for i in range(self.world):
            if self.peer_gh[i] is None:
                raise RuntimeError(f"rank {self.rank}: peer {i} not linked")
            ga.gh[i], ga.gs[i], ga.flag[i] = self.peer_gh[i], self.peer_gs[i], self.peer_flag[i]
        ga.epoch, ga.done = self.epoch, self.done

    def close(self) -> None:
        from . import _lib

        lib = _lib.load()
        for p in self._opened:
            lib.qs_ipc_close(p)
        for p in self._own:
            lib.qs_dev_free(p)
        self._opened, self._own = [], []
