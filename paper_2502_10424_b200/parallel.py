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
