"""World-size-2 test of the multi-GPU host path on CPU (gloo backend):
batch partition + job-level accounting (sum of tokens, max of per-rank time),
exactly what bench.py does under torchrun with nccl."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, batch, q):
    import torch.distributed as dist

    from paper_2502_10424_b200.parallel import job_throughput, partition

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = partition(batch, world, rank)
        # each "sequence" emits (index + 1) tokens; ranks take different times
        tokens = sum(i + 1 for i in mine)
        seconds = 1.0 + rank
        jt = job_throughput(tokens, seconds)
        q.put((rank, list(mine), jt.total_units, jt.max_seconds, jt.world))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("batch", [8, 5])
def test_batch_partition_and_job_accounting_world2(batch):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, batch, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(world))
    owned = [i for _, m, *_ in res for i in m]
    assert owned == list(range(batch))
    want_tokens = sum(i + 1 for i in range(batch))
    for _, _, total, mx, w in res:
        assert total == want_tokens
        assert mx == 2.0
        assert w == world
