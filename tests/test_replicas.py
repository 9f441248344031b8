"""Multi-GPU path of bench.py (replicas) on CPU with gloo,
world_size 2: the job time is the max over ranks and the aggregate
throughput counts every rank's maps."""
from __future__ import annotations

import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    local = 100.0 + 50.0 * rank          # rank 1 is the slow replica
    tmax = bench.max_over_ranks(local, world, "cpu")
    value = bench.job_throughput(1000, 4, world, tmax)
    dist.barrier()
    q.put((rank, tmax, value))
    dist.destroy_process_group()


def test_max_over_ranks_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(world))
    for _, tmax, value in res:
        assert tmax == 150.0
        assert value == pytest.approx(1000 * 4 * 2 / 0.150)
