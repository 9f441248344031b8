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
    js = bench.gather_lists([10 * rank + i for i in range(rank + 1)], world)
    dist.barrier()
    q.put((rank, tmax, value, js))
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
    for _, tmax, value, js in res:
        assert tmax == 150.0
        assert value == pytest.approx(1000 * 4 * 2 / 0.150)
        # config-5 results gathered over the gloo group in rank order
        assert js == [0, 10, 11]


# ---------------------------------------------------------------------------
# config-5 replica runner (paper_2510_12196_b200/replicas.py): job split and
# aggregation across spawned processes, no NCCL

def _fake_child(rank, gpu, seeds, logn, concurrency, barrier, q):
    """Stands in for the GPU mapper: every 'map' of seed s takes 20 ms and
    reports J = 1000 + s; rank 1 starts late to exercise the wall span."""
    import time
    barrier.wait()
    if rank == 1:
        time.sleep(0.05)
    t0 = time.time()
    jobs = []
    for s in seeds:
        time.sleep(0.02 / max(concurrency, 1))
        jobs.append({"seed": s, "J": 1000 + s, "ms": 20.0, "balanced": True})
    q.put({"rank": rank, "t_start": t0, "t_end": time.time(), "jobs": jobs, "m": 500})


def test_split_jobs_covers_every_seed_once():
    from paper_2510_12196_b200.replicas import split_jobs
    for g in (1, 2, 3, 4, 8):
        parts = split_jobs(list(range(64)), g)
        assert sorted(s for p in parts for s in p) == list(range(64))
        assert max(map(len, parts)) - min(map(len, parts)) <= 1


def test_replica_runner_processes_aggregate():
    import math

    from paper_2510_12196_b200 import replicas
    out = replicas.run(gpus=2, jobs=10, concurrency=2, logn=10, child=_fake_child)
    assert out["maps"] == 10 and out["gpus"] == 2 and out["jobs"] == 10
    assert out["edges_per_s"] == pytest.approx(10 * 500 / out["wall_s"])
    assert out["wall_s"] >= 0.05  # spans the late rank
    assert out["J_geomean"] == pytest.approx(math.exp(sum(math.log(1000 + s)
                                                          for s in range(10)) / 10))
    assert out["balanced"]
