"""Config-5 replica runner: many independent GPU-IM maps over the GPUs of one box.

SURVEY.md §8(e) / BASELINE.json configs[4]: 64 independent jobs (mapping
seeds 0..63 of the rgg 2^22 instance, H=4:8:6) split evenly over G GPUs, one
host process per GPU, no NCCL and no inter-GPU traffic (one mapping needs
the whole graph for refinement; it does not shard).  Inside a process,
`concurrency` maps run at once on separate CUDA streams from separate host
threads, so one map's latency-bound coarse levels and initial multisection
overlap another's bandwidth-bound finest levels.  The parent gathers the
results over multiprocessing queues and reports aggregate edges/s = sum of
the edges mapped / (last end - first start).

    python -m paper_2510_12196_b200.replicas --gpus 8 --jobs 64 --concurrency 3

Every per-call switch travels in the call's own parameters (run contexts,
include/gpuim.h `run_flags`), so concurrent maps in one process are
independent; `tests/test_gpu_runtime.py` checks that two concurrent maps
equal the serial ones.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import queue
import threading
import time

H = (4, 8, 6)
DIST = (1, 10, 100)
EPS = 0.03


def split_jobs(jobs: list, workers: int) -> list[list]:
    """Round-robin split of the job list over `workers` processes (every
    worker gets floor or ceil of len/workers jobs, seeds interleaved)."""
    return [jobs[i::workers] for i in range(workers)]


def aggregate(results: list[dict], m: int) -> dict:
    """Whole-job numbers from the per-process records: edges mapped by all
    processes over the wall span from the first start to the last end."""
    t0 = min(r["t_start"] for r in results)
    t1 = max(r["t_end"] for r in results)
    maps = sum(len(r["jobs"]) for r in results)
    js = [j["J"] for r in results for j in r["jobs"]]
    return {"maps": maps, "wall_s": t1 - t0, "edges_per_s": maps * m / (t1 - t0),
            "J_geomean": math.exp(sum(math.log(x) for x in js) / len(js)) if js else None,
            "balanced": all(j["balanced"] for r in results for j in r["jobs"])}


class DeviceRunner:
    """`concurrency` host threads, each driving its own CUDA stream, mapping
    seeds on one resident graph.  The streams persist across warm() and
    run(), so the library's per-stream scratch caches are warm when timed."""

    def __init__(self, dg, concurrency: int, hierarchy=H, distances=DIST, eps=EPS):
        import torch

        self.dg, self.h, self.d, self.eps = dg, hierarchy, distances, eps
        self.streams = [torch.cuda.Stream(device=dg.device) for _ in range(max(concurrency, 1))]

    def warm(self, rounds: int = 1) -> None:
        self.run([10**6 + i for i in range(rounds * len(self.streams))])

    def run(self, seeds: list[int]) -> dict:
        """Map every seed; returns {t_start, t_end, jobs: [{seed, J, ms, balanced}]}."""
        import torch

        from . import device as D

        dev = self.dg.device
        work: queue.Queue = queue.Queue()
        for s in seeds:
            work.put(s)
        out: list[dict] = []
        lock = threading.Lock()
        errs: list[BaseException] = []

        def worker(st):
            torch.cuda.set_device(dev)
            with torch.cuda.stream(st):
                while True:
                    try:
                        s = work.get_nowait()
                    except queue.Empty:
                        return
                    try:
                        t0 = time.perf_counter()
                        _, _, stt = D.integrated_map_device(self.dg, self.h, self.d, self.eps, s)
                        ms = (time.perf_counter() - t0) * 1e3
                    except BaseException as e:  # noqa: BLE001 - re-raised below
                        errs.append(e)
                        return
                    with lock:
                        out.append({"seed": s, "J": stt["final_j"], "ms": ms,
                                    "balanced": stt["max_block_weight"] <= stt["l_max"]})

        torch.cuda.synchronize(dev)
        t_start = time.time()
        threads = [threading.Thread(target=worker, args=(st,)) for st in self.streams]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        torch.cuda.synchronize(dev)
        t_end = time.time()
        if errs:
            raise errs[0]
        out.sort(key=lambda r: r["seed"])
        return {"t_start": t_start, "t_end": t_end, "jobs": out}


def _child(rank: int, gpu: int, seeds: list[int], logn: int, concurrency: int, barrier, q):
    os.environ["CUDA_VISIBLE_DEVICES"] = str(gpu)  # before CUDA initialises here
    try:
        import torch

        from . import device as D
        from .generators import gen_rgg

        torch.cuda.set_device(0)
        g = gen_rgg(1 << logn, 0.55, 1)  # generated and uploaded outside the timing
        dg = D.DeviceGraph.from_host(g)
        runner = DeviceRunner(dg, concurrency)
        runner.warm()
        barrier.wait()
        res = runner.run(seeds)
        barrier.wait()
        res["rank"] = rank
        res["m"] = g.m
        q.put(res)
    except BaseException as e:  # noqa: BLE001 - reported to the parent
        q.put({"rank": rank, "error": repr(e)})
        barrier.abort()


def run(gpus: int, jobs: int, concurrency: int, logn: int = 22, child=None) -> dict:
    """Config 5 on `gpus` GPUs: one spawned process per GPU, no NCCL.
    `child(rank, gpu, seeds, logn, concurrency, barrier, queue)` is the
    per-process body (default: the GPU mapper)."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    parts = split_jobs(list(range(jobs)), gpus)
    barrier = ctx.Barrier(gpus)
    q = ctx.Queue()
    procs = [ctx.Process(target=child or _child,
                         args=(r, r, parts[r], logn, concurrency, barrier, q))
             for r in range(gpus)]
    for p in procs:
        p.start()
    results = [q.get() for _ in procs]
    for p in procs:
        p.join()
    bad = [r for r in results if "error" in r]
    if bad:
        raise RuntimeError(f"replica process failed: {bad[0]}")
    m = results[0]["m"]
    agg = aggregate(results, m)
    agg.update({"gpus": gpus, "jobs": jobs, "concurrency": concurrency, "m": m,
                "n": 1 << logn, "per_process_wall_s": sorted(
                    r["t_end"] - r["t_start"] for r in results)})
    return agg


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--jobs", type=int, default=64)
    ap.add_argument("--concurrency", type=int, default=3)
    ap.add_argument("--logn", type=int, default=22)
    a = ap.parse_args()
    print(json.dumps(run(a.gpus, a.jobs, a.concurrency, a.logn)), flush=True)


if __name__ == "__main__":
    main()
