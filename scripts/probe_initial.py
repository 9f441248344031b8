"""Probe the initial-mapping phase (hierarchical multisection of the coarsest
graph): wall time with/without sibling fan-out, single partitioner calls at
the sizes the multisection sees, and (--kineto) the device-busy share from a
torch.profiler (CUPTI) trace — how much of the wall time is kernels vs host
latency (launch + sync)."""
import argparse
import json
import time

import torch

from paper_2510_12196_b200 import device as D
from paper_2510_12196_b200.generators import gen_rgg

H, DIST = (4, 8, 6), (1, 10, 100)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3


def kineto(fn, label, trace=None):
    from torch.profiler import ProfilerActivity, profile
    fn()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
    if trace:
        prof.export_chrome_trace(trace)
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    busy = sum(e.device_time for e in ev) / 1e3
    by = {}
    for e in ev:
        k = e.name.split("(")[0][:60]
        c, t = by.get(k, (0, 0.0))
        by[k] = (c + 1, t + e.device_time / 1e3)
    top = sorted(by.items(), key=lambda kv: -kv[1][1])[:25]
    print(json.dumps({"probe": label, "wall_ms_profiled": wall, "kernels": len(ev),
                      "device_busy_ms": busy,
                      "top": [{"k": k, "n": c, "ms": round(t, 3)} for k, (c, t) in top]}),
          flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="+", default=[24000, 4000, 500])
    ap.add_argument("--kineto", action="store_true")
    ap.add_argument("--trace", default="", help="chrome-trace prefix (under gpurun_out/)")
    args = ap.parse_args()
    for n in args.n:
        g = gen_rgg(n, 0.55, 1)
        dg = D.DeviceGraph.from_host(g)
        parts = {24000: 6, 4000: 8, 500: 4}.get(n, 6)
        r = {"n": n, "m": g.m, "parts": parts}
        r["partitioner_ms"] = timed(lambda: D.internal_partitioner(dg, parts, 0.03, 1))
        if n >= 4000:
            D.set_fanout(True)
            r["multisection_fanout_ms"] = timed(
                lambda: D.hierarchical_multisection(dg, H, DIST, 0.03, 1))
            D.set_fanout(False)
            r["multisection_serial_ms"] = timed(
                lambda: D.hierarchical_multisection(dg, H, DIST, 0.03, 1))
            D.set_fanout(True)
        print(json.dumps(r), flush=True)
        if args.kineto:
            tr = f"{args.trace}_part{n}.json" if args.trace else None
            kineto(lambda: D.internal_partitioner(dg, parts, 0.03, 1), f"partitioner n={n}", tr)
            if n >= 4000:
                D.set_fanout(False)
                kineto(lambda: D.hierarchical_multisection(dg, H, DIST, 0.03, 1),
                       f"multisection serial n={n}")
                D.set_fanout(True)
                tr = f"{args.trace}_ms{n}.json" if args.trace else None
                kineto(lambda: D.hierarchical_multisection(dg, H, DIST, 0.03, 1),
                       f"multisection fanout n={n}", tr)


if __name__ == "__main__":
    main()
