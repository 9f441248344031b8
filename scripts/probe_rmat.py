"""R-MAT probe: per-kernel device time of one integrated_map (torch.profiler /
CUPTI), with launch counts and the longest single launch per kernel."""
import argparse
import json
import time
from collections import defaultdict

import torch
from torch.profiler import ProfilerActivity, profile

from paper_2510_12196_b200 import device as D
from paper_2510_12196_b200.generators import gen_rmat

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=17)
ap.add_argument("--top", type=int, default=25)
ap.add_argument("--trace", default="", help="chrome trace output path")
args = ap.parse_args()
g = gen_rmat(args.scale)
dg = D.DeviceGraph.from_host(g)
h, d = (4, 8, 8), (1, 10, 100)
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    a, bw, st = D.integrated_map_device(dg, h, d, 0.03, 0)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
if args.trace:
    prof.export_chrome_trace(args.trace)
by = defaultdict(lambda: [0, 0.0, 0.0])
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        k = e.name.split("(")[0][-48:]
        r = by[k]
        r[0] += 1
        r[1] += e.device_time / 1e3
        r[2] = max(r[2], e.device_time / 1e3)
print(json.dumps({"scale": args.scale, "n": g.n, "m": g.m, "wall_ms": wall * 1e3,
                  **{k: round(st[k], 1) for k in ("ms_coarsen", "ms_initial", "ms_refine")},
                  "level_n": st["level_n"]}))
for k, (c, t, mx) in sorted(by.items(), key=lambda kv: -kv[1][1])[:args.top]:
    print(f"{k:50s} {c:7d} {t:10.2f} ms  max {mx:8.2f} ms")
