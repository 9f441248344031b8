"""Timeline of one integrated_map (fan-out on) under torch.profiler (CUPTI):
exports a chrome trace to analyse GPU-busy fractions and host gaps per phase."""
import argparse
import json
import time

import torch
from torch.profiler import ProfilerActivity, profile

from paper_2510_12196_b200 import device as D
from paper_2510_12196_b200.generators import gen_rgg

H, DIST = (4, 8, 6), (1, 10, 100)
ap = argparse.ArgumentParser()
ap.add_argument("--logn", type=int, default=22)
ap.add_argument("--out", default="gpurun_out/timeline.json")
ap.add_argument("--seed", type=int, default=0)
ap.add_argument("--warm-seeds", type=int, default=2)
args = ap.parse_args()
g = gen_rgg(1 << args.logn, 0.55, 1)
dg = D.DeviceGraph.from_host(g)
for s in range(args.warm_seeds):
    D.integrated_map_device(dg, H, DIST, 0.03, s)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    a, bw, st = D.integrated_map_device(dg, H, DIST, 0.03, args.seed)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
prof.export_chrome_trace(args.out)
print(json.dumps({"wall_ms": wall * 1e3, **{k: st[k] for k in ("ms_coarsen", "ms_initial",
                                                               "ms_refine", "ms_total")}}))
