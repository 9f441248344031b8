"""Per-refinement trace (GIM_TRACE_REFINE=1 prints n, grid, mode, iterations,
ms per refine launch to stderr) for one partitioner call and one
integrated_map with the multisection fan-out off (serialised, so per-launch
times are not inflated by concurrency)."""
import argparse

import torch

from paper_2510_12196_b200 import device as D
from paper_2510_12196_b200.generators import gen_rgg

H, DIST = (4, 8, 6), (1, 10, 100)

ap = argparse.ArgumentParser()
ap.add_argument("--part-n", type=int, default=24000)
ap.add_argument("--logn", type=int, default=22)
args = ap.parse_args()
g = gen_rgg(args.part_n, 0.55, 1)
dg = D.DeviceGraph.from_host(g)
D.internal_partitioner(dg, 6, 0.03, 1)
torch.cuda.synchronize()
import sys
print("---- partitioner", args.part_n, file=sys.stderr, flush=True)
D.internal_partitioner(dg, 6, 0.03, 1)
torch.cuda.synchronize()
if args.logn:
    g = gen_rgg(1 << args.logn, 0.55, 1)
    dg = D.DeviceGraph.from_host(g)
    D.set_fanout(False)
    D.integrated_map_device(dg, H, DIST, 0.03, 0)
    torch.cuda.synchronize()
    print("---- integrated_map 2^%d" % args.logn, file=sys.stderr, flush=True)
    a, bw, st = D.integrated_map_device(dg, H, DIST, 0.03, 0)
    torch.cuda.synchronize()
    print({k: st[k] for k in ("ms_coarsen", "ms_initial", "ms_refine", "ms_total")}, file=sys.stderr)
