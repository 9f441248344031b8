"""Kernel-time breakdown of one R-MAT integrated_map (torch.profiler)."""
import collections
import json
import sys

import torch
from torch.profiler import ProfilerActivity, profile

from paper_2510_12196_b200 import device as D
from paper_2510_12196_b200.generators import gen_rmat

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 18
g = gen_rmat(scale)
dg = D.DeviceGraph.from_host(g)
h, d = (4, 8, 8), (1, 10, 100)
D.integrated_map_device(dg, h, d, 0.03, 0)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    a, bw, st = D.integrated_map_device(dg, h, d, 0.03, 1)
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for e in prof.events():
    if e.device_type != torch.autograd.DeviceType.CUDA:
        continue
    k = e.name.split("(")[0][-50:]
    agg[k][0] += 1
    agg[k][1] += e.device_time / 1e3
    agg[k][2] = max(agg[k][2], e.device_time / 1e3)
print(json.dumps({k: st[k] for k in ("ms_coarsen", "ms_initial", "ms_refine", "n_levels")}))
for k, (c, t, mx) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:15]:
    print(f"{k:52s} {c:6d} {t:10.2f} ms  max {mx:8.2f}")
