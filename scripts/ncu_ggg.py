"""ncu target: one large-graph greedy growing (k_ggg_large) on an R-MAT graph."""
import sys

import torch

from paper_2510_12196_b200 import device as D
from paper_2510_12196_b200.generators import gen_rmat

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 17
k = int(sys.argv[2]) if len(sys.argv) > 2 else 8
g = gen_rmat(scale)
dg = D.DeviceGraph.from_host(g)
torch.cuda.synchronize()
import time
t0 = time.perf_counter()
D.greedy_graph_growing(dg, k)
torch.cuda.synchronize()
print("ggg ms", (time.perf_counter() - t0) * 1e3, "n", g.n, "m2", len(g.edge_targets))
