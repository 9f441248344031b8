"""ncu target: internal_partitioner calls on a small rgg graph (the
multisection leaves' size) — k_refine_smem / k_ggg launches."""
import sys

import torch

from paper_2510_12196_b200 import device as D
from paper_2510_12196_b200.generators import gen_rgg

n = int(sys.argv[1]) if len(sys.argv) > 1 else 500
parts = int(sys.argv[2]) if len(sys.argv) > 2 else 4
g = gen_rgg(n, 0.55, 1)
dg = D.DeviceGraph.from_host(g)
D.internal_partitioner(dg, parts, 0.03, 1)
torch.cuda.synchronize()
torch.cuda.profiler.start()
D.internal_partitioner(dg, parts, 0.03, 1)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
