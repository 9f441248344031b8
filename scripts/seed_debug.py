"""Per-seed phase times and batch-path fallbacks of one rgg map (GIM_BATCH_DEBUG
prints general-path / strong-pass events of the batched multisection)."""
import sys

import torch

from paper_2510_12196_b200 import device as D
from paper_2510_12196_b200.generators import gen_rgg

logn = int(sys.argv[1]) if len(sys.argv) > 1 else 20
g = gen_rgg(1 << logn, 0.55, 1)
dg = D.DeviceGraph.from_host(g)
H, DIST = (4, 8, 6), (1, 10, 100)
for s in range(3):
    D.integrated_map_device(dg, H, DIST, 0.03, 1000 + s)
for seed in [int(x) for x in sys.argv[2:]] or [0, 3]:
    torch.cuda.synchronize()
    print(f"---- seed {seed}", file=sys.stderr, flush=True)
    a, bw, st = D.integrated_map_device(dg, H, DIST, 0.03, seed)
    torch.cuda.synchronize()
    print(seed, {k: round(st[k], 2) for k in ("ms_coarsen", "ms_initial", "ms_refine")},
          "init_iters", st["init_refine_iterations"], "strong", st["strong_passes"],
          "calls", st["partitioner_calls"], file=sys.stderr, flush=True)
