"""One shared-memory-resident refinement (k_refine_smem, n <= 1000) on its
own, for ncu: rgg n=2^9, k=4 flat topology, a random start partition."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2510_12196_b200 import device as D  # noqa: E402
from paper_2510_12196_b200.generators import gen_rgg  # noqa: E402

logn = int(sys.argv[1]) if len(sys.argv) > 1 else 9
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
g = gen_rgg(1 << logn, 0.55, 3)
dg = D.DeviceGraph.from_host(g)
rng = np.random.default_rng(1)
for rep in range(2):
    a = torch.from_numpy(rng.integers(0, k, g.n).astype(np.int32)).cuda()
    bw = D.block_weights(dg, a, k)
    torch.cuda.synchronize()
    if rep == 1:
        torch.cuda.profiler.start()
    D.refine(dg, (k,), (1,), a, bw, i_max=12, i_w_max=2, sigma_fraction=0.03, jet=True,
             seed=7, l_max=1.03 * g.n / k)
    torch.cuda.synchronize()
    if rep == 1:
        torch.cuda.profiler.stop()
print("n", g.n, "m2", 2 * g.m)
