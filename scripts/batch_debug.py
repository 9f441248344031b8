"""Compare batched vs general multisection on small rgg graphs (GIM_BATCH_DEBUG=1
prints per-job level-stack / partition comparisons)."""
import numpy as np
import torch

from paper_2510_12196_b200 import device as D
from paper_2510_12196_b200.generators import gen_rgg

for n in (3000, 6000):
    g = gen_rgg(n, 0.55, 1)
    dg = D.DeviceGraph.from_host(g)
    D.set_batch(False)
    a = D.hierarchical_multisection(dg, (4, 8, 6), (1, 10, 100), 0.03, 1).cpu().numpy()
    D.set_batch(True)
    b = D.hierarchical_multisection(dg, (4, 8, 6), (1, 10, 100), 0.03, 1).cpu().numpy()
    torch.cuda.synchronize()
    print(n, "equal" if np.array_equal(a, b) else f"DIFF {(a != b).sum()}", flush=True)
