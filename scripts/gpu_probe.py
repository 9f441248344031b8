"""Quick GPU probe: J-eval and block weights vs numpy on a few graphs."""
import time

import numpy as np
import torch

from paper_2510_12196_b200 import device as D
from paper_2510_12196_b200.generators import gen_grid, gen_rgg


def np_dist(h, d, x, y):
    top = np.full(x.shape, -1)
    x = x.copy(); y = y.copy()
    for i, a in enumerate(h):
        top[(x % a) != (y % a)] = i
        x //= a; y //= a
    dv = np.asarray(d)
    return np.where(top >= 0, dv[np.maximum(top, 0)], 0)


def main():
    print(torch.cuda.get_device_name(0))
    for g, h, d in [(gen_grid(128, 128), (4, 8, 2), (1, 10, 100)),
                    (gen_rgg(1 << 16, 0.55, 1), (4, 8, 6), (1, 10, 100))]:
        k = int(np.prod(h))
        a = np.random.default_rng(0).integers(0, k, g.n)
        ref = int((np_dist(h, d, a[g.edge_sources], a[g.edge_targets]) * g.edge_weights).sum())
        dg = D.DeviceGraph.from_host(g)
        at = torch.from_numpy(a).cuda()
        j = D.total_cost(dg, at, h, d)
        bw = D.block_weights(dg, at, k).cpu().numpy()
        bw_ref = np.bincount(a, weights=g.vertex_weights, minlength=k).astype(np.int64)
        print(g.n, ref, j, ref == j, np.array_equal(bw, bw_ref))


if __name__ == "__main__":
    main()
