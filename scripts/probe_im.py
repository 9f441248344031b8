"""Probe: run integrated_map on rgg graphs, print timing + stats; optionally
compare with the oracle (slow)."""
import argparse
import json
import time

import numpy as np
import torch

from paper_2510_12196_b200 import device as D
from paper_2510_12196_b200.generators import gen_rgg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--logn", type=int, nargs="+", default=[16, 20])
    ap.add_argument("--oracle", type=int, default=16, help="compare with oracle up to this logn")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--no-fanout", action="store_true")
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--seeds", type=int, nargs="+", default=[0])
    ap.add_argument("--no-host", action="store_true")
    args = ap.parse_args()
    D.set_fanout(not args.no_fanout)
    D.set_profiling(args.profile)
    h, d = (4, 8, 6), (1, 10, 100)
    for logn in args.logn:
        t0 = time.time()
        g = gen_rgg(1 << logn, 0.55, 1)
        print(f"gen 2^{logn}: n={g.n} m={g.m} {time.time()-t0:.1f}s", flush=True)
        dg = D.DeviceGraph.from_host(g)
        for seed in args.seeds:
            for r in range(args.reps):
                torch.cuda.synchronize()
                t0 = time.time()
                a, bw, st = D.integrated_map_device(dg, h, d, 0.03, seed)
                torch.cuda.synchronize()
                wall = time.time() - t0
                print(json.dumps({"logn": logn, "seed": seed, "rep": r, "wall_s": wall, **st}),
                      flush=True)
        if args.no_host:
            continue
        t0 = time.time()
        ah, bwh, st = D.integrated_map_host(g.offsets, g.edge_targets, g.edge_weights,
                                            g.vertex_weights, h, d, 0.03, 0)
        print(f"host-API e2e {time.time()-t0:.3f}s J={st['final_j']}", flush=True)
        assert np.array_equal(ah, a.cpu().numpy())
        if logn <= args.oracle:
            import sys
            sys.path.insert(0, ".")
            from oracle import promap_np as O
            t0 = time.time()
            ao, bwo, l_max = O.integrated_map(g, O.OTopology(h, d), 0.03, 0)
            print(f"oracle {time.time()-t0:.1f}s J={O.total_cost(g, O.OTopology(h, d), ao)} "
                  f"equal={np.array_equal(ao, ah)}", flush=True)


if __name__ == "__main__":
    main()
