"""ncu targets (run under `ncu --profile-from-start off ...`).

  --mode step : warm-up map, then ONE integrated_map inside the capture
                window (launch list / per-kernel share of a step)
  --mode lp   : warm-up map, then the level-0 LP / J / HEM / contraction
                kernels on the final mapping inside the window (full sets)
  --mode refine0 : warm-up map, then ONE device-resident Alg. 4 refinement
                (k_refine_fused) of the finest level inside the window,
                started from the final mapping with 2% of the vertices moved
                to random blocks (LP + weak-rebalance work as on level 0)
"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2510_12196_b200 import device as D  # noqa: E402
from paper_2510_12196_b200.generators import gen_rgg  # noqa: E402

H, DIST = (4, 8, 6), (1, 10, 100)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", choices=["step", "lp", "refine0"], default="step")
    ap.add_argument("--logn", type=int, default=20)
    ap.add_argument("--graph", choices=["rgg", "rmat"], default="rgg",
                    help="rmat: R-MAT scale --logn, H=4:8:8 (config 3)")
    ap.add_argument("--cache", default="", help="npz cache of the generated graph")
    ap.add_argument("--level", type=int, default=0,
                    help="refine0: refine this level of the stack instead of level 0")
    args = ap.parse_args()
    global H
    if args.graph == "rmat":
        import os
        import numpy as np
        from paper_2510_12196_b200.generators import HostGraph, gen_rmat
        H = (4, 8, 8)
        if args.cache and os.path.exists(args.cache):
            z = np.load(args.cache)
            g = HostGraph(z["o"], z["t"], z["w"], z["vw"])
        else:
            g = gen_rmat(args.logn)
            if args.cache:
                np.savez(args.cache, o=g.offsets, t=g.edge_targets, w=g.edge_weights,
                         vw=g.vertex_weights)
    else:
        g = gen_rgg(1 << args.logn, 0.55, 1)
    dg = D.DeviceGraph.from_host(g)
    if args.mode == "refine0" and args.level > 0:
        k0 = 1
        for x in H:
            k0 *= x
        l_max0 = 1.03 * dg.total_weight / k0
        for li in range(args.level):  # coarsen down to the requested level
            partner = D.match_graph(dg, l_max0, 1000 + li)
            cmap, n_c = D.coarse_map(partner)
            dg = D.contract(dg, cmap, n_c)
        print("level", args.level, "n", dg.n, "m2", dg.m2)
    a, bw, st = D.integrated_map_device(dg, H, DIST, 0.03, 0)
    torch.cuda.synchronize()
    prof = torch.cuda.profiler
    if args.mode == "step":
        prof.start()
        D.integrated_map_device(dg, H, DIST, 0.03, 1)
        torch.cuda.synchronize()
        prof.stop()
    elif args.mode == "refine0":
        k = 1
        for x in H:
            k *= x
        gen = torch.Generator(device="cuda").manual_seed(5)
        idx = torch.randperm(dg.n, device="cuda", generator=gen)[: dg.n // 50]
        a = a.clone()
        a[idx] = torch.randint(0, k, (idx.numel(),), device="cuda", dtype=torch.int32,
                               generator=gen)
        bw2 = D.block_weights(dg, a, k)
        l_max = 1.03 * dg.total_weight / k
        torch.cuda.synchronize()
        prof.start()
        D.refine(dg, H, DIST, a, bw2, i_max=12 + args.level,
                 i_w_max=10 if args.level == 0 else 2,
                 sigma_fraction=0.005 if args.level == 0 else 0.03, seed=3, l_max=l_max)
        torch.cuda.synchronize()
        prof.stop()
    else:
        locked = torch.zeros(dg.n, dtype=torch.uint8, device="cuda")
        prof.start()
        for _ in range(3):
            D.lp_pass(dg, a, locked, H, DIST)
        D.total_cost(dg, a, H, DIST)
        partner = torch.full((dg.n,), -1, dtype=torch.int32, device="cuda")
        D.hem_round(dg, partner, 1e9, 12345, 0)
        cmap, n_c = D.coarse_map(partner)
        D.contract(dg, cmap, n_c)
        torch.cuda.synchronize()
        prof.stop()
    print("done", st["final_j"])


if __name__ == "__main__":
    main()
