"""Run the BASELINE configs 3 and 4 (R-MAT scale 22 -> H=4:8:8, 3D grid
256^3 -> H=4:16:8) through integrated_map_device: time, balance, J."""
import argparse
import json
import time

import torch

from paper_2510_12196_b200 import device as D
from paper_2510_12196_b200.generators import gen_grid3d, gen_rmat

ap = argparse.ArgumentParser()
ap.add_argument("--which", nargs="+", default=["rmat", "grid3d"])
ap.add_argument("--rmat-scale", type=int, default=22)
ap.add_argument("--grid", type=int, default=256)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--profile", action="store_true", help="serialised per-class device times")
ap.add_argument("--isolated", nargs="+", default=["keep"], choices=["keep", "strip"],
                help="isolated-vertex modes to run (R-MAT: strip = tolerance-parity mode)")
ap.add_argument("--cache", default="", help="npz path: reuse the generated graph across runs")
args = ap.parse_args()
D.set_profiling(args.profile)
for w in args.which:
    t0 = time.time()
    if w == "rmat":
        import os
        import numpy as np
        from paper_2510_12196_b200.generators import HostGraph
        if args.cache and os.path.exists(args.cache):
            z = np.load(args.cache)
            g = HostGraph(z["o"], z["t"], z["w"], z["vw"])
        else:
            g = gen_rmat(args.rmat_scale)
            if args.cache:
                np.savez(args.cache, o=g.offsets, t=g.edge_targets, w=g.edge_weights,
                         vw=g.vertex_weights)
        h, d = (4, 8, 8), (1, 10, 100)
    else:
        g = gen_grid3d(args.grid, args.grid, args.grid)
        h, d = (4, 16, 8), (1, 10, 100)
    print(f"{w}: n={g.n} m={g.m} gen {time.time() - t0:.1f}s", flush=True)
    dg = D.DeviceGraph.from_host(g)
    for iso, r in [(i, r) for i in args.isolated for r in range(args.reps)]:
        torch.cuda.synchronize()
        t0 = time.time()
        a, bw, st = D.integrated_map_device(dg, h, d, 0.03, r, isolated_vertices=iso)
        torch.cuda.synchronize()
        print(json.dumps({"cfg": w, "isolated": iso, "rep": r, "wall_ms": (time.time() - t0) * 1e3,
                          "isolated_vertices": st["isolated_vertices"],
                          "J": st["final_j"], "maxw": st["max_block_weight"],
                          "l_max": st["l_max"], "balanced": st["max_block_weight"] <= st["l_max"],
                          "levels": st["n_levels"], "level_n": st["level_n"],
                          **{k: round(st[k], 1) for k in ("ms_coarsen", "ms_initial",
                                                          "ms_refine")},
                          "profile": {k: round(v["ms"], 1) for k, v in st.get("profile", {}).items()},
                          "top_launch": st.get("top_launch")}), flush=True)
