"""METIS input timing (the paper's "I/O = 74.9 % of GPU-IM
time"): write the bench graph (rgg 2^logn) as a METIS file, then time the
native loader (paper_2510_12196_b200.load_metis, C++ in libgpuim.so) and the
reference's pure-Python promap.graph.load_metis (graph.py:185-294, from
baseline/_ref) on the same file; both must return the identical CSR.

    python scripts/bench_metis.py --logn 22 [--no-ref]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def write_metis(g, path: str) -> None:
    n = len(g.offsets) - 1
    off = g.offsets
    tg = (g.edge_targets + 1).astype(np.int64)
    with open(path, "w") as fh:
        fh.write(f"{n} {len(tg) // 2}\n")
        step = 1 << 16
        for a in range(0, n, step):
            b = min(n, a + step)
            rows = np.split(tg[off[a]:off[b]], (off[a + 1:b] - off[a]))
            fh.write("\n".join(" ".join(map(str, r.tolist())) for r in rows))
            fh.write("\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--logn", type=int, default=22)
    ap.add_argument("--no-ref", action="store_true")
    args = ap.parse_args()
    from paper_2510_12196_b200 import load_metis
    from paper_2510_12196_b200.generators import gen_rgg
    g = gen_rgg(1 << args.logn, 0.55, 1)
    fd, path = tempfile.mkstemp(suffix=".metis")
    os.close(fd)
    t0 = time.perf_counter()
    write_metis(g, path)
    out = {"graph": f"rgg 2^{args.logn} (graph seed 1)", "n": g.n, "m": g.m,
           "file_bytes": os.path.getsize(path), "write_s": time.perf_counter() - t0}
    load_metis(path)  # page cache warm
    t0 = time.perf_counter()
    mine = load_metis(path)
    out["native_s"] = time.perf_counter() - t0
    ok = np.array_equal(mine.offsets, g.offsets) and np.array_equal(mine.edge_targets,
                                                                      g.edge_targets)
    out["native_equals_generator"] = bool(ok)
    # straight to a device CSR (parse + narrow + upload), the mapping's input
    import torch
    from paper_2510_12196_b200.metis import load_metis_device
    load_metis_device(path)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dg = load_metis_device(path)
    torch.cuda.synchronize()
    out["native_to_device_s"] = time.perf_counter() - t0
    out["device_csr_equal"] = bool(np.array_equal(dg.offsets.cpu().numpy(), g.offsets) and
                                   np.array_equal(dg.targets.cpu().numpy(), g.edge_targets))
    ref_dir = ROOT / "baseline" / "_ref"
    if not args.no_ref and (ref_dir / "promap").is_dir():
        sys.path.insert(0, str(ref_dir))
        from promap.graph import load_metis as ref_load
        t0 = time.perf_counter()
        ref = ref_load(path)
        out["reference_s"] = time.perf_counter() - t0
        out["identical_csr"] = bool(
            np.array_equal(ref.offsets, mine.offsets) and
            np.array_equal(ref.edge_targets, mine.edge_targets) and
            np.array_equal(ref.edge_weights, mine.edge_weights) and
            np.array_equal(ref.vertex_weights, mine.vertex_weights))
        out["speedup"] = out["reference_s"] / out["native_s"]
    os.unlink(path)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
