"""Golden fixtures for the multisection plugin seam (pipelines.py:49-110),
made by running the REFERENCE package: trace records with the built-in
partitioner and mappings + traces with a deterministic custom partitioner
(vertex-index blocks), for the GPU-HM plugin tests.

    python scripts/make_golden_plugin.py   ->  tests/golden/plugin.npz
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from promap.graph import gen_grid, gen_rgg  # noqa: E402
from promap.pipelines import hierarchical_multisection  # noqa: E402
from promap.topology import Topology  # noqa: E402

OUT = Path(__file__).resolve().parents[1] / "tests" / "golden" / "plugin.npz"


def index_blocks(sub, parts, eps_local, seed):
    """A deterministic custom partitioner: contiguous vertex-index blocks,
    rotated by the node seed (exercises the seed argument)."""
    n = sub.n
    base = (np.arange(n, dtype=np.int64) * parts) // max(n, 1)
    return (base + seed % parts) % parts


def run(tag, g, t, partitioner, bag):
    trace = []
    m = hierarchical_multisection(g, t, 0.03, partitioner=partitioner, seed=5, trace=trace)
    bag[f"{tag}/assignment"] = m.assignment
    bag[f"{tag}/block_weights"] = m.block_weights
    bag[f"{tag}/trace_level"] = np.asarray([r.level for r in trace])
    bag[f"{tag}/trace_ident"] = np.asarray(["/".join(map(str, r.identifier)) for r in trace])
    bag[f"{tag}/trace_parts"] = np.asarray([r.parts for r in trace])
    bag[f"{tag}/trace_eps"] = np.asarray([r.eps_local for r in trace])
    bag[f"{tag}/trace_weight"] = np.asarray([r.subgraph_weight for r in trace])
    bag[f"{tag}/trace_bw"] = np.asarray([",".join(map(str, r.block_weights)) for r in trace])
    bag[f"{tag}/trace_met"] = np.asarray([r.budget_met for r in trace])
    print(tag, len(trace), "records")


bag = {}
for tag, g, h in [("grid", gen_grid(24, 24), (2, 2, 2)), ("rgg", gen_rgg(1500, 0.55, 3), (4, 3))]:
    t = Topology(h, (1, 10, 100)[:len(h)])
    bag[f"{tag}/offsets"] = g.offsets
    bag[f"{tag}/targets"] = g.edge_targets
    bag[f"{tag}/weights"] = g.edge_weights
    bag[f"{tag}/vweights"] = g.vertex_weights
    bag[f"{tag}/hierarchy"] = np.asarray(h)
    run(f"{tag}/builtin", g, t, None, bag)
    run(f"{tag}/custom", g, t, index_blocks, bag)
np.savez_compressed(OUT, **bag)
