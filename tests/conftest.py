"""Shared pytest setup: the `gpu` marker, repo on sys.path, golden loaders."""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libgpuim.so")


class Case(dict):
    """One golden case: dict of arrays plus a graph builder."""

    def graph(self):
        from oracle.promap_np import OGraph
        return OGraph(self["offsets"], self["targets"], self["weights"], self["vweights"])

    def topology(self):
        from oracle.promap_np import OTopology
        return OTopology(tuple(int(x) for x in self["hierarchy"]),
                         tuple(int(x) for x in self["distances"]))

    def scalar(self, key):
        return self[key].item()


def load_golden(name: str) -> list[Case]:
    z = np.load(GOLDEN / f"{name}.npz")
    cases = [Case() for _ in range(int(z["count"]))]
    for key in z.files:
        if key == "count":
            continue
        i, field = key.split("/", 1)
        cases[int(i)][field] = z[key]
    return cases


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = load_golden(name)
        return cache[name]
    return get


def csr_digest(g) -> np.ndarray:
    """Order-sensitive uint64 digests of (offsets, targets, weights, vweights);
    the same function scripts/make_golden_scale.py stored with each fixture."""
    out = []
    for a in (g.offsets, g.edge_targets, g.edge_weights, g.vertex_weights):
        a = np.asarray(a, dtype=np.uint64)
        mult = (np.arange(len(a), dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
                + np.uint64(1))
        with np.errstate(over="ignore"):
            out.append(np.uint64(np.sum(a * mult, dtype=np.uint64)))
    return np.asarray(out, dtype=np.uint64)


def load_npz(name: str) -> dict:
    z = np.load(GOLDEN / f"{name}.npz")
    return {k: z[k] for k in z.files}
