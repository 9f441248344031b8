"""GPU-HM's plugin seam and trace records (pipelines.py:49-110), pinned to the
reference's own outputs (tests/golden/plugin.npz, scripts/make_golden_plugin.py):
the built-in partitioner's trace records, a custom partitioner's mapping and
trace (called per node in the reference's depth-first order), and the
reference's error wrapping for failing / invalid partitioners."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import load_npz

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def Z():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return load_npz("plugin")


class Topo:
    def __init__(self, h):
        self.hierarchy = tuple(int(x) for x in h)
        self.distances = (1, 10, 100)[:len(self.hierarchy)]


def index_blocks(sub, parts, eps_local, seed):
    n = sub.n if hasattr(sub, "n") else len(sub.offsets) - 1
    base = (np.arange(n, dtype=np.int64) * parts) // max(n, 1)
    return (base + seed % parts) % parts


def graph(Z, tag):
    from paper_2510_12196_b200.generators import HostGraph
    return HostGraph(Z[f"{tag}/offsets"], Z[f"{tag}/targets"], Z[f"{tag}/weights"],
                     Z[f"{tag}/vweights"])


def check_trace(Z, key, trace):
    assert [r.level for r in trace] == list(Z[f"{key}/trace_level"])
    assert ["/".join(map(str, r.identifier)) for r in trace] == list(Z[f"{key}/trace_ident"])
    assert [r.parts for r in trace] == list(Z[f"{key}/trace_parts"])
    assert [r.eps_local for r in trace] == list(Z[f"{key}/trace_eps"])
    assert [r.subgraph_weight for r in trace] == list(Z[f"{key}/trace_weight"])
    assert [",".join(map(str, r.block_weights)) for r in trace] == list(Z[f"{key}/trace_bw"])
    assert [r.budget_met for r in trace] == list(Z[f"{key}/trace_met"])


@pytest.mark.parametrize("tag", ["grid", "rgg"])
@pytest.mark.parametrize("which", ["builtin", "custom"])
def test_multisection_plugin_and_trace_match_reference(Z, tag, which):
    from paper_2510_12196_b200 import hierarchical_multisection
    g = graph(Z, tag)
    t = Topo(Z[f"{tag}/hierarchy"])
    trace: list = []
    calls: list = []

    def custom(sub, parts, eps_local, seed):
        calls.append((sub.n, parts))
        return index_blocks(sub, parts, eps_local, seed)

    m = hierarchical_multisection(g, t, 0.03, partitioner=custom if which == "custom" else None,
                                  seed=5, trace=trace)
    key = f"{tag}/{which}"
    assert np.array_equal(m.assignment, Z[f"{key}/assignment"])
    assert np.array_equal(m.block_weights, Z[f"{key}/block_weights"])
    check_trace(Z, key, trace)
    if which == "custom":  # one call per node with parts > 1, depth-first
        assert len(calls) == sum(1 for p in Z[f"{key}/trace_parts"] if p > 1)


def test_partitioner_errors_wrapped_like_reference(Z):
    from paper_2510_12196_b200 import hierarchical_multisection
    g = graph(Z, "grid")
    t = Topo(Z["grid/hierarchy"])

    def boom(sub, parts, eps_local, seed):
        raise KeyError("user bug")

    with pytest.raises(RuntimeError, match=r"partitioner failed at hierarchy node \[\]") as ei:
        hierarchical_multisection(g, t, 0.03, partitioner=boom)
    assert isinstance(ei.value.__cause__, KeyError)

    def bad(sub, parts, eps_local, seed):
        return np.full(sub.n, parts, dtype=np.int64)  # out of range

    with pytest.raises(RuntimeError, match=r"invalid assignment at node \[\]"):
        hierarchical_multisection(g, t, 0.03, partitioner=bad)

    def short(sub, parts, eps_local, seed):
        return np.zeros(max(sub.n - 1, 0), dtype=np.int64)

    with pytest.raises(RuntimeError, match="invalid assignment"):
        hierarchical_multisection(g, t, 0.03, partitioner=short)
