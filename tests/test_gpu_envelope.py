"""The reference's interface beyond integral distances and short hierarchies,
pinned to the reference's own outputs (tests/golden/scale_envelope.npz,
scripts/make_golden_scale.py `envelope`):

* non-integral distances (topology.py:56-58, mapping.py:76-91 float path):
  dyadic distances (1.5:10.25:100, 0.5:2.25:7.125, 1:10.5:100) run as exact
  scaled integers, so the mapping, the float J and the LP proposals equal the
  reference's; non-dyadic ones (0.7:3.3, 1.1:9.9:101.3) run on distances
  rounded to 2^-s and are held to tolerance parity (balanced, J within 10 %
  of the reference's, float J of a fixed mapping within 1e-12);
* hierarchies of 9-11 levels (topology.py:25-40 has no cap);
* vertex / edge weights whose totals exceed 2^31 (graph.py:21-24 int64).
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import load_npz

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def D():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2510_12196_b200 import device
    return device


@pytest.fixture(scope="module")
def Z():
    return load_npz("scale_envelope")


class Topo:
    def __init__(self, h, d):
        self.hierarchy = tuple(int(x) for x in h)
        self.distances = tuple(d)


def case(Z, i):
    from paper_2510_12196_b200.generators import HostGraph
    g = HostGraph(Z[f"{i}/offsets"], Z[f"{i}/targets"], Z[f"{i}/weights"], Z[f"{i}/vweights"])
    d = [float(x) for x in Z[f"{i}/distances"]]
    if bool(Z[f"{i}/integral"]):
        d = [int(x) for x in d]
    elif str(Z[f"{i}/kind"]) == "float_d" and d == [1.0, 10.5, 100.0]:
        d = [1, 10.5, 100]  # as the generator wrote it (mixed int / float)
    return g, Topo(Z[f"{i}/hierarchy"], d)


def indices(Z, kind):
    return [i for i in range(int(Z["count"])) if str(Z[f"{i}/kind"]) == kind]


def test_float_distance_scale(D):
    assert D.topology_scale((2, 2, 2), (1.5, 10.25, 100.0)) == (2, True)
    assert D.topology_scale((2, 3, 2), (0.5, 2.25, 7.125)) == (3, True)
    assert D.topology_scale((4, 8, 6), (1, 10, 100)) == (0, True)
    s, exact = D.topology_scale((4, 4), (0.7, 3.3))
    assert not exact and s >= 20


@pytest.mark.parametrize("kind", ["float_d", "float_d_units"])
def test_float_distances_integrated_map(D, Z, kind):
    from paper_2510_12196_b200 import integrated_map
    for i in indices(Z, kind):
        g, t = case(Z, i)
        _, exact = D.topology_scale(t.hierarchy, t.distances)
        st: dict = {}
        m = integrated_map(g, t, float(Z[f"{i}/eps"]), int(Z[f"{i}/seed"]),
                           coarsest_factor=int(Z[f"{i}/coarsest_factor"]), stats=st)
        ref = Z[f"{i}/assignment"]
        j_ref = float(Z[f"{i}/j"])
        assert isinstance(st["J"], float)
        k = int(np.prod(t.hierarchy))
        l_max = 1.03 * g.total_weight / k
        ref_max = int(np.bincount(ref, weights=g.vertex_weights, minlength=k).max())
        # balanced wherever the reference is; never worse where it is not
        assert m.max_block_weight() <= max(l_max, ref_max), (i, m.max_block_weight(), ref_max)
        if exact:
            assert np.array_equal(m.assignment, ref), f"case {i}"
            assert st["J"] == j_ref
        else:
            assert st["J"] <= 1.10 * j_ref, (i, st["J"], j_ref)
            if np.array_equal(m.assignment, ref):
                assert st["J"] == pytest.approx(j_ref, rel=1e-12)


def test_float_distances_units(D, Z):
    """total_cost (float J) and label_propagation_pass of a fixed random
    mapping, both filter modes (the locked masks replay the generator's rng)."""
    rng = np.random.default_rng(7)
    for i in indices(Z, "float_d_units"):
        g, t = case(Z, i)
        k = int(np.prod(t.hierarchy))
        a = rng.integers(0, k, size=g.n)
        assert np.array_equal(a, Z[f"{i}/unit_assignment"])
        dg = D.DeviceGraph.from_host(g)
        j = D.total_cost(dg, a, t.hierarchy, t.distances)
        assert isinstance(j, float)
        assert j == pytest.approx(float(Z[f"{i}/unit_j"]), rel=1e-12)
        _, exact = D.topology_scale(t.hierarchy, t.distances)
        for mode in ("nonneg", "jet"):
            locked = rng.random(g.n) < 0.2
            cand, dest, tm = D.lp_pass(dg, a, locked, t.hierarchy, t.distances,
                                       jet=mode == "jet")
            got = (cand.cpu().numpy().astype(bool), dest.cpu().numpy(),
                   tm.cpu().numpy().astype(bool))
            want = (Z[f"lp{i}_{mode}/cand"], Z[f"lp{i}_{mode}/dest"], Z[f"lp{i}_{mode}/to_move"])
            if exact:
                assert np.array_equal(got[0], want[0]), (i, mode)
                assert np.array_equal(got[1][want[0]], want[1][want[0]]), (i, mode)
                assert np.array_equal(got[2], want[2]), (i, mode)
            else:  # rounded distances: near-ties may flip, the bulk must agree
                assert (got[0] != want[0]).mean() < 0.02, (i, mode)


def test_deep_hierarchies(D, Z):
    from paper_2510_12196_b200 import integrated_map
    for i in indices(Z, "deep"):
        g, t = case(Z, i)
        assert len(t.hierarchy) >= 9
        st: dict = {}
        m = integrated_map(g, t, float(Z[f"{i}/eps"]), int(Z[f"{i}/seed"]),
                           coarsest_factor=int(Z[f"{i}/coarsest_factor"]), stats=st)
        assert np.array_equal(m.assignment, Z[f"{i}/assignment"]), f"case {i}"
        assert st["J"] == int(Z[f"{i}/j"])


@pytest.mark.xfail(reason="int64 device weights not built yet (GIM_E_OVERFLOW)", strict=False)
def test_int64_weights(D, Z):
    from paper_2510_12196_b200 import integrated_map
    for i in indices(Z, "int64_w"):
        g, t = case(Z, i)
        assert g.total_weight >= 2**31
        st: dict = {}
        m = integrated_map(g, t, float(Z[f"{i}/eps"]), int(Z[f"{i}/seed"]),
                           coarsest_factor=int(Z[f"{i}/coarsest_factor"]), stats=st)
        assert np.array_equal(m.assignment, Z[f"{i}/assignment"]), f"case {i}"
        assert st["J"] == int(Z[f"{i}/j"])
