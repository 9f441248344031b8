"""The reference's hand-built known-answer cases, run on the GPU through the C
ABI (paper_2510_12196_b200.device wraps include/gpuim.h).

Each test cites the reference test it ports; the expected values are the
reference test's own assertions.
"""
from __future__ import annotations

import logging

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

FLAT2 = ((2,), (1,))


@pytest.fixture(scope="module")
def D():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2510_12196_b200 import device
    return device


def edge_list(n, triples, vweights=None):
    """from_edge_list (graph.py:102-126)."""
    from paper_2510_12196_b200.generators import from_pairs
    if triples:
        u, v, w = (np.asarray(x, dtype=np.int64) for x in zip(*triples))
    else:
        u = v = w = np.empty(0, np.int64)
    return from_pairs(n, u, v, w, None if vweights is None else np.asarray(vweights, np.int64))


def ring(n):
    return edge_list(n, [(i, (i + 1) % n, 1) for i in range(n)])


def overload_instance(n_over=6, n_under=2):
    """test_refinement.py:243-250: path, first block overloaded."""
    n = n_over + n_under
    return edge_list(n, [(i, i + 1, 1) for i in range(n - 1)]), np.array([0] * n_over +
                                                                        [1] * n_under)


def random_graph(rng, n, p=0.35, wmax=9):
    """conftest.py:140-156 shape: spanning path + random edges, unit vertex
    weights."""
    edges = {}
    for v in range(1, n):
        edges[(int(rng.integers(0, v)), v)] = int(rng.integers(1, wmax + 1))
    for u in range(n):
        for v in range(u + 1, n):
            if (u, v) not in edges and rng.random() < p:
                edges[(u, v)] = int(rng.integers(1, wmax + 1))
    return edge_list(n, [(u, v, w) for (u, v), w in sorted(edges.items())])


def host(t):
    return t.cpu().numpy().astype(np.int64)


def bw_of(g, a, k):
    return np.bincount(a, weights=g.vertex_weights, minlength=k).astype(np.int64)


def test_lp_all_locked_moves_nothing(D):
    """test_refinement.py:123-130."""
    g = ring(8)
    dg = D.DeviceGraph.from_host(g)
    cand, dest, tm = D.lp_pass(dg, [0, 1] * 4, np.ones(8, bool), *FLAT2)
    assert not host(cand).any() and not host(tm).any()


def test_lp_single_positive_vertex_moves(D):
    """test_refinement.py:133-142."""
    g = edge_list(3, [(0, 1, 2)])
    dg = D.DeviceGraph.from_host(g)
    cand, dest, tm = D.lp_pass(dg, [0, 1, 0], np.array([False, True, False]), *FLAT2)
    cand, dest, tm = host(cand), host(dest), host(tm)
    assert tm[0] and dest[0] == 1
    assert not tm[2]
    assert (tm <= cand).all()


def test_lp_ord_keeps_the_earlier_of_a_swap_pair(D):
    """test_refinement.py:145-155: both middle vertices want to swap; only the
    lower id survives the second filter."""
    g = edge_list(4, [(0, 1, 1), (1, 2, 5), (2, 3, 1)])
    dg = D.DeviceGraph.from_host(g)
    cand, dest, tm = (host(x) for x in D.lp_pass(dg, [0, 0, 1, 1], np.zeros(4, bool), *FLAT2))
    assert cand[1] and cand[2]
    assert dest[1] == 1 and dest[2] == 0
    assert tm[1] and not tm[2]


def test_lp_jet_filter_admits_small_losses_only(D):
    """test_refinement.py:158-178: gain -1 passes the jet filter
    (floor(0.25*9) = 2), -2 does not; nonneg rejects any loss."""
    locked = np.array([False, True, True])

    def run(other, jet):
        g = edge_list(3, [(0, 1, 9), (0, 2, other)])
        dg = D.DeviceGraph.from_host(g)
        return [host(x) for x in D.lp_pass(dg, [0, 0, 1], locked, *FLAT2, jet=jet, jet_c=0.25)]

    cand, _, tm = run(8, True)
    assert cand[0] and not tm[0]
    cand, _, _ = run(7, True)
    assert not cand[0]
    cand, _, _ = run(8, False)
    assert not cand[0]


def test_weak_rebalance_moves_exactly_the_excess(D):
    """test_refinement.py:252-262."""
    g, a = overload_instance(6, 2)
    dg = D.DeviceGraph.from_host(g)
    bw = bw_of(g, a, 2)
    cand, dest, tm, inc = D.rebalance(dg, a, bw, *FLAT2, False, 5.0 * 0.995, 5.0, 2, 0, 0)
    assert int(host(tm).sum()) == 1
    assert not inc
    at = torch.from_numpy(a.astype(np.int32)).cuda()
    bwt = torch.from_numpy(bw).cuda()
    D.apply_moves(dg, at, bwt, tm, dest, *FLAT2)
    assert list(host(bwt)) == [5, 3]


def test_weak_rebalance_noop_when_balanced(D):
    """test_refinement.py:265-270."""
    g, a = overload_instance(4, 4)
    dg = D.DeviceGraph.from_host(g)
    cand, dest, tm, inc = D.rebalance(dg, a, bw_of(g, a, 2), *FLAT2, False, 4.0, 4.12, 2, 0, 0)
    assert not host(cand).any() and not host(tm).any()


def test_weak_rebalance_falls_back_to_hashed_block(D):
    """test_refinement.py:273-285: the only eligible block is not adjacent."""
    g = edge_list(5, [(0, 1, 1), (1, 2, 1), (0, 2, 1)])
    a = np.array([0, 0, 0, 1, 1])
    dg = D.DeviceGraph.from_host(g)
    cand, dest, tm, inc = D.rebalance(dg, a, bw_of(g, a, 2), *FLAT2, False, 2.9, 2.5, 2, 5, 0)
    tm, dest = host(tm).astype(bool), host(dest)
    assert tm.any()
    assert (dest[tm] == 1).all()
    assert not inc


def test_weak_rebalance_flags_incomplete_when_no_block_fits(D):
    """test_refinement.py:288-294."""
    g, a = overload_instance(6, 2)
    dg = D.DeviceGraph.from_host(g)
    cand, dest, tm, inc = D.rebalance(dg, a, bw_of(g, a, 2), *FLAT2, False, 1.0, 5.0, 2, 0, 0)
    assert inc
    assert not host(tm).any()


def test_strong_rebalance_restores_balance_in_one_pass(D):
    """test_refinement.py:296-305: the target absorbs all its room (3 moves)."""
    g, a = overload_instance(6, 2)
    dg = D.DeviceGraph.from_host(g)
    bw = bw_of(g, a, 2)
    cand, dest, tm, inc = D.rebalance(dg, a, bw, *FLAT2, True, 5.0 * 0.995, 5.0, 2, 0, 0)
    assert int(host(tm).sum()) == 3
    at = torch.from_numpy(a.astype(np.int32)).cuda()
    bwt = torch.from_numpy(bw).cuda()
    D.apply_moves(dg, at, bwt, tm, dest, *FLAT2)
    assert host(bwt).max() <= 5.0


def test_strong_rebalance_targets_never_overshoot(D):
    """test_refinement.py:315-333."""
    rng = np.random.default_rng(2)
    topo = ((4,), (1,))
    checked = 0
    for _ in range(20):
        g = random_graph(rng, 20)
        a = rng.integers(0, 4, size=20)
        l_max = 1.03 * g.total_weight / 4
        before = bw_of(g, a, 4)
        if before.max() <= l_max:
            continue
        dg = D.DeviceGraph.from_host(g)
        cand, dest, tm, inc = D.rebalance(dg, a, before, *topo, True, l_max * 0.995, l_max, 2,
                                          0, 0)
        at = torch.from_numpy(a.astype(np.int32)).cuda()
        bwt = torch.from_numpy(before.copy()).cuda()
        D.apply_moves(dg, at, bwt, tm, dest, *topo)
        after = host(bwt)
        for b in range(4):
            if before[b] <= l_max:
                assert after[b] <= l_max
        checked += 1
    assert checked > 0


def _refine(D, g, a, topo, l_max, seed=0):
    dg = D.DeviceGraph.from_host(g)
    k = int(np.prod(topo[0]))
    at = torch.from_numpy(np.asarray(a, np.int32)).cuda()
    bwt = torch.from_numpy(bw_of(g, np.asarray(a), k)).cuda()
    D.refine(dg, *topo, at, bwt, i_max=12, i_w_max=2, sigma_fraction=0.005, seed=seed,
             l_max=l_max)
    return host(at), host(bwt)


def test_refine_keeps_locally_optimal_input(D):
    """test_refinement.py:339-345: the 4-cycle split stays at J = 4."""
    from oracle import promap_np as O
    g = edge_list(4, [(0, 1, 1), (1, 2, 1), (2, 3, 1), (0, 3, 1)])
    a, _ = _refine(D, g, [0, 0, 1, 1], FLAT2, 2.06)
    assert O.total_cost(g, O.OTopology(*FLAT2), a) == 4


def test_refine_rebalances_path_split(D):
    """test_refinement.py:348-353."""
    g, a0 = overload_instance(6, 2)
    a, bw = _refine(D, g, a0, FLAT2, 4.12)
    assert bw.max() <= 4.12
    assert np.array_equal(bw, bw_of(g, a, 2))


def test_refine_unsatisfiable_balance_terminates_least_loaded(D):
    """test_refinement.py:369-377: the heavy vertex pins the bound."""
    g = edge_list(3, [(0, 1, 1), (1, 2, 1)], vweights=[10, 1, 1])
    a, bw = _refine(D, g, [0, 0, 0], FLAT2, 6.18)
    assert 10 <= bw.max() <= 12
    assert bw.max() > 6.18


def test_refine_monotone_on_ring_from_random_balanced_starts(D):
    """test_refinement.py:356-366 (balanced starts drawn by the oracle)."""
    from oracle import promap_np as O
    g = ring(16)
    topo = ((4,), (1,))
    l_max = 1.03 * 16 / 4
    rng = np.random.default_rng(0)
    for seed in range(20):
        a0 = np.repeat(np.arange(4), 4)[rng.permutation(16)]
        j_in = O.total_cost(g, O.OTopology(*topo), a0)
        a, bw = _refine(D, g, a0, topo, l_max, seed)
        assert bw.max() <= l_max
        assert O.total_cost(g, O.OTopology(*topo), a) <= j_in


def test_integrated_map_warns_when_balance_unreachable(D, caplog):
    """test_pipelines.py:218-224: an imbalanced result is returned with a
    warning on logger promap.pipelines."""
    from paper_2510_12196_b200 import integrated_map

    class T:
        hierarchy, distances = FLAT2
    g = edge_list(3, [(0, 1, 1), (1, 2, 1)], vweights=[10, 1, 1])
    with caplog.at_level(logging.WARNING, logger="promap.pipelines"):
        m = integrated_map(g, T(), 0.03, seed=0)
    assert "imbalanced" in caplog.text
    assert m.max_block_weight() >= 10


def test_integrated_map_empty_graph_rejected(D):
    """test_pipelines.py:227-229."""
    from paper_2510_12196_b200 import integrated_map

    class T:
        hierarchy, distances = FLAT2
    with pytest.raises(ValueError):
        integrated_map(edge_list(0, []), T(), 0.03)
