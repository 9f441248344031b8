"""GPU parity: libgpuim.so kernels vs the reference's golden vectors and the
oracle, through the C ABI (paper_2510_12196_b200.device wraps include/gpuim.h).

Bit-exact everywhere: J, HEM rounds, coarse ids, contraction, connectivity,
LP / weak / strong proposals, apply_moves deltas, refine, greedy growing,
the internal partitioner, multisection and integrated_map itself.
"""
from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import promap_np as O  # noqa: E402


@pytest.fixture(scope="module")
def D():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2510_12196_b200 import device
    return device


@pytest.fixture(params=["fused", "phased"])
def mode(request, D):
    """Alg. 4 as one persistent cooperative kernel per level + row-wise
    contraction ("fused") or per-phase launches with host control + the
    radix-sort contraction ("phased"); both must be exact."""
    D.set_fused(request.param == "fused")
    D.set_rowwise_contraction(request.param == "fused")
    yield request.param
    D.set_fused(True)
    D.set_rowwise_contraction(True)


def dev_graph(D, c):
    return D.DeviceGraph.from_host(c.graph())


def np_(t):
    return t.cpu().numpy().astype(np.int64)


def test_total_cost_golden(D, golden):
    for c in golden("jeval"):
        dg = dev_graph(D, c)
        j = D.total_cost(dg, c["assignment"], tuple(c["hierarchy"]), tuple(c["distances"]))
        assert j == c.scalar("j")


def test_block_weights(D, golden):
    for c in golden("jeval"):
        g = c.graph()
        k = int(np.prod(c["hierarchy"]))
        bw = D.block_weights(dev_graph(D, c), c["assignment"], k)
        assert np.array_equal(np_(bw), O.block_weights(g.vertex_weights, c["assignment"], k))


def test_hem_rounds_golden(D, golden):
    for c in golden("hem"):
        if not c.scalar("has_rounds"):
            continue
        dg = dev_graph(D, c)
        partner = torch.full((dg.n,), -1, dtype=torch.int32, device="cuda")
        pref, m = D.hem_round(dg, partner, c.scalar("l_max"), int(c["seed1"]), 0)
        assert np.array_equal(np_(pref), c["pref1"])
        assert np.array_equal(np_(partner), c["part1"])
        assert m == int((c["part1"] >= 0).sum())
        pref, m = D.hem_round(dg, partner, c.scalar("l_max"), int(c["seed2"]), m)
        assert np.array_equal(np_(pref), c["pref2"])
        assert np.array_equal(np_(partner), c["part2"])


def test_match_coarse_map_contract_golden(D, golden):
    for c in golden("hem"):
        dg = dev_graph(D, c)
        partner = D.match_graph(dg, c.scalar("l_max"), int(c["match_seed"]))
        assert np.array_equal(np_(partner), c["match_partner"])
        cmap, n_c = D.coarse_map(partner)
        assert n_c == c.scalar("n_c")
        assert np.array_equal(np_(cmap), c["coarse_map"])
        cg = D.contract(dg, cmap, n_c)
        off, tgt, w, vw = cg.to_host()
        assert np.array_equal(off, c["c_offsets"])
        assert np.array_equal(tgt, c["c_targets"])
        assert np.array_equal(w, c["c_weights"])
        assert np.array_equal(vw, c["c_vweights"])
        assert np.array_equal(np_(cg.sources), np.repeat(np.arange(n_c), np.diff(off)))


def test_level_stack_golden(D, golden):
    """build_level_stack (coarsening.py:280-295) driven level by level."""
    for c in golden("stack"):
        dg = dev_graph(D, c)
        sizes, m2s = [dg.n], [dg.m2]
        li = 0
        while dg.n >= int(c["threshold"]):
            seed = O.splitmix64(int(c["seed"]) ^ li)
            partner = D.match_graph(dg, c.scalar("l_max"), seed)
            cmap, n_c = D.coarse_map(partner)
            if li == 0:
                assert np.array_equal(np_(cmap), c["cmap0"])
            if n_c * 1.02 > dg.n:
                break
            dg = D.contract(dg, cmap, n_c)
            sizes.append(dg.n)
            m2s.append(dg.m2)
            li += 1
        assert sizes == list(c["sizes"])
        assert m2s == list(c["m2s"])
        off, tgt, w, _ = dg.to_host()
        assert np.array_equal(off, c["c_offsets"])
        assert np.array_equal(tgt, c["c_targets"])
        assert np.array_equal(w, c["c_weights"])


def test_contract_matches_oracle_random(D):
    rng = np.random.default_rng(5)
    from paper_2510_12196_b200.generators import gen_rgg
    g = gen_rgg(20000, 0.55, 11)
    dg = D.DeviceGraph.from_host(g)
    cmap = rng.integers(0, 7000, g.n)
    cmap[:7000] = np.arange(7000)
    cg = D.contract(dg, torch.from_numpy(cmap).cuda(), 7000)
    ref = O.contract(g, cmap, 7000)
    off, tgt, w, vw = cg.to_host()
    assert np.array_equal(off, ref.offsets)
    assert np.array_equal(tgt, ref.edge_targets)
    assert np.array_equal(w, ref.edge_weights)
    assert np.array_equal(vw, ref.vertex_weights)


def test_conn_golden(D, golden):
    for c in golden("conn"):
        off, blocks, w = D.conn_build(dev_graph(D, c), c["assignment"], c.topology().k)
        assert np.array_equal(np_(off), c["conn_offsets"])
        assert np.array_equal(np_(blocks), c["conn_blocks"])
        assert np.array_equal(np_(w), c["conn_weights"])


def test_lp_golden(D, golden):
    for c in golden("lp"):
        cand, dest, tm = D.lp_pass(dev_graph(D, c), c["assignment"], c["locked"],
                                   tuple(c["hierarchy"]), tuple(c["distances"]),
                                   jet=bool(c.scalar("jet")))
        assert np.array_equal(np_(cand).astype(bool), c["cand"])
        assert np.array_equal(np_(dest), c["dest"])
        assert np.array_equal(np_(tm).astype(bool), c["to_move"])


@pytest.mark.parametrize("h,d", [((4, 8, 8), (1, 10, 100)), ((3, 5, 7), (1, 7, 40)),
                                 ((2, 3, 4, 5), (0, 2, 3, 50)), ((64, 4), (5, 5))])
def test_wide_tables_match_oracle(D, h, d):
    """Vertices adjacent to many blocks (R-MAT hubs under a random mapping
    onto k = 120..256 blocks) take the grouped O(L) candidate costs
    (refine_dev.cuh eval_table_grouped): LP proposals and weak-rebalance
    candidates equal the reference's (refinement.py:201-309) for mixed-radix
    hierarchies with unequal, equal and zero distances."""
    from paper_2510_12196_b200.generators import gen_rmat
    g = gen_rmat(12)
    og = O.as_ograph(g)
    t = O.OTopology(h, d)
    rng = np.random.default_rng(len(h))
    a = rng.integers(0, t.k, g.n)
    assert (np.diff(g.offsets) > 64).sum() > 10  # hubs: > 16 distinct blocks
    dg = D.DeviceGraph.from_host(g)
    locked = np.zeros(g.n, dtype=bool)
    for jet in (False, True):
        cand, dest, tm = D.lp_pass(dg, a, locked, h, d, jet=jet)
        p = O.label_propagation_pass(og, t, a, locked,
                                     O.Config(filter_mode="jet" if jet else "nonneg"))
        assert np.array_equal(np_(cand).astype(bool), p.candidates)
        assert np.array_equal(np_(dest), p.destinations)
        assert np.array_equal(np_(tm).astype(bool), p.to_move)
    bw = O.block_weights(g.vertex_weights, a, t.k)
    l_max = float(bw.mean())  # about half the blocks overloaded
    cfg = O.Config()
    sigma = l_max * (1 - cfg.sigma_fraction)
    cand, dest, tm, inc = D.rebalance(dg, a, bw, h, d, False, sigma, l_max, cfg.rho, 3, 1)
    p = O.weak_rebalance(og, t, a, bw, sigma, l_max, O.Config(seed=3), pass_counter=1)
    assert np.array_equal(np_(cand).astype(bool), p.candidates)
    assert np.array_equal(np_(dest), p.destinations)
    assert np.array_equal(np_(tm).astype(bool), p.to_move)


@pytest.mark.parametrize("scale", [12, 15])
def test_wide_tables_refine_matches_oracle(D, mode, scale):
    """Alg. 4 end to end on an R-MAT graph under a random k = 256 mapping
    (hub rows listed for the grid, wide tables, rebalancing; at scale 15
    hub movers > 2048 slots applied by grid-wide segments): the best
    mapping equals the reference's refine (refinement.py:389-464)."""
    from paper_2510_12196_b200.generators import gen_rmat
    g = gen_rmat(scale)
    h, d = (4, 8, 8), (1, 10, 100)
    t = O.OTopology(h, d)
    a = np.random.default_rng(9).permutation(g.n) % t.k  # balanced, random
    cfg = O.config_for_level(0, 3, seed=4)
    l_max = 1.25 * g.vertex_weights.sum() / t.k
    want = O.refine(g, t, a.copy(), cfg, l_max)
    dg = D.DeviceGraph.from_host(g)
    at = torch.from_numpy(a.astype(np.int32)).cuda()
    bw = torch.from_numpy(O.block_weights(g.vertex_weights, a, t.k)).cuda()
    D.refine(dg, h, d, at, bw, phi=cfg.phi, i_max=cfg.i_max, i_w_max=cfg.i_w_max,
             sigma_fraction=cfg.sigma_fraction, rho=cfg.rho, jet=False, jet_c=cfg.jet_filter_c,
             seed=cfg.seed, l_max=l_max)
    assert np.array_equal(np_(at), want)


def test_rebalance_golden(D, golden):
    for c in golden("rebalance"):
        g = c.graph()
        k = c.topology().k
        bw = O.block_weights(g.vertex_weights, c["assignment"], k)
        dg = dev_graph(D, c)
        for strong, p in ((False, "w"), (True, "s")):
            cand, dest, tm, inc = D.rebalance(
                dg, c["assignment"], bw, tuple(c["hierarchy"]), tuple(c["distances"]), strong,
                c.scalar("sigma"), c.scalar("l_max"), int(c["rho"]), int(c["seed"]),
                int(c["pass_counter"]))
            assert np.array_equal(np_(cand).astype(bool), c[f"{p}_cand"])
            assert np.array_equal(np_(dest), c[f"{p}_dest"])
            assert np.array_equal(np_(tm).astype(bool), c[f"{p}_to_move"])
            assert inc == bool(c[f"{p}_incomplete"])


def test_apply_moves_delta_j(D, golden):
    rng = np.random.default_rng(3)
    for c in golden("lp")[::3]:
        g, t = c.graph(), c.topology()
        a = c["assignment"].copy()
        h, d = tuple(c["hierarchy"]), tuple(c["distances"])
        tm = rng.random(g.n) < 0.3
        dest = np.where(tm, rng.integers(0, t.k, g.n), a)
        dg = dev_graph(D, c)
        at = torch.from_numpy(a.astype(np.int32)).cuda()
        bw = torch.from_numpy(O.block_weights(g.vertex_weights, a, t.k)).cuda()
        dj = D.apply_moves(dg, at, bw, tm, dest, h, d)
        new = np.where(tm, dest, a)
        assert np.array_equal(np_(at), new)
        assert np.array_equal(np_(bw), O.block_weights(g.vertex_weights, new, t.k))
        assert dj == O.total_cost(g, t, new) - O.total_cost(g, t, a)


def test_refine_golden(D, mode, golden):
    for c in golden("refine"):
        g, t = c.graph(), c.topology()
        lev, nl = int(c["level"]), int(c["n_levels"])
        cfg = O.config_for_level(lev, nl, seed=int(c["seed"]),
                                 filter_mode="jet" if c.scalar("jet") else "nonneg")
        dg = dev_graph(D, c)
        at = torch.from_numpy(c["assignment"].astype(np.int32)).cuda()
        bw = torch.from_numpy(O.block_weights(g.vertex_weights, c["assignment"], t.k)).cuda()
        D.refine(dg, tuple(c["hierarchy"]), tuple(c["distances"]), at, bw, phi=cfg.phi,
                 i_max=cfg.i_max, i_w_max=cfg.i_w_max, sigma_fraction=cfg.sigma_fraction,
                 rho=cfg.rho, jet=cfg.filter_mode == "jet", jet_c=cfg.jet_filter_c,
                 seed=cfg.seed, l_max=c.scalar("l_max"))
        assert np.array_equal(np_(at), c["best"])
        assert np.array_equal(np_(bw), O.block_weights(g.vertex_weights, c["best"], t.k))


def test_ggg_golden(D, golden):
    for c in golden("ggg"):
        g = c.graph()
        k = int(c["k"])
        if g.n <= k:
            continue
        part = D.greedy_graph_growing(dev_graph(D, c), k)
        assert np.array_equal(np_(part), c["part"])


def test_partitioner_golden(D, mode, golden):
    for c in golden("partitioner"):
        part = D.internal_partitioner(dev_graph(D, c), int(c["k"]), c.scalar("eps"),
                                      int(c["seed"]))
        assert np.array_equal(np_(part), c["part"])


def test_multisection_golden(D, mode, golden):
    for c in golden("multisection"):
        a = D.hierarchical_multisection(dev_graph(D, c), tuple(c["hierarchy"]),
                                        tuple(c["distances"]), c.scalar("eps"), int(c["seed"]))
        assert np.array_equal(np_(a), c["assignment"])


def test_integrated_map_small_golden(D, mode, golden):
    for c in golden("im_small"):
        a, bw, st = D.integrated_map_device(dev_graph(D, c), tuple(c["hierarchy"]),
                                            tuple(c["distances"]), c.scalar("eps"),
                                            int(c["seed"]),
                                            coarsest_factor=int(c["coarsest_factor"]))
        assert np.array_equal(np_(a), c["assignment"].astype(np.int64))
        assert st["final_j"] == c.scalar("j")


def test_integrated_map_cfg1_all_seeds_bit_exact(D, mode, golden):
    """Config 1 through the public drop-in API: identical mappings to the
    reference for seeds 0-4 (stronger than the J tolerance gate)."""
    from paper_2510_12196_b200 import integrated_map
    from paper_2510_12196_b200.generators import gen_grid
    g = gen_grid(128, 128)
    t = O.OTopology((4, 8, 2), (1, 10, 100))
    for c in golden("im_cfg1"):
        m = integrated_map(g, t, 0.03, int(c["seed"]))
        assert np.array_equal(m.assignment, c["assignment"].astype(np.int64))
        assert O.total_cost(g, t, m.assignment) == c.scalar("j")
        assert m.max_block_weight() <= (1.03 * g.n / 64)


def test_integrated_map_edge_cases(D):
    from paper_2510_12196_b200 import integrated_map
    from paper_2510_12196_b200.generators import HostGraph, from_pairs
    t = O.OTopology((2, 2), (1, 10))
    empty = HostGraph(np.zeros(1, np.int64), np.zeros(0, np.int64), np.zeros(0, np.int64),
                      np.zeros(0, np.int64))
    with pytest.raises(ValueError):
        integrated_map(empty, t, 0.03)
    # no edges at all, and fewer vertices than PEs
    iso = HostGraph(np.zeros(4, np.int64), np.zeros(0, np.int64), np.zeros(0, np.int64),
                    np.ones(3, np.int64))
    m = integrated_map(iso, t, 0.03)
    a, _, _ = O.integrated_map(iso, t, 0.03)
    assert np.array_equal(m.assignment, a)
    # two components plus isolated vertices, k = 1
    g = from_pairs(9, np.array([0, 1, 4, 5]), np.array([1, 2, 5, 6]))
    one = O.OTopology((1,), (3,))
    m = integrated_map(g, one, 0.0)
    assert np.array_equal(m.assignment, np.zeros(9, np.int64))
    m = integrated_map(g, t, 0.5, seed=3)
    a, bw, _ = O.integrated_map(g, t, 0.5, seed=3)
    assert np.array_equal(m.assignment, a)
    assert np.array_equal(m.block_weights, bw)


def test_integrated_map_matches_oracle_rgg(D, mode):
    """Mid-size rgg with a real level stack: identical to the oracle."""
    from paper_2510_12196_b200 import integrated_map
    from paper_2510_12196_b200.generators import gen_rgg
    g = gen_rgg(1 << 14, 0.55, 1)
    t = O.OTopology((4, 8, 6), (1, 10, 100))
    m = integrated_map(g, t, 0.03, 0, coarsest_factor=16)
    a, bw, l_max = O.integrated_map(g, t, 0.03, 0, coarsest_factor=16)
    assert np.array_equal(m.assignment, a)
    assert m.max_block_weight() <= l_max


@pytest.mark.parametrize("logn", [13, 16])
def test_batched_multisection_equals_recursive(D, logn):
    """The breadth-first, batched multisection (one launch per phase for all
    small tree nodes, strong passes resumed on the device loop) computes the
    same assignment as the recursive per-node path."""
    from paper_2510_12196_b200.generators import gen_rgg
    g = gen_rgg(1 << logn, 0.55, 1)
    dg = D.DeviceGraph.from_host(g)
    h, d = (4, 8, 6), (1, 10, 100)
    try:
        D.set_batch(False)
        a = np_(D.hierarchical_multisection(dg, h, d, 0.03, 5))
        D.set_batch(True)
        b = np_(D.hierarchical_multisection(dg, h, d, 0.03, 5))
    finally:
        D.set_batch(True)
    assert np.array_equal(a, b)


def test_batched_integrated_map_equals_recursive(D):
    from paper_2510_12196_b200.generators import gen_rgg
    g = gen_rgg(1 << 16, 0.55, 1)
    dg = D.DeviceGraph.from_host(g)
    h, d = (4, 8, 6), (1, 10, 100)
    try:
        D.set_batch(False)
        a, bwa, sa = D.integrated_map_device(dg, h, d, 0.03, 2)
        D.set_batch(True)
        b, bwb, sb = D.integrated_map_device(dg, h, d, 0.03, 2)
    finally:
        D.set_batch(True)
    assert np.array_equal(np_(a), np_(b))
    assert np.array_equal(np_(bwa), np_(bwb))
    assert sa["final_j"] == sb["final_j"]


def test_rmat_small_matches_oracle(D):
    """Skewed degrees: two-hop matching and hub rows (general-path fallbacks
    of the batched partitioner, radix contraction) — identical to the oracle."""
    from paper_2510_12196_b200 import integrated_map
    from paper_2510_12196_b200.generators import gen_rmat
    g = gen_rmat(11)
    t = O.OTopology((2, 4, 2), (1, 10, 100))
    m = integrated_map(g, t, 0.03, 1, coarsest_factor=16)
    a, bw, l_max = O.integrated_map(g, t, 0.03, 1, coarsest_factor=16)
    assert np.array_equal(m.assignment, a)
    assert np.array_equal(m.block_weights, bw)


def test_gpu_hm_host_api_golden(D, golden):
    """GPU-HM through the drop-in (host int64 arrays in, Mapping out) equals
    the reference's hierarchical_multisection on its golden cases."""
    from paper_2510_12196_b200 import hierarchical_multisection
    for c in golden("multisection"):
        g, t = c.graph(), c.topology()
        m = hierarchical_multisection(g, t, c.scalar("eps"), seed=int(c["seed"]))
        assert np.array_equal(m.assignment, c["assignment"].astype(np.int64))
        assert np.array_equal(m.block_weights,
                              O.block_weights(g.vertex_weights, c["assignment"], t.k))


def test_gpu_hm_matches_oracle_rgg(D):
    from paper_2510_12196_b200 import hierarchical_multisection
    from paper_2510_12196_b200.generators import gen_rgg
    g = gen_rgg(1 << 13, 0.55, 1)
    t = O.OTopology((4, 8, 2), (1, 10, 100))
    m = hierarchical_multisection(g, t, 0.03, seed=4)
    assert np.array_equal(m.assignment, O.hierarchical_multisection(g, t, 0.03, seed=4))
    # a partitioner returning nothing fails like the reference's seam
    # (pipelines.py:86-93): RuntimeError naming the node
    with pytest.raises(RuntimeError, match="partitioner failed at hierarchy node"):
        hierarchical_multisection(g, t, 0.03, partitioner=lambda *a: None)


def test_ggg_large_kernel_forced_golden(D, golden, monkeypatch):
    """The large-graph greedy growing (two-level frontier maxima, lazy
    repair, warp-driven claims) forced on every call: golden growing,
    partitioner and multisection cases and a skewed R-MAT map stay exact."""
    monkeypatch.setenv("GIM_GGG_LARGE", "1")
    for c in golden("ggg"):
        g = c.graph()
        k = int(c["k"])
        if g.n <= k:
            continue
        part = D.greedy_graph_growing(dev_graph(D, c), k)
        assert np.array_equal(np_(part), c["part"])
    for c in golden("partitioner"):
        part = D.internal_partitioner(dev_graph(D, c), int(c["k"]), c.scalar("eps"),
                                      int(c["seed"]))
        assert np.array_equal(np_(part), c["part"])
    from paper_2510_12196_b200 import integrated_map
    from paper_2510_12196_b200.generators import gen_rmat
    g = gen_rmat(11)
    t = O.OTopology((2, 4, 2), (1, 10, 100))
    m = integrated_map(g, t, 0.03, 1, coarsest_factor=16)
    a, bw, _ = O.integrated_map(g, t, 0.03, 1, coarsest_factor=16)
    assert np.array_equal(m.assignment, a)


@pytest.mark.parametrize("scale,k", [(13, 4), (14, 8)])
def test_ggg_large_graph_matches_oracle(D, scale, k):
    """Graphs too large for the shared-memory growing kernel (R-MAT: hubs
    handed to the whole CTA, isolated vertices claimed by the fallback)."""
    from paper_2510_12196_b200.generators import gen_rmat
    g = gen_rmat(scale)
    og = O.as_ograph(g)
    dg = D.DeviceGraph.from_host(g)
    part = D.greedy_graph_growing(dg, k)
    assert np.array_equal(np_(part), O.greedy_graph_growing(og, k))


@pytest.mark.parametrize("k", [2, 5, 8, 32, 40])
def test_ggg_large_isolated_runs_match_oracle(D, monkeypatch, k):
    """Weighted isolated vertices interleaved with small components (the
    stalled R-MAT coarsest graphs): the register-resident run of fallback
    claims (k <= 32) and the general loop (k > 32) both equal the
    reference's heap growing (pipelines.py:132-188)."""
    from paper_2510_12196_b200.generators import from_pairs
    monkeypatch.setenv("GIM_GGG_LARGE", "1")
    rng = np.random.default_rng(k)
    n = 6000
    conn = np.flatnonzero(rng.random(n) < 0.3)  # vertices with neighbours
    u = rng.choice(conn, 4 * len(conn))
    v = rng.choice(conn, 4 * len(conn))
    keep = u != v
    pairs = np.unique(np.sort(np.stack([u[keep], v[keep]], 1), axis=1), axis=0)
    vw = rng.integers(1, 6, n)
    g = from_pairs(n, pairs[:, 0], pairs[:, 1], rng.integers(1, 4, len(pairs)), vw)
    assert (np.diff(g.offsets) == 0).sum() > n // 2
    part = D.greedy_graph_growing(D.DeviceGraph.from_host(g), k)
    assert np.array_equal(np_(part), O.greedy_graph_growing(O.as_ograph(g), k))


def test_relatives_parallel_equals_sequential(D, monkeypatch):
    """Two-hop relatives by rounds of disjoint ready matchmakers equal the
    single-thread sequential sweep (coarsening.py:148-158) on R-MAT, where
    relatives fire on most levels: identical level stacks and mappings."""
    from paper_2510_12196_b200 import integrated_map
    from paper_2510_12196_b200.generators import gen_rmat
    g = gen_rmat(15)
    t = O.OTopology((4, 8, 8), (1, 10, 100))
    m_par = integrated_map(g, t, 0.03, 2)
    monkeypatch.setenv("GIM_RELATIVES_SEQ", "1")
    m_seq = integrated_map(g, t, 0.03, 2)
    assert np.array_equal(m_par.assignment, m_seq.assignment)
    assert np.array_equal(m_par.block_weights, m_seq.block_weights)


def test_host_upload_constant_weight_chunks(D):
    """The host entry fills constant weight chunks on the device instead of
    copying them: mappings equal the device-array path for unit vertex
    weights + varied edge weights and for constant non-unit edge weights +
    varied vertex weights, and bytes_h2d counts exactly what was copied."""
    from paper_2510_12196_b200 import integrated_map
    from paper_2510_12196_b200.generators import HostGraph, gen_rgg
    g = gen_rgg(1 << 16, 0.55, 1)
    src = np.repeat(np.arange(g.n), np.diff(g.offsets))
    lo, hi = np.minimum(src, g.edge_targets), np.maximum(src, g.edge_targets)
    varied_ew = 1 + (lo * 7 + hi * 13) % 5           # symmetric
    varied_vw = 1 + np.arange(g.n) % 3
    h, d = (4, 8, 6), (1, 10, 100)
    t = O.OTopology(h, d)
    cases = [(varied_ew, np.ones(g.n, np.int64), 4 * (g.n + 1) + 8 * len(g.edge_targets)),
             (np.full(len(g.edge_targets), 7), varied_vw,
              4 * (g.n + 1) + 4 * len(g.edge_targets) + 4 * g.n)]
    for ew, vw, want_h2d in cases:
        hg = HostGraph(g.offsets, g.edge_targets, ew, vw)
        st: dict = {}
        m = integrated_map(hg, t, 0.03, 1, stats=st)
        a, bw, _ = D.integrated_map_device(D.DeviceGraph.from_host(hg), h, d, 0.03, 1)
        assert np.array_equal(m.assignment, np_(a))
        assert np.array_equal(m.block_weights, np_(bw))
        assert st["bytes_h2d"] == want_h2d
        assert st["bytes_d2h"] == 4 * g.n + 8 * 192


def test_hem_hub_rows_match_oracle(D):
    """Rows longer than 1024 slots (R-MAT hubs) are rated by one CTA each:
    two HEM rounds equal the oracle's (coarsening.py:63-95), with vertex
    weights that make some hub candidates ineligible."""
    from paper_2510_12196_b200.generators import HostGraph, gen_rmat
    g0 = gen_rmat(14)
    assert np.diff(g0.offsets).max() > 1024
    vw = 1 + np.arange(g0.n) % 4
    g = HostGraph(g0.offsets, g0.edge_targets, g0.edge_weights, vw)
    og = O.as_ograph(g)
    dg = D.DeviceGraph.from_host(g)
    l_max = 6.0
    partner = torch.full((dg.n,), -1, dtype=torch.int32, device="cuda")
    op = np.full(g.n, -1, np.int64)
    m = 0
    for seed in (11, 12):
        pref, m = D.hem_round(dg, partner, l_max, seed, m)
        op, opref = O.hem_round(og, op, l_max, seed)
        assert np.array_equal(np_(pref), opref)
        assert np.array_equal(np_(partner), op)


_HUB_CHILD = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r})
from paper_2510_12196_b200 import integrated_map, device as D
from paper_2510_12196_b200.generators import gen_rgg, gen_rmat
from oracle import promap_np as O
D.set_batch(False)
for name, g in (("rmat", gen_rmat(11)), ("rgg", gen_rgg(2048, 0.55, 1))):
    t = O.OTopology((2, 4, 2), (1, 10, 100))
    m = integrated_map(g, t, 0.03, 1, coarsest_factor=16)
    np.save({out!r} + name + ".npy", m.assignment)
"""


@pytest.mark.parametrize("list_deg,hub_deg", [("8", "8"), ("8", "70")])
def test_listed_rows_grid_evaluation_matches_oracle(D, tmp_path, list_deg, hub_deg):
    """Long rows listed by the first filter / rebalance-candidate passes and
    evaluated by the grid afterwards (medium rows one warp each, hub rows by
    segments accumulated into per-hub conn tables): every refinement forced
    onto the cooperative grid, small thresholds so most rows take these
    paths; mappings identical to the oracle."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    from paper_2510_12196_b200.generators import gen_rgg, gen_rmat
    root = str(Path(__file__).resolve().parents[1])
    env = dict(os.environ, GIM_SMEM_MAXN="0", GIM_CLUSTER_VPC="1", GIM_HUB_DEG=hub_deg,
               GIM_LIST_DEG=list_deg)
    code = _HUB_CHILD.format(root=root, out=str(tmp_path / "hub_"))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    t = O.OTopology((2, 4, 2), (1, 10, 100))
    for name, g in (("rmat", gen_rmat(11)), ("rgg", gen_rgg(2048, 0.55, 1))):
        a, _, _ = O.integrated_map(g, t, 0.03, 1, coarsest_factor=16)
        assert np.array_equal(np.load(tmp_path / f"hub_{name}.npy"), a), name
