"""Pin the CPU oracle (oracle/promap_np.py) to the reference's own outputs.

Every golden vector in tests/golden/ was produced by running the reference
package (scripts/make_golden.py); these tests must pass before the oracle is
trusted as the checker for the CUDA path.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import promap_np as O


def test_jeval_golden(golden):
    for c in golden("jeval"):
        assert O.total_cost(c.graph(), c.topology(), c["assignment"]) == c.scalar("j")


def test_hem_rounds_golden(golden):
    for c in golden("hem"):
        if not c.scalar("has_rounds"):
            continue
        g = c.graph()
        part = np.full(g.n, -1, dtype=np.int64)
        part, pref = O.hem_round(g, part, c.scalar("l_max"), int(c["seed1"]))
        assert np.array_equal(pref, c["pref1"])
        assert np.array_equal(part, c["part1"])
        part, pref = O.hem_round(g, part, c.scalar("l_max"), int(c["seed2"]))
        assert np.array_equal(pref, c["pref2"])
        assert np.array_equal(part, c["part2"])


def test_match_and_contract_golden(golden):
    for c in golden("hem"):
        g = c.graph()
        part = O.match_graph(g, c.scalar("l_max"), int(c["match_seed"]))
        assert np.array_equal(part, c["match_partner"])
        cmap, n_c = O.coarse_map_from_matching(part)
        assert n_c == c.scalar("n_c")
        assert np.array_equal(cmap, c["coarse_map"])
        cg = O.contract(g, cmap, n_c)
        assert np.array_equal(cg.offsets, c["c_offsets"])
        assert np.array_equal(cg.edge_targets, c["c_targets"])
        assert np.array_equal(cg.edge_weights, c["c_weights"])
        assert np.array_equal(cg.vertex_weights, c["c_vweights"])


def test_level_stack_golden(golden):
    for c in golden("stack"):
        st = O.build_level_stack(c.graph(), c.scalar("l_max"), int(c["threshold"]),
                                 int(c["seed"]))
        assert [lv.graph.n for lv in st] == list(c["sizes"])
        assert [len(lv.graph.edge_targets) for lv in st] == list(c["m2s"])
        assert np.array_equal(st[0].coarse_map, c["cmap0"])
        last = st[-1].graph
        assert np.array_equal(last.offsets, c["c_offsets"])
        assert np.array_equal(last.edge_targets, c["c_targets"])
        assert np.array_equal(last.edge_weights, c["c_weights"])


def test_conn_golden(golden):
    for c in golden("conn"):
        off, blocks, w, _ = O.conn_table(c.graph(), c["assignment"], c.topology().k)
        assert np.array_equal(off, c["conn_offsets"])
        assert np.array_equal(blocks, c["conn_blocks"])
        assert np.array_equal(w, c["conn_weights"])


def test_lp_golden(golden):
    for c in golden("lp"):
        cfg = O.Config(filter_mode="jet" if c.scalar("jet") else "nonneg")
        p = O.label_propagation_pass(c.graph(), c.topology(), c["assignment"], c["locked"], cfg)
        assert np.array_equal(p.candidates, c["cand"])
        assert np.array_equal(p.destinations, c["dest"])
        assert np.array_equal(p.to_move, c["to_move"])


def test_rebalance_golden(golden):
    for c in golden("rebalance"):
        g, t = c.graph(), c.topology()
        a = c["assignment"]
        bw = O.block_weights(g.vertex_weights, a, t.k)
        cfg = O.Config(seed=int(c["seed"]), rho=int(c["rho"]))
        args = (g, t, a, bw, c.scalar("sigma"), c.scalar("l_max"), cfg, int(c["pass_counter"]))
        pw = O.weak_rebalance(*args)
        assert np.array_equal(pw.candidates, c["w_cand"])
        assert np.array_equal(pw.destinations, c["w_dest"])
        assert np.array_equal(pw.to_move, c["w_to_move"])
        assert pw.incomplete == bool(c["w_incomplete"])
        ps = O.strong_rebalance(*args)
        assert np.array_equal(ps.candidates, c["s_cand"])
        assert np.array_equal(ps.destinations, c["s_dest"])
        assert np.array_equal(ps.to_move, c["s_to_move"])
        assert ps.incomplete == bool(c["s_incomplete"])


def test_refine_golden(golden):
    for c in golden("refine"):
        lev, nl = int(c["level"]), int(c["n_levels"])
        cfg = O.config_for_level(lev, nl, seed=int(c["seed"]),
                                 filter_mode="jet" if c.scalar("jet") else "nonneg")
        best = O.refine(c.graph(), c.topology(), c["assignment"], cfg, c.scalar("l_max"))
        assert np.array_equal(best, c["best"])


def test_ggg_golden(golden):
    for c in golden("ggg"):
        assert np.array_equal(O.greedy_graph_growing(c.graph(), int(c["k"])), c["part"])


def test_partitioner_golden(golden):
    for c in golden("partitioner"):
        p = O.internal_partitioner(c.graph(), int(c["k"]), c.scalar("eps"), int(c["seed"]))
        assert np.array_equal(p, c["part"])


def test_multisection_golden(golden):
    for c in golden("multisection"):
        a = O.hierarchical_multisection(c.graph(), c.topology(), c.scalar("eps"),
                                        int(c["seed"]))
        assert np.array_equal(a, c["assignment"])


def test_integrated_map_small_golden(golden):
    for c in golden("im_small"):
        g, t = c.graph(), c.topology()
        a, bw, l_max = O.integrated_map(g, t, c.scalar("eps"), int(c["seed"]),
                                        coarsest_factor=int(c["coarsest_factor"]))
        assert np.array_equal(a, c["assignment"].astype(np.int64))
        assert O.total_cost(g, t, a) == c.scalar("j")


@pytest.mark.slow
def test_integrated_map_cfg1_golden(golden):
    """Config 1 (grid 128x128, H=4:8:2, D=1:10:100, eps=0.03), seed 0."""
    from paper_2510_12196_b200.generators import gen_grid
    c = golden("im_cfg1")[0]
    g = gen_grid(128, 128)
    t = O.OTopology((4, 8, 2), (1, 10, 100))
    a, _, _ = O.integrated_map(g, t, 0.03, int(c["seed"]))
    assert np.array_equal(a, c["assignment"].astype(np.int64))
