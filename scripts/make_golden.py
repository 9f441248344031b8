"""Generate tests/golden/*.npz by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python scripts/make_golden.py

The fixtures pin the oracle (oracle/promap_np.py) and the CUDA path to the
reference's own outputs on identical inputs.  /root/reference is read-only
and is only read here; the fixtures are committed so the GPU box never needs
it.
"""
from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))

from promap.coarsening import (  # noqa: E402
    MatchingState, build_level_stack, coarse_map_from_matching, contract,
    heavy_edge_matching_round, match_graph, two_hop_matching)
from promap.graph import Graph, from_edge_list, gen_grid, gen_rgg  # noqa: E402
from promap.mapping import BlockConnectivity, Mapping, total_cost  # noqa: E402
from promap.pipelines import (  # noqa: E402
    greedy_graph_growing, hierarchical_multisection, integrated_map,
    internal_partitioner)
from promap.refinement import (  # noqa: E402
    RefinementConfig, config_for_level, label_propagation_pass, refine,
    strong_rebalance, weak_rebalance)
from promap.topology import Topology, flat_topology  # noqa: E402
from promap.util import hash2  # noqa: E402
from conftest import random_assignment, random_graph, random_hierarchy  # noqa: E402

OUT = Path(__file__).resolve().parents[1] / "tests" / "golden"


class Bag:
    """Flat npz writer: case i's arrays under keys f"{i}/{name}"."""

    def __init__(self):
        self.d: dict[str, np.ndarray] = {}
        self.n = 0

    def add(self, **arrays):
        for k, v in arrays.items():
            self.d[f"{self.n}/{k}"] = np.asarray(v)
        self.n += 1

    def save(self, name):
        self.d["count"] = np.asarray(self.n)
        np.savez_compressed(OUT / f"{name}.npz", **self.d)
        print(f"{name}: {self.n} cases, {(OUT / f'{name}.npz').stat().st_size} bytes")


def gfields(g: Graph) -> dict:
    return dict(offsets=g.offsets, targets=g.edge_targets, weights=g.edge_weights,
                vweights=g.vertex_weights)


def weighted_grid(rng, r, c, wmax=4):
    g = gen_grid(r, c)
    ew = {}
    for u, v in zip(g.edge_sources, g.edge_targets):
        if u < v:
            ew[(int(u), int(v))] = int(rng.integers(1, wmax + 1))
    edges = [(u, v, w) for (u, v), w in sorted(ew.items())]
    return from_edge_list(g.n, edges, rng.integers(1, wmax + 1, size=g.n))


def graphs(rng):
    out = [random_graph(rng, int(rng.integers(8, 40)), p=0.2) for _ in range(6)]
    out += [gen_grid(12, 12), weighted_grid(rng, 10, 14), gen_rgg(600, 1.0, 3)]
    out += [random_graph(rng, 60, p=0.05, wmax=3, unit_vertex_weights=True)]
    return out


def make_jeval(rng):
    bag = Bag()
    for _ in range(60):
        n = int(rng.integers(2, 30))
        g = random_graph(rng, n, p=0.3)
        h, d = random_hierarchy(rng, max_levels=4)
        t = Topology(h, d)
        a = random_assignment(rng, n, t.k)
        bag.add(**gfields(g), hierarchy=h, distances=d, assignment=a,
                j=total_cost(g, t, a))
    for g, h in [(gen_grid(40, 40), (4, 8, 6)), (gen_rgg(3000, 0.55, 1), (4, 8, 6)),
                 (weighted_grid(rng, 30, 31), (2, 3, 4, 2))]:
        t = Topology(h, (1, 10, 100, 1000)[:len(h)])
        a = random_assignment(rng, g.n, t.k)
        bag.add(**gfields(g), hierarchy=h, distances=t.distances, assignment=a,
                j=total_cost(g, t, a))
    bag.save("jeval")


def make_hem(rng):
    bag = Bag()
    for g in graphs(rng):
        for seed in (0, 12345):
            l_max = 1.03 * g.total_weight / 4
            st = MatchingState.empty(g.n)
            s1 = int(rng.integers(0, 2**63))
            heavy_edge_matching_round(g, st, l_max, s1)
            pref1, part1 = st.preferred.copy(), st.matched_partner.copy()
            s2 = int(rng.integers(0, 2**63))
            heavy_edge_matching_round(g, st, l_max, s2)
            full = match_graph(g, l_max, seed)
            cmap, n_c = coarse_map_from_matching(full)
            cg = contract(g, cmap, n_c)
            # reference rows are in hash order: store them sorted by target
            order = np.lexsort((cg.edge_targets, cg.edge_sources))
            bag.add(**gfields(g), has_rounds=1, l_max=l_max, seed1=np.uint64(s1),
                    seed2=np.uint64(s2),
                    pref1=pref1, part1=part1, pref2=st.preferred, part2=st.matched_partner,
                    match_seed=seed, match_partner=full.matched_partner, coarse_map=cmap,
                    n_c=n_c, c_offsets=cg.offsets, c_targets=cg.edge_targets[order],
                    c_weights=cg.edge_weights[order], c_vweights=cg.vertex_weights)
    # two-hop heavy: stars and leaves
    star = from_edge_list(9, [(0, i, 1) for i in range(1, 9)])
    twins = from_edge_list(8, [(0, 2, 1), (1, 2, 1), (0, 3, 1), (1, 3, 1), (4, 5, 2),
                               (5, 6, 1), (6, 7, 3)])
    for g in (star, twins):
        l_max = 100.0
        full = match_graph(g, l_max, 5)
        cmap, n_c = coarse_map_from_matching(full)
        cg = contract(g, cmap, n_c)
        order = np.lexsort((cg.edge_targets, cg.edge_sources))
        z = np.zeros(g.n, np.int64)
        bag.add(**gfields(g), has_rounds=0, l_max=l_max, seed1=np.uint64(1),
                seed2=np.uint64(2),
                pref1=z - 9, part1=z - 9, pref2=z - 9, part2=z - 9, match_seed=5,
                match_partner=full.matched_partner, coarse_map=cmap, n_c=n_c,
                c_offsets=cg.offsets, c_targets=cg.edge_targets[order],
                c_weights=cg.edge_weights[order], c_vweights=cg.vertex_weights)
    bag.save("hem")


def make_stack(rng):
    bag = Bag()
    for g, k, seed in [(gen_grid(48, 48), 4, 0), (gen_rgg(4096, 0.55, 2), 8, 3),
                       (weighted_grid(rng, 30, 30), 6, 9)]:
        l_max = 1.03 * g.total_weight / k
        st = build_level_stack(g, l_max, 64, seed)
        sizes = [lv.graph.n for lv in st.levels]
        m2s = [len(lv.graph.edge_targets) for lv in st.levels]
        c = st.levels[-1].graph
        order = np.lexsort((c.edge_targets, c.edge_sources))
        bag.add(**gfields(g), l_max=l_max, seed=seed, threshold=64, sizes=sizes, m2s=m2s,
                c_offsets=c.offsets, c_targets=c.edge_targets[order],
                c_weights=c.edge_weights[order], c_vweights=c.vertex_weights,
                cmap0=st.levels[0].coarse_map)
    bag.save("stack")


def conn_csr(conn: BlockConnectivity, n):
    dicts = conn.as_dicts()
    off = [0]
    blocks, ws = [], []
    for v in range(n):
        for b in sorted(dicts[v]):
            blocks.append(b)
            ws.append(dicts[v][b])
        off.append(len(blocks))
    return np.asarray(off), np.asarray(blocks, dtype=np.int64), np.asarray(ws, dtype=np.int64)


def make_refinement(rng):
    lp, rb, rf, cn = Bag(), Bag(), Bag(), Bag()
    topos = [Topology((4, 8, 6), (1, 10, 100)), Topology((2, 3), (1, 7)), flat_topology(5),
             Topology((3, 2, 2), (0, 4, 9))]
    for gi, g in enumerate(graphs(rng) + [gen_grid(24, 24), gen_rgg(2000, 0.55, 4)]):
        for t in topos:
            k = t.k
            a = random_assignment(rng, g.n, k)
            # skew half the vertices into block 0 for imbalance
            skew = a.copy()
            skew[rng.random(g.n) < 0.5] = 0
            conn = BlockConnectivity(g, a, k)
            off, blocks, ws = conn_csr(conn, g.n)
            cn.add(**gfields(g), hierarchy=t.hierarchy, distances=t.distances,
                   assignment=a, conn_offsets=off, conn_blocks=blocks, conn_weights=ws)
            locked = rng.random(g.n) < 0.2
            for mode in ("nonneg", "jet"):
                cfg = RefinementConfig(filter_mode=mode)
                m = Mapping.from_assignment(g, a.copy(), k)
                p = label_propagation_pass(g, t, m, conn, locked, cfg)
                lp.add(**gfields(g), hierarchy=t.hierarchy, distances=t.distances,
                       assignment=a, locked=locked, jet=int(mode == "jet"),
                       cand=p.candidates, dest=p.destinations, to_move=p.to_move)
            for eps in (0.03, 0.3):
                l_max = (1.0 + eps) * g.total_weight / k
                for frac in (0.005, 0.065):
                    sigma = l_max * (1.0 - frac)
                    seed = int(rng.integers(0, 2**62))
                    pc = int(rng.integers(0, 5))
                    cfg = RefinementConfig(seed=seed, sigma_fraction=frac)
                    m = Mapping.from_assignment(g, skew.copy(), k)
                    c2 = BlockConnectivity(g, skew, k)
                    pw = weak_rebalance(g, t, m, c2, sigma, l_max, cfg, pc)
                    ps = strong_rebalance(g, t, m, c2, sigma, l_max, cfg, pc)
                    rb.add(**gfields(g), hierarchy=t.hierarchy, distances=t.distances,
                           assignment=skew, l_max=l_max, sigma=sigma, seed=np.uint64(seed),
                           pass_counter=pc, rho=2,
                           w_cand=pw.candidates, w_dest=pw.destinations,
                           w_to_move=pw.to_move, w_incomplete=pw.incomplete,
                           s_cand=ps.candidates, s_dest=ps.destinations,
                           s_to_move=ps.to_move, s_incomplete=ps.incomplete)
            if gi % 2 == 0:
                for start, lev, nl in ((a, 0, 3), (skew, 2, 3)):
                    l_max = 1.03 * g.total_weight / k
                    cfg = config_for_level(lev, nl, seed=hash2(7, 211, lev),
                                           filter_mode="jet" if lev else "nonneg")
                    m = Mapping.from_assignment(g, start.copy(), k)
                    best = refine(g, t, m, BlockConnectivity(g, start, k), cfg, l_max)
                    rf.add(**gfields(g), hierarchy=t.hierarchy, distances=t.distances,
                           assignment=start, level=lev, n_levels=nl,
                           seed=np.uint64(cfg.seed), jet=int(cfg.filter_mode == "jet"),
                           l_max=l_max, best=best.assignment)
    cn.save("conn")
    lp.save("lp")
    rb.save("rebalance")
    rf.save("refine")


def make_initial(rng):
    gg, ip, hm = Bag(), Bag(), Bag()
    gs = graphs(rng)
    disc = from_edge_list(10, [(0, 1, 1), (1, 2, 1), (5, 6, 2), (7, 8, 1)])
    for g in gs + [disc]:
        for k in (2, 3, 5):
            gg.add(**gfields(g), k=k, part=greedy_graph_growing(g, k))
    for g in gs + [gen_grid(30, 30), gen_rgg(3000, 0.55, 5)]:
        for k, eps in ((2, 0.03), (4, 0.1), (6, 0.0)):
            seed = int(rng.integers(0, 2**40))
            ip.add(**gfields(g), k=k, eps=eps, seed=seed,
                   part=internal_partitioner(g, k, eps, seed))
    for g, h in [(gen_grid(20, 20), (2, 2)), (gen_grid(32, 32), (4, 8, 2)),
                 (gen_rgg(2500, 0.55, 6), (4, 3, 2)), (weighted_grid(rng, 16, 18), (3, 4))]:
        t = Topology(h, (1, 10, 100)[:len(h)])
        seed = int(rng.integers(0, 2**40))
        m = hierarchical_multisection(g, t, 0.03, seed=seed)
        hm.add(**gfields(g), hierarchy=h, distances=t.distances, eps=0.03, seed=seed,
               assignment=m.assignment)
    gg.save("ggg")
    ip.save("partitioner")
    hm.save("multisection")


def make_im(rng):
    bag = Bag()
    cases = [(gen_grid(32, 32), (2, 2, 2), 16, 0), (gen_rgg(2000, 0.55, 7), (4, 4), 8, 1),
             (weighted_grid(rng, 24, 24), (2, 3, 2), 8, 2), (gen_grid(64, 64), (4, 8, 2), 16, 3)]
    for g, h, cf, seed in cases:
        t = Topology(h, (1, 10, 100)[:len(h)])
        t0 = time.time()
        m = integrated_map(g, t, 0.03, seed, coarsest_factor=cf)
        bag.add(**gfields(g), hierarchy=h, distances=t.distances, eps=0.03, seed=seed,
                coarsest_factor=cf, assignment=m.assignment.astype(np.int16),
                j=total_cost(g, t, m.assignment), seconds=time.time() - t0)
    bag.save("im_small")
    # config 1: grid 128x128 -> H=4:8:2, D=1:10:100, eps=0.03, seeds 0..4
    cfg1 = Bag()
    g = gen_grid(128, 128)
    t = Topology((4, 8, 2), (1, 10, 100))
    for seed in range(5):
        t0 = time.time()
        m = integrated_map(g, t, 0.03, seed)
        cfg1.add(seed=seed, assignment=m.assignment.astype(np.uint8),
                 j=total_cost(g, t, m.assignment), seconds=time.time() - t0)
        print("cfg1 seed", seed, total_cost(g, t, m.assignment), time.time() - t0)
    cfg1.save("im_cfg1")


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    which = set(sys.argv[1:]) or {"jeval", "hem", "stack", "refinement", "initial", "im"}
    rng = np.random.default_rng(20251017)
    for name, fn in [("jeval", make_jeval), ("hem", make_hem), ("stack", make_stack),
                     ("refinement", make_refinement), ("initial", make_initial),
                     ("im", make_im)]:
        sub = np.random.default_rng(rng.integers(0, 2**63))
        if name in which:
            t0 = time.time()
            fn(sub)
            print(f"  [{name}] {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
