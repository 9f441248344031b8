"""Reference-generated goldens at BASELINE scale (round 2).

Runs the REFERENCE package itself (/root/reference/pkg/src, read-only) on the
benchmark shapes and stores its mappings so the GPU path can be pinned to them
byte for byte on the box (where /root/reference does not exist):

    python scripts/make_golden_scale.py rgg16 rgg18 rgg20 grid3d52 rmat14 \
        relatives envelope

Every case is one process (run them in parallel); each writes
tests/golden/scale_<case>.npz.  Graph inputs are regenerated on the box from
the recipe (graph seed, generator) — the arrays are not stored — and the
fixture keeps a checksum of the CSR so a generator drift is caught.
"""
from __future__ import annotations

import logging
import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(ROOT))

import promap.coarsening as C  # noqa: E402
from promap.coarsening import (  # noqa: E402
    build_level_stack, coarse_map_from_matching, contract, match_graph)
from promap.graph import Graph, from_edge_list, gen_grid, gen_rgg  # noqa: E402
from promap.mapping import BlockConnectivity, Mapping, total_cost  # noqa: E402
from promap.pipelines import integrated_map  # noqa: E402
from promap.refinement import (  # noqa: E402
    RefinementConfig, config_for_level, label_propagation_pass, refine)
from promap.topology import Topology  # noqa: E402

from paper_2510_12196_b200 import generators as G  # noqa: E402

OUT = ROOT / "tests" / "golden"


def csr_digest(g) -> np.ndarray:
    """Order-sensitive 64-bit digests of the CSR arrays (uint64 wraparound)."""
    out = []
    for a in (g.offsets, g.edge_targets, g.edge_weights, g.vertex_weights):
        a = np.asarray(a, dtype=np.uint64)
        mult = (np.arange(len(a), dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
                + np.uint64(1))
        with np.errstate(over="ignore"):
            out.append(np.uint64(np.sum(a * mult, dtype=np.uint64)))
    return np.asarray(out, dtype=np.uint64)


def to_ref(h) -> Graph:
    return Graph(h.offsets, h.edge_targets, h.edge_weights, h.vertex_weights)


class WarnCatcher(logging.Handler):
    def __init__(self):
        super().__init__()
        self.msgs = []

    def emit(self, record):
        self.msgs.append(record.getMessage())


def im_case(name, g, h, d, eps, seeds, recipe):
    t = Topology(h, d)
    catcher = WarnCatcher()
    logging.getLogger("promap.pipelines").addHandler(catcher)
    bag = {"recipe": np.asarray(recipe), "hierarchy": np.asarray(h),
           "distances": np.asarray(d), "eps": np.asarray(eps), "digest": csr_digest(g),
           "n": np.asarray(g.n), "m": np.asarray(g.m), "seeds": np.asarray(seeds)}
    dt = np.uint8 if t.k <= 256 else np.uint16
    for s in seeds:
        catcher.msgs.clear()
        t0 = time.time()
        m = integrated_map(g, t, eps, s)
        sec = time.time() - t0
        l_max = (1.0 + eps) * g.total_weight / t.k
        bag[f"{s}/assignment"] = m.assignment.astype(dt)
        bag[f"{s}/j"] = np.asarray(total_cost(g, t, m.assignment))
        bag[f"{s}/seconds"] = np.asarray(sec)
        bag[f"{s}/balanced"] = np.asarray(m.is_balanced(l_max))
        bag[f"{s}/max_block_weight"] = np.asarray(m.max_block_weight())
        bag[f"{s}/warning"] = np.asarray("\n".join(catcher.msgs))
        print(f"{name} seed {s}: J={int(bag[f'{s}/j'])} balanced={m.is_balanced(l_max)} "
              f"{sec:.1f}s warn={catcher.msgs}", flush=True)
    np.savez_compressed(OUT / f"scale_{name}.npz", **bag)


def rgg(logn, seeds, name=None):
    g = gen_rgg(1 << logn, 0.55, 1)
    im_case(name or f"rgg{logn}", g, (4, 8, 6), (1, 10, 100), 0.03, seeds,
            f"gen_rgg(2^{logn}, 0.55, seed=1)")


def grid3d52():
    g = to_ref(G.gen_grid3d(52, 52, 52))
    im_case("grid3d52", g, (4, 16, 8), (1, 10, 100), 0.03, [0], "gen_grid3d(52,52,52)")


def rmat14():
    g = to_ref(G.gen_rmat(14, seed=1))
    im_case("rmat14", g, (4, 8, 8), (1, 10, 100), 0.03, [0], "gen_rmat(14, seed=1)")


def relatives():
    """match_graph / build_level_stack on skewed graphs where two-hop
    relatives (coarsening.py:148-160) actually pair vertices."""
    calls = {"rel": 0}
    orig = C._pair_up

    def spy(state, group, vw, l_max):
        before = int((state.matched_partner >= 0).sum())
        orig(state, group, vw, l_max)
        if "mm" in sys._getframe(1).f_locals and int((state.matched_partner >= 0).sum()) > before:
            calls["rel"] += 1
    C._pair_up = spy
    bag, i = {}, 0
    for scale in (9, 10, 11, 12):
        for gseed in (1, 2, 3):
            g = to_ref(G.gen_rmat(scale, edge_factor=8, seed=gseed))
            for k in (16, 256):
                l_max = 1.03 * g.total_weight / k
                for mseed in (0, 99):
                    calls["rel"] = 0
                    st = match_graph(g, l_max, mseed)
                    if calls["rel"] == 0:
                        continue
                    cmap, n_c = coarse_map_from_matching(st)
                    bag[f"{i}/recipe"] = np.asarray([scale, 8, gseed])
                    bag[f"{i}/l_max"] = np.asarray(l_max)
                    bag[f"{i}/seed"] = np.asarray(mseed)
                    bag[f"{i}/partner"] = st.matched_partner.astype(np.int32)
                    bag[f"{i}/coarse_map"] = cmap.astype(np.int32)
                    bag[f"{i}/n_c"] = np.asarray(n_c)
                    bag[f"{i}/relative_pairings"] = np.asarray(calls["rel"])
                    bag[f"{i}/digest"] = csr_digest(g)
                    print("relatives", scale, gseed, k, mseed, calls["rel"], flush=True)
                    i += 1
    # a whole level stack where relatives fire on several levels
    g = to_ref(G.gen_rmat(13, edge_factor=8, seed=4))
    l_max = 1.03 * g.total_weight / 64
    calls["rel"] = 0
    st = build_level_stack(g, l_max, 64 * 8, 5)
    bag["stack/recipe"] = np.asarray([13, 8, 4])
    bag["stack/l_max"] = np.asarray(l_max)
    bag["stack/sizes"] = np.asarray([lv.graph.n for lv in st.levels])
    bag["stack/m2s"] = np.asarray([len(lv.graph.edge_targets) for lv in st.levels])
    bag["stack/relative_pairings"] = np.asarray(calls["rel"])
    for li, lv in enumerate(st.levels[:-1]):
        bag[f"stack/cmap{li}"] = lv.coarse_map.astype(np.int32)
    c = st.levels[-1].graph
    order = np.lexsort((c.edge_targets, c.edge_sources))
    bag["stack/c_offsets"] = c.offsets
    bag["stack/c_targets"] = c.edge_targets[order].astype(np.int32)
    bag["stack/c_weights"] = c.edge_weights[order]
    bag["stack/c_vweights"] = c.vertex_weights
    bag["count"] = np.asarray(i)
    C._pair_up = orig
    print("stack relatives", calls["rel"], bag["stack/sizes"])
    np.savez_compressed(OUT / "scale_relatives.npz", **bag)


def envelope():
    """Inputs outside the int32 / integral-D / <= 8-level envelope of round 1:
    non-integral distances (float J and gains), vertex and edge weights whose
    totals exceed 2^31, hierarchies of 9-11 levels."""
    rng = np.random.default_rng(7)
    bag, i = {}, 0

    def add(kind, g, h, d, eps, seed, cf, **extra):
        nonlocal i
        t = Topology(h, d)
        t0 = time.time()
        m = integrated_map(g, t, eps, seed, coarsest_factor=cf)
        bag[f"{i}/kind"] = np.asarray(kind)
        bag[f"{i}/offsets"] = g.offsets
        bag[f"{i}/targets"] = g.edge_targets
        bag[f"{i}/weights"] = g.edge_weights
        bag[f"{i}/vweights"] = g.vertex_weights
        bag[f"{i}/hierarchy"] = np.asarray(h)
        bag[f"{i}/distances"] = np.asarray(d, dtype=np.float64)
        bag[f"{i}/integral"] = np.asarray(t.integral_distances)
        bag[f"{i}/eps"] = np.asarray(eps)
        bag[f"{i}/seed"] = np.asarray(seed)
        bag[f"{i}/coarsest_factor"] = np.asarray(cf)
        bag[f"{i}/assignment"] = m.assignment
        bag[f"{i}/j"] = np.asarray(total_cost(g, t, m.assignment), dtype=np.float64
                                   if not t.integral_distances else np.int64)
        for k2, v in extra.items():
            bag[f"{i}/{k2}"] = np.asarray(v)
        print(kind, i, h, d, bag[f"{i}/j"], f"{time.time() - t0:.1f}s", flush=True)
        i += 1

    # float distances: J and all gains in float64
    for g, h, d, cf in [(gen_grid(24, 24), (2, 2, 2), (1.5, 10.25, 100.0), 16),
                        (gen_rgg(1500, 0.55, 3), (4, 4), (0.7, 3.3), 8),
                        (gen_grid(32, 32), (4, 8, 2), (1, 10.5, 100), 16)]:
        for seed in (0, 1):
            add("float_d", g, h, d, 0.03, seed, cf)
    # float-D J and LP pass (the unit-level float goldens)
    for g, h, d in [(gen_grid(20, 20), (2, 3, 2), (0.5, 2.25, 7.125)),
                    (gen_rgg(800, 0.55, 8), (4, 8, 6), (1.1, 9.9, 101.3))]:
        t = Topology(h, d)
        a = rng.integers(0, t.k, size=g.n)
        conn = BlockConnectivity(g, a, t.k)
        for mode in ("nonneg", "jet"):
            p = label_propagation_pass(g, t, Mapping.from_assignment(g, a.copy(), t.k), conn,
                                       rng.random(g.n) < 0.2, RefinementConfig(filter_mode=mode))
            bag[f"lp{i}_{mode}/dest"] = p.destinations
            bag[f"lp{i}_{mode}/cand"] = p.candidates
            bag[f"lp{i}_{mode}/to_move"] = p.to_move
        add("float_d_units", g, h, d, 0.03, 0, 8, unit_assignment=a,
            unit_j=total_cost(g, t, a))
    # int64 weights: totals above 2^31 (vertex weights ~2^27, edge weights ~2^26)
    for g0, h in [(gen_grid(16, 16), (2, 2, 2)), (gen_rgg(1000, 0.55, 9), (4, 4))]:
        vw = rng.integers(1 << 26, 1 << 27, size=g0.n)
        edges = []
        for u, v in zip(g0.edge_sources, g0.edge_targets):
            if u < v:
                edges.append((int(u), int(v), int(rng.integers(1 << 25, 1 << 26))))
        g = from_edge_list(g0.n, edges, vw)
        add("int64_w", g, h, (1, 10, 100)[:len(h)], 0.03, 0, 8)
    # deep hierarchies (9..11 levels)
    for g, h in [(gen_grid(48, 48), (2,) * 9), (gen_rgg(4000, 0.55, 10), (2, 2, 2, 2, 2, 2, 2, 2, 2, 2)),
                 (gen_grid(40, 40), (2, 3, 2, 2, 2, 2, 2, 2, 2, 2, 2))]:
        d = tuple(int(x) for x in np.cumsum(np.arange(1, len(h) + 1)))
        add("deep", g, h, d, 0.03, 0, 4)
    bag["count"] = np.asarray(i)
    np.savez_compressed(OUT / "scale_envelope.npz", **bag)


def kat():
    """SPEC criterion 7 (test_acceptance.py:216-242): 30 tiny instances with
    the reference's brute-force optimum and its integrated_map mapping."""
    sys.path.insert(0, str(REF / "tests"))
    from conftest import random_graph
    from promap.mapping import brute_force_map
    from promap.topology import flat_topology
    rng = np.random.default_rng(1007)
    specs = [(12 + 2 * (i % 4), flat_topology(2)) for i in range(12)]
    specs += [(12, flat_topology(3))] * 6 + [(8, Topology((2, 2), (1, 10)))] * 6
    specs += [(8, flat_topology(4))] * 6
    bag = {}
    for idx, (n, t) in enumerate(specs):
        g = random_graph(rng, n, p=0.3, unit_vertex_weights=True)
        _, opt_j = brute_force_map(g, t, 0.03)
        m = integrated_map(g, t, 0.03, seed=idx)
        bag[f"{idx}/offsets"] = g.offsets
        bag[f"{idx}/targets"] = g.edge_targets
        bag[f"{idx}/weights"] = g.edge_weights
        bag[f"{idx}/vweights"] = g.vertex_weights
        bag[f"{idx}/hierarchy"] = np.asarray(t.hierarchy)
        bag[f"{idx}/distances"] = np.asarray(t.distances)
        bag[f"{idx}/seed"] = np.asarray(idx)
        bag[f"{idx}/opt_j"] = np.asarray(opt_j)
        bag[f"{idx}/assignment"] = m.assignment
    bag["count"] = np.asarray(len(specs))
    np.savez_compressed(OUT / "scale_kat.npz", **bag)


CASES = {"kat": kat, "rgg16": lambda: rgg(16, [0, 1, 2]), "rgg18": lambda: rgg(18, [0]),
         "rgg20": lambda: rgg(20, [0]), "rgg22": lambda: rgg(22, [0]),
         "grid3d52": grid3d52, "rmat14": rmat14,
         "relatives": relatives, "envelope": envelope}

# one seed per process (rgg 2^20 ~ 9 min, 2^22 ~ 45 min of one core each)
for _s in range(1, 5):
    CASES[f"rgg20s{_s}"] = (lambda s: lambda: rgg(20, [s], f"rgg20s{s}"))(_s)
for _s in range(0, 3):
    CASES[f"rgg22s{_s}"] = (lambda s: lambda: rgg(22, [s], f"rgg22s{s}"))(_s)

if __name__ == "__main__":
    for c in sys.argv[1:]:
        t0 = time.time()
        CASES[c]()
        print(f"[{c}] {time.time() - t0:.1f}s", flush=True)
