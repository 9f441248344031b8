"""Drop-in `integrated_map` with the reference signature, plus `install()`.

Reference boundary: promap.pipelines.integrated_map (pipelines.py:221-269).
Same arguments, same return type (a `Mapping` with int64 `assignment[n]` and
`block_weights[k]`), same errors (ValueError on an empty graph, ValueError
for invalid refinement knobs as RefinementConfig raises them,
refinement.py:61-71) and the same imbalance warning on logger
"promap.pipelines" (pipelines.py:264-268).  The whole computation runs in
libgpuim.so on the current CUDA device; there is no CPU fallback.
"""
from __future__ import annotations

import logging
from dataclasses import dataclass

import numpy as np

log = logging.getLogger("promap.pipelines")


@dataclass
class Mapping:
    """Mirror of promap.mapping.Mapping (mapping.py:46-73), used when the
    reference package is not importable."""

    assignment: np.ndarray
    block_weights: np.ndarray

    @property
    def k(self) -> int:
        return len(self.block_weights)

    def copy(self) -> "Mapping":
        return Mapping(self.assignment.copy(), self.block_weights.copy())

    def max_block_weight(self) -> int:
        return int(self.block_weights.max()) if len(self.block_weights) else 0

    def is_balanced(self, l_max: float) -> bool:
        return self.max_block_weight() <= l_max


def _mapping_type():
    try:
        from promap.mapping import Mapping as RefMapping  # reference type when present
        return RefMapping
    except Exception:  # noqa: BLE001 - reference absent (e.g. on the GPU box)
        return Mapping


def _validate(phi, rho, filter_mode, sigma_coarse, sigma_fine, iw_max_finest):
    # the same checks RefinementConfig.__post_init__ applies (refinement.py:61-71)
    if not (0 < phi <= 1):
        raise ValueError(f"phi must be in (0,1], got {phi}")
    if rho < 1:
        raise ValueError(f"rho must be >= 1, got {rho}")
    for f in (sigma_coarse, sigma_fine):
        if not (0 <= f < 1):
            raise ValueError(f"sigma_fraction must be in [0,1), got {f}")
    if filter_mode not in ("nonneg", "jet"):
        raise ValueError(f"unknown filter_mode {filter_mode!r}")
    if iw_max_finest < 1:
        raise ValueError("iteration caps must be >= 1")


def integrated_map(g, t, eps: float, seed: int = 0, *, coarsest_factor: int = 128,
                   phi: float = 0.999, rho: int = 2, filter_mode: str = "nonneg",
                   jet_filter_c: float = 0.25, sigma_coarse: float = 0.065,
                   sigma_fine: float = 0.005, iw_max_finest: int = 10, stats: dict | None = None,
                   isolated_vertices: str = "keep"):
    """GPU-IM: coarsen, map the coarsest graph, refine upward — on the B200.

    `g` is any object with the reference Graph's int64 CSR arrays
    (offsets, edge_targets, edge_weights, vertex_weights); `t` any object
    with `hierarchy` and `distances`.  If `stats` is a dict it receives the
    run counters (levels, iterations, device milliseconds, launches).

    `isolated_vertices="strip"` (not in the reference) maps the graph without
    its degree-0 vertices and water-fills them into the lightest blocks
    afterwards (include/gpuim.h GIM_ISOLATED_STRIP): on skewed graphs whose
    isolated vertices stall the coarsening (R-MAT) this is much faster; it is
    held to tolerance parity (balanced, J by geometric mean), not bit-exact.
    """
    from . import device as D

    n = len(g.offsets) - 1
    if n == 0:
        raise ValueError("cannot map an empty graph")
    _validate(phi, rho, filter_mode, sigma_coarse, sigma_fine, iw_max_finest)
    a, bw, st = D.integrated_map_host(
        g.offsets, g.edge_targets, g.edge_weights, g.vertex_weights, tuple(t.hierarchy),
        tuple(t.distances), eps, seed, coarsest_factor=coarsest_factor, phi=phi, rho=rho,
        filter_mode=filter_mode, jet_filter_c=jet_filter_c, sigma_coarse=sigma_coarse,
        sigma_fine=sigma_fine, iw_max_finest=iw_max_finest, isolated_vertices=isolated_vertices)
    # J as the reference types it (mapping.py:76-91): int for integral
    # distances, else float (the device works on d * 2^dist_shift)
    st["J"] = st["final_j"] if D.integral_distances(t.distances) else st["final_j_f64"]
    if stats is not None:
        stats.update(st)
    m = _mapping_type()(a, bw)
    l_max = st["l_max"]
    if not m.is_balanced(l_max):
        log.warning(
            "integrated mapping left imbalanced: max block weight %d > L_max %.3f",
            m.max_block_weight(), l_max,
        )
    return m


@dataclass
class SplitRecord:
    """Mirror of promap.pipelines.SplitRecord (pipelines.py:36-47), used when
    the reference package is not importable."""

    level: int
    identifier: tuple
    parts: int
    eps_local: float
    subgraph_weight: int
    block_weights: list
    budget_met: bool


def _split_record_type():
    try:
        from promap.pipelines import SplitRecord as RefSplitRecord
        return RefSplitRecord
    except Exception:  # noqa: BLE001 - reference absent
        return SplitRecord


def _graph_type():
    try:
        from promap.graph import Graph as RefGraph
        return RefGraph
    except Exception:  # noqa: BLE001 - reference absent
        from .generators import HostGraph
        return HostGraph


def hierarchical_multisection(g, t, eps: float, partitioner=None, seed: int = 0,
                              trace: list | None = None):
    """GPU-HM: recursive multisection along the machine hierarchy
    (pipelines.py:49-110) of the whole graph on the B200.  Same signature,
    return type and errors as the reference, including its plugin seam: a
    `partitioner(sub, parts, eps_local, seed)` callable is called per tree
    node in the reference's depth-first order with the node's subgraph (a
    reference `Graph`), its exceptions surface as `RuntimeError("partitioner
    failed at hierarchy node [...]")` and invalid outputs as
    `RuntimeError("partitioner returned an invalid assignment at node
    [...]")`; `trace` receives one SplitRecord per partitioning step.  The
    tree (extraction, block weights, the built-in partitioner) runs on the
    GPU; only the caller's own partitioner runs on the host."""
    from . import _lib
    from . import device as D

    n = len(g.offsets) - 1
    if n == 0:
        raise ValueError("cannot map an empty graph")
    if partitioner is None and trace is None:
        a, bw = D.hierarchical_multisection_host(g.offsets, g.edge_targets, g.edge_weights,
                                                 g.vertex_weights, tuple(t.hierarchy),
                                                 tuple(t.distances), eps, seed)
        return _mapping_type()(a, bw)
    failure: list = []
    part_cb = trace_cb = None
    if partitioner is not None:
        Graph = _graph_type()

        def _part(_user, nn, off, tgt, ew, vw, parts, eps_local, node_seed, ident, ilen, out):
            try:
                ids = [ident[i] for i in range(ilen)]
                o = np.ctypeslib.as_array(off, shape=(nn + 1,)).copy()
                m2 = int(o[-1])
                arr = (lambda p: np.ctypeslib.as_array(p, shape=(m2,)).copy()) if m2 else \
                    (lambda p: np.zeros(0, dtype=np.int64))
                sub = Graph(o, arr(tgt), arr(ew), np.ctypeslib.as_array(vw, shape=(nn,)).copy())
                try:
                    part = np.asarray(partitioner(sub, int(parts), float(eps_local),
                                                  int(node_seed)), dtype=np.int64)
                except Exception as exc:  # noqa: BLE001 - wrapped like the reference
                    err = RuntimeError(f"partitioner failed at hierarchy node {ids}")
                    err.__cause__ = exc
                    failure.append(err)
                    return 1
                if len(part) != nn or part.min() < 0 or part.max() >= parts:
                    failure.append(RuntimeError(
                        f"partitioner returned an invalid assignment at node {ids}"))
                    return 1
                np.ctypeslib.as_array(out, shape=(nn,))[:] = part
                return 0
            except BaseException as exc:  # noqa: BLE001 - re-raised after the call
                failure.append(exc)
                return 1
        part_cb = _lib.PARTITION_FN(_part)
    if trace is not None:
        Rec = _split_record_type()

        def _trace(_user, level, ident, ilen, parts, eps_local, sub_weight, bws, met):
            trace.append(Rec(int(level), tuple(ident[i] for i in range(ilen)), int(parts),
                             float(eps_local), int(sub_weight),
                             [int(bws[i]) for i in range(parts)], bool(met)))
        trace_cb = _lib.TRACE_FN(_trace)
    try:
        a, bw = D.hierarchical_multisection_plugin(
            g.offsets, g.edge_targets, g.edge_weights, g.vertex_weights, tuple(t.hierarchy),
            tuple(t.distances), eps, seed, part_cb, trace_cb)
    except _lib.GimError as exc:
        if exc.status == _lib.GIM_E_CALLBACK and failure:
            raise failure[0] from failure[0].__cause__
        raise
    return _mapping_type()(a, bw)


def empty_cache() -> None:
    """Release the device scratch libgpuim caches across calls (per device,
    stream and size class) back to the CUDA pools, e.g. before handing the
    GPU memory to other torch code."""
    from . import device as D

    D.release_cached_memory()


_INSTALL_SITES = ("promap.pipelines", "promap.estimators", "promap.cli", "promap.bench", "promap",
                  "promap.graph")
_NAMES = ("integrated_map", "hierarchical_multisection", "load_metis")


def install() -> list[str]:
    """Rebind `integrated_map`, `hierarchical_multisection` and
    `load_metis` in every reference module that imported them (pipelines,
    graph, estimators.py:17, cli.py:31-33, bench.py:23-25, __init__.py), so
    the reference's estimators (IntegratedMapper, MultisectionMapper), CLI
    (`--algo im|hm`, METIS input) and bench run on the native path
    unchanged.  Returns the patched module names."""
    import importlib

    from .metis import load_metis

    ours = {"integrated_map": integrated_map,
            "hierarchical_multisection": hierarchical_multisection,
            "load_metis": load_metis}
    patched = []
    for name in _INSTALL_SITES:
        mod = importlib.import_module(name)
        hit = False
        for fn in _NAMES:
            if hasattr(mod, fn):
                if not hasattr(mod, f"_cpu_{fn}"):
                    setattr(mod, f"_cpu_{fn}", getattr(mod, fn))
                setattr(mod, fn, ours[fn])
                hit = True
        if hit:
            patched.append(name)
    return patched


def uninstall() -> None:
    import importlib
    import sys

    for name in _INSTALL_SITES:
        mod = sys.modules.get(name) or importlib.import_module(name)
        for fn in _NAMES:
            if hasattr(mod, f"_cpu_{fn}"):
                setattr(mod, fn, getattr(mod, f"_cpu_{fn}"))
