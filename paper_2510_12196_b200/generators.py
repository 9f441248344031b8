"""Vectorized synthetic task-graph generators (measurement inputs).

`gen_grid` / `gen_rgg` produce arrays identical to the reference generators
(graph.py:316-350, rows sorted by target via `from_edge_list`, graph.py:102-126);
`gen_grid3d` and `gen_rmat` build the config-3/4 shapes of SURVEY.md §8(d).
Host-side numpy only: graph generation is outside every timed region.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass
class HostGraph:
    """Reference-layout CSR (int64 numpy), duck-compatible with promap.Graph."""

    offsets: np.ndarray
    edge_targets: np.ndarray
    edge_weights: np.ndarray
    vertex_weights: np.ndarray
    edge_sources: np.ndarray = field(default=None)

    def __post_init__(self):
        self.offsets = np.ascontiguousarray(self.offsets, dtype=np.int64)
        self.edge_targets = np.ascontiguousarray(self.edge_targets, dtype=np.int64)
        self.edge_weights = np.ascontiguousarray(self.edge_weights, dtype=np.int64)
        self.vertex_weights = np.ascontiguousarray(self.vertex_weights, dtype=np.int64)
        if self.edge_sources is None:
            self.edge_sources = np.repeat(np.arange(self.n, dtype=np.int64),
                                          np.diff(self.offsets))
        else:
            self.edge_sources = np.ascontiguousarray(self.edge_sources, dtype=np.int64)

    @property
    def n(self) -> int:
        return len(self.offsets) - 1

    @property
    def m(self) -> int:
        return len(self.edge_targets) // 2

    @property
    def total_weight(self) -> int:
        return int(self.vertex_weights.astype(object).sum()) if self.n else 0

    def neighbors(self, v: int) -> np.ndarray:
        return self.edge_targets[self.offsets[v]:self.offsets[v + 1]]

    def neighbor_weights(self, v: int) -> np.ndarray:
        return self.edge_weights[self.offsets[v]:self.offsets[v + 1]]


def from_pairs(n: int, u: np.ndarray, v: np.ndarray, w: np.ndarray | None = None,
               vertex_weights=None) -> HostGraph:
    """Vectorized `from_edge_list` (graph.py:102-126): both directions, rows
    sorted by target.  Pairs must be unique, u != v."""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    w = np.ones(len(u), dtype=np.int64) if w is None else np.asarray(w, dtype=np.int64)
    if np.any(u == v):
        raise ValueError("self-loop")
    srcs = np.empty(2 * len(u), dtype=np.int64)
    tgts = np.empty(2 * len(u), dtype=np.int64)
    wgts = np.empty(2 * len(u), dtype=np.int64)
    srcs[0::2], srcs[1::2] = u, v
    tgts[0::2], tgts[1::2] = v, u
    wgts[0::2], wgts[1::2] = w, w
    order = np.lexsort((tgts, srcs))
    srcs, tgts, wgts = srcs[order], tgts[order], wgts[order]
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(srcs, minlength=n), out=offsets[1:])
    vw = np.ones(n, dtype=np.int64) if vertex_weights is None else vertex_weights
    return HostGraph(offsets, tgts, wgts, np.asarray(vw, dtype=np.int64), srcs)


def gen_grid(rows: int, cols: int) -> HostGraph:
    """2D 4-neighbour grid, unit weights (graph.py:316-328)."""
    if rows < 1 or cols < 1:
        raise ValueError("grid dimensions must be positive")
    idx = np.arange(rows * cols, dtype=np.int64).reshape(rows, cols)
    u = np.concatenate([idx[:, :-1].ravel(), idx[:-1, :].ravel()])
    v = np.concatenate([idx[:, 1:].ravel(), idx[1:, :].ravel()])
    return from_pairs(rows * cols, u, v)


def gen_grid3d(nx: int, ny: int, nz: int) -> HostGraph:
    """3D 6-neighbour grid, unit weights (config 4 shape)."""
    idx = np.arange(nx * ny * nz, dtype=np.int64).reshape(nx, ny, nz)
    u = np.concatenate([idx[:-1].ravel(), idx[:, :-1].ravel(), idx[:, :, :-1].ravel()])
    v = np.concatenate([idx[1:].ravel(), idx[:, 1:].ravel(), idx[:, :, 1:].ravel()])
    return from_pairs(nx * ny * nz, u, v)


def gen_rgg(n: int, radius_factor: float = 1.0, seed: int = 0) -> HostGraph:
    """Random geometric graph on the unit square (graph.py:331-350)."""
    if n < 1:
        raise ValueError("n must be positive")
    from scipy.spatial import cKDTree

    rng = np.random.default_rng(seed)
    points = rng.random((n, 2))
    radius = radius_factor * math.sqrt(math.log(max(n, 2)) / n)
    tree = cKDTree(points)
    pairs = tree.query_pairs(radius, output_type="ndarray")
    if len(pairs):
        dist = np.linalg.norm(points[pairs[:, 0]] - points[pairs[:, 1]], axis=1)
        pairs = pairs[dist < radius]
    return from_pairs(n, pairs[:, 0], pairs[:, 1]) if len(pairs) else from_pairs(
        n, np.empty(0, np.int64), np.empty(0, np.int64))


def gen_rmat(scale: int, edge_factor: int = 16, a=0.57, b=0.19, c=0.19,
             seed: int = 1) -> HostGraph:
    """Graph500-style R-MAT: one rng.random(E) per
    bit, self-loops dropped, undirected pairs deduplicated, unit weights."""
    n = 1 << scale
    E = edge_factor * n
    rng = np.random.default_rng(seed)
    u = np.zeros(E, dtype=np.int64)
    v = np.zeros(E, dtype=np.int64)
    for bit in range(scale):
        r = rng.random(E)
        ubit = r >= a + b            # quadrants c, d set the row bit
        vbit = ((r >= a) & (r < a + b)) | (r >= a + b + c)
        u |= ubit.astype(np.int64) << bit
        v |= vbit.astype(np.int64) << bit
    keep = u != v
    lo = np.minimum(u[keep], v[keep])
    hi = np.maximum(u[keep], v[keep])
    key = np.unique(lo * n + hi)
    return from_pairs(n, key // n, key % n)
