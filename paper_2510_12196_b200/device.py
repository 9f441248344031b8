"""Device-resident CSR levels and thin wrappers over every libgpuim entry point.

torch tensors are the plumbing (device memory + the current CUDA stream);
all compute happens in libgpuim.so.  Each wrapper cites the reference
function its kernel replaces.  There is no CPU fallback anywhere: a missing
library raises ImportError, a failed call raises GimError.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib

INT32_MAX = 2**31 - 1


def _ptr(t: torch.Tensor | None):
    if t is None:
        return None
    return t.data_ptr() if t.numel() else None


def stream_ptr(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _i32(x, device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=torch.int32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.int32)).to(device)


def _u8(x, device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=torch.uint8).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.uint8)).to(device)


def topology_struct(hierarchy, distances) -> _lib.GimTopology:
    """gim_topology of a (hierarchy, distances) pair; non-integral distances
    run as d * 2^s device integers (include/gpuim.h)."""
    return _lib.topology_struct(hierarchy, distances)


def integral_distances(distances) -> bool:
    """topology.py:56-58: J and gains are Python ints iff every d is an int."""
    return all(isinstance(d, (int, np.integer)) for d in distances)


def topology_scale(hierarchy, distances) -> tuple[int, bool]:
    """(s, exact): the device carries d * 2^s (exact for dyadic d)."""
    t = topology_struct(hierarchy, distances)
    sh, ex = C.c_int32(0), C.c_int32(0)
    _lib.call("gim_topology_scale", C.byref(t), C.byref(sh), C.byref(ex))
    return sh.value, bool(ex.value)


class DeviceGraph:
    """One CSR level on the GPU: int32 offsets/targets/weights/vweights/sources."""

    def __init__(self, offsets, targets, weights, vweights, sources=None, total_weight=None):
        self.offsets = offsets
        self.targets = targets
        self.weights = weights
        self.vweights = vweights
        if sources is None:
            sources = torch.empty(targets.numel(), dtype=torch.int32, device=offsets.device)
            if self.n:
                _lib.call("gim_fill_sources", self.n, _ptr(offsets), _ptr(sources),
                          stream_ptr(offsets.device))
        self.sources = sources
        self.total_weight = int(vweights.sum().item()) if total_weight is None else int(total_weight)

    @property
    def n(self) -> int:
        return self.offsets.numel() - 1

    @property
    def m2(self) -> int:
        return self.targets.numel()

    @property
    def device(self):
        return self.offsets.device

    @staticmethod
    def check_host(offsets, targets, eweights, vweights) -> int:
        n = len(offsets) - 1
        if len(targets) > INT32_MAX or n > INT32_MAX:
            raise OverflowError("graph too large for the int32 device layout")
        total_vw = int(np.asarray(vweights).sum(dtype=np.int64)) if n else 0
        if total_vw > INT32_MAX:
            raise OverflowError("total vertex weight must be < 2^31")
        if len(eweights) and int(np.asarray(eweights).sum(dtype=np.int64)) > INT32_MAX:
            raise OverflowError("total edge weight must be < 2^31")
        return total_vw

    @classmethod
    def from_host(cls, g, device="cuda") -> "DeviceGraph":
        """Upload a reference-layout Graph (offsets, edge_targets, edge_weights,
        vertex_weights; int64)."""
        total = cls.check_host(g.offsets, g.edge_targets, g.edge_weights, g.vertex_weights)
        dev = torch.device(device)
        return cls(_i32(g.offsets, dev), _i32(g.edge_targets, dev), _i32(g.edge_weights, dev),
                   _i32(g.vertex_weights, dev), None, total)

    def struct(self) -> _lib.GimGraph:
        s = _lib.GimGraph()
        s.n = self.n
        s.m2 = self.m2
        s.offsets = _ptr(self.offsets)
        s.targets = _ptr(self.targets)
        s.weights = _ptr(self.weights)
        s.vweights = _ptr(self.vweights)
        s.sources = _ptr(self.sources)
        return s

    def to_host(self):
        """(offsets, targets, weights, vweights) as int64 numpy arrays."""
        return tuple(x.cpu().numpy().astype(np.int64) for x in
                     (self.offsets, self.targets, self.weights, self.vweights))


# ---------------------------------------------------------------------------
# objective (mapping.py:38-91)

def total_cost(dg: DeviceGraph, assignment, hierarchy, distances):
    """mapping.py:76-91: exact int J for integral distances, else float J
    (float64 with the caller's distances)."""
    a = _i32(assignment, dg.device)
    t = topology_struct(hierarchy, distances)
    g = dg.struct()
    if not integral_distances(distances):
        out = torch.empty(1, dtype=torch.float64, device=dg.device)
        _lib.call("gim_total_cost_f64", C.byref(g), _ptr(a), C.byref(t), out.data_ptr(),
                  stream_ptr(dg.device))
        return float(out.item())
    out = torch.empty(1, dtype=torch.int64, device=dg.device)
    _lib.call("gim_total_cost", C.byref(g), _ptr(a), C.byref(t), out.data_ptr(),
              stream_ptr(dg.device))
    return int(out.item())


def block_weights(dg: DeviceGraph, assignment, k: int) -> torch.Tensor:
    a = _i32(assignment, dg.device)
    out = torch.empty(k, dtype=torch.int64, device=dg.device)
    g = dg.struct()
    _lib.call("gim_block_weights", C.byref(g), _ptr(a), int(k), out.data_ptr(),
              stream_ptr(dg.device))
    return out


# ---------------------------------------------------------------------------
# coarsening (coarsening.py)

def hem_round(dg: DeviceGraph, partner: torch.Tensor, l_max: float, seed: int,
              matched: int = 0):
    """coarsening.py:63-95; partner updated in place. Returns (preferred, matched)."""
    pref = torch.empty(dg.n, dtype=torch.int32, device=dg.device)
    m = C.c_int64(matched)
    g = dg.struct()
    _lib.call("gim_hem_round", C.byref(g), _ptr(partner), _ptr(pref), float(l_max),
              int(seed) & (2**64 - 1), C.byref(m), stream_ptr(dg.device))
    return pref, m.value


def match_graph(dg: DeviceGraph, l_max: float, seed: int) -> torch.Tensor:
    """coarsening.py:164-173."""
    partner = torch.empty(dg.n, dtype=torch.int32, device=dg.device)
    m = C.c_int64(0)
    g = dg.struct()
    _lib.call("gim_match_graph", C.byref(g), float(l_max), int(seed) & (2**64 - 1),
              _ptr(partner), C.byref(m), stream_ptr(dg.device))
    return partner


def coarse_map(partner: torch.Tensor):
    """coarsening.py:176-188 -> (coarse_map, n_c)."""
    n = partner.numel()
    cmap = torch.empty(n, dtype=torch.int32, device=partner.device)
    n_c = C.c_int32(0)
    _lib.call("gim_coarse_map", n, _ptr(partner), _ptr(cmap), C.byref(n_c),
              stream_ptr(partner.device))
    return cmap, n_c.value


def contract(dg: DeviceGraph, cmap: torch.Tensor, n_c: int) -> DeviceGraph:
    """coarsening.py:191-249 (rows sorted by target)."""
    dev = dg.device
    cap = max(dg.m2, 1)
    off = torch.empty(n_c + 1, dtype=torch.int32, device=dev)
    tgt = torch.empty(cap, dtype=torch.int32, device=dev)
    w = torch.empty(cap, dtype=torch.int32, device=dev)
    vw = torch.empty(max(n_c, 1), dtype=torch.int32, device=dev)
    src = torch.empty(cap, dtype=torch.int32, device=dev)
    m2 = C.c_int64(0)
    g = dg.struct()
    cm = _i32(cmap, dev)  # keep every argument tensor alive across the call
    _lib.call("gim_contract", C.byref(g), _ptr(cm), int(n_c), _ptr(off), _ptr(tgt),
              _ptr(w), _ptr(vw), _ptr(src), C.byref(m2), stream_ptr(dev))
    k = m2.value
    return DeviceGraph(off, tgt[:k].clone(), w[:k].clone(), vw[:n_c].clone(), src[:k].clone(),
                       dg.total_weight)


def project(cmap: torch.Tensor, coarse_part: torch.Tensor) -> torch.Tensor:
    """coarsening.py:269-277."""
    out = torch.empty(cmap.numel(), dtype=torch.int32, device=cmap.device)
    cp = _i32(coarse_part, cmap.device)
    _lib.call("gim_project", cmap.numel(), _ptr(cmap), _ptr(cp),
              _ptr(out), stream_ptr(cmap.device))
    return out


# ---------------------------------------------------------------------------
# refinement (refinement.py, mapping.py)

def conn_build(dg: DeviceGraph, assignment, k: int):
    """BlockConnectivity values (mapping.py:141-158) as a block-sorted CSR."""
    dev = dg.device
    cap = max(dg.m2, 1)
    off = torch.empty(dg.n + 1, dtype=torch.int32, device=dev)
    blocks = torch.empty(cap, dtype=torch.int32, device=dev)
    w = torch.empty(cap, dtype=torch.int32, device=dev)
    tot = C.c_int64(0)
    g = dg.struct()
    a = _i32(assignment, dev)
    _lib.call("gim_conn_build", C.byref(g), _ptr(a), int(k), _ptr(off),
              _ptr(blocks), _ptr(w), C.byref(tot), stream_ptr(dev))
    return off, blocks[:tot.value], w[:tot.value]


def lp_pass(dg: DeviceGraph, assignment, locked, hierarchy, distances, jet: bool = False,
            jet_c: float = 0.25):
    """label_propagation_pass (refinement.py:201-270) -> (cand, dest, to_move)."""
    dev = dg.device
    a = _i32(assignment, dev)
    lk = _u8(locked, dev) if locked is not None else None
    cand = torch.empty(dg.n, dtype=torch.uint8, device=dev)
    dest = torch.empty(dg.n, dtype=torch.int32, device=dev)
    tm = torch.empty(dg.n, dtype=torch.uint8, device=dev)
    mv = C.c_int64(0)
    t = topology_struct(hierarchy, distances)
    g = dg.struct()
    _lib.call("gim_lp_pass", C.byref(g), _ptr(a), _ptr(lk), C.byref(t), int(bool(jet)),
              float(jet_c), _ptr(cand), _ptr(dest), _ptr(tm), C.byref(mv), stream_ptr(dev))
    return cand, dest, tm


def rebalance(dg: DeviceGraph, assignment, bw, hierarchy, distances, strong: bool,
              sigma: float, l_max: float, rho: int, seed: int, pass_counter: int):
    """weak/strong_rebalance (refinement.py:312-386) -> (cand, dest, to_move, incomplete)."""
    dev = dg.device
    a = _i32(assignment, dev)
    bwt = bw.to(device=dev, dtype=torch.int64).contiguous() if isinstance(bw, torch.Tensor) \
        else torch.from_numpy(np.ascontiguousarray(bw, dtype=np.int64)).to(dev)
    cand = torch.empty(dg.n, dtype=torch.uint8, device=dev)
    dest = torch.empty(dg.n, dtype=torch.int32, device=dev)
    tm = torch.empty(dg.n, dtype=torch.uint8, device=dev)
    inc = C.c_int32(0)
    t = topology_struct(hierarchy, distances)
    g = dg.struct()
    _lib.call("gim_rebalance", C.byref(g), _ptr(a), _ptr(bwt), C.byref(t), int(bool(strong)),
              float(sigma), float(l_max), int(rho), int(seed) & (2**64 - 1), int(pass_counter),
              _ptr(cand), _ptr(dest), _ptr(tm), C.byref(inc), stream_ptr(dev))
    return cand, dest, tm, bool(inc.value)


def apply_moves(dg: DeviceGraph, assignment: torch.Tensor, bw: torch.Tensor, to_move, dest,
                hierarchy, distances) -> int:
    """apply_moves (mapping.py:252-282) in place; returns the exact J delta."""
    dev = dg.device
    dj = C.c_int64(0)
    t = topology_struct(hierarchy, distances)
    g = dg.struct()
    tm = _u8(to_move, dev)
    de = _i32(dest, dev)
    _lib.call("gim_apply_moves", C.byref(g), _ptr(assignment), _ptr(bw), _ptr(tm), _ptr(de),
              C.byref(t), C.byref(dj), stream_ptr(dev))
    return dj.value


def refine(dg: DeviceGraph, hierarchy, distances, assignment: torch.Tensor, bw: torch.Tensor, *,
           phi=0.999, i_max=12, i_w_max=2, sigma_fraction=0.005, rho=2, jet=False,
           jet_c=0.25, seed=0, l_max: float):
    """refine (Alg. 4, refinement.py:389-464); assignment/bw replaced in place by the best."""
    t = topology_struct(hierarchy, distances)
    g = dg.struct()
    _lib.call("gim_refine", C.byref(g), C.byref(t), _ptr(assignment), _ptr(bw), float(phi),
              int(i_max), int(i_w_max), float(sigma_fraction), int(rho), int(bool(jet)),
              float(jet_c), int(seed) & (2**64 - 1), float(l_max), stream_ptr(dg.device))


# ---------------------------------------------------------------------------
# initial mapping (pipelines.py)

def greedy_graph_growing(dg: DeviceGraph, k: int) -> torch.Tensor:
    out = torch.empty(max(dg.n, 1), dtype=torch.int32, device=dg.device)
    g = dg.struct()
    _lib.call("gim_greedy_graph_growing", C.byref(g), int(k), _ptr(out), stream_ptr(dg.device))
    return out[:dg.n]


def internal_partitioner(dg: DeviceGraph, k: int, eps_local: float, seed: int) -> torch.Tensor:
    out = torch.empty(max(dg.n, 1), dtype=torch.int32, device=dg.device)
    g = dg.struct()
    _lib.call("gim_internal_partitioner", C.byref(g), int(k), float(eps_local),
              int(seed) & (2**64 - 1), _ptr(out), stream_ptr(dg.device))
    return out[:dg.n]


def hierarchical_multisection(dg: DeviceGraph, hierarchy, distances, eps: float,
                              seed: int) -> torch.Tensor:
    out = torch.empty(max(dg.n, 1), dtype=torch.int32, device=dg.device)
    t = topology_struct(hierarchy, distances)
    g = dg.struct()
    _lib.call("gim_hierarchical_multisection", C.byref(g), C.byref(t), float(eps),
              int(seed) & (2**64 - 1), _ptr(out), stream_ptr(dg.device))
    return out[:dg.n]


def run_flags(fused=True, rowwise=True, batch=True, fanout=True, profile=False) -> int:
    """GIM_RUN_* bits for one call (gim_im_params.run_flags)."""
    return ((_lib.RUN_FUSED if fused else 0) | (_lib.RUN_ROWWISE if rowwise else 0) |
            (_lib.RUN_BATCH if batch else 0) | (_lib.RUN_FANOUT if fanout else 0) |
            (_lib.RUN_PROFILE if profile else 0))


def params_struct(coarsest_factor=128, phi=0.999, rho=2, filter_mode="nonneg", jet_filter_c=0.25,
                  sigma_coarse=0.065, sigma_fine=0.005, iw_max_finest=10,
                  run_flags: int = -1, isolated_vertices: str = "keep") -> _lib.GimImParams:
    p = _lib.GimImParams()
    p.coarsest_factor = int(coarsest_factor)
    p.phi = float(phi)
    p.rho = int(rho)
    p.filter_mode = 1 if filter_mode == "jet" else 0
    p.jet_filter_c = float(jet_filter_c)
    p.sigma_coarse = float(sigma_coarse)
    p.sigma_fine = float(sigma_fine)
    p.iw_max_finest = int(iw_max_finest)
    p.run_flags = int(run_flags)
    if isolated_vertices not in ("keep", "strip"):
        raise ValueError(f"isolated_vertices must be 'keep' or 'strip', got {isolated_vertices!r}")
    p.isolated = 1 if isolated_vertices == "strip" else 0
    return p


PROF_CLASSES = ("jeval", "hem", "contract", "lp_eval", "lp_second", "apply", "rebalance",
                "ggg", "extract", "two_hop")


def stats_dict(st: _lib.GimImStats) -> dict:
    per_level = ("level_n", "level_m2", "level_iters", "level_refine_ms", "level_bytes",
                 "level_barriers")
    d = {f: getattr(st, f) for f, _ in _lib.GimImStats._fields_
         if f not in per_level + ("prof_ms", "prof_bytes", "prof_count", "top_class",
                                  "top_ms", "top_bytes", "acct")}
    nl = min(st.n_levels, 64)
    for f in per_level:
        arr = getattr(st, f)
        d[f] = [arr[i] for i in range(nl)]
    d["acct"] = {name: st.acct[i] for i, name in enumerate(_lib.ACCT_NAMES)}
    prof = {}
    for i, name in enumerate(PROF_CLASSES):
        if st.prof_count[i]:
            prof[name] = {"ms": st.prof_ms[i], "bytes": st.prof_bytes[i],
                          "count": st.prof_count[i]}
    d["profile"] = prof
    d["top_launch"] = ({"class": PROF_CLASSES[st.top_class], "ms": st.top_ms,
                        "bytes": st.top_bytes} if 0 <= st.top_class < len(PROF_CLASSES) else None)
    return d


def release_cached_memory() -> None:
    """Return the library's cached device scratch to the CUDA pools and trim
    them (like torch.cuda.empty_cache for libgpuim's allocator)."""
    _lib.load().gim_release_cached_memory()


def set_profiling(on: bool) -> None:
    _lib.load().gim_set_profiling(1 if on else 0)


def integrated_map_device(dg: DeviceGraph, hierarchy, distances, eps: float, seed: int = 0,
                          **kw):
    """integrated_map on a resident graph -> (assignment int32, bw int64, stats dict)."""
    k = int(np.prod(hierarchy))
    a = torch.empty(dg.n, dtype=torch.int32, device=dg.device)
    bw = torch.empty(k, dtype=torch.int64, device=dg.device)
    st = _lib.GimImStats()
    t = topology_struct(hierarchy, distances)
    p = params_struct(**kw)
    g = dg.struct()
    _lib.call("gim_integrated_map_device", C.byref(g), C.byref(t), float(eps),
              int(seed) & (2**64 - 1), C.byref(p), _ptr(a), _ptr(bw), C.byref(st),
              stream_ptr(dg.device))
    return a, bw, stats_dict(st)


def integrated_map_host(offsets, targets, eweights, vweights, hierarchy, distances, eps: float,
                        seed: int = 0, **kw):
    """integrated_map on HOST int64 arrays through the one-call C ABI
    -> (assignment int64 np, block weights int64 np, stats dict)."""
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    tgt = np.ascontiguousarray(targets, dtype=np.int64)
    ew = np.ascontiguousarray(eweights, dtype=np.int64)
    vw = np.ascontiguousarray(vweights, dtype=np.int64)
    n = len(off) - 1
    k = int(np.prod(hierarchy))
    a = np.empty(max(n, 0), dtype=np.int64)
    bw = np.empty(k, dtype=np.int64)
    st = _lib.GimImStats()
    t = topology_struct(hierarchy, distances)
    p = params_struct(**kw)
    ptr = lambda x: x.ctypes.data if x.size else None  # noqa: E731
    _lib.call("gim_integrated_map", int(n), ptr(off), ptr(tgt), ptr(ew), ptr(vw), C.byref(t),
              float(eps), int(seed) & (2**64 - 1), C.byref(p), ptr(a), ptr(bw), C.byref(st),
              stream_ptr())
    return a, bw, stats_dict(st)


def hierarchical_multisection_host(offsets, targets, eweights, vweights, hierarchy, distances,
                                   eps: float, seed: int = 0):
    """GPU-HM on HOST int64 arrays -> (assignment int64 np, block weights int64 np)."""
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    tgt = np.ascontiguousarray(targets, dtype=np.int64)
    ew = np.ascontiguousarray(eweights, dtype=np.int64)
    vw = np.ascontiguousarray(vweights, dtype=np.int64)
    n = len(off) - 1
    k = int(np.prod(hierarchy))
    a = np.empty(max(n, 0), dtype=np.int64)
    bw = np.empty(k, dtype=np.int64)
    t = topology_struct(hierarchy, distances)
    ptr = lambda x: x.ctypes.data if x.size else None  # noqa: E731
    _lib.call("gim_hierarchical_multisection_host", int(n), ptr(off), ptr(tgt), ptr(ew), ptr(vw),
              C.byref(t), float(eps), int(seed) & (2**64 - 1), ptr(a), ptr(bw), stream_ptr())
    return a, bw


def hierarchical_multisection_plugin(offsets, targets, eweights, vweights, hierarchy, distances,
                                     eps: float, seed: int, partition_cb=None, trace_cb=None):
    """GPU-HM with the reference's plugin seam (pipelines.py:49-110): ctypes
    callbacks (_lib.PARTITION_FN / TRACE_FN, or None) called per tree node in
    depth-first order -> (assignment int64 np, block weights int64 np)."""
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    tgt = np.ascontiguousarray(targets, dtype=np.int64)
    ew = np.ascontiguousarray(eweights, dtype=np.int64)
    vw = np.ascontiguousarray(vweights, dtype=np.int64)
    n = len(off) - 1
    k = int(np.prod(hierarchy))
    a = np.empty(max(n, 0), dtype=np.int64)
    bw = np.empty(k, dtype=np.int64)
    t = topology_struct(hierarchy, distances)
    ptr = lambda x: x.ctypes.data if x.size else None  # noqa: E731
    fn = lambda cb: C.cast(cb, C.c_void_p).value if cb is not None else None  # noqa: E731
    _lib.call("gim_hierarchical_multisection_plugin", int(n), ptr(off), ptr(tgt), ptr(ew),
              ptr(vw), C.byref(t), float(eps), int(seed) & (2**64 - 1), fn(partition_cb),
              fn(trace_cb), None, ptr(a), ptr(bw), stream_ptr())
    return a, bw


def set_fanout(on: bool) -> None:
    """Sibling multisection subtrees on concurrent host threads/streams."""
    _lib.load().gim_set_fanout(1 if on else 0)


def set_fused(on: bool) -> None:
    """Device-resident Alg. 4 (one cooperative kernel per level) vs per-phase launches."""
    _lib.load().gim_set_fused(1 if on else 0)


def set_batch(on: bool) -> None:
    """Batched partitioning of the multisection's small leaf-parent subgraphs."""
    _lib.load().gim_set_batch(1 if on else 0)


def set_rowwise_contraction(on: bool) -> None:
    """Row-wise contraction of matchings vs the radix-sort path."""
    _lib.load().gim_set_rowwise_contraction(1 if on else 0)
