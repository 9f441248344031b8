"""Device-resident CSR levels (torch tensors as plumbing, int32 layout).

`DeviceGraph.from_host` performs the one host->device upload of the
reference `Graph` arrays (graph.py:17-39, int64) with the overflow checks
the int32 device layout needs.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib

INT32_MAX = 2**31 - 1


def _ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    return t.data_ptr() if t.numel() else None


class DeviceGraph:
    """One CSR level on the GPU: offsets/targets/weights/vweights/sources."""

    def __init__(self, offsets, targets, weights, vweights, sources, total_weight: int):
        self.offsets = offsets
        self.targets = targets
        self.weights = weights
        self.vweights = vweights
        self.sources = sources
        self.total_weight = int(total_weight)

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
    def check_host(offsets: np.ndarray, targets: np.ndarray, eweights: np.ndarray,
                   vweights: np.ndarray) -> int:
        n = len(offsets) - 1
        if n < 0:
            raise ValueError("offsets must have n+1 entries")
        if len(targets) > INT32_MAX or n > INT32_MAX:
            raise OverflowError("graph too large for the int32 device layout")
        total_vw = int(vweights.sum(dtype=np.int64)) if n else 0
        if total_vw > INT32_MAX:
            raise OverflowError("total vertex weight must be < 2^31")
        if len(eweights) and int(eweights.sum(dtype=np.int64)) > INT32_MAX:
            raise OverflowError("total edge weight must be < 2^31")
        return total_vw

    @classmethod
    def from_host(cls, g, device="cuda") -> "DeviceGraph":
        """Upload a reference-style Graph (attributes offsets, edge_targets,
        edge_weights, vertex_weights, optional edge_sources)."""
        off = np.ascontiguousarray(g.offsets, dtype=np.int64)
        tgt = np.ascontiguousarray(g.edge_targets, dtype=np.int64)
        ew = np.ascontiguousarray(g.edge_weights, dtype=np.int64)
        vw = np.ascontiguousarray(g.vertex_weights, dtype=np.int64)
        total = cls.check_host(off, tgt, ew, vw)
        dev = torch.device(device)
        t_off = torch.from_numpy(off).to(dev, non_blocking=False).to(torch.int32)
        t_tgt = torch.from_numpy(tgt).to(dev).to(torch.int32)
        t_w = torch.from_numpy(ew).to(dev).to(torch.int32)
        t_vw = torch.from_numpy(vw).to(dev).to(torch.int32)
        n = len(off) - 1
        deg = t_off[1:] - t_off[:-1]
        t_src = torch.repeat_interleave(torch.arange(n, device=dev, dtype=torch.int32),
                                        deg.to(torch.int64), output_size=len(tgt))
        return cls(t_off, t_tgt, t_w, t_vw, t_src, total)

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


def stream_ptr(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def total_cost(dg: DeviceGraph, assignment: torch.Tensor, hierarchy, distances) -> int:
    """J(C, D, Pi) on the device (mapping.py:76-91), exact int64."""
    a = assignment.to(device=dg.device, dtype=torch.int32).contiguous()
    out = torch.empty(1, dtype=torch.int64, device=dg.device)
    t = _lib.topology_struct(hierarchy, distances)
    g = dg.struct()
    _lib.call("gim_total_cost", C.byref(g), _ptr(a), C.byref(t), out.data_ptr(),
              stream_ptr(dg.device))
    return int(out.item())


def block_weights(dg: DeviceGraph, assignment: torch.Tensor, k: int) -> torch.Tensor:
    a = assignment.to(device=dg.device, dtype=torch.int32).contiguous()
    out = torch.empty(k, dtype=torch.int64, device=dg.device)
    g = dg.struct()
    _lib.call("gim_block_weights", C.byref(g), _ptr(a), int(k), out.data_ptr(),
              stream_ptr(dg.device))
    return out
