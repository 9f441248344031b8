"""Native METIS reader: drop-in for `promap.graph.load_metis`
(graph.py:185-294).  Parsing and validation run in libgpuim.so (C++, mmap,
worker threads); the result is the reference's `Graph` (its own type when
`promap` is importable) with the same CSR, and malformed files raise
`MetisFormatError` (a `ValueError`) with the reference's message."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib


def _error_type():
    try:
        from promap.graph import MetisFormatError as Ref  # the reference's class
        return Ref
    except Exception:  # noqa: BLE001
        return MetisFormatError


class MetisFormatError(ValueError):
    """Mirror of promap.graph.MetisFormatError (graph.py:170-171)."""


def load_metis(path: str):
    lib = _lib.load()
    h = C.c_void_p()
    n = C.c_int64()
    m2 = C.c_int64()
    rc = lib.gim_metis_load(str(path).encode(), C.byref(h), C.byref(n), C.byref(m2))
    if rc == _lib.GIM_E_FORMAT:
        raise _error_type()(lib.gim_last_error().decode())
    if rc == _lib.GIM_E_IO:
        raise FileNotFoundError(lib.gim_last_error().decode())
    _lib.check(rc)
    n, m2 = n.value, m2.value
    off = np.empty(n + 1, np.int64)
    tgt = np.empty(m2, np.int64)
    ew = np.empty(m2, np.int64)
    vw = np.empty(n, np.int64)
    src = np.empty(m2, np.int64)
    ptr = lambda x: x.ctypes.data if x.size else None  # noqa: E731
    _lib.check(lib.gim_metis_fetch(h, ptr(off), ptr(tgt), ptr(ew), ptr(vw), ptr(src)))
    try:
        from promap.graph import Graph  # reference type when present
        return Graph(off, tgt, ew, vw, src)
    except Exception:  # noqa: BLE001
        from .generators import HostGraph
        return HostGraph(off, tgt, ew, vw, src)


def load_metis_device(path: str, device="cuda"):
    """A METIS file straight to a device-resident CSR (`device.DeviceGraph`):
    parsed natively (same rules and `MetisFormatError` messages as
    `load_metis`), narrowed to int32 and uploaded by the library's
    multi-threaded upload path — no int64 host Graph in between."""
    import torch

    from . import device as D
    lib = _lib.load()
    h = C.c_void_p()
    n = C.c_int64()
    m2 = C.c_int64()
    rc = lib.gim_metis_load(str(path).encode(), C.byref(h), C.byref(n), C.byref(m2))
    if rc == _lib.GIM_E_FORMAT:
        raise _error_type()(lib.gim_last_error().decode())
    if rc == _lib.GIM_E_IO:
        raise FileNotFoundError(lib.gim_last_error().decode())
    _lib.check(rc)
    n, m2 = n.value, m2.value
    dev = torch.device(device)
    i32 = dict(dtype=torch.int32, device=dev)
    off = torch.empty(n + 1, **i32)
    tgt = torch.empty(max(m2, 1), **i32)
    w = torch.empty(max(m2, 1), **i32)
    vw = torch.empty(max(n, 1), **i32)
    src = torch.empty(max(m2, 1), **i32)
    tot = C.c_int64(0)
    _lib.call("gim_metis_upload", h, off.data_ptr(), tgt.data_ptr(), w.data_ptr(), vw.data_ptr(),
              src.data_ptr(), C.byref(tot), D.stream_ptr(dev))
    return D.DeviceGraph(off, tgt[:m2], w[:m2], vw[:n], src[:m2], tot.value)
