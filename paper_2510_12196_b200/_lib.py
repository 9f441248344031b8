"""ctypes binding of libgpuim.so (include/gpuim.h).

The product path has no CPU fallback: if the shared library is missing or a
call fails, this module raises.  Build with `python -m paper_2510_12196_b200.build`.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / os.environ.get("GIM_LIB_NAME", "libgpuim.so")
MAX_LEVELS = 32

GIM_OK = 0
GIM_E_INVALID = 1
GIM_E_CUDA = 2
GIM_E_UNSUPPORTED = 3
GIM_E_OVERFLOW = 4
GIM_E_INTERNAL = 5
GIM_E_EMPTY = 6
GIM_E_FORMAT = 7
GIM_E_IO = 8
GIM_E_CALLBACK = 9


class GimGraph(C.Structure):
    _fields_ = [
        ("n", C.c_int32),
        ("m2", C.c_int64),
        ("offsets", C.c_void_p),
        ("targets", C.c_void_p),
        ("weights", C.c_void_p),
        ("vweights", C.c_void_p),
        ("sources", C.c_void_p),
    ]


class GimTopology(C.Structure):
    _fields_ = [
        ("levels", C.c_int32),
        ("hierarchy", C.c_int64 * MAX_LEVELS),
        ("distances", C.c_double * MAX_LEVELS),
    ]


class GimImParams(C.Structure):
    _fields_ = [
        ("coarsest_factor", C.c_int64),
        ("phi", C.c_double),
        ("rho", C.c_int32),
        ("filter_mode", C.c_int32),
        ("jet_filter_c", C.c_double),
        ("sigma_coarse", C.c_double),
        ("sigma_fine", C.c_double),
        ("iw_max_finest", C.c_int32),
        ("run_flags", C.c_int32),
        ("isolated", C.c_int32),
    ]


RUN_DEFAULT = -1
RUN_FUSED, RUN_ROWWISE, RUN_BATCH, RUN_FANOUT, RUN_PROFILE = 1, 2, 4, 8, 16
ACCT_NAMES = ("scan", "bnd", "eval_v", "eval_slots", "eval_S", "cand_v", "cand_slots",
              "mov_v", "mov_slots", "ovl_v", "ovl_slots", "ovl_S", "lp_it", "weak_it",
              "barriers", "sweeps")


class GimImStats(C.Structure):
    _fields_ = [
        ("n_levels", C.c_int32),
        ("level_n", C.c_int64 * 64),
        ("level_m2", C.c_int64 * 64),
        ("refine_iterations", C.c_int64),
        ("lp_passes", C.c_int64),
        ("weak_passes", C.c_int64),
        ("strong_passes", C.c_int64),
        ("init_refine_iterations", C.c_int64),
        ("partitioner_calls", C.c_int64),
        ("kernel_launches", C.c_int64),
        ("final_j", C.c_int64),
        ("max_block_weight", C.c_int64),
        ("l_max", C.c_double),
        ("ms_coarsen", C.c_double),
        ("ms_initial", C.c_double),
        ("ms_refine", C.c_double),
        ("ms_total", C.c_double),
        ("prof_ms", C.c_double * 16),
        ("prof_bytes", C.c_double * 16),
        ("prof_count", C.c_int64 * 16),
        ("top_class", C.c_int32),
        ("top_ms", C.c_double),
        ("top_bytes", C.c_double),
        ("ms_upload", C.c_double),
        ("ms_download", C.c_double),
        ("bytes_h2d", C.c_int64),
        ("bytes_d2h", C.c_int64),
        ("level_iters", C.c_int64 * 64),
        ("level_refine_ms", C.c_double * 64),
        ("level_bytes", C.c_double * 64),
        ("level_barriers", C.c_int64 * 64),
        ("acct", C.c_int64 * 16),
        ("dist_shift", C.c_int32),
        ("dist_exact", C.c_int32),
        ("final_j_f64", C.c_double),
        ("isolated_vertices", C.c_int64),
    ]


P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
U64 = C.c_uint64
DBL = C.c_double
GP = C.POINTER(GimGraph)
TP = C.POINTER(GimTopology)

# name -> argtypes; every symbol declared in include/gpuim.h appears here
PI32 = C.POINTER(C.c_int32)
PI64 = C.POINTER(C.c_int64)
PARP = C.POINTER(GimImParams)
PSTP = C.POINTER(GimImStats)

SIGNATURES: dict[str, list] = {
    "gim_version": [],
    "gim_last_error": [],
    "gim_total_cost": [GP, P, TP, P, P],
    "gim_total_cost_f64": [GP, P, TP, P, P],
    "gim_topology_scale": [TP, PI32, PI32],
    "gim_block_weights": [GP, P, I32, P, P],
    "gim_hem_round": [GP, P, P, DBL, U64, PI64, P],
    "gim_match_graph": [GP, DBL, U64, P, PI64, P],
    "gim_coarse_map": [I32, P, P, PI32, P],
    "gim_contract": [GP, P, I32, P, P, P, P, P, PI64, P],
    "gim_project": [I32, P, P, P, P],
    "gim_conn_build": [GP, P, I32, P, P, P, PI64, P],
    "gim_lp_pass": [GP, P, P, TP, I32, DBL, P, P, P, PI64, P],
    "gim_rebalance": [GP, P, P, TP, I32, DBL, DBL, I32, U64, I64, P, P, P, PI32, P],
    "gim_apply_moves": [GP, P, P, P, P, TP, PI64, P],
    "gim_refine": [GP, TP, P, P, DBL, I32, I32, DBL, I32, I32, DBL, U64, DBL, P],
    "gim_greedy_graph_growing": [GP, I32, P, P],
    "gim_internal_partitioner": [GP, I32, DBL, U64, P, P],
    "gim_hierarchical_multisection": [GP, TP, DBL, U64, P, P],
    "gim_hierarchical_multisection_host": [I64, P, P, P, P, TP, DBL, U64, P, P, P],
    "gim_default_params": [PARP],
    "gim_metis_upload": [P, P, P, P, P, P, PI64, P],
    "gim_hierarchical_multisection_plugin": [I64, P, P, P, P, TP, DBL, U64, P, P, P, P, P, P],
    "gim_integrated_map_device": [GP, TP, DBL, U64, PARP, P, P, PSTP, P],
    "gim_integrated_map": [I64, P, P, P, P, TP, DBL, U64, PARP, P, P, PSTP, P],
    "gim_fill_sources": [I32, P, P, P],
    "gim_set_profiling": [I32],
    "gim_set_fanout": [I32],
    "gim_set_fused": [I32],
    "gim_set_batch": [I32],
    "gim_set_rowwise_contraction": [I32],
    "gim_launch_count": [],
    "gim_reset_launch_count": [],
    "gim_release_cached_memory": [],
    "gim_metis_load": [C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(C.c_int64),
                       C.POINTER(C.c_int64)],
    "gim_metis_fetch": [C.c_void_p, P, P, P, P, P],
}
RESTYPES = {"gim_last_error": C.c_char_p, "gim_launch_count": C.c_int64,
            "gim_reset_launch_count": None, "gim_set_profiling": None,
            "gim_release_cached_memory": None,
            "gim_set_fanout": None, "gim_set_fused": None, "gim_set_batch": None,
            "gim_set_rowwise_contraction": None}

_lib = None


# plugin-seam callbacks (include/gpuim.h gim_partition_fn / gim_trace_fn)
PARTITION_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.POINTER(C.c_int64),
                           C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                           C.c_int32, C.c_double, C.c_uint64, C.POINTER(C.c_int32), C.c_int32,
                           C.POINTER(C.c_int64))
TRACE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int32, C.POINTER(C.c_int32), C.c_int32, C.c_int32,
                       C.c_double, C.c_int64, C.POINTER(C.c_int64), C.c_int32)


class GimError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"libgpuim error {status}: {msg}")
        self.status = status


def load():
    """Load libgpuim.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2510_12196_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH), mode=os.RTLD_LOCAL if hasattr(os, "RTLD_LOCAL") else 0)
    for name, argtypes in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = RESTYPES.get(name, C.c_int)
    _lib = lib
    return lib


def check(status: int) -> None:
    if status != GIM_OK:
        msg = load().gim_last_error()
        msg = msg.decode() if msg else ""
        if status == GIM_E_EMPTY:
            raise ValueError(msg)
        raise GimError(status, msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def topology_struct(hierarchy, distances) -> GimTopology:
    if len(hierarchy) > MAX_LEVELS:
        raise ValueError(f"at most {MAX_LEVELS} hierarchy levels are supported")
    t = GimTopology()
    t.levels = len(hierarchy)
    for i, (a, d) in enumerate(zip(hierarchy, distances)):
        t.hierarchy[i] = int(a)
        t.distances[i] = float(d)
        if int(d) == d and abs(d) >= 2**53:
            raise OverflowError("integral distances must be < 2^53")
    return t
