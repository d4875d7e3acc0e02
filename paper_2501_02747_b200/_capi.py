"""ctypes binding of include/visrt.h (the product C-ABI).

This is the ONLY way the Python layer reaches the hot path: there is no CPU
fallback. If ``libvisrt_cuda.so`` is missing or fails to load, every call
raises — on a GPU box a missing extension is an error, never a silent
downgrade.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libvisrt_cuda.so")

_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_i8p = np.ctypeslib.ndpointer(dtype=np.int8, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")

# every symbol include/visrt.h declares (checked by tests/test_capi_symbols.py)
EXPORTS = [
    "visrt_last_error", "visrt_version", "visrt_scene_create", "visrt_scene_destroy",
    "visrt_scene_nfaces", "visrt_scene_ingest", "visrt_scene_upload_bytes", "visrt_measure_peaks",
    "visrt_pair_visibility", "visrt_pair_visibility_rows", "visrt_matrix_bits_device",
    "visrt_candidates", "visrt_pair_detail", "visrt_point_regions", "visrt_point_tables", "visrt_segments_clear",
    "visrt_chain_reach", "visrt_trajectory_table", "visrt_mobile_table_rows", "visrt_mobile_table_destroy",
    "visrt_chain_triples", "visrt_tracer_create",
    "visrt_tracer_destroy", "visrt_trace", "visrt_trace_results", "visrt_image_tree", "visrt_closest_edges",
    "visrt_tracer_set_edges", "visrt_trace_snapshot_edges", "visrt_resolve_keys",
    "visrt_cache_save", "visrt_cache_load", "visrt_ray_gains", "visrt_channel_stats",
    "visrt_triples_feasible",
]

VISRT_PAIRS_ALL = 0x1
VISRT_PAIRS_PREFILTERED = 0x2


class visrt_facets_v1(C.Structure):
    _fields_ = [("nfaces", C.c_int32), ("vert_off", C.c_void_p), ("verts", C.c_void_p),
                ("building", C.c_void_p)]


class visrt_stats(C.Structure):
    _fields_ = [("pairs", C.c_int64), ("candidates", C.c_int64), ("admitted", C.c_int64),
                ("tests_alg", C.c_double), ("tests_exec", C.c_int64), ("ms", C.c_float),
                ("sweeps", C.c_int64), ("tiles", C.c_int64)]


class visrt_region(C.Structure):
    _fields_ = [("present", C.c_int8), ("has", C.c_int8 * 3), ("clipped", C.c_int8 * 3),
                ("pad", C.c_int8), ("sub", C.c_double * 6)]


class visrt_names(C.Structure):
    _fields_ = [("key_rank", C.c_void_p), ("parent_rank", C.c_void_p), ("building_rank", C.c_void_p)]


class visrt_path(C.Structure):
    _fields_ = [("nrefl", C.c_int32), ("faces", C.c_int32 * 4), ("edge", C.c_int32), ("snap", C.c_int32),
                ("pad", C.c_int32), ("points", C.c_double * 21), ("length", C.c_double)]


class visrt_seqkey(C.Structure):
    _fields_ = [("nrefl", C.c_int32), ("faces", C.c_int32 * 4), ("edge", C.c_int32)]


class visrt_em_config(C.Structure):
    _fields_ = [("frequency", C.c_double), ("tx_gain_dbi", C.c_double), ("rx_gain_dbi", C.c_double),
                ("polarization", C.c_int32), ("pad", C.c_int32)]


class visrt_trace_stats(C.Structure):
    _fields_ = [("nodes", C.c_int64), ("sequences", C.c_int64), ("paths", C.c_int64),
                ("leg_tests", C.c_int64), ("ms", C.c_float)]


class VisrtError(RuntimeError):
    code = 0


class VisibilityError(VisrtError):
    code = 1


class PlacementError(VisrtError):
    code = 2


class SceneError(VisrtError):
    code = 3


class CudaError(VisrtError):
    code = 4


class UsageError(VisrtError):
    code = 5


_ERR = {1: VisibilityError, 2: PlacementError, 3: SceneError, 4: CudaError, 5: UsageError}
_lib = None


def lib():
    """Load the product library (raises when it is absent — no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                          "(nvcc -gencode arch=compute_100a,code=sm_100a); there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    L.visrt_last_error.restype = C.c_char_p
    L.visrt_version.restype = C.c_int
    L.visrt_scene_create.argtypes = [C.POINTER(visrt_facets_v1), C.c_int, C.POINTER(C.c_void_p)]
    L.visrt_scene_destroy.argtypes = [C.c_void_p]
    L.visrt_scene_nfaces.argtypes = [C.c_void_p]
    L.visrt_scene_ingest.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    L.visrt_scene_upload_bytes.restype = C.c_int64
    L.visrt_scene_upload_bytes.argtypes = [C.c_void_p]
    L.visrt_measure_peaks.argtypes = [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.visrt_pair_visibility.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.POINTER(visrt_stats),
                                        C.c_void_p]
    L.visrt_pair_visibility_rows.argtypes = [C.c_void_p, C.c_uint32, C.c_int32, C.c_int32, C.c_void_p,
                                             C.POINTER(visrt_stats), C.c_void_p]
    L.visrt_matrix_bits_device.restype = C.c_void_p
    L.visrt_matrix_bits_device.argtypes = [C.c_void_p]
    L.visrt_candidates.restype = C.c_int64
    L.visrt_candidates.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    L.visrt_pair_detail.argtypes = [C.c_void_p, C.c_int64, _i32p, _i32p, _i8p, _i64p, C.c_void_p,
                                    C.c_int64, C.POINTER(visrt_stats), C.c_void_p]
    L.visrt_point_regions.argtypes = [C.c_void_p, C.c_int64, _f64p, C.POINTER(visrt_region),
                                      C.POINTER(visrt_stats), C.c_void_p]
    L.visrt_point_tables.argtypes = [C.c_void_p, C.c_int64, _f64p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.POINTER(visrt_stats), C.c_void_p]
    L.visrt_segments_clear.argtypes = [C.c_void_p, C.c_int64, _f64p, _f64p, C.c_void_p, C.POINTER(visrt_stats),
                                       C.c_void_p]
    L.visrt_chain_reach.argtypes = [C.c_void_p, C.c_int64, _f64p, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.POINTER(visrt_stats), C.c_void_p]
    L.visrt_trajectory_table.argtypes = [C.c_void_p, C.c_int32, _f64p, C.c_int64, C.c_void_p, C.c_int32,
                                         C.POINTER(visrt_names), C.POINTER(C.c_void_p), C.POINTER(visrt_stats),
                                         C.c_void_p]
    L.visrt_mobile_table_rows.restype = C.c_int64
    L.visrt_mobile_table_rows.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
    L.visrt_mobile_table_destroy.argtypes = [C.c_void_p]
    L.visrt_chain_triples.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_int64),
                                      C.POINTER(visrt_stats), C.c_void_p]
    L.visrt_tracer_create.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_void_p,
                                      C.POINTER(C.c_void_p)]
    L.visrt_tracer_destroy.argtypes = [C.c_void_p]
    L.visrt_trace.argtypes = [C.c_void_p, C.c_int64, _f64p, _f64p, C.c_int, C.POINTER(visrt_trace_stats),
                              C.c_void_p]
    L.visrt_image_tree.argtypes = [C.c_void_p, _f64p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_int64, C.POINTER(C.c_int64), C.POINTER(visrt_stats), C.c_void_p]
    L.visrt_closest_edges.argtypes = [C.c_void_p, C.c_int64, _f64p, C.c_int32, C.c_void_p, C.c_void_p, _i32p,
                                      C.POINTER(visrt_stats), C.c_void_p]
    L.visrt_resolve_keys.argtypes = [C.c_void_p, C.c_int64, _f64p, _f64p, C.c_int, C.c_void_p, C.c_void_p,
                                     C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(visrt_stats),
                                     C.c_void_p]
    L.visrt_ray_gains.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, _f64p, C.c_int32, C.c_void_p, C.c_void_p,
                                  C.POINTER(visrt_em_config), C.c_void_p, C.c_void_p, C.POINTER(visrt_stats),
                                  C.c_void_p]
    L.visrt_channel_stats.argtypes = [C.c_void_p, C.c_int64, _i64p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p]
    L.visrt_triples_feasible.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
    L.visrt_cache_save.argtypes = [C.c_char_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int64, C.c_void_p]
    L.visrt_cache_load.argtypes = [C.c_char_p, C.c_void_p, C.POINTER(C.c_int32), C.c_void_p, C.c_void_p, C.c_int64,
                                   C.POINTER(C.c_int64)]
    L.visrt_trace_snapshot_edges.restype = C.c_int64
    L.visrt_trace_snapshot_edges.argtypes = [C.c_void_p, C.c_void_p]
    L.visrt_tracer_set_edges.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]
    L.visrt_trace_results.restype = C.c_int64
    L.visrt_trace_results.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
    _lib = L
    return L


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().visrt_last_error().decode()
        raise _ERR.get(rc, VisrtError)(msg)


def last_error() -> str:
    return lib().visrt_last_error().decode()
