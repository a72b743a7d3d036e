"""ctypes binding of the engine's C ABI (include/geosink_b200.h -> lib/libgeosink_b200.so).

The product path: there is no fallback. If the shared library is missing or no CUDA device is
visible, every entry point raises instead of computing anything on the CPU.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libgeosink_b200.so")

GS_OK = 0
GS_ERR_CUDA = 100
GS_ERR_NCCL = 101
GS_ERR_UNSUPPORTED = 102
GS_MEM_HOST = 0
GS_MEM_DEVICE = 1
GS_FLAG_SINGLE = 1
GS_FLAG_NO_STAGNATION_ABORT = 2
GS_FLAG_FP32 = 4

# (name, restype, argtypes) for every symbol declared in include/geosink_b200.h
_vp = C.c_void_p
_i = C.c_int
_i64 = C.c_int64
_d = C.c_double
_pi = C.POINTER(C.c_int)
_pi64 = C.POINTER(C.c_int64)
_pd = C.POINTER(C.c_double)
_pvp = C.POINTER(C.c_void_p)

ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_void_p)
ALLTOALLV_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64), C.c_void_p,
                           C.POINTER(C.c_int64), C.c_int, C.c_void_p)


GS_COMM_GRAPH_SAFE = 1
GS_NCCL_UNIQUE_ID_BYTES = 128


class GsComm(C.Structure):
    _fields_ = [("allreduce", ALLREDUCE_FN), ("user", C.c_void_p), ("alltoallv", ALLTOALLV_FN),
                ("flags", C.c_int)]


SIGNATURES = {
    "gs_nccl_unique_id": (_i, [_vp]),
    "gs_nccl_comm_create": (_i, [_vp, _vp, _i, _i, _pvp]),
    "gs_nccl_comm_destroy": (None, [_vp]),
    "gs_nccl_comm_calls": (_i64, [_vp]),
    "gs_win_bisect_order_host": (_i, [_i, _vp, _vp, _i, _vp]),
    "gs_win_plan_host": (_i, [_i, _vp, _vp, _i, _i, _pvp, _vp]),
    "gs_win_plan_arrays": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "gs_win_plan_destroy": (None, [_vp]),
    "gs_ctx_create": (_i, [_i, _pvp]),
    "gs_ctx_destroy": (None, [_vp]),
    "gs_last_error": (C.c_char_p, [_vp]),
    "gs_ctx_synchronize": (_i, [_vp]),
    "gs_ctx_set_stream": (_i, [_vp, _vp]),
    "gs_ctx_stream": (_vp, [_vp]),
    "gs_ctx_set_timing": (_i, [_vp, _i]),
    "gs_ctx_timing": (_i, [_vp, _i, _pi64, _pd]),
    "gs_ctx_launch_count": (_i64, [_vp]),
    "gs_ctx_knn_fallback": (_i64, [_vp]),
    "gs_graph_from_triplets": (_i, [_vp, _i, _i64, _vp, _vp, _vp, _i, _pvp]),
    "gs_graph_from_csr": (_i, [_vp, _i, _i64, _vp, _vp, _vp, _i, _pvp]),
    "gs_graph_destroy": (None, [_vp]),
    "gs_graph_info": (_i, [_vp, _pi, _pi64]),
    "gs_graph_download": (_i, [_vp, _vp, _vp, _vp, _vp, _i]),
    "gs_graph_multiply": (_i, [_vp, _vp, _vp, _vp, _i, _i]),
    "gs_graph_gershgorin": (_i, [_vp, _vp, _pd]),
    "gs_knn": (_i, [_vp, _vp, _i, _i, _i, _i, _vp, _vp]),
    "gs_knn_graph": (_i, [_vp, _vp, _i, _i, _i, _i, _d, _i, _pvp, _pd]),
    "gs_laplacian": (_i, [_vp, _vp, _i, _pvp, _pd, _pi]),
    "gs_lambda_max": (_i, [_vp, _vp, _pd, _pi]),
    "gs_heat_coefficients": (_i, [_vp, _d, _i, _vp]),
    "gs_filter_create": (_i, [_vp, _vp, _i, _d, _d, _i, _pvp]),
    "gs_filter_destroy": (None, [_vp]),
    "gs_filter_info": (_i, [_vp, _pi, _pd, _pd, _pd, _pi, _pi]),
    "gs_filter_coefficients": (_i, [_vp, _vp]),
    "gs_filter_scaled": (_vp, [_vp]),
    "gs_filter_order": (_i, [_vp, _vp, _vp, _i]),
    "gs_filter_set_order": (_i, [_vp, _vp, _i, _vp, _i]),
    "gs_dense_sinkhorn": (_i, [_vp, _vp, _i, _i, _vp, _vp, _d, _i, _d, _i, _vp, _vp, _vp, _vp,
                               _vp, _vp, _vp]),
    "gs_dense_sinkhorn_groups": (_i, [_vp, _vp, _i, _i, _vp, _vp, _i, _vp, _vp, _i, _i, _d, _i,
                                      _d, _vp, _vp, _vp, _vp, _vp, _pi]),
    "gs_filter_apply": (_i, [_vp, _vp, _vp, _vp, _i, _i]),
    "gs_filter_apply_ex": (_i, [_vp, _vp, _vp, _vp, _i, _i, _i]),
    "gs_sinkhorn": (_i, [_vp, _vp, _vp, _vp, _vp, _i, _i, _d, _i, _i, _vp, _vp, _vp, _vp, _vp,
                         _vp, _vp, _pi, _pi]),
    "gs_barycenter": (_i, [_vp, _vp, _vp, _vp, _i, _vp, _i, _d, _i, _vp, _vp, _vp, _vp, _vp,
                           _vp, _vp]),
    "gs_barycenter_ex": (_i, [_vp, _vp, _vp, _vp, _i, _vp, _i, _d, _i, _vp, _i, _vp, _vp, _vp,
                              _vp, _vp, _vp]),
    "gs_plan_rows": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _vp]),
    "gs_graph_save": (_i, [_vp, _vp, C.c_char_p]),
    "gs_graph_load": (_i, [_vp, C.c_char_p, _pvp]),
    "gs_part_create": (_i, [_vp, _vp, _i, _i, _pvp]),
    "gs_part_destroy": (None, [_vp]),
    "gs_part_info": (_i, [_vp, _pi, _pi, _pi, _pi64, _pi]),
    "gs_part_counts": (_i, [_vp, _vp, _vp]),
    "gs_part_interior": (_i, [_vp, _pi, _pi]),
    "gs_part_vertices": (_i, [_vp, _vp, _vp, _i]),
    "gs_part_filter_apply": (_i, [_vp, _vp, _vp, _vp, _vp, _i, _i, _i]),
    "gs_part_sinkhorn": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _d, _i, _i, _vp, _vp, _vp,
                              _vp, _vp, _vp, _vp, _pi, _pi]),
    "gs_euler_create": (_i, [_vp, _vp, _d, _i, _pvp]),
    "gs_euler_create_ex": (_i, [_vp, _vp, _d, _i, _i, _pvp]),
    "gs_euler_destroy": (None, [_vp]),
    "gs_euler_system": (_vp, [_vp]),
    "gs_euler_apply": (_i, [_vp, _vp, _vp, _vp, _i, _i, _pi]),
    "gs_euler_sinkhorn": (_i, [_vp, _vp, _vp, _vp, _vp, _i, _i, _d, _i, _i, _vp, _vp, _vp, _vp,
                               _vp, _vp, _vp, _pi, _pi]),
    "gs_rng_create": (_vp, [C.c_uint64]),
    "gs_rng_destroy": (None, [_vp]),
    "gs_rng_bits": (C.c_uint64, [_vp]),
    "gs_rng_uniform": (_d, [_vp]),
    "gs_rng_uniform_range": (_d, [_vp, _d, _d]),
    "gs_rng_normal": (_d, [_vp]),
    "gs_rng_below": (C.c_uint64, [_vp, C.c_uint64]),
    "gs_rng_seed_mix": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "gs_rng_fill_pattern": (None, [_vp, _vp, _i64, _vp, _vp, _vp, _i]),
}

_LIB = None


class EngineUnavailable(RuntimeError):
    """The CUDA engine cannot run here (library missing or no device). Never falls back."""


def load(path: str | None = None):
    """Load the shared library (no device needed) and declare every exported symbol."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = path or os.environ.get("GS_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise EngineUnavailable(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib
