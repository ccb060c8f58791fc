"""ctypes declarations of the C ABI in include/coopcg_gpu.h.

This is the binding a maintainer of a Python caller would write (the same
shape as INTEGRATION.md's cgo/ctypes stubs).  The library must exist: there is
no CPU fallback anywhere in the product path -- a missing or unloadable .so
raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

from . import build as _build

# COOPCG_LIB_PATH: an alternative build of the same library (A/B timing of
# build-time variants, tools/variants.sh); the default is the in-tree build.
LIB_PATH = os.environ.get("COOPCG_LIB_PATH") or _build.LIB


class coopcg_opts(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iters", C.c_int),
                ("recompute_residual_every", C.c_int), ("rank_rel_tol", C.c_double), ("algo", C.c_int)]


class coopcg_trace(C.Structure):
    _fields_ = [("capacity", C.c_int),
                ("residual_norms", C.POINTER(C.c_double)),
                ("minres", C.POINTER(C.c_double)),
                ("wall_ns", C.POINTER(C.c_uint64)),
                ("initial_residual_norms", C.POINTER(C.c_double)),
                ("final_x", C.POINTER(C.c_double)),
                ("final_residual_norms", C.POINTER(C.c_double)),
                ("status", C.c_int), ("converged_agent", C.c_int), ("iterations", C.c_int),
                ("initial_minres", C.c_double), ("final_minres", C.c_double),
                ("loop_wall_ns", C.c_uint64), ("exact_rank_checks", C.c_int),
                ("active_agents", C.POINTER(C.c_int)), ("n_active", C.c_int)]


class coopcg_timing(C.Structure):
    _fields_ = [("matvec_launches", C.c_int), ("matvec_ms_total", C.c_double),
                ("run_ms", C.c_double), ("loop_ms", C.c_double),
                ("kernel_launches", C.c_longlong), ("a_l2_resident_bytes", C.c_double)]


# Every symbol include/coopcg_gpu.h declares: (name, restype, argtypes).
_VP = C.c_void_p
_I = C.c_int
SIGNATURES = [
    ("coopcg_gpu_version", C.c_char_p, []),
    ("coopcg_gpu_create", _I, [_I, _I, _I, _I, C.POINTER(_VP)]),
    ("coopcg_gpu_create_shard", _I, [_I, _I, _I, _I, _I, _I, C.POINTER(_VP)]),
    ("coopcg_gpu_destroy", _I, [_VP]),
    ("coopcg_gpu_last_error", _I, [_VP, C.c_char_p, C.c_size_t]),
    ("coopcg_gpu_set_A", _I, [_VP, _VP]),
    ("coopcg_gpu_gen_A", _I, [_VP, _I, C.c_uint64, _I, C.c_double]),
    ("coopcg_gpu_get_A", _I, [_VP, _VP]),
    ("coopcg_gpu_get_A_rows", _I, [_VP, _I, _I, _VP]),
    ("coopcg_gpu_gen_householder_begin", _I, [_VP, C.c_uint64, _I, C.c_double]),
    ("coopcg_gpu_gen_householder_local", _I, [_VP, _I]),
    ("coopcg_gpu_gen_householder_rest", _I, [_VP, _I]),
    ("coopcg_gpu_gen_householder_end", _I, [_VP]),
    ("coopcg_gen_rhs", _I, [_I, _I, C.c_uint64, _VP]),
    ("coopcg_gen_starts", _I, [_I, _I, C.c_uint64, _VP]),
    ("coopcg_gen_householder_factors", _I, [_I, _I, C.c_double, C.c_uint64, _VP, _VP]),
    ("coopcg_gen_random_spd_spectrum", _I, [_I, C.c_double, C.c_uint64, _VP]),
    ("coopcg_gen_reference_rhs_starts", _I, [_I, _I, C.c_uint64, _VP, _VP]),
    ("coopcg_gpu_upload", _I, [_VP, _VP, _VP]),
    ("coopcg_gpu_run", _I, [_VP, C.POINTER(coopcg_opts), C.POINTER(coopcg_trace)]),
    ("coopcg_gpu_solve", _I, [_VP, _VP, _VP, C.POINTER(coopcg_opts), C.POINTER(coopcg_trace)]),
    ("coopcg_gpu_set_verification", _I, [_VP, _I, _VP]),
    ("coopcg_gpu_history_count", _I, [_VP, C.POINTER(C.c_int)]),
    ("coopcg_gpu_get_history", _I, [_VP, _I, _VP, _VP, _VP]),
    ("coopcg_gpu_get_anorm_errors", _I, [_VP, _I, _VP]),
    ("coopcg_gpu_timing", _I, [_VP, C.POINTER(coopcg_timing)]),
    ("coopcg_gpu_stream", _VP, [_VP]),
    ("coopcg_gpu_matvec_block", _I, [_VP, _VP, _VP]),
    ("coopcg_gpu_numerical_rank", _I, [_VP, _VP, C.c_double, C.POINTER(_I)]),
    ("coopcg_gpu_numerical_rank_ex", _I, [_VP, _VP, C.c_double, _I, C.POINTER(_I)]),
    ("coopcg_gpu_begin", _I, [_VP, C.POINTER(coopcg_opts)]),
    ("coopcg_gpu_phase", _I, [_VP, _I, _I]),
    ("coopcg_gpu_recompute_at", _I, [_VP, _I]),
    ("coopcg_gpu_block", _I, [_VP, _I, _I, C.POINTER(_VP), C.POINTER(_I)]),
    ("coopcg_gpu_state", _I, [_VP, C.POINTER(_I), C.POINTER(_I)]),
    ("coopcg_gpu_mccg_resume", _I, [_VP, C.POINTER(_I)]),
    ("coopcg_gpu_end", _I, [_VP, C.POINTER(coopcg_trace)]),
    ("coopcg_gpu_ipc_handles", _I, [_VP, _VP]),
    ("coopcg_gpu_set_peers", _I, [_VP, _I, _I, _VP]),
    ("coopcg_row_split", _I, [_I, _I, _I, C.POINTER(_I), C.POINTER(_I)]),
    ("coopcg_gpu_create_multi", _I, [_I, _I, _I, C.POINTER(_I), _I, C.POINTER(_VP)]),
    ("coopcg_nccl_unique_id", _I, [_VP]),
    ("coopcg_gpu_create_rank", _I, [_I, _I, _I, _I, _I, _I, _VP, C.POINTER(_VP)]),
    ("coopcg_gpu_shards", _I, [_VP, _I, C.POINTER(_I), C.POINTER(_I), C.POINTER(_I), C.POINTER(_I)]),
]
NCCL_ID_BYTES = 128

PH_SETUP_LOCAL, PH_SETUP_REST, PH_ITER_LOCAL, PH_ITER_MID, PH_ITER_REST, PH_FINAL_LOCAL, PH_FINAL_REST, PH_MCCG_SETUP = range(8)
BLOCK_X, BLOCK_R, BLOCK_D, BLOCK_Q, BLOCK_S, BLOCK_W = range(6)

_lib = None


def lib() -> C.CDLL:
    """Load the CUDA library (fails loudly if it is missing)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"CUDA library {LIB_PATH} is missing; build it with "
                "`python -m paper_1204_0069_b200.build` (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib
