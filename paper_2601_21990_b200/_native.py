"""ctypes binding of the C-ABI in include/batchlp_cuda.h.

The shared library is built in-tree (paper_2601_21990_b200/lib/) by
``paper_2601_21990_b200.build.build()``. There is no fallback: importing the
solver without the library raises, and every entry point runs on the GPU.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# BATCHLP_LIB selects an alternative in-tree build (tuning variants under
# lib/variants/); it is still this package's CUDA library, never a fallback.
LIB_PATH = os.environ.get("BATCHLP_LIB") or os.path.join(_HERE, "lib", "libbatchlp_cuda.so")

# enum values (batchlp_cuda.h)
BL_OK = 0
BL_ERR_INVALID_ARGUMENT = 1
BL_ERR_OUT_OF_RANGE = 2
BL_ERR_DOMAIN = 3
BL_ERR_LOGIC = 4
BL_ERR_CUDA = 5

BL_VECTORS_NONE = 0
BL_VECTORS_SOLUTION = 1
BL_VECTORS_CERTIFICATE = 2


class bl_config(C.Structure):
    _fields_ = [
        ("eps_opt", C.c_double),
        ("eps_infeas", C.c_double),
        ("eps_dual", C.c_double),
        ("theta", C.c_double),
        ("beta_sufficient", C.c_double),
        ("beta_necessary", C.c_double),
        ("beta_artificial", C.c_double),
        ("max_iterations", C.c_int64),
        ("termination_check_period", C.c_int64),
        ("w_init", C.c_double),
        ("robust_bound_contribution", C.c_int32),
        ("average_over_all_columns", C.c_int32),
        ("trace_iterates", C.c_int32),
        ("vectors", C.c_int32),
        ("eta", C.c_double),
    ]


class bl_override(C.Structure):
    _fields_ = [
        ("column", C.c_int32),
        ("kind", C.c_int32),
        ("variable", C.c_int32),
        ("reserved", C.c_int32),
        ("value", C.c_double),
    ]


class bl_column_result(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("restarts", C.c_int32),
        ("iterations", C.c_int64),
        ("objective", C.c_double),
        ("gap", C.c_double),
        ("primal", C.c_double),
        ("dual", C.c_double),
        ("fixed_point", C.c_double),
        ("bound_support", C.c_double),
        ("row_support", C.c_double),
        ("base_bound_support", C.c_double),
        ("has_solution", C.c_int32),
        ("has_certificate", C.c_int32),
        ("certificate_kind", C.c_int32),
        ("vectors_exist", C.c_int32),
    ]


class bl_restart_event(C.Structure):
    _fields_ = [
        ("at_iteration", C.c_int64),
        ("reason", C.c_int32),
        ("reserved", C.c_int32),
        ("residual", C.c_double),
        ("anchor_residual", C.c_double),
    ]


class bl_summary(C.Structure):
    _fields_ = [
        ("iterations", C.c_int64),
        ("restarts", C.c_int32),
        ("restart_log_size", C.c_int32),
        ("sparse_products", C.c_int64),
        ("trajectory_hash", C.c_uint64),
        ("eta", C.c_double),
        ("device_ms", C.c_double),
        ("kernel_launches", C.c_int64),
        ("loop_passes", C.c_int64),
    ]


class bl_kernel_stat(C.Structure):
    _fields_ = [
        ("name", C.c_char * 16),
        ("launches", C.c_double),
        ("total_ns", C.c_double),
        ("alg_bytes", C.c_double),
    ]


class bl_instance(C.Structure):
    _fields_ = [
        ("m", C.c_int32),
        ("n", C.c_int32),
        ("nnz", C.c_int64),
        ("rowptr", C.POINTER(C.c_int32)),
        ("col", C.POINTER(C.c_int32)),
        ("val", C.POINTER(C.c_double)),
        ("t_rowptr", C.POINTER(C.c_int32)),
        ("t_col", C.POINTER(C.c_int32)),
        ("t_val", C.POINTER(C.c_double)),
        ("objective", C.POINTER(C.c_double)),
        ("var_lower", C.POINTER(C.c_double)),
        ("var_upper", C.POINTER(C.c_double)),
        ("row_lower", C.POINTER(C.c_double)),
        ("row_upper", C.POINTER(C.c_double)),
    ]


_P = C.c_void_p
_DP = C.POINTER(C.c_double)
_IP = C.POINTER(C.c_int32)

# name -> (restype, argtypes); every symbol declared in include/batchlp_cuda.h
SIGNATURES = {
    "bl_config_default": (None, [C.POINTER(bl_config)]),
    "bl_abi_version": (C.c_int, []),
    "bl_ctx_create": (C.c_int, [C.c_int, C.POINTER(_P)]),
    "bl_ctx_destroy": (None, [_P]),
    "bl_last_error": (C.c_char_p, [_P]),
    "bl_problem_upload": (
        C.c_int,
        [_P, C.c_int32, C.c_int32, C.c_int64, _IP, _IP, _DP, _IP, _IP, _DP,
         _DP, _DP, _DP, _DP, _DP, C.POINTER(_P)],
    ),
    "bl_problem_free": (None, [_P]),
    "bl_problem_assign": (
        C.c_int,
        [_P, _P, C.c_int32, C.c_int32, C.c_int64, _IP, _IP, _DP, _IP, _IP, _DP,
         _DP, _DP, _DP, _DP, _DP],
    ),
    "bl_spectral_norm": (C.c_int, [_P, _P, _DP]),
    "bl_spmm": (C.c_int, [_P, _P, C.c_int, C.c_int32, C.c_int32, _DP, _DP]),
    "bl_csr_apply": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int64, _IP, _IP, _DP, _DP, _DP]),
    "bl_measure_spmm": (C.c_int, [_P, _P, C.c_int32, C.c_int32, _DP, _DP,
                                  C.POINTER(C.c_int32)]),
    "bl_solve_batch_sharded": (
        C.c_int,
        [C.POINTER(_P), C.POINTER(_P), C.c_int32, C.c_int32, C.c_int32, _P, C.c_int32, _P,
         _IP, C.c_int32, _DP, _P, _P],
    ),
    "bl_solve_batch": (
        C.c_int,
        [_P, _P, C.c_int32, C.c_int32, C.POINTER(bl_override), C.c_int32,
         C.POINTER(bl_config), _IP, C.c_int32, _DP, _DP, _DP,
         C.POINTER(bl_summary), C.POINTER(bl_column_result)],
    ),
    "bl_fetch_solution": (C.c_int, [_P, C.c_int32, _DP, _DP, _DP]),
    "bl_fetch_certificate": (C.c_int, [_P, C.c_int32, _DP, _DP, _DP]),
    "bl_fetch_profile": (
        C.c_int, [_P, C.POINTER(bl_kernel_stat), C.c_int32, _IP]),
    "bl_fetch_restart_log": (
        C.c_int, [_P, C.POINTER(bl_restart_event), C.c_int32, _IP]),
    "bl_gen_set_cover": (
        C.c_int, [C.c_int32, C.c_int32, C.c_double, C.c_uint64, C.POINTER(bl_instance)]),
    "bl_gen_sparse_cover": (
        C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_uint64, C.POINTER(bl_instance)]),
    "bl_gen_boxed_feasible": (
        C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_uint64, C.POINTER(bl_instance)]),
    "bl_instance_free": (None, [C.POINTER(bl_instance)]),
}

_lib = None
_lock = threading.Lock()


def lib() -> C.CDLL:
    """The loaded C-ABI library; raises if it has not been built."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"batchlp CUDA library not built: {LIB_PATH} is missing "
                    "(run __graft_entry__.build()); there is no CPU fallback")
            L = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
        return _lib


def dptr(a):
    """double* of a contiguous float64 numpy array (or None)."""
    if a is None:
        return None
    return a.ctypes.data_as(_DP)


def iptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(_IP)
