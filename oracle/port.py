"""TEST INFRASTRUCTURE ONLY: ctypes access to the plain-C restatement
(oracle/batchlp_oracle.c -> oracle/_build/libbatchlp_oracle.so).

Used by tests/ (pinned against oracle/_ref and tests/golden/) and as the
CPU-side checker where the compiled reference is unavailable. The product
never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libbatchlp_oracle.so")
sys.path.insert(0, os.path.dirname(HERE))
from paper_2601_21990_b200 import _native as N  # noqa: E402  (struct layouts only)

_DP = C.POINTER(C.c_double)
_IP = C.POINTER(C.c_int32)


class orc_lp(C.Structure):
    _fields_ = [("m", C.c_int), ("n", C.c_int), ("rp", _IP), ("ci", _IP), ("trp", _IP),
                ("tci", _IP), ("cv", _DP), ("tcv", _DP), ("c", _DP), ("xl", _DP),
                ("xu", _DP), ("rl", _DP), ("ru", _DP)]


_lib = None


def available() -> bool:
    return os.path.exists(LIB)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB)
        L.orc_spmm.argtypes = [C.POINTER(orc_lp), C.c_int, C.c_int, C.c_int, _DP, _DP]
        L.orc_spectral_norm.argtypes = [C.POINTER(orc_lp)]
        L.orc_spectral_norm.restype = C.c_double
        L.orc_solve_batch.argtypes = [C.POINTER(orc_lp), C.c_int, C.c_int,
                                      C.POINTER(N.bl_override), C.c_int,
                                      C.POINTER(N.bl_config), _IP, C.c_int, _DP,
                                      C.POINTER(N.bl_summary),
                                      C.POINTER(N.bl_column_result), _DP, _DP, _DP]
        L.orc_solve_batch.restype = C.c_int
        _lib = L
    return _lib


class _Lp:
    """Keeps the numpy arrays alive for the duration of a call."""

    def __init__(self, p):
        A = p.A
        self.keep = [np.ascontiguousarray(a) for a in (
            A.row_offsets, A.col_indices, A.t_row_offsets, A.t_col_indices)]
        self.keepd = [np.ascontiguousarray(a, dtype=np.float64) for a in (
            A.values, A.t_values, p.objective, p.var_bounds.lower, p.var_bounds.upper,
            p.row_bounds.lower, p.row_bounds.upper)]
        ip = lambda a: a.ctypes.data_as(_IP)  # noqa: E731
        dp = lambda a: a.ctypes.data_as(_DP)  # noqa: E731
        k, d = self.keep, self.keepd
        self.s = orc_lp(A.n_rows(), A.n_cols(), ip(k[0]), ip(k[1]), ip(k[2]), ip(k[3]),
                        dp(d[0]), dp(d[1]), dp(d[2]), dp(d[3]), dp(d[4]), dp(d[5]), dp(d[6]))


def spmm(p, X, transpose=False, active=-1, out=None):
    lp = _Lp(p)
    width = X.shape[1]
    rout = p.A.n_cols() if transpose else p.A.n_rows()
    xc = np.ascontiguousarray(X.T, dtype=np.float64)
    oc = np.ascontiguousarray((np.zeros((rout, width)) if out is None else out).T)
    lib().orc_spmm(C.byref(lp.s), int(transpose), width, width if active < 0 else active,
                   xc.ctypes.data_as(_DP), oc.ctypes.data_as(_DP))
    return oc.T.copy()


def spectral_norm(p) -> float:
    lp = _Lp(p)
    return lib().orc_spectral_norm(C.byref(lp.s))


def solve_batch(p, width, mode=0, overrides=(), cfg=None, presets=(), initial_weights=None,
                vectors=False):
    """Same contract as oracle.ref.solve_batch (presets: (column, status,
    objective)); returns (summary, results list, x, y, r)."""
    from paper_2601_21990_b200.solver import SolverConfig
    lp = _Lp(p)
    cfg = cfg or SolverConfig()
    c = cfg.to_c()
    ov = (N.bl_override * max(len(overrides), 1))()
    for k, o in enumerate(overrides):
        ov[k].column, ov[k].kind, ov[k].variable, ov[k].value = (
            o.column, int(o.kind), o.variable, o.value)
    pc = np.array([q[0] for q in presets], np.int32)
    w0 = None if initial_weights is None else np.ascontiguousarray(initial_weights, np.float64)
    summ = N.bl_summary()
    res = (N.bl_column_result * max(width, 1))()
    n, m = p.num_cols(), p.num_rows()
    xs = np.zeros(max(width * n, 1)) if vectors else None
    ys = np.zeros(max(width * m, 1)) if vectors else None
    rs = np.zeros(max(width * n, 1)) if vectors else None
    dp = lambda a: None if a is None else a.ctypes.data_as(_DP)  # noqa: E731
    rc = lib().orc_solve_batch(C.byref(lp.s), width, mode, ov, len(overrides), C.byref(c),
                               pc.ctypes.data_as(_IP) if len(pc) else None, len(pc), dp(w0),
                               C.byref(summ), res, dp(xs), dp(ys), dp(rs))
    if rc != 0:
        raise RuntimeError(f"oracle port: code {rc}")
    for q in presets:  # the caller's preset results pass through
        res[q[0]].status = q[1]
        res[q[0]].objective = q[2]
    return summ, [res[j] for j in range(width)], xs, ys, rs
