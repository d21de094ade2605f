"""TEST INFRASTRUCTURE ONLY: ctypes access to the compiled reference.

oracle/_ref/libbatchlp_ref.so is the unmodified reference (headers under
/root/reference/proj/include, compiled by oracle/Makefile) behind the C shim
oracle/ref_shim.cpp. Only tests/, __graft_entry__.smoke() and bench.py's
CPU-baseline / --impl reference legs may import this module; the product
never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libbatchlp_ref.so")

import sys as _sys

_sys.path.insert(0, os.path.dirname(HERE))
from paper_2601_21990_b200 import _native as N  # noqa: E402  (struct layouts only)

_DP = C.POINTER(C.c_double)
_IP = C.POINTER(C.c_int32)
_LP = C.POINTER(C.c_int64)
_P = C.c_void_p

_lib = None


def available() -> bool:
    return os.path.exists(REF_LIB)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference oracle not built: {REF_LIB}")
        L = C.CDLL(REF_LIB)
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_lp_create": (_P, [C.c_int32, C.c_int32, C.c_int64, _IP, _IP, _DP, _DP, _DP,
                                   _DP, _DP, _DP]),
            "ref_lp_free": (None, [_P]),
            "ref_lp_dims": (None, [_P, _IP, _IP, _LP]),
            "ref_lp_export": (None, [_P, _IP, _IP, _DP, _IP, _IP, _DP, _DP, _DP, _DP, _DP,
                                     _DP]),
            "ref_gen_set_cover": (_P, [C.c_int32, C.c_int32, C.c_double, C.c_uint64]),
            "ref_gen_family": (_P, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_uint64,
                                    _IP, _IP]),
            "ref_test_lp": (_P, [C.c_int32, C.c_uint64]),
            "ref_append_cutoff": (_P, [_P, C.c_double]),
            "ref_spectral_norm": (C.c_int, [_P, _DP]),
            "ref_spmm": (C.c_int, [_P, C.c_int, C.c_int32, C.c_int32, _DP, _DP]),
            "ref_solve_batch": (C.c_int, [
                _P, C.c_int32, C.c_int32, C.POINTER(N.bl_override), C.c_int32, C.c_int32,
                C.c_double, C.POINTER(N.bl_config), _IP, _IP, _DP, C.c_int32, _DP,
                C.POINTER(N.bl_summary), C.POINTER(N.bl_column_result), _DP, _DP, _DP,
                C.POINTER(N.bl_restart_event), C.c_int32]),
            "ref_solve": (C.c_int, [_P, C.POINTER(N.bl_config), _DP, _DP,
                                    C.POINTER(N.bl_summary), C.POINTER(N.bl_column_result),
                                    _DP, _DP, _DP, C.POINTER(N.bl_restart_event),
                                    C.c_int32]),
            "ref_solve_certificate": (C.c_int, [_P, C.POINTER(N.bl_config), _DP, _DP, _DP,
                                                _IP]),
            "ref_run_fsb": (C.c_int, [_P, _DP, _IP, C.c_int32, C.c_double,
                                      C.POINTER(N.bl_config), C.c_double, _IP, _IP, _DP,
                                      _DP, _LP, _LP, _DP, _DP, _IP, _IP, _DP, _DP, _LP,
                                      _LP]),
            "ref_run_obbt": (C.c_int, [_P, C.c_double, C.c_double, C.c_double, C.c_int64,
                                       C.c_int32, C.c_double, C.c_int32,
                                       C.POINTER(N.bl_config), _DP, _DP, _IP, _IP, _DP,
                                       _DP, _IP, _IP, _IP, _DP, _LP]),
            "ref_oracle_solve": (C.c_int, [_P, _IP, _DP, _DP]),
        }
        for k, (r, a) in sig.items():
            f = getattr(L, k)
            f.restype = r
            f.argtypes = a
        _lib = L
    return _lib


def _dp(a):
    return None if a is None else a.ctypes.data_as(_DP)


def _ip(a):
    return None if a is None else a.ctypes.data_as(_IP)


def _chk(rc):
    if rc != 0:
        raise RuntimeError(f"reference raised (code {rc}): {lib().ref_last_error().decode()}")


class RefLp:
    """Owning handle to a reference LpProblem."""

    def __init__(self, handle):
        if not handle:
            raise RuntimeError("reference: " + lib().ref_last_error().decode())
        self.h = handle
        m, n, nnz = C.c_int32(), C.c_int32(), C.c_int64()
        lib().ref_lp_dims(self.h, C.byref(m), C.byref(n), C.byref(nnz))
        self.m, self.n, self.nnz = m.value, n.value, nnz.value

    @classmethod
    def from_problem(cls, p) -> "RefLp":
        A = p.A
        arrs = [np.ascontiguousarray(a) for a in (A.row_offsets, A.col_indices, A.values)]
        vec = [np.ascontiguousarray(a, dtype=np.float64) for a in (
            p.objective, p.var_bounds.lower, p.var_bounds.upper, p.row_bounds.lower,
            p.row_bounds.upper)]
        return cls(lib().ref_lp_create(A.n_rows(), A.n_cols(), A.nnz(), _ip(arrs[0]),
                                       _ip(arrs[1]), _dp(arrs[2]), *[_dp(v) for v in vec]))

    def to_problem(self):
        from paper_2601_21990_b200.problem import Bounds, LpProblem, SparseMatrix
        m, n, nnz = self.m, self.n, self.nnz
        rp = np.zeros(m + 1, np.int32)
        ci = np.zeros(max(nnz, 1), np.int32)
        cv = np.zeros(max(nnz, 1))
        trp = np.zeros(n + 1, np.int32)
        tci = np.zeros(max(nnz, 1), np.int32)
        tcv = np.zeros(max(nnz, 1))
        c, xl, xu = np.zeros(n), np.zeros(n), np.zeros(n)
        rl, ru = np.zeros(m), np.zeros(m)
        lib().ref_lp_export(self.h, _ip(rp), _ip(ci), _dp(cv), _ip(trp), _ip(tci), _dp(tcv),
                            _dp(c), _dp(xl), _dp(xu), _dp(rl), _dp(ru))
        A = SparseMatrix(m, n, rp, ci[:nnz], cv[:nnz], trp, tci[:nnz], tcv[:nnz])
        return LpProblem(A, c, Bounds.from_arrays(rl, ru), Bounds.from_arrays(xl, xu))

    def __del__(self):
        try:
            if self.h:
                lib().ref_lp_free(self.h)
        except Exception:
            pass


def test_lp(shape: int, seed: int):
    """testsupport fixtures: 0 feasible, 1 primal infeasible, 2 dual infeasible,
    10 two_var_lp, 11 knapsack_lp (tests/support/instances.hpp)."""
    return RefLp(lib().ref_test_lp(shape, seed)).to_problem()


def gen_set_cover(rows, cols, density, seed):
    return RefLp(lib().ref_gen_set_cover(rows, cols, density, seed)).to_problem()


def gen_family(family, a, b, c, seed):
    """0 set cover (density c/100), 1 comb auction, 2 max ind set, 3 facility."""
    ic = np.zeros(100000, np.int32)
    ni = C.c_int32()
    h = RefLp(lib().ref_gen_family(family, a, b, c, seed, _ip(ic), C.byref(ni)))
    return h.to_problem(), list(ic[:ni.value])


def append_cutoff(p, alpha):
    h = RefLp.from_problem(p)
    return RefLp(lib().ref_append_cutoff(h.h, alpha)).to_problem()


def spectral_norm(p) -> float:
    out = C.c_double()
    h = RefLp.from_problem(p)
    _chk(lib().ref_spectral_norm(h.h, C.byref(out)))
    return out.value


def spmm(p, X: np.ndarray, transpose: bool = False, active: int = -1,
         out: Optional[np.ndarray] = None) -> np.ndarray:
    """X rows x width (numpy); returns op(A) X with trailing columns of `out`
    untouched."""
    h = RefLp.from_problem(p)
    width = X.shape[1]
    rout = p.A.n_cols() if transpose else p.A.n_rows()
    xc = np.ascontiguousarray(X.T, dtype=np.float64)
    oc = np.ascontiguousarray((np.zeros((rout, width)) if out is None else out).T)
    _chk(lib().ref_spmm(h.h, int(transpose), width, width if active < 0 else active,
                        _dp(xc), _dp(oc)))
    return oc.T.copy()


@dataclass
class RefColumn:
    status: int
    objective: float
    iterations: int
    restarts: int
    gap: float
    primal: float
    dual: float
    fixed_point: float
    bound_support: float
    row_support: float
    base_bound_support: float
    has_solution: int
    certificate_kind: int
    x: Optional[np.ndarray] = None
    y: Optional[np.ndarray] = None
    reduced: Optional[np.ndarray] = None


@dataclass
class RefSummary:
    iterations: int
    restarts: int
    sparse_products: int
    trajectory_hash: int
    eta: float
    per_problem: List[RefColumn] = field(default_factory=list)
    restart_log: list = field(default_factory=list)


def _cfg(cfg) -> N.bl_config:
    if cfg is None:
        from paper_2601_21990_b200.solver import SolverConfig
        cfg = SolverConfig()
    return cfg.to_c()


def _collect(summ, res, width, n, m, xs, ys, rs, log) -> RefSummary:
    out = RefSummary(int(summ.iterations), int(summ.restarts), int(summ.sparse_products),
                     int(summ.trajectory_hash), summ.eta)
    for j in range(width):
        r = res[j]
        col = RefColumn(r.status, r.objective, int(r.iterations), int(r.restarts), r.gap,
                        r.primal, r.dual, r.fixed_point, r.bound_support, r.row_support,
                        r.base_bound_support, r.has_solution, r.certificate_kind)
        if r.has_solution and xs is not None:
            col.x = xs[j * n:(j + 1) * n].copy()
            col.y = ys[j * m:(j + 1) * m].copy()
            col.reduced = rs[j * n:(j + 1) * n].copy()
        out.per_problem.append(col)
    k = min(int(summ.restart_log_size), len(log))
    out.restart_log = [(int(e.at_iteration), int(e.reason), e.residual, e.anchor_residual)
                       for e in log[:k]]
    return out


def solve_batch(p, width: int, mode: int = 0, overrides: Sequence = (), cfg=None,
                presets: Sequence = (), initial_weights=None, cutoff=None,
                vectors: bool = True) -> RefSummary:
    """The reference solve_batch on the same arrays. presets: (column, status,
    objective) tuples. overrides: ColumnOverride-like objects."""
    h = RefLp.from_problem(p)
    n, m = h.n, h.m + (1 if cutoff is not None else 0)
    ov = (N.bl_override * max(len(overrides), 1))()
    for k, o in enumerate(overrides):
        ov[k].column, ov[k].kind, ov[k].variable, ov[k].value = (
            o.column, int(o.kind), o.variable, o.value)
    pc = np.array([q[0] for q in presets], np.int32)
    ps = np.array([q[1] for q in presets], np.int32)
    po = np.array([q[2] for q in presets], np.float64)
    w0 = None if initial_weights is None else np.ascontiguousarray(initial_weights, np.float64)
    summ = N.bl_summary()
    res = (N.bl_column_result * max(width, 1))()
    xs = np.zeros(max(width * n, 1)) if vectors else None
    ys = np.zeros(max(width * m, 1)) if vectors else None
    rs = np.zeros(max(width * n, 1)) if vectors else None
    log = (N.bl_restart_event * 65536)()
    c = _cfg(cfg)
    _chk(lib().ref_solve_batch(h.h, width, mode, ov, len(overrides), int(cutoff is not None),
                               0.0 if cutoff is None else cutoff, C.byref(c),
                               _ip(pc) if len(pc) else None, _ip(ps) if len(ps) else None,
                               _dp(po) if len(po) else None, len(pc), _dp(w0), C.byref(summ),
                               res, _dp(xs), _dp(ys), _dp(rs), log, 65536))
    return _collect(summ, res, width, n, m, xs, ys, rs, log)


def solve(p, cfg=None, warm=None) -> RefSummary:
    h = RefLp.from_problem(p)
    n, m = h.n, h.m
    summ = N.bl_summary()
    res = (N.bl_column_result * 1)()
    xs, ys, rs = np.zeros(max(n, 1)), np.zeros(max(m, 1)), np.zeros(max(n, 1))
    log = (N.bl_restart_event * 65536)()
    c = _cfg(cfg)
    wx = None if warm is None else np.ascontiguousarray(warm.x, np.float64)
    wy = None if warm is None else np.ascontiguousarray(warm.y, np.float64)
    _chk(lib().ref_solve(h.h, C.byref(c), _dp(wx), _dp(wy), C.byref(summ), res, _dp(xs),
                         _dp(ys), _dp(rs), log, 65536))
    return _collect(summ, res, 1, n, m, xs, ys, rs, log)


def certificate(p, cfg=None):
    h = RefLp.from_problem(p)
    dx, dy, dr = np.zeros(max(h.n, 1)), np.zeros(max(h.m, 1)), np.zeros(max(h.n, 1))
    kind = C.c_int32()
    c = _cfg(cfg)
    _chk(lib().ref_solve_certificate(h.h, C.byref(c), _dp(dx), _dp(dy), _dp(dr),
                                     C.byref(kind)))
    return kind.value, dx[:h.n], dy[:h.m], dr[:h.n]


def run_fsb(p, x_rel, frac, cfg=None, integrality_tol=1e-6, infeasible_delta=1e20) -> dict:
    h = RefLp.from_problem(p)
    k = len(frac)
    f = np.ascontiguousarray(frac, np.int32)
    xr = np.ascontiguousarray(x_rel, np.float64)
    i32 = lambda: np.zeros(max(k, 1), np.int32)  # noqa: E731
    f64 = lambda: np.zeros(max(k, 1), np.float64)  # noqa: E731
    i64 = lambda: np.zeros(max(k, 1), np.int64)  # noqa: E731
    us, ds, uo, do, ui, di, du, dd, uf, df, sc = (i32(), i32(), f64(), f64(), i64(), i64(),
                                                  f64(), f64(), i32(), i32(), f64())
    root, it, sp = C.c_double(), C.c_int64(), C.c_int64()
    c = _cfg(cfg)
    lp = lambda a: a.ctypes.data_as(_LP)  # noqa: E731
    _chk(lib().ref_run_fsb(h.h, _dp(xr), _ip(f), k, integrality_tol, C.byref(c),
                           infeasible_delta, _ip(us), _ip(ds), _dp(uo), _dp(do), lp(ui),
                           lp(di), _dp(du), _dp(dd), _ip(uf), _ip(df), _dp(sc),
                           C.byref(root), C.byref(it), C.byref(sp)))
    return dict(up_status=us[:k], down_status=ds[:k], up_objective=uo[:k],
                down_objective=do[:k], up_iterations=ui[:k], down_iterations=di[:k],
                delta_up=du[:k], delta_down=dd[:k], up_flagged=uf[:k], down_flagged=df[:k],
                score=sc[:k], root_objective=root.value, iterations=it.value,
                sparse_products=sp.value)


def run_obbt(p, eps_opt=1e-4, eps_dual=1e-8, min_improvement=1e-4, max_iterations=100000,
             cutoff=None, lenient=False, solver_cfg=None) -> dict:
    h = RefLp.from_problem(p)
    n = h.n
    nl, nu = np.zeros(n), np.zeros(n)
    lc, uc = np.zeros(n, np.int32), np.zeros(n, np.int32)
    lm, um = np.zeros(n), np.zeros(n)
    ls, us = np.zeros(n, np.int32), np.zeros(n, np.int32)
    counts = np.zeros(3, np.int32)
    mr, it = C.c_double(), C.c_int64()
    c = _cfg(solver_cfg)
    _chk(lib().ref_run_obbt(h.h, eps_opt, eps_dual, min_improvement, max_iterations,
                            int(cutoff is not None), 0.0 if cutoff is None else cutoff,
                            int(lenient), C.byref(c), _dp(nl), _dp(nu), _ip(lc), _ip(uc),
                            _dp(lm), _dp(um), _ip(ls), _ip(us), _ip(counts), C.byref(mr),
                            C.byref(it)))
    return dict(new_lower=nl, new_upper=nu, lower_changed=lc, upper_changed=uc,
                lower_margin=lm, upper_margin=um, lower_status=ls, upper_status=us,
                changed_count=int(counts[0]), solved_count=int(counts[1]),
                limit_count=int(counts[2]), mean_reduction_pct=mr.value,
                iterations=it.value)


def oracle_solve(p):
    """Vertex enumeration ground truth (oracle.hpp:164-306) for n + m <= 16.
    status 0 optimal, 1 infeasible, 2 unbounded."""
    h = RefLp.from_problem(p)
    st, obj = C.c_int32(), C.c_double()
    v = np.zeros(max(h.n, 1))
    _chk(lib().ref_oracle_solve(h.h, C.byref(st), C.byref(obj), _dp(v)))
    return st.value, obj.value, v[:h.n]
