"""Batched PDHG solver API over the CUDA C-ABI.

Mirrors the reference's public solver surface (same names, argument meaning
and exceptions):
  SolverConfig / SolveStatus / RestartReason / RestartEvent / Residuals /
  InfeasibilityProbe / SolveResult / WarmStart      solver.hpp:51-145,529-531
  PresetColumn / BatchSolveSummary / BatchWorkspace batch_solver.hpp:45-67
  solve_batch                                       batch_solver.hpp:78-355
  solve                                             solver.hpp:569-703
  spmm / spmv / spectral_norm / step_size_for       sparse.hpp:185-319,
                                                    solver.hpp:62-64
Every call goes through include/batchlp_cuda.h into the sm_100a kernels; there
is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import threading
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import _native as N
from .errors import BY_CODE, DeviceError, InvalidArgument
from .problem import BatchProblem, LpProblem, ObjectiveMode, SparseMatrix, kInf


# Shared read-only empty vector: the default of every result vector, so that
# building K results does not allocate 6K numpy arrays.
_EMPTY = np.zeros(0)
_EMPTY.setflags(write=False)


def _empty() -> np.ndarray:
    return _EMPTY


class SolveStatus(enum.IntEnum):
    kOptimal = 0
    kPrimalInfeasible = 1
    kDualInfeasible = 2
    kIterationLimit = 3


class RestartReason(enum.IntEnum):
    kSufficientDecay = 0
    kNecessaryNoProgress = 1
    kArtificial = 2


class Vectors(enum.IntEnum):
    """What a solve copies back (extension; the reference always copies)."""
    NONE = 0
    SOLUTION = 1
    CERTIFICATE = 2


@dataclass
class SolverConfig:
    """solver.hpp:66-103"""
    eps_opt: float = 1e-4
    eps_infeas: float = 1e-8
    eps_dual: float = -1.0
    theta: float = 0.5
    beta_sufficient: float = 0.2
    beta_necessary: float = 0.8
    beta_artificial: float = 0.36
    max_iterations: int = 100000
    termination_check_period: int = 64
    w_init: float = 1.0
    robust_bound_contribution: bool = False
    average_over_all_columns: bool = False
    trace_iterates: bool = False

    def effective_eps_dual(self) -> float:
        return self.eps_opt if self.eps_dual < 0.0 else self.eps_dual

    def check(self) -> None:
        if not (0.0 < self.beta_sufficient < self.beta_necessary < 1.0):
            raise InvalidArgument("config: need 0 < beta_s < beta_n < 1")
        if not (0.0 < self.theta <= 1.0):
            raise InvalidArgument("config: need 0 < theta <= 1")
        if self.termination_check_period < 1:
            raise InvalidArgument("config: check period must be >= 1")
        if self.max_iterations < 0:
            raise InvalidArgument("config: negative iteration limit")
        if not (self.eps_opt > 0.0) or not (self.eps_infeas > 0.0):
            raise InvalidArgument("config: tolerances must be positive")

    def to_c(self, vectors: int = Vectors.SOLUTION, eta: float = 0.0) -> N.bl_config:
        c = N.bl_config()
        c.eps_opt = self.eps_opt
        c.eps_infeas = self.eps_infeas
        c.eps_dual = self.eps_dual
        c.theta = self.theta
        c.beta_sufficient = self.beta_sufficient
        c.beta_necessary = self.beta_necessary
        c.beta_artificial = self.beta_artificial
        c.max_iterations = int(self.max_iterations)
        c.termination_check_period = int(self.termination_check_period)
        c.w_init = self.w_init
        c.robust_bound_contribution = int(bool(self.robust_bound_contribution))
        c.average_over_all_columns = int(bool(self.average_over_all_columns))
        c.trace_iterates = int(bool(self.trace_iterates))
        c.vectors = int(vectors)
        c.eta = float(eta)
        return c


@dataclass
class RestartEvent:
    at_iteration: int = 0
    reason: RestartReason = RestartReason.kSufficientDecay
    residual: float = 0.0
    anchor_residual: float = 0.0


@dataclass
class Residuals:
    gap: float = kInf
    primal: float = kInf
    dual: float = kInf
    fixed_point: float = kInf


@dataclass
class InfeasibilityProbe:
    delta_x: np.ndarray = field(default_factory=_empty)
    delta_y: np.ndarray = field(default_factory=_empty)
    delta_r: np.ndarray = field(default_factory=_empty)


# The (empty) certificate of every result without one; results that carry a
# certificate get their own InfeasibilityProbe.
_NO_CERTIFICATE = InfeasibilityProbe()


@dataclass
class SolveResult:
    """solver.hpp:134-145 (plus the device-computed support sums)."""
    status: SolveStatus = SolveStatus.kIterationLimit
    objective: float = math.nan
    x: np.ndarray = field(default_factory=_empty)
    y: np.ndarray = field(default_factory=_empty)
    reduced_costs: np.ndarray = field(default_factory=_empty)
    residuals: Residuals = field(default_factory=Residuals)
    iterations: int = 0
    restarts: int = 0
    certificate: InfeasibilityProbe = field(default_factory=InfeasibilityProbe)
    restart_log: List[RestartEvent] = field(default_factory=list)
    trajectory_hash: int = 1469598103934665603
    sparse_products: int = 0
    # extension: OptimalityReport supports of the returned triple
    bound_support: float = 0.0
    row_support: float = 0.0
    base_bound_support: float = 0.0
    vectors_exist: bool = False


@dataclass
class WarmStart:
    x: np.ndarray
    y: np.ndarray


@dataclass
class PresetColumn:
    column: int = 0
    result: SolveResult = field(default_factory=SolveResult)


@dataclass
class BatchSolveSummary:
    per_problem: List[SolveResult] = field(default_factory=list)
    iterations: int = 0
    restarts: int = 0
    sparse_products: int = 0
    restart_log: List[RestartEvent] = field(default_factory=list)
    trajectory_hash: int = 1469598103934665603
    # extension
    eta: float = 0.0
    device_ms: float = 0.0
    kernel_launches: int = 0
    loop_passes: int = 0
    profile: Dict[str, tuple] = field(default_factory=dict)  # kind -> (launches, ns, bytes)
    shards: List[dict] = field(default_factory=list)  # per-shard scalars (sharded solves)


# ---------------------------------------------------------------------------
# device contexts and resident problems
# ---------------------------------------------------------------------------
def _check(ctx, rc: int) -> None:
    if rc != N.BL_OK:
        msg = N.lib().bl_last_error(ctx).decode()
        raise BY_CODE.get(rc, DeviceError)(msg)


class DeviceContext:
    """One bl_ctx: a CUDA stream + grow-only workspace on one device."""

    def __init__(self, device: int = 0):
        L = N.lib()
        h = C.c_void_p()
        _check(None, L.bl_ctx_create(int(device), C.byref(h)))
        self.handle = h
        self.device = device

    def close(self) -> None:
        if self.handle:
            N.lib().bl_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass


class DeviceProblem:
    """An LpProblem resident in HBM (bl_problem)."""

    def __init__(self, ctx: DeviceContext, p: LpProblem):
        self.ctx = ctx
        self.handle = None
        self.assign(p)

    @staticmethod
    def _arrays(p: LpProblem):
        A = p.A
        m, n = A.n_rows(), A.n_cols()
        if len(p.objective) != n or p.row_bounds.size() != m or p.var_bounds.size() != n:
            raise InvalidArgument("solve: inconsistent problem dimensions")
        ints = [np.ascontiguousarray(a) for a in (
            A.row_offsets, A.col_indices, A.values, A.t_row_offsets, A.t_col_indices,
            A.t_values)]
        vec = [np.ascontiguousarray(a, dtype=np.float64) for a in (
            p.objective, p.var_bounds.lower, p.var_bounds.upper, p.row_bounds.lower,
            p.row_bounds.upper)]
        k = ints
        args = (m, n, A.nnz(), N.iptr(k[0]), N.iptr(k[1]), N.dptr(k[2]), N.iptr(k[3]),
                N.iptr(k[4]), N.dptr(k[5]), *[N.dptr(v) for v in vec])
        return m, n, args, (ints, vec)

    def assign(self, p: LpProblem) -> None:
        """(Re)uploads p; re-uploading keeps the device buffers (grow-only),
        so the solver's captured graphs stay valid (bl_problem_assign)."""
        m, n, args, keep = self._arrays(p)
        L = N.lib()
        if self.handle is None:
            h = C.c_void_p()
            _check(self.ctx.handle, L.bl_problem_upload(self.ctx.handle, *args, C.byref(h)))
            self.handle = h
        else:
            _check(self.ctx.handle, L.bl_problem_assign(self.ctx.handle, self.handle, *args))
        del keep
        self.m, self.n = m, n

    def close(self) -> None:
        if self.handle:
            N.lib().bl_problem_free(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


class BatchWorkspace:
    """Caller-owned device state reused across solves (batch_solver.hpp:61-67):
    the CUDA context (grow-only buffers) and a cache of resident problems."""

    def __init__(self, device: int = 0):
        self.ctx = DeviceContext(device)
        self._problems: Dict[int, tuple] = {}
        self._scratch: Optional[DeviceProblem] = None

    @staticmethod
    def _vectors(p: LpProblem):
        return (p.objective, p.var_bounds.lower, p.var_bounds.upper, p.row_bounds.lower,
                p.row_bounds.upper)

    def resident(self, p: LpProblem, cache: bool = True) -> DeviceProblem:
        """The device copy of p. A cached entry is reused only for the same
        (immutable) matrix AND the same objective and bounds BY VALUE, as
        the C++ drop-in does (include/batchlp/device.hpp): the reference
        passes the LpProblem by value, so an edited bound must be seen."""
        key = id(p.A)
        hit = self._problems.get(key)
        if cache and hit is not None and hit[0] is p.A:
            vec = self._vectors(p)
            if all(a.shape == b.shape and np.array_equal(a, b, equal_nan=True)
                   for a, b in zip(vec, hit[2])):
                return hit[1]
            # same matrix, new vectors: re-upload into the same device problem
            hit[1].assign(p)
            self._problems[key] = (p.A, hit[1], tuple(np.array(v, copy=True) for v in vec))
            return hit[1]
        if not cache:
            # a fresh upload every call (the caller's arrays may have changed),
            # into one reusable device problem of this workspace
            if self._scratch is None:
                self._scratch = DeviceProblem(self.ctx, p)
            else:
                self._scratch.assign(p)
            return self._scratch
        dp = DeviceProblem(self.ctx, p)
        if cache:
            if len(self._problems) > 8:
                self._problems.clear()
            self._problems[key] = (p.A, dp,
                                   tuple(np.array(v, copy=True) for v in self._vectors(p)))
        return dp


_tls = threading.local()


def default_workspace(device: int = 0) -> BatchWorkspace:
    ws = getattr(_tls, "ws", None)
    if ws is None:
        ws = {}
        _tls.ws = ws
    if device not in ws:
        ws[device] = BatchWorkspace(device)
    return ws[device]


# ---------------------------------------------------------------------------
# solve_batch / solve
# ---------------------------------------------------------------------------
_STATUS = list(SolveStatus)
_RESULT_DTYPE = None


def _result_view(res, width: int) -> np.ndarray:
    """Zero-copy structured view of a bl_column_result array."""
    global _RESULT_DTYPE
    if _RESULT_DTYPE is None:
        _RESULT_DTYPE = np.ctypeslib.as_array((N.bl_column_result * 1)()).dtype
    return np.frombuffer(res, dtype=_RESULT_DTYPE, count=width)


def _results_from_c(res, width: int) -> list:
    """Per-LP SolveResults from the bl_column_result array, via one numpy
    view (attribute access on 10^3-10^4 ctypes structs dominates otherwise)."""
    a = _result_view(res, width)
    c = {name: a[name].tolist() for name in a.dtype.names}
    new = object.__new__
    out = []
    # instances are filled through __dict__ (dataclass __init__ with its
    # default factories costs microseconds per object)
    for st, ob, ga, pr, du, fp, it, rs, bs, rw, bb, ve in zip(
            c["status"], c["objective"], c["gap"], c["primal"], c["dual"], c["fixed_point"],
            c["iterations"], c["restarts"], c["bound_support"], c["row_support"],
            c["base_bound_support"], c["vectors_exist"]):
        res_ = new(Residuals)
        res_.__dict__.update(gap=ga, primal=pr, dual=du, fixed_point=fp)
        r = new(SolveResult)
        r.__dict__.update(status=_STATUS[st], objective=ob, x=_EMPTY, y=_EMPTY,
                          reduced_costs=_EMPTY, residuals=res_, iterations=it, restarts=rs,
                          certificate=_NO_CERTIFICATE, restart_log=[],
                          trajectory_hash=1469598103934665603,
                          sparse_products=0, bound_support=bs, row_support=rw,
                          base_bound_support=bb, vectors_exist=bool(ve))
        out.append(r)
    return out


def _result_from_c(r: N.bl_column_result) -> SolveResult:
    out = SolveResult()
    out.status = SolveStatus(r.status)
    out.objective = r.objective
    out.residuals = Residuals(r.gap, r.primal, r.dual, r.fixed_point)
    out.iterations = int(r.iterations)
    out.restarts = int(r.restarts)
    out.bound_support = r.bound_support
    out.row_support = r.row_support
    out.base_bound_support = r.base_bound_support
    out.vectors_exist = bool(r.vectors_exist)
    return out


def solve_batch(batch: BatchProblem, cfg: Optional[SolverConfig] = None,
                presets: Sequence[PresetColumn] = (), workspace: Optional[BatchWorkspace] = None,
                initial_weights: Optional[Sequence[float]] = None, *,
                vectors: int = Vectors.SOLUTION, eta: float = 0.0,
                warm_start: Optional[Sequence[WarmStart]] = None,
                cache_problem: bool = True) -> BatchSolveSummary:
    """batch_solver.hpp:78-355 on the GPU. `vectors` (extension) selects what
    is copied back; `eta` > 0 overrides the power-iteration step size."""
    cfg = cfg or SolverConfig()
    ws = workspace or default_workspace()
    L = N.lib()
    width = batch.batch_width()
    base = batch.base()
    n, m = base.num_cols(), base.num_rows()
    dp = ws.resident(base, cache=cache_problem)
    ovs = batch.overrides()
    ov_arr = (N.bl_override * max(len(ovs), 1))()
    for k, o in enumerate(ovs):
        ov_arr[k].column = o.column
        ov_arr[k].kind = int(o.kind)
        ov_arr[k].variable = o.variable
        ov_arr[k].value = o.value
    pcols = np.array([p.column for p in presets], dtype=np.int32)
    w0 = None
    if initial_weights is not None and len(initial_weights) > 0:
        if len(initial_weights) != width:
            # the reference checks this after its preset checks and the
            # width == 0 early return (batch_solver.hpp:100,116-118)
            cfg.check()
            if width == 0:
                return BatchSolveSummary()
            raise InvalidArgument("solve_batch: initial weight count mismatch")
        w0 = np.ascontiguousarray(initial_weights, dtype=np.float64)
    wx = wy = None
    if warm_start is not None:
        wx = np.ascontiguousarray(np.stack([np.asarray(w.x, np.float64) for w in warm_start]))
        wy = np.ascontiguousarray(np.stack([np.asarray(w.y, np.float64) for w in warm_start]))
        if wx.shape != (width, n) or wy.shape != (width, m):
            raise InvalidArgument("solve: warm start dimension mismatch")
    ccfg = cfg.to_c(vectors, eta)
    summ = N.bl_summary()
    res = (N.bl_column_result * max(width, 1))()
    _check(ws.ctx.handle, L.bl_solve_batch(
        ws.ctx.handle, dp.handle, width, int(batch.objective_mode()), ov_arr, len(ovs),
        C.byref(ccfg), N.iptr(pcols) if len(pcols) else None, len(pcols), N.dptr(w0),
        N.dptr(wx), N.dptr(wy), C.byref(summ), res))
    out = BatchSolveSummary()
    out.iterations = int(summ.iterations)
    out.restarts = int(summ.restarts)
    out.sparse_products = int(summ.sparse_products)
    out.trajectory_hash = int(summ.trajectory_hash)
    out.eta = summ.eta
    out.device_ms = summ.device_ms
    out.kernel_launches = int(summ.kernel_launches)
    out.loop_passes = int(summ.loop_passes)
    if width == 0:
        return out
    stats = (N.bl_kernel_stat * 16)()
    got = C.c_int32()
    _check(ws.ctx.handle, L.bl_fetch_profile(ws.ctx.handle, stats, 16, C.byref(got)))
    out.profile = {st.name.decode(): (st.launches, st.total_ns, st.alg_bytes)
                   for st in stats[:got.value]}
    if summ.restart_log_size > 0:
        ev = (N.bl_restart_event * summ.restart_log_size)()
        got = C.c_int32()
        _check(ws.ctx.handle, L.bl_fetch_restart_log(ws.ctx.handle, ev, summ.restart_log_size,
                                                     C.byref(got)))
        out.restart_log = [RestartEvent(int(e.at_iteration), RestartReason(e.reason),
                                        e.residual, e.anchor_residual)
                           for e in ev[:got.value]]
    preset_of = {p.column: p for p in presets}
    converted = _results_from_c(res, width)
    a = _result_view(res, width)
    has_sol = a["has_solution"].tolist()
    has_cert = a["has_certificate"].tolist()
    for j in range(width):
        if j in preset_of:
            out.per_problem.append(preset_of[j].result)
            continue
        r = converted[j]
        if has_sol[j]:
            x = np.empty(n)
            y = np.empty(m)
            red = np.empty(n)
            _check(ws.ctx.handle, L.bl_fetch_solution(ws.ctx.handle, j, N.dptr(x), N.dptr(y),
                                                      N.dptr(red)))
            r.x, r.y, r.reduced_costs = x, y, red
        if has_cert[j]:
            dx = np.empty(n)
            dy = np.empty(m)
            dr = np.empty(n)
            _check(ws.ctx.handle, L.bl_fetch_certificate(ws.ctx.handle, j, N.dptr(dx),
                                                         N.dptr(dy), N.dptr(dr)))
            if res[j].certificate_kind == 1:
                r.certificate = InfeasibilityProbe(dx, dy, dr)
            else:
                r.certificate = InfeasibilityProbe(dx, np.zeros(0), np.zeros(0))
        out.per_problem.append(r)
    return out


def solve_batch_sharded(batch: BatchProblem, cfg: Optional[SolverConfig] = None,
                        presets: Sequence[PresetColumn] = (),
                        workspaces: Sequence[BatchWorkspace] = (),
                        initial_weights: Optional[Sequence[float]] = None, *,
                        vectors: int = Vectors.NONE) -> BatchSolveSummary:
    """The batch sharded over several device contexts in one process
    (bl_solve_batch_sharded): one workspace per shard --
    normally one per GPU -- each holding a replica of the problem and solving
    one contiguous column slice with no exchange while iterating. Results are
    in original column order; the summary merges the shards (iterations of
    the longest, restarts / products summed, restart logs concatenated).
    Equals the reference's solve_batch run slice by slice."""
    cfg = cfg or SolverConfig()
    if len(workspaces) < 1:
        raise InvalidArgument("solve_batch_sharded: need at least one workspace")
    L = N.lib()
    width = batch.batch_width()
    base = batch.base()
    G = len(workspaces)
    dps = [ws.resident(base) for ws in workspaces]
    ctxs = (C.c_void_p * G)(*[ws.ctx.handle for ws in workspaces])
    probs = (C.c_void_p * G)(*[dp.handle for dp in dps])
    ovs = batch.overrides()
    ov_arr = (N.bl_override * max(len(ovs), 1))()
    for k, o in enumerate(ovs):
        ov_arr[k].column, ov_arr[k].kind = o.column, int(o.kind)
        ov_arr[k].variable, ov_arr[k].value = o.variable, o.value
    pcols = np.array([q.column for q in presets], dtype=np.int32)
    w0 = None
    if initial_weights is not None and len(initial_weights) > 0:
        if len(initial_weights) != width:
            raise InvalidArgument("solve_batch: initial weight count mismatch")
        w0 = np.ascontiguousarray(initial_weights, dtype=np.float64)
    ccfg = cfg.to_c(vectors)
    sums = (N.bl_summary * G)()
    res = (N.bl_column_result * max(width, 1))()
    _check(workspaces[0].ctx.handle, L.bl_solve_batch_sharded(
        ctxs, probs, G, width, int(batch.objective_mode()), C.cast(ov_arr, C.c_void_p),
        len(ovs), C.cast(C.pointer(ccfg), C.c_void_p),
        N.iptr(pcols) if len(pcols) else None, len(pcols), N.dptr(w0),
        C.cast(sums, C.c_void_p), C.cast(res, C.c_void_p)))
    out = BatchSolveSummary()
    for q in sums:
        out.iterations = max(out.iterations, int(q.iterations))
        out.restarts += int(q.restarts)
        out.sparse_products += int(q.sparse_products)
        out.device_ms = max(out.device_ms, q.device_ms)
        out.kernel_launches += int(q.kernel_launches)
        out.loop_passes = max(out.loop_passes, int(q.loop_passes))
        out.eta = q.eta
        out.shards.append({"iterations": int(q.iterations), "restarts": int(q.restarts),
                           "device_ms": q.device_ms, "loop_passes": int(q.loop_passes)})
    if width == 0:
        return out
    preset_of = {q.column: q for q in presets}
    converted = _results_from_c(res, width)
    out.per_problem = [preset_of[j].result if j in preset_of else converted[j]
                       for j in range(width)]
    return out


def solve(p: LpProblem, cfg: Optional[SolverConfig] = None, warm: Optional[WarmStart] = None,
          *, workspace: Optional[BatchWorkspace] = None, vectors: int = Vectors.CERTIFICATE,
          eta: float = 0.0) -> SolveResult:
    """Single LP (solver.hpp:569-703) as a width-1 batch on the GPU; the
    reference's width-1 batch is bit-identical to it (batch_solver.hpp:22-24)."""
    cfg = cfg or SolverConfig()
    cfg.check()
    if (len(p.objective) != p.num_cols() or p.row_bounds.size() != p.num_rows()
            or p.var_bounds.size() != p.num_cols()):
        raise InvalidArgument("solve: inconsistent problem dimensions")
    if warm is not None and (len(warm.x) != p.num_cols() or len(warm.y) != p.num_rows()):
        raise InvalidArgument("solve: warm start dimension mismatch")
    b = BatchProblem(p, 1, ObjectiveMode.kSharedObjective, [])
    s = solve_batch(b, cfg, (), workspace, None, vectors=vectors, eta=eta,
                    warm_start=[warm] if warm is not None else None)
    r = s.per_problem[0]
    r.restart_log = s.restart_log
    r.trajectory_hash = s.trajectory_hash
    r.sparse_products = s.sparse_products
    return r


def spectral_norm(A: SparseMatrix, *, workspace: Optional[BatchWorkspace] = None) -> float:
    """||A||_2 estimate x 1.01 by the device power iteration (sparse.hpp:297-319)."""
    if A.nnz() == 0:
        raise InvalidArgument("spectral_norm: zero matrix")
    ws = workspace or default_workspace()
    p = LpProblem(A, np.zeros(A.n_cols()), _bounds(A.n_rows()), _bounds(A.n_cols()))
    dp = DeviceProblem(ws.ctx, p)
    out = C.c_double()
    _check(ws.ctx.handle, N.lib().bl_spectral_norm(ws.ctx.handle, dp.handle, C.byref(out)))
    dp.close()
    return out.value


def step_size_for(A: SparseMatrix, **kw) -> float:
    """solver.hpp:62-64"""
    return 0.998 / (1.0 if A.nnz() == 0 else spectral_norm(A, **kw))


def _bounds(n):
    from .problem import Bounds
    return Bounds(n)


def spmm(A: SparseMatrix, X: np.ndarray, out: Optional[np.ndarray] = None,
         transpose_a: bool = False, active_width: int = -1, *,
         workspace: Optional[BatchWorkspace] = None) -> np.ndarray:
    """out[:, j] = op(A) X[:, j] for the leading active_width columns; trailing
    columns of `out` untouched (sparse.hpp:213-238). X is rows x width (numpy
    2-D, any order); entries are bit-identical to the reference csr_apply."""
    rin = A.n_rows() if transpose_a else A.n_cols()
    rout = A.n_cols() if transpose_a else A.n_rows()
    X = np.asarray(X, dtype=np.float64)
    if X.ndim == 1:
        X = X[:, None]
    if X.shape[0] != rin:
        raise InvalidArgument("spmm: dimension mismatch")
    width = X.shape[1]
    if out is None:
        out = np.zeros((rout, width))
    if out.shape != (rout, width):
        raise InvalidArgument("spmm: dimension mismatch")
    active = width if active_width < 0 else active_width
    if active > width:
        raise InvalidArgument("spmm: active width too large")
    ws = workspace or default_workspace()
    p = LpProblem(A, np.zeros(A.n_cols()), _bounds(A.n_rows()), _bounds(A.n_cols()))
    dp = ws.resident(p, cache=False)
    xc = np.ascontiguousarray(X.T)          # column j contiguous
    oc = np.ascontiguousarray(out.T)
    _check(ws.ctx.handle, N.lib().bl_spmm(ws.ctx.handle, dp.handle, int(bool(transpose_a)),
                                          width, active, N.dptr(xc), N.dptr(oc)))
    out[:, :] = oc.T
    return out


def spmv(A: SparseMatrix, x: np.ndarray, transpose_a: bool = False, **kw) -> np.ndarray:
    """sparse.hpp:185-192"""
    return spmm(A, np.asarray(x, np.float64)[:, None], None, transpose_a, -1, **kw)[:, 0]
