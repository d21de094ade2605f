"""The reference's callers of the hot path: full strong branching and OBBT.

Mirrors proj/include/batchlp/strong_branching.hpp and obbt.hpp (same names,
argument meaning, exceptions and constants). Each round is ONE batched GPU
solve (solver.solve_batch); FSB needs only per-LP status / objective /
iterations and OBBT only the objective, dual residual and the two support
sums, so both solve with vectors=NONE and nothing but scalars crosses PCIe.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from .errors import InvalidArgument, OutOfRange
from .problem import (BatchProblem, ColumnOverride, LpProblem, ObjectiveMode, OverrideKind,
                      kInf)
from .solver import (BatchSolveSummary, BatchWorkspace, PresetColumn, SolverConfig,
                     SolveResult, SolveStatus, Vectors, solve_batch)


# ---------------------------------------------------------------------------
# strong branching (strong_branching.hpp)
# ---------------------------------------------------------------------------
@dataclass
class FsbRequest:
    problem: LpProblem
    x_rel: np.ndarray
    fractional_indices: List[int]
    integrality_tol: float = 1e-6


@dataclass
class FsbBatch:
    batch: BatchProblem
    presets: List[PresetColumn]


@dataclass
class FsbBranch:
    variable: int = 0
    up_status: SolveStatus = SolveStatus.kIterationLimit
    down_status: SolveStatus = SolveStatus.kIterationLimit
    up_objective: float = 0.0
    down_objective: float = 0.0
    delta_up: float = 0.0
    delta_down: float = 0.0
    up_flagged: bool = False
    down_flagged: bool = False
    up_iterations: int = 0
    down_iterations: int = 0
    score: float = 0.0


@dataclass
class FsbOutcome:
    root_objective: float = 0.0
    branches: List[FsbBranch] = field(default_factory=list)
    iterations: int = 0
    sparse_products: int = 0


def validate_fsb_request(req: FsbRequest) -> None:
    """strong_branching.hpp:73-92"""
    n = req.problem.num_cols()
    if len(req.x_rel) != n:
        raise InvalidArgument("fsb: relaxation point has wrong dimension")
    for i in req.fractional_indices:
        if i < 0 or i >= n:
            raise OutOfRange("fsb: fractional index out of range")
        v = float(req.x_rel[i])
        if abs(v - _cpp_round(v)) <= req.integrality_tol:
            raise InvalidArgument(f"fsb: variable {i} is not fractional")
        b = req.problem.var_bounds.at(i)
        if b.is_fixed():
            raise InvalidArgument(f"fsb: variable {i} is fixed; fixing contradicts fractionality")
        if v < b.lower - req.integrality_tol or v > b.upper + req.integrality_tol:
            raise InvalidArgument(f"fsb: relaxation value of variable {i} violates its bounds")


def _cpp_round(v: float) -> float:
    """std::round: half away from zero."""
    return math.floor(v + 0.5) if v >= 0 else -math.floor(-v + 0.5)


def build_fsb_batch(req: FsbRequest) -> FsbBatch:
    """2p columns: j raises var_j's lower bound to the ceiling, p + j lowers its
    upper bound to the floor (strong_branching.hpp:97-127)."""
    validate_fsb_request(req)
    p = len(req.fractional_indices)
    overrides: List[ColumnOverride] = []
    presets: List[PresetColumn] = []
    for j, var in enumerate(req.fractional_indices):
        base = req.problem.var_bounds.at(var)
        up = math.ceil(float(req.x_rel[var]))
        down = math.floor(float(req.x_rel[var]))
        if up > base.upper:
            presets.append(PresetColumn(j, SolveResult(status=SolveStatus.kPrimalInfeasible)))
        else:
            overrides.append(ColumnOverride(j, OverrideKind.kVariableLower, var, float(up)))
        if down < base.lower:
            presets.append(PresetColumn(p + j, SolveResult(status=SolveStatus.kPrimalInfeasible)))
        else:
            overrides.append(ColumnOverride(p + j, OverrideKind.kVariableUpper, var, float(down)))
    return FsbBatch(BatchProblem(req.problem, 2 * p, ObjectiveMode.kSharedObjective, overrides),
                    presets)


class FsbDriver:
    """Keeps the device workspace across branching rounds
    (strong_branching.hpp:131-179)."""

    def __init__(self, workspace: Optional[BatchWorkspace] = None):
        self.workspace = workspace

    def run(self, req: FsbRequest, cfg: Optional[SolverConfig] = None,
            infeasible_delta: float = 1e20) -> FsbOutcome:
        cfg = cfg or SolverConfig()
        p = len(req.fractional_indices)
        out = FsbOutcome()
        root = 0.0
        for i in range(req.problem.num_cols()):
            root += float(req.problem.objective[i]) * float(req.x_rel[i])
        out.root_objective = root
        if p == 0:
            return out
        fsb = build_fsb_batch(req)
        s = solve_batch(fsb.batch, cfg, fsb.presets, self.workspace, vectors=Vectors.NONE)
        out.iterations = s.iterations
        out.sparse_products = s.sparse_products
        for j in range(p):
            br = FsbBranch(variable=req.fractional_indices[j])
            up, down = s.per_problem[j], s.per_problem[p + j]
            br.up_status, br.down_status = up.status, down.status
            br.up_objective, br.down_objective = up.objective, down.objective
            br.up_iterations, br.down_iterations = up.iterations, down.iterations
            if up.status == SolveStatus.kPrimalInfeasible:
                br.delta_up, br.up_flagged = infeasible_delta, True
            else:
                br.delta_up = up.objective - root
            if down.status == SolveStatus.kPrimalInfeasible:
                br.delta_down, br.down_flagged = infeasible_delta, True
            else:
                br.delta_down = down.objective - root
            br.score = _cpp_max(br.delta_down, 1e-6) * _cpp_max(br.delta_up, 1e-6)
            out.branches.append(br)
        return out


def _cpp_max(a: float, b: float) -> float:
    return b if a < b else a


def run_fsb(req: FsbRequest, cfg: Optional[SolverConfig] = None,
            infeasible_delta: float = 1e20, workspace: Optional[BatchWorkspace] = None) -> FsbOutcome:
    return FsbDriver(workspace).run(req, cfg, infeasible_delta)


def score_branching(outcome: FsbOutcome, score_eps: float = 1e-6) -> List[int]:
    """Product rule, descending, ties to the smaller index
    (strong_branching.hpp:189-207)."""
    scored = [(_cpp_max(b.delta_down, score_eps) * _cpp_max(b.delta_up, score_eps), b.variable)
              for b in outcome.branches]
    scored.sort(key=lambda t: (-t[0], t[1]))
    return [v for _, v in scored]


# ---------------------------------------------------------------------------
# OBBT (obbt.hpp)
# ---------------------------------------------------------------------------
@dataclass
class ObbtConfig:
    eps_opt: float = 1e-4
    eps_dual: float = 1e-8
    min_improvement: float = 1e-4
    max_iterations: int = 100000
    cutoff: Optional[float] = None
    lenient_iteration_limit: bool = False
    solver: SolverConfig = field(default_factory=SolverConfig)

    def check(self) -> None:
        if self.eps_dual > self.eps_opt:
            raise InvalidArgument("obbt: eps_dual must not exceed eps_opt")
        if not (self.min_improvement > 0.0):
            raise InvalidArgument("obbt: min_improvement must be positive")

    def solver_config(self) -> SolverConfig:
        import dataclasses
        c = dataclasses.replace(self.solver)
        c.eps_opt = self.eps_opt
        c.eps_dual = self.eps_dual
        c.max_iterations = self.max_iterations
        return c


@dataclass
class ObbtVariable:
    variable: int = 0
    old_lower: float = -kInf
    old_upper: float = kInf
    new_lower: float = -kInf
    new_upper: float = kInf
    lower_changed: bool = False
    upper_changed: bool = False
    lower_margin: float = 0.0
    upper_margin: float = 0.0
    lower_status: SolveStatus = SolveStatus.kIterationLimit
    upper_status: SolveStatus = SolveStatus.kIterationLimit

    def changed(self) -> bool:
        return self.lower_changed or self.upper_changed


@dataclass
class ObbtOutcome:
    variables: List[ObbtVariable] = field(default_factory=list)
    changed_count: int = 0
    solved_count: int = 0
    limit_count: int = 0
    mean_reduction_pct: float = 0.0
    iterations: int = 0
    sparse_products: int = 0


@dataclass
class ObbtBatch:
    batch: BatchProblem
    presets: List[PresetColumn]


def build_obbt_batch(p: LpProblem, cfg: ObbtConfig) -> ObbtBatch:
    """Column i minimizes x_i, column n + i minimizes -x_i; fixed variables
    are preset (obbt.hpp:95-114)."""
    cfg.check()
    n = p.num_cols()
    presets: List[PresetColumn] = []
    for i in range(n):
        b = p.var_bounds.at(i)
        if not b.is_fixed():
            continue
        presets.append(PresetColumn(i, SolveResult(status=SolveStatus.kOptimal, objective=b.lower)))
        presets.append(PresetColumn(n + i, SolveResult(status=SolveStatus.kOptimal,
                                                       objective=-b.lower)))
    return ObbtBatch(BatchProblem(p, 2 * n, ObjectiveMode.kSignedUnitColumns, [], cfg.cutoff),
                     presets)


def _support_terms(r: SolveResult):
    # The device returns the two support sums of the returned triple; the
    # reference recomputes them from the vectors (obbt.hpp:123-127,133-136).
    return r.base_bound_support, r.row_support


def obbt_margin(base: LpProblem, r: SolveResult, eps: float) -> float:
    """eps (1 + |objective| + |dual support terms|), obbt.hpp:121-129."""
    if len(r.reduced_costs) or len(r.y):
        sup_r = _support(r.reduced_costs, base.var_bounds.lower, base.var_bounds.upper)
        sup_y = _support(r.y, base.row_bounds.lower, base.row_bounds.upper)
    else:
        sup_r, sup_y = _support_terms(r)
    return eps * (1.0 + abs(r.objective) + abs(sup_r + sup_y))


def obbt_dual_objective(base: LpProblem, r: SolveResult) -> float:
    """obbt.hpp:131-137"""
    if len(r.reduced_costs) or len(r.y):
        sup_r = _support(r.reduced_costs, base.var_bounds.lower, base.var_bounds.upper)
        sup_y = _support(r.y, base.row_bounds.lower, base.row_bounds.upper)
    else:
        sup_r, sup_y = _support_terms(r)
    return -(sup_r + sup_y)


def _support(v, lo, hi) -> float:
    t = 0.0
    for i in range(len(v)):
        x = float(v[i])
        t += (float(hi[i]) * x) if x > 0.0 else ((float(lo[i]) * x) if x < 0.0 else 0.0)
    return t


def certified_value(base: LpProblem, r: SolveResult, cfg: ObbtConfig) -> Optional[float]:
    """obbt.hpp:141-152"""
    if r.status == SolveStatus.kOptimal:
        return r.objective - obbt_margin(base, r, cfg.eps_opt)
    has_y = len(r.y) > 0 or r.vectors_exist
    if (cfg.lenient_iteration_limit and r.status == SolveStatus.kIterationLimit and has_y
            and r.residuals.dual <= cfg.eps_dual * 2.0):
        dual = obbt_dual_objective(base, r)
        if math.isfinite(dual):
            return dual - obbt_margin(base, r, cfg.eps_opt)
    return None


def run_obbt(p: LpProblem, cfg: Optional[ObbtConfig] = None,
             ws: Optional[BatchWorkspace] = None) -> ObbtOutcome:
    """obbt.hpp:156-223"""
    cfg = cfg or ObbtConfig()
    cfg.check()
    n = p.num_cols()
    built = build_obbt_batch(p, cfg)
    s: BatchSolveSummary = solve_batch(built.batch, cfg.solver_config(), built.presets, ws,
                                       vectors=Vectors.NONE)
    out = ObbtOutcome(iterations=s.iterations, sparse_products=s.sparse_products)
    for r in s.per_problem:
        if r.status == SolveStatus.kIterationLimit:
            out.limit_count += 1
        else:
            out.solved_count += 1
    base = built.batch.base()
    red_sum, red_cnt = 0.0, 0
    for i in range(n):
        v = ObbtVariable(variable=i, old_lower=float(p.var_bounds.lower[i]),
                         old_upper=float(p.var_bounds.upper[i]))
        v.new_lower, v.new_upper = v.old_lower, v.old_upper
        lo, hi = s.per_problem[i], s.per_problem[n + i]
        v.lower_status, v.upper_status = lo.status, hi.status
        cv = certified_value(base, lo, cfg)
        if cv is not None:
            v.lower_margin = lo.objective - cv
            if math.isfinite(cv) and cv > v.old_lower + cfg.min_improvement:
                v.new_lower, v.lower_changed = cv, True
        cv = certified_value(base, hi, cfg)
        if cv is not None:
            v.upper_margin = -cv - (-hi.objective)
            if math.isfinite(cv) and -cv < v.old_upper - cfg.min_improvement:
                v.new_upper, v.upper_changed = -cv, True
        if v.changed():
            out.changed_count += 1
            old_w = v.old_upper - v.old_lower
            if math.isfinite(old_w) and old_w > 0.0:
                red_sum += 100.0 * (old_w - (v.new_upper - v.new_lower)) / old_w
                red_cnt += 1
        out.variables.append(v)
    out.mean_reduction_pct = red_sum / red_cnt if red_cnt > 0 else 0.0
    return out


def domain_reduction_stats(o: ObbtOutcome):
    return o.changed_count, o.mean_reduction_pct
