"""batchlp-b200: B200-native batched PDHG LP solving (strong branching / OBBT).

A drop-in for the reference's hot path ``batchlp::solve_batch``: the same
API surface (problem.py, solver.py, drivers.py) over a C-ABI
(include/batchlp_cuda.h) whose implementation is hand-written sm_100a CUDA
(csrc/). There is no CPU fallback.
"""
from .errors import DeviceError, DomainError, InvalidArgument, LogicError, OutOfRange
from .problem import (BatchProblem, Bounds, ColumnOverride, ColumnView, Interval, LpProblem,
                      ObjectiveMode, OverrideKind, SparseMatrix, Triplet, append_cutoff_row,
                      kInf, make_problem, resolve_column, validate)
from .solver import (BatchSolveSummary, BatchWorkspace, InfeasibilityProbe, PresetColumn,
                     Residuals, RestartEvent, RestartReason, SolveResult, SolverConfig,
                     SolveStatus, Vectors, WarmStart, solve, solve_batch, solve_batch_sharded,
                     spectral_norm, spmm, spmv, step_size_for)
from .drivers import (FsbBranch, FsbDriver, FsbOutcome, FsbRequest, ObbtConfig, ObbtOutcome,
                      ObbtVariable, build_fsb_batch, build_obbt_batch, certified_value,
                      run_fsb, run_obbt, score_branching)

from .tuner import (TuneEntry, TuneReport, choose_width, default_tune_widths, measure_spmm,
                    tune_batch_width, write_tune_csv)

__all__ = [n for n in dir() if not n.startswith("_")]
