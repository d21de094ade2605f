"""Batch-width tuning on the device (reference tuner.hpp:33-139).

Same entries, report, tie rule and CSV as the reference. The timed products
are the solver's own device SpMM kernels (bl_measure_spmm: CUDA-event time
of R products A X plus R products A'Y per candidate width), so the chosen
width is the cheapest per column on this GPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import IO, List, Optional, Sequence, Tuple

import numpy as np

from . import _native as N
from .errors import InvalidArgument, LogicError
from .problem import LpProblem, SparseMatrix
from .solver import BatchWorkspace, _bounds, _check, default_workspace


@dataclass
class TuneEntry:
    width: int = 0
    total_s: float = 0.0       # R products A X plus R products A'Y
    per_column_s: float = 0.0  # total_s / width


def choose_width(entries: Sequence[TuneEntry]) -> int:
    """Lowest time per column; exact ties go to the larger width
    (tuner.hpp:42-51)."""
    if not entries:
        raise InvalidArgument("tuner: no candidates")
    best = entries[0]
    for e in entries[1:]:
        if (e.per_column_s, -e.width) < (best.per_column_s, -best.width):
            best = e
    return best.width


@dataclass
class TuneReport:
    entries: List[TuneEntry] = field(default_factory=list)
    chosen_width: int = 0
    repetitions: int = 10
    overhead_clamped: bool = False

    def validate(self) -> None:
        """tuner.hpp:59-65."""
        if choose_width(self.entries) != self.chosen_width:
            raise LogicError("tuner: chosen width inconsistent with entries")
        if any(e.total_s < 0.0 or e.per_column_s < 0.0 for e in self.entries):
            raise LogicError("tuner: negative measured time")


def measure_spmm(a: SparseMatrix, width: int, repetitions: int = 10, *,
                 workspace: Optional[BatchWorkspace] = None) -> Tuple[float, float, bool]:
    """(total seconds, seconds per column, overhead clamped) of `repetitions`
    products each way on the device (tuner.hpp:71-108)."""
    if width < 1:
        raise InvalidArgument("tuner: width must be >= 1")
    if repetitions < 3:
        raise InvalidArgument("tuner: need >= 3 repetitions")
    ws = workspace or default_workspace()
    p = LpProblem(a, np.zeros(a.n_cols()), _bounds(a.n_rows()), _bounds(a.n_cols()))
    dp = ws.resident(p, cache=False)
    total, per_col, clamped = C.c_double(), C.c_double(), C.c_int32()
    _check(ws.ctx.handle, N.lib().bl_measure_spmm(ws.ctx.handle, dp.handle, int(width),
                                                  int(repetitions), C.byref(total),
                                                  C.byref(per_col), C.byref(clamped)))
    return total.value, per_col.value, bool(clamped.value)


def tune_batch_width(a: SparseMatrix, candidates: Sequence[int], repetitions: int = 10, *,
                     workspace: Optional[BatchWorkspace] = None) -> TuneReport:
    """tuner.hpp:110-126."""
    if not candidates:
        raise InvalidArgument("tuner: no candidates")
    report = TuneReport(repetitions=repetitions)
    for w in candidates:
        total, per_col, clamped = measure_spmm(a, w, repetitions, workspace=workspace)
        report.overhead_clamped = report.overhead_clamped or clamped
        report.entries.append(TuneEntry(int(w), total, per_col))
    report.chosen_width = choose_width(report.entries)
    report.validate()
    return report


def default_tune_widths() -> List[int]:
    return [32, 64, 128, 256, 512, 1024, 2048]


def write_tune_csv(os: IO[str], report: TuneReport) -> None:
    """tuner.hpp:132-139 (C++ ostream formatting of doubles: 6 significant digits)."""
    os.write("width,total_s,per_column_s,chosen\n")
    for e in report.entries:
        os.write(f"{e.width},{e.total_s:.6g},{e.per_column_s:.6g},"
                 f"{1 if e.width == report.chosen_width else 0}\n")
