"""Problem model: the reference's LpProblem / BatchProblem layer.

Mirrors proj/include/batchlp/problem.hpp and the data side of sparse.hpp
(same names, argument meaning and exceptions): SparseMatrix with an eager
explicit transpose (sparse.hpp:93-171), LpProblem (problem.hpp:32-40),
ColumnOverride / ObjectiveMode / BatchProblem (problem.hpp:124-195),
append_cutoff_row (problem.hpp:104-122) and resolve_column
(problem.hpp:199-252). All of this is host-side data; the solve itself runs
on the GPU (solver.py).
"""
from __future__ import annotations

import enum
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from .errors import InvalidArgument, OutOfRange

kInf = math.inf


@dataclass(frozen=True)
class Triplet:
    row: int
    col: int
    value: float


@dataclass
class Interval:
    """One component of a hyperrectangle (bounds.hpp:31-41)."""
    lower: float = -kInf
    upper: float = kInf

    def valid(self) -> bool:
        return (not math.isnan(self.lower) and not math.isnan(self.upper)
                and self.lower < kInf and self.upper > -kInf
                and self.lower <= self.upper)

    def is_fixed(self) -> bool:
        return self.lower == self.upper

    def is_free(self) -> bool:
        return self.lower == -kInf and self.upper == kInf


class Bounds:
    """Parallel lower/upper arrays (bounds.hpp:45-63)."""

    def __init__(self, n: int = 0, fill: Interval = Interval()):
        self.lower = np.full(n, fill.lower, dtype=np.float64)
        self.upper = np.full(n, fill.upper, dtype=np.float64)

    @classmethod
    def from_arrays(cls, lower, upper) -> "Bounds":
        b = cls(0)
        b.lower = np.ascontiguousarray(lower, dtype=np.float64).copy()
        b.upper = np.ascontiguousarray(upper, dtype=np.float64).copy()
        return b

    def size(self) -> int:
        return int(self.lower.shape[0])

    def at(self, i: int) -> Interval:
        return Interval(float(self.lower[i]), float(self.upper[i]))

    def set(self, i: int, v: Interval) -> None:
        self.lower[i] = v.lower
        self.upper[i] = v.upper

    def push_back(self, v: Interval) -> None:
        self.lower = np.append(self.lower, v.lower)
        self.upper = np.append(self.upper, v.upper)

    def copy(self) -> "Bounds":
        return Bounds.from_arrays(self.lower, self.upper)


_INT32_MAX = 2**31 - 1


def _index_array(a, what: str) -> np.ndarray:
    """int32 copy of an index array; values beyond int32 raise (the device
    CSR is int32, nnz <= INT32_MAX)."""
    a = np.asarray(a)
    if a.dtype.kind not in "iu":
        if a.size and not np.all(np.floor(a) == a):
            raise InvalidArgument(f"sparse: non-integer {what}")
    if a.size and (int(a.max()) > _INT32_MAX or int(a.min()) < -_INT32_MAX - 1):
        raise InvalidArgument(f"sparse: {what} exceed int32 (nnz above INT32_MAX)")
    return np.ascontiguousarray(a, dtype=np.int32)


def _check_csr(ptr: np.ndarray, idx: np.ndarray, val: np.ndarray, rows: int, cols: int):
    """Invariants of detail/csr.hpp from_csr: rows + 1 monotone offsets from
    0 to nnz, one value per index (InvalidArgument); column indices inside
    [0, cols) (OutOfRange)."""
    if (ptr.shape[0] != rows + 1 or idx.shape[0] != val.shape[0] or int(ptr[0]) != 0
            or int(ptr[-1]) != idx.shape[0] or (rows > 0 and bool(np.any(np.diff(ptr) < 0)))):
        raise InvalidArgument("sparse: malformed CSR arrays")
    if idx.size and (int(idx.min()) < 0 or int(idx.max()) >= cols):
        raise OutOfRange("sparse: column index out of range")


class SparseMatrix:
    """CSR matrix with an explicit transpose (sparse.hpp:93-171). Immutable."""

    def __init__(self, n_rows, n_cols, offsets, cols, values, t_offsets, t_cols, t_values):
        self._n_rows = int(n_rows)
        self._n_cols = int(n_cols)
        if self._n_rows < 0 or self._n_cols < 0:
            raise InvalidArgument("sparse: negative dimension")
        # the arrays are uploaded to the device as they are: check the CSR
        # invariants first (detail/csr.hpp from_csr), so malformed input
        # raises instead of reading out of bounds on the GPU
        self.row_offsets = _index_array(offsets, "offsets")
        self.col_indices = _index_array(cols, "column indices")
        self.values = np.ascontiguousarray(values, dtype=np.float64)
        self.t_row_offsets = _index_array(t_offsets, "transpose offsets")
        self.t_col_indices = _index_array(t_cols, "transpose column indices")
        self.t_values = np.ascontiguousarray(t_values, dtype=np.float64)
        _check_csr(self.row_offsets, self.col_indices, self.values, self._n_rows,
                   self._n_cols)
        _check_csr(self.t_row_offsets, self.t_col_indices, self.t_values, self._n_cols,
                   self._n_rows)
        if self.t_values.shape[0] != self.values.shape[0]:
            raise InvalidArgument("sparse: malformed CSR arrays")
        for a in (self.row_offsets, self.col_indices, self.values, self.t_row_offsets,
                  self.t_col_indices, self.t_values):
            a.flags.writeable = False

    @staticmethod
    def from_triplets(triplets: Sequence, n_rows: int, n_cols: int) -> "SparseMatrix":
        """Duplicates summed in stored order, exact zeros dropped
        (sparse.hpp:99-134). Accepts Triplet objects or (row, col, value)."""
        if n_rows < 0 or n_cols < 0:
            raise InvalidArgument("sparse: negative dimension")
        if len(triplets):
            t = np.array([(t.row, t.col, t.value) if isinstance(t, Triplet) else tuple(t)
                          for t in triplets], dtype=np.float64).reshape(-1, 3)
            r = t[:, 0].astype(np.int64)
            c = t[:, 1].astype(np.int64)
            v = t[:, 2].copy()
        else:
            r = np.zeros(0, np.int64)
            c = np.zeros(0, np.int64)
            v = np.zeros(0, np.float64)
        return SparseMatrix.from_coo(r, c, v, n_rows, n_cols)

    @staticmethod
    def from_coo(r, c, v, n_rows: int, n_cols: int) -> "SparseMatrix":
        r = np.asarray(r, dtype=np.int64)
        c = np.asarray(c, dtype=np.int64)
        v = np.asarray(v, dtype=np.float64)
        bad = (r < 0) | (r >= n_rows) | (c < 0) | (c >= n_cols)
        if bad.any():
            k = int(np.argmax(bad))
            raise OutOfRange(f"sparse: triplet index ({r[k]}, {c[k]}) out of range")
        order = np.lexsort((c, r))  # stable: row, then col, then input order
        r, c, v = r[order], c[order], v[order]
        if r.size:
            key = r * max(n_cols, 1) + c
            start = np.flatnonzero(np.r_[True, key[1:] != key[:-1]])
            end = np.r_[start[1:], key.size]
            sums = 0.0 + v[start]
            multi = np.flatnonzero(end - start > 1)
            for g in multi:  # sequential sum, as the reference loop does
                s = 0.0
                for k in range(start[g], end[g]):
                    s += float(v[k])
                sums[g] = s
            keep = sums != 0.0
            rr, cc, vv = r[start][keep], c[start][keep], sums[keep]
        else:
            rr, cc, vv = r, c, v
        offsets = np.zeros(n_rows + 1, dtype=np.int64)
        np.add.at(offsets, rr + 1, 1)
        offsets = np.cumsum(offsets)
        # transpose by a stable counting pass in row order (sparse.hpp:148-163)
        t_order = np.argsort(cc, kind="stable")
        t_offsets = np.zeros(n_cols + 1, dtype=np.int64)
        np.add.at(t_offsets, cc + 1, 1)
        t_offsets = np.cumsum(t_offsets)
        return SparseMatrix(n_rows, n_cols, offsets, cc, vv, t_offsets, rr[t_order],
                            vv[t_order])

    @staticmethod
    def from_csr(n_rows, n_cols, offsets, cols, values, t_offsets=None, t_cols=None,
                 t_values=None) -> "SparseMatrix":
        """Adopts an already canonical CSR (sorted, no duplicates, no zeros)."""
        if t_offsets is None:
            offsets = np.asarray(offsets, dtype=np.int64)
            rows = np.repeat(np.arange(n_rows, dtype=np.int64), np.diff(offsets))
            cols = np.asarray(cols, dtype=np.int64)
            values = np.asarray(values, dtype=np.float64)
            t_order = np.argsort(cols, kind="stable")
            t_offsets = np.zeros(n_cols + 1, dtype=np.int64)
            np.add.at(t_offsets, cols + 1, 1)
            t_offsets = np.cumsum(t_offsets)
            t_cols, t_values = rows[t_order], values[t_order]
        return SparseMatrix(n_rows, n_cols, offsets, cols, values, t_offsets, t_cols,
                            t_values)

    def n_rows(self) -> int:
        return self._n_rows

    def n_cols(self) -> int:
        return self._n_cols

    def nnz(self) -> int:
        return int(self.values.shape[0])

    def view(self):
        return (self._n_rows, self._n_cols, self.row_offsets, self.col_indices, self.values)

    def transpose_view(self):
        return (self._n_cols, self._n_rows, self.t_row_offsets, self.t_col_indices,
                self.t_values)

    def triplets(self):
        rows = np.repeat(np.arange(self._n_rows), np.diff(self.row_offsets))
        return rows, self.col_indices.astype(np.int64), self.values


@dataclass
class LpProblem:
    """min c'x s.t. l <= Ax <= u, xl <= x <= xu (problem.hpp:32-40)."""
    A: SparseMatrix
    objective: np.ndarray
    row_bounds: Bounds
    var_bounds: Bounds

    def num_rows(self) -> int:
        return self.A.n_rows()

    def num_cols(self) -> int:
        return self.A.n_cols()

    def copy(self) -> "LpProblem":
        return LpProblem(self.A, np.array(self.objective, dtype=np.float64),
                         self.row_bounds.copy(), self.var_bounds.copy())


def make_problem(triplets, m, n, objective, rows: Sequence, vars_: Sequence) -> LpProblem:
    """testsupport::make_problem (tests/support/instances.hpp:41-53)."""
    A = SparseMatrix.from_triplets(triplets, m, n)
    rb = Bounds(m)
    for i, iv in enumerate(rows):
        rb.set(i, iv if isinstance(iv, Interval) else Interval(*iv))
    vb = Bounds(n)
    for i, iv in enumerate(vars_):
        vb.set(i, iv if isinstance(iv, Interval) else Interval(*iv))
    return LpProblem(A, np.asarray(objective, dtype=np.float64), rb, vb)


@dataclass
class Diagnostics:
    errors: List[str] = field(default_factory=list)
    warnings: List[str] = field(default_factory=list)

    def ok(self) -> bool:
        return not self.errors


def validate(p: LpProblem) -> Diagnostics:
    """Structural checks (problem.hpp:67-100)."""
    d = Diagnostics()
    m, n = p.num_rows(), p.num_cols()
    if len(p.objective) != n:
        d.errors.append(f"objective length {len(p.objective)} does not match column count {n}")
    if p.row_bounds.size() != m:
        d.errors.append(f"row bound count {p.row_bounds.size()} does not match row count {m}")
    if p.var_bounds.size() != n:
        d.errors.append(f"variable bound count {p.var_bounds.size()} does not match column count {n}")
    for i in range(p.row_bounds.size()):
        if not p.row_bounds.at(i).valid():
            d.errors.append(f"inverted interval, row {i}")
    for i in range(p.var_bounds.size()):
        if not p.var_bounds.at(i).valid():
            d.errors.append(f"inverted interval, variable {i}")
    for i, c in enumerate(p.objective):
        if not math.isfinite(c):
            d.errors.append(f"non-finite objective entry {i}")
    for r in np.flatnonzero(np.diff(p.A.row_offsets) == 0):
        d.warnings.append(f"row {r} has no nonzeros")
    for c in np.flatnonzero(np.diff(p.A.t_row_offsets) == 0):
        d.warnings.append(f"column {c} has no nonzeros")
    return d


def append_cutoff_row(p: LpProblem, alpha: float) -> LpProblem:
    """Appends c'x <= alpha as a new last row (problem.hpp:104-122)."""
    rows, cols, vals = p.A.triplets()
    nz = np.flatnonzero(np.asarray(p.objective) != 0.0)
    r = np.concatenate([rows, np.full(nz.size, p.num_rows(), dtype=np.int64)])
    c = np.concatenate([cols, nz.astype(np.int64)])
    v = np.concatenate([vals, np.asarray(p.objective, dtype=np.float64)[nz]])
    A = SparseMatrix.from_coo(r, c, v, p.num_rows() + 1, p.num_cols())
    rb = p.row_bounds.copy()
    rb.push_back(Interval(-kInf, alpha))
    return LpProblem(A, np.array(p.objective, dtype=np.float64), rb, p.var_bounds.copy())


class OverrideKind(enum.IntEnum):
    kObjectiveEntry = 0
    kVariableLower = 1
    kVariableUpper = 2


class ObjectiveMode(enum.IntEnum):
    kSharedObjective = 0
    kSignedUnitColumns = 1


@dataclass
class ColumnOverride:
    column: int = 0
    kind: OverrideKind = OverrideKind.kVariableLower
    variable: int = 0
    value: float = 0.0


class BatchProblem:
    """N problems sharing one A (problem.hpp:141-195)."""

    def __init__(self, base: LpProblem, batch_width: int, mode: ObjectiveMode,
                 overrides: Sequence[ColumnOverride] = (), cutoff: Optional[float] = None):
        if batch_width < 0:
            raise InvalidArgument("batch: negative width")
        if mode == ObjectiveMode.kSignedUnitColumns and batch_width != 2 * base.num_cols():
            raise InvalidArgument("batch: signed unit columns require width 2n")
        self._base = append_cutoff_row(base, cutoff) if cutoff is not None else base
        self._width = int(batch_width)
        self._mode = ObjectiveMode(mode)
        self._cutoff = cutoff
        n = self._base.num_cols()
        vb = self._base.var_bounds
        for o in overrides:
            if o.column < 0 or o.column >= batch_width:
                raise OutOfRange("batch: override column out of range")
            if o.variable < 0 or o.variable >= n:
                raise OutOfRange("batch: override variable out of range")
            eff = vb.at(o.variable)
            if o.kind == OverrideKind.kVariableLower:
                eff.lower = o.value
            if o.kind == OverrideKind.kVariableUpper:
                eff.upper = o.value
            if o.kind != OverrideKind.kObjectiveEntry and not eff.valid():
                raise InvalidArgument(
                    f"batch: override inverts the bound interval of variable {o.variable}")
        self._overrides = sorted(overrides, key=lambda o: o.column)  # stable
        self._offsets = np.zeros(batch_width + 1, dtype=np.int64)
        for o in self._overrides:
            self._offsets[o.column + 1] += 1
        self._offsets = np.cumsum(self._offsets)

    def base(self) -> LpProblem:
        return self._base

    def batch_width(self) -> int:
        return self._width

    def objective_mode(self) -> ObjectiveMode:
        return self._mode

    def cutoff(self) -> Optional[float]:
        return self._cutoff

    def overrides(self) -> List[ColumnOverride]:
        return list(self._overrides)

    def overrides_for(self, column: int) -> List[ColumnOverride]:
        return self._overrides[self._offsets[column]:self._offsets[column + 1]]


class ColumnView:
    """Effective cost and bounds of one batch column (problem.hpp:199-245)."""

    def __init__(self, base: LpProblem, mode=ObjectiveMode.kSharedObjective, column=0,
                 overrides: Sequence[ColumnOverride] = ()):
        self._base = base
        self._mode = mode
        self._column = column
        self._ov = list(overrides)

    def cost(self, i: int) -> float:
        if self._mode == ObjectiveMode.kSharedObjective:
            c = float(self._base.objective[i])
        else:
            n = self._base.num_cols()
            if self._column < n:
                c = 1.0 if i == self._column else 0.0
            else:
                c = -1.0 if i == self._column - n else 0.0
        for o in self._ov:
            if o.kind == OverrideKind.kObjectiveEntry and o.variable == i:
                c = o.value
        return c

    def lower(self, i: int) -> float:
        v = float(self._base.var_bounds.lower[i])
        for o in self._ov:
            if o.kind == OverrideKind.kVariableLower and o.variable == i:
                v = o.value
        return v

    def upper(self, i: int) -> float:
        v = float(self._base.var_bounds.upper[i])
        for o in self._ov:
            if o.kind == OverrideKind.kVariableUpper and o.variable == i:
                v = o.value
        return v

    def problem(self) -> LpProblem:
        return self._base


def resolve_column(b: BatchProblem, column: int) -> ColumnView:
    if column < 0 or column >= b.batch_width():
        raise OutOfRange("resolve_column: column out of range")
    return ColumnView(b.base(), b.objective_mode(), column, b.overrides_for(column))
