"""Multi-GPU batched solve: column sharding with one final gather.

One process per GPU (torch.distributed). The batch's LP columns are split
into contiguous slices, one per rank; A is replicated; each rank runs its own
device-resident solve_batch with no collective in the iteration loop; at the
end one all_gather of the per-LP scalars (status, iterations, restarts,
objective, residuals, supports) reassembles the batch in original column
order on every rank.

Semantics: restarts synchronize on the SLICE's averaged residual, so a
G-slice run equals G independent reference solve_batch runs on the same
slices (the parity definition for G > 1), not one whole-batch run.

Signed-unit batches (OBBT, problem.hpp:134-137) are sliced by rewriting the
slice as a shared-objective batch with a zero base objective and one
objective-entry override per column (+1 / -1 on its variable): the same LPs,
expressible for any column subset.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from .problem import BatchProblem, ColumnOverride, LpProblem, ObjectiveMode, OverrideKind
from .solver import (BatchSolveSummary, PresetColumn, Residuals, SolverConfig, SolveResult,
                     SolveStatus, Vectors)


def column_slices(width: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous near-equal slices [start, stop) of range(width)."""
    base, extra = divmod(width, world)
    out, s = [], 0
    for r in range(world):
        e = s + base + (1 if r < extra else 0)
        out.append((s, e))
        s = e
    return out


@dataclass
class Shard:
    batch: BatchProblem
    presets: List[PresetColumn]
    start: int
    stop: int


def shard_batch(batch: BatchProblem, presets: Sequence[PresetColumn], rank: int,
                world: int) -> Shard:
    """This rank's slice of the batch as a standalone BatchProblem."""
    start, stop = column_slices(batch.batch_width(), world)[rank]
    width = stop - start
    base = batch.base()
    ovs: List[ColumnOverride] = []
    if batch.objective_mode() == ObjectiveMode.kSignedUnitColumns:
        n = base.num_cols()
        zero = LpProblem(base.A, np.zeros(n), base.row_bounds, base.var_bounds)
        for j in range(start, stop):
            var, sign = (j, 1.0) if j < n else (j - n, -1.0)
            ovs.append(ColumnOverride(j - start, OverrideKind.kObjectiveEntry, var, sign))
        for o in batch.overrides():
            if start <= o.column < stop:
                ovs.append(ColumnOverride(o.column - start, o.kind, o.variable, o.value))
        sub = BatchProblem(zero, width, ObjectiveMode.kSharedObjective, ovs)
    else:
        for o in batch.overrides():
            if start <= o.column < stop:
                ovs.append(ColumnOverride(o.column - start, o.kind, o.variable, o.value))
        sub = BatchProblem(base, width, ObjectiveMode.kSharedObjective, ovs)
    pre = [PresetColumn(p.column - start, p.result) for p in presets
           if start <= p.column < stop]
    return Shard(sub, pre, start, stop)


# per-LP scalar record exchanged by the final gather
_FIELDS = ("status", "iterations", "restarts", "objective", "gap", "primal", "dual",
           "fixed_point", "bound_support", "row_support", "base_bound_support",
           "vectors_exist")


def pack(results: Sequence[SolveResult]) -> np.ndarray:
    a = np.zeros((len(results), len(_FIELDS)), dtype=np.float64)
    for i, r in enumerate(results):
        a[i] = (int(r.status), r.iterations, r.restarts, r.objective, r.residuals.gap,
                r.residuals.primal, r.residuals.dual, r.residuals.fixed_point,
                r.bound_support, r.row_support, r.base_bound_support, float(r.vectors_exist))
    return a


def unpack(a: np.ndarray) -> List[SolveResult]:
    out = []
    for row in a:
        r = SolveResult()
        r.status = SolveStatus(int(row[0]))
        r.iterations = int(row[1])
        r.restarts = int(row[2])
        r.objective = float(row[3])
        r.residuals = Residuals(float(row[4]), float(row[5]), float(row[6]), float(row[7]))
        r.bound_support, r.row_support, r.base_bound_support = (float(row[8]), float(row[9]),
                                                                float(row[10]))
        r.vectors_exist = bool(row[11])
        out.append(r)
    return out


def gather_results(local: np.ndarray, slices: Sequence[Tuple[int, int]], device=None,
                   group=None) -> np.ndarray:
    """all_gather of the per-LP records (one collective, after the loop).
    Ranks hold unequal slices; each pads to the largest slice."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rows = max(e - s for s, e in slices)
    buf = np.zeros((rows, len(_FIELDS)), dtype=np.float64)
    buf[:local.shape[0]] = local
    t = torch.from_numpy(buf)
    if device is not None:
        t = t.to(device)
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t, group=group)
    parts = [o.cpu().numpy()[:e - s] for o, (s, e) in zip(outs, slices)]
    return np.concatenate(parts, axis=0)


def solve_batch_sharded(batch: BatchProblem, cfg: Optional[SolverConfig] = None,
                        presets: Sequence[PresetColumn] = (), *, rank: int, world: int,
                        solver=None, device=None, group=None) -> BatchSolveSummary:
    """Runs this rank's slice and returns the whole batch's per-LP scalars on
    every rank. `solver(shard, cfg)` defaults to the GPU solve_batch with
    vectors=NONE; tests substitute the reference to check the plumbing."""
    shard = shard_batch(batch, presets, rank, world)
    if solver is None:
        from .solver import solve_batch
        local = solve_batch(shard.batch, cfg, shard.presets, vectors=Vectors.NONE)
    else:
        local = solver(shard, cfg)
    slices = column_slices(batch.batch_width(), world)
    allrec = gather_results(pack(local.per_problem), slices, device, group)
    out = BatchSolveSummary()
    out.per_problem = unpack(allrec)
    import torch
    import torch.distributed as dist
    its = torch.tensor([local.iterations, local.restarts, local.sparse_products],
                       dtype=torch.int64, device=device)
    dist.all_reduce(its, op=dist.ReduceOp.MAX, group=group)
    out.iterations, out.restarts, out.sparse_products = (int(v) for v in its.cpu())
    return out
