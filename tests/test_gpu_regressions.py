"""GPU regressions for round-1 advisor findings, against the compiled
reference (oracle/_ref)."""
import numpy as np
import pytest

import paper_2601_21990_b200 as bl
from paper_2601_21990_b200 import instances as I

pytestmark = pytest.mark.gpu


def _presets(ps):
    return [(q.column, int(q.result.status), q.result.objective) for q in ps]


def _same(got, want, exact_iterations=True):
    if exact_iterations:
        assert got.iterations == want.iterations
    for g, w in zip(got.per_problem, want.per_problem):
        assert int(g.status) == w.status
        assert abs(g.iterations - w.iterations) <= 0.1 * max(w.iterations, 1)
        if w.status in (0, 3):
            assert abs(g.objective - w.objective) <= 1e-6 * (1 + abs(w.objective))


def test_tall_wide_batch_sizes_the_partials(ref):
    """m >> n with K = 1024 on a fresh context: the initial AX = A X picks
    more work items per column block than the row kernels do, and its
    partials must fit (the buffer used to be sized from the row kernels
    only). Capped at 70 iterations (one termination check) vs the reference."""
    p = I.boxed_feasible(50000, 1000, 10, 3)
    x, frac = I.synthetic_branch_point(p, 512)
    fb = bl.build_fsb_batch(bl.FsbRequest(p, x, frac))
    cfg = bl.SolverConfig()
    cfg.max_iterations = 70
    ws = bl.BatchWorkspace(0)  # fresh context: buffers sized by this solve
    got = bl.solve_batch(fb.batch, cfg, fb.presets, ws, vectors=bl.Vectors.NONE)
    want = ref.solve_batch(p, fb.batch.batch_width(), 0, fb.batch.overrides(), cfg,
                           _presets(fb.presets), vectors=False)
    assert fb.batch.batch_width() == 1024
    _same(got, want)


def test_cached_problem_sees_edited_bounds(ref):
    """A workspace caches the device copy of a problem; a solve after an
    in-place bound edit (same A and objective objects) must use the new
    bounds, as the reference (LpProblem by value) does."""
    p = I.set_cover(60, 90, 0.08, 4)
    ws = bl.BatchWorkspace(0)
    cfg = bl.SolverConfig()
    batch = bl.BatchProblem(p, 4, bl.ObjectiveMode.kSharedObjective)
    first = bl.solve_batch(batch, cfg, (), ws, vectors=bl.Vectors.NONE)
    p.var_bounds.set(0, bl.Interval(1.0, 1.0))  # fix x0 = 1 in place
    p.var_bounds.set(1, bl.Interval(0.0, 0.0))
    p.row_bounds.set(2, bl.Interval(2.0, bl.kInf))
    batch2 = bl.BatchProblem(p, 4, bl.ObjectiveMode.kSharedObjective)
    got = bl.solve_batch(batch2, cfg, (), ws, vectors=bl.Vectors.NONE)
    want = ref.solve_batch(p, 4, 0, [], cfg, [], vectors=False)
    _same(got, want)
    assert any(g.objective != f.objective for g, f in zip(got.per_problem, first.per_problem))
