"""CPU: host-side logic mirroring the reference's problem / driver tests
(test_problem.cpp, test_sparse.cpp:44-88, test_strong_branching.cpp:25-195,
test_obbt.cpp:25-63,162-188). No GPU calls."""
import math

import numpy as np
import pytest

import paper_2601_21990_b200 as bl
from paper_2601_21990_b200 import drivers as D
from paper_2601_21990_b200.problem import Interval, kInf


def test_from_triplets_sums_duplicates_drops_zeros_and_sorts():
    A = bl.SparseMatrix.from_triplets(
        [(1, 2, 1.0), (0, 1, 2.0), (1, 2, 3.0), (0, 0, 5.0), (1, 0, 1.0), (1, 0, -1.0)], 2, 3)
    assert list(A.row_offsets) == [0, 2, 3]
    assert list(A.col_indices) == [0, 1, 2]
    assert list(A.values) == [5.0, 2.0, 4.0]
    # explicit transpose (sparse.hpp:148-163)
    assert list(A.t_row_offsets) == [0, 1, 2, 3]
    assert list(A.t_col_indices) == [0, 0, 1]
    with pytest.raises(bl.OutOfRange):
        bl.SparseMatrix.from_triplets([(2, 0, 1.0)], 2, 3)
    with pytest.raises(bl.InvalidArgument):
        bl.SparseMatrix.from_triplets([], -1, 3)


def test_from_triplets_matches_reference_csr(ref):
    rng = np.random.default_rng(5)
    t = [(int(rng.integers(0, 30)), int(rng.integers(0, 40)), float(rng.integers(-3, 4)))
         for _ in range(400)]
    A = bl.SparseMatrix.from_triplets(t, 30, 40)
    p = bl.LpProblem(A, np.zeros(40), bl.Bounds(30), bl.Bounds(40))
    # rebuild from the triplet list inside the reference
    r = ref.RefLp.from_problem(p).to_problem()
    for a, b in ((A.row_offsets, r.A.row_offsets), (A.col_indices, r.A.col_indices),
                 (A.values, r.A.values), (A.t_col_indices, r.A.t_col_indices),
                 (A.t_values, r.A.t_values)):
        assert np.array_equal(a, b)


def test_batch_problem_validation_messages():
    p = bl.make_problem([(0, 0, 1.0), (0, 1, 1.0)], 1, 2, [-1.0, -1.0], [(-kInf, 1.0)],
                        [(0.0, 1.0), (0.0, 1.0)])
    with pytest.raises(bl.InvalidArgument, match="negative width"):
        bl.BatchProblem(p, -1, bl.ObjectiveMode.kSharedObjective)
    with pytest.raises(bl.InvalidArgument, match="require width 2n"):
        bl.BatchProblem(p, 3, bl.ObjectiveMode.kSignedUnitColumns)
    with pytest.raises(bl.OutOfRange, match="override column"):
        bl.BatchProblem(p, 2, bl.ObjectiveMode.kSharedObjective,
                        [bl.ColumnOverride(2, bl.OverrideKind.kVariableLower, 0, 0.5)])
    with pytest.raises(bl.OutOfRange, match="override variable"):
        bl.BatchProblem(p, 2, bl.ObjectiveMode.kSharedObjective,
                        [bl.ColumnOverride(0, bl.OverrideKind.kVariableLower, 5, 0.5)])
    with pytest.raises(bl.InvalidArgument, match="inverts the bound interval of variable 1"):
        bl.BatchProblem(p, 2, bl.ObjectiveMode.kSharedObjective,
                        [bl.ColumnOverride(1, bl.OverrideKind.kVariableLower, 1, 2.0)])


def test_column_view_applies_overrides_in_list_order():
    p = bl.make_problem([(0, 0, 1.0)], 1, 2, [3.0, 4.0], [(-kInf, 1.0)],
                        [(0.0, 5.0), (0.0, 5.0)])
    b = bl.BatchProblem(p, 3, bl.ObjectiveMode.kSharedObjective, [
        bl.ColumnOverride(2, bl.OverrideKind.kVariableUpper, 0, 2.0),
        bl.ColumnOverride(1, bl.OverrideKind.kObjectiveEntry, 1, -7.0),
        bl.ColumnOverride(2, bl.OverrideKind.kVariableUpper, 0, 1.5)])
    v = bl.resolve_column(b, 2)
    assert v.upper(0) == 1.5 and v.lower(0) == 0.0 and v.cost(0) == 3.0
    assert bl.resolve_column(b, 1).cost(1) == -7.0
    s = bl.BatchProblem(p, 4, bl.ObjectiveMode.kSignedUnitColumns)
    assert [bl.resolve_column(s, 1).cost(i) for i in range(2)] == [0.0, 1.0]
    assert [bl.resolve_column(s, 2).cost(i) for i in range(2)] == [-1.0, 0.0]


def test_append_cutoff_row_matches_reference(ref):
    p = ref.test_lp(0, 7)
    a = bl.append_cutoff_row(p, 2.5)
    b = ref.append_cutoff(p, 2.5)
    assert a.num_rows() == p.num_rows() + 1
    assert np.array_equal(a.A.col_indices, b.A.col_indices)
    assert np.array_equal(a.A.values, b.A.values)
    assert np.array_equal(a.row_bounds.upper, b.row_bounds.upper)


def knapsack():
    return bl.make_problem([(0, 0, 2.0), (0, 1, 3.0), (0, 2, 1.0)], 1, 3, [-3.0, -4.0, -2.0],
                           [(-kInf, 4.0)], [(0.0, 1.0)] * 3)


def test_fsb_batch_layout_ups_first_downs_second():
    """test_strong_branching.cpp:25-51"""
    p = knapsack()
    req = bl.FsbRequest(p, np.array([1.0, 2.0 / 3.0, 0.4]), [1, 2])
    fb = bl.build_fsb_batch(req)
    assert fb.batch.batch_width() == 4 and not fb.presets
    for j, (kind, var, val) in enumerate([(bl.OverrideKind.kVariableLower, 1, 1.0),
                                          (bl.OverrideKind.kVariableLower, 2, 1.0),
                                          (bl.OverrideKind.kVariableUpper, 1, 0.0),
                                          (bl.OverrideKind.kVariableUpper, 2, 0.0)]):
        ov = fb.batch.overrides_for(j)
        assert len(ov) == 1 and (ov[0].kind, ov[0].variable, ov[0].value) == (kind, var, val)


def test_fsb_request_validation():
    """test_strong_branching.cpp:53-92"""
    p = knapsack()
    with pytest.raises(bl.InvalidArgument, match="wrong dimension"):
        bl.build_fsb_batch(bl.FsbRequest(p, np.zeros(2), [0]))
    with pytest.raises(bl.OutOfRange):
        bl.build_fsb_batch(bl.FsbRequest(p, np.zeros(3), [3]))
    with pytest.raises(bl.InvalidArgument, match="not fractional"):
        bl.build_fsb_batch(bl.FsbRequest(p, np.array([0.0, 1.0, 0.5]), [1]))
    q = knapsack()
    q.var_bounds.set(1, Interval(0.5, 0.5))
    with pytest.raises(bl.InvalidArgument, match="is fixed"):
        bl.build_fsb_batch(bl.FsbRequest(q, np.array([0.0, 0.5, 0.0]), [1]))
    # a rounded bound past the base interval is preset infeasible
    r = bl.make_problem([(0, 0, 1.0)], 1, 1, [1.0], [(-kInf, 5.0)], [(0.2, 0.7)])
    fb = bl.build_fsb_batch(bl.FsbRequest(r, np.array([0.5]), [0]))
    assert sorted(pc.column for pc in fb.presets) == [0, 1]
    assert all(pc.result.status == bl.SolveStatus.kPrimalInfeasible for pc in fb.presets)


def test_score_branching_product_rule_and_ties():
    """test_strong_branching.cpp:168-195"""
    o = D.FsbOutcome()
    for var, du, dd in ((3, 2.0, 2.0), (1, 4.0, 1.0), (2, 0.0, 100.0), (0, 1e20, 0.5)):
        o.branches.append(D.FsbBranch(variable=var, delta_up=du, delta_down=dd))
    # scores: 4, 4, 1e-6*100, 0.5e20 -> var 0 first, then the tie 1 < 3
    assert bl.score_branching(o) == [0, 1, 3, 2]


def test_obbt_batch_layout_fixed_presets_and_cutoff():
    """test_obbt.cpp:25-63"""
    p = bl.make_problem([(0, 0, 1.0), (0, 1, 1.0), (0, 2, 1.0)], 1, 3, [1.0, 2.0, 0.0],
                        [(-kInf, 4.0)], [(0.0, 3.0), (1.5, 1.5), (0.0, 2.0)])
    ob = bl.build_obbt_batch(p, bl.ObbtConfig())
    assert ob.batch.batch_width() == 6
    assert ob.batch.objective_mode() == bl.ObjectiveMode.kSignedUnitColumns
    pre = {pc.column: pc.result for pc in ob.presets}
    assert sorted(pre) == [1, 4]
    assert pre[1].objective == 1.5 and pre[4].objective == -1.5
    cut = bl.build_obbt_batch(p, bl.ObbtConfig(cutoff=3.0))
    assert cut.batch.base().num_rows() == 2
    assert cut.batch.base().row_bounds.upper[1] == 3.0
    with pytest.raises(bl.InvalidArgument, match="eps_dual"):
        bl.ObbtConfig(eps_opt=1e-6, eps_dual=1e-5).check()


def test_obbt_lenient_certified_value_kat():
    """test_obbt.cpp:162-188: dual objective 0 minus eps (1 + |0.3| + 0)."""
    p = bl.make_problem([(0, 0, 1.0), (0, 1, 1.0)], 1, 2, [1.0, 1.0], [(-kInf, 1.0)],
                        [(0.0, 10.0), (0.0, 10.0)])
    r = bl.SolveResult(status=bl.SolveStatus.kIterationLimit, objective=0.3)
    r.y = np.array([0.0])
    r.reduced_costs = np.array([-1.0, 0.0])
    r.residuals.dual = 1e-12
    assert D.certified_value(p, r, bl.ObbtConfig()) is None
    v = D.certified_value(p, r, bl.ObbtConfig(lenient_iteration_limit=True))
    assert v == pytest.approx(-1.3e-4, rel=1e-9)
    r.residuals.dual = 1e-3
    assert D.certified_value(p, r, bl.ObbtConfig(lenient_iteration_limit=True)) is None


def test_solver_config_check_messages():
    c = bl.SolverConfig(beta_sufficient=0.9)
    with pytest.raises(bl.InvalidArgument, match="beta_s < beta_n"):
        c.check()
    with pytest.raises(bl.InvalidArgument, match="theta"):
        bl.SolverConfig(theta=0.0).check()
    with pytest.raises(bl.InvalidArgument, match="check period"):
        bl.SolverConfig(termination_check_period=0).check()
    with pytest.raises(bl.InvalidArgument, match="negative iteration"):
        bl.SolverConfig(max_iterations=-1).check()
    with pytest.raises(bl.InvalidArgument, match="tolerances"):
        bl.SolverConfig(eps_opt=0.0).check()
    assert bl.SolverConfig(eps_dual=-1.0, eps_opt=3e-4).effective_eps_dual() == 3e-4


def test_column_slices_cover_the_batch():
    from paper_2601_21990_b200.distributed import column_slices
    for width, world in ((10, 3), (4000, 8), (3, 4), (0, 2)):
        s = column_slices(width, world)
        assert len(s) == world and s[0][0] == 0 and s[-1][1] == width
        assert all(a[1] == b[0] for a, b in zip(s, s[1:]))
        assert max(e - b for b, e in s) - min(e - b for b, e in s) <= 1


def test_sparse_matrix_rejects_malformed_csr():
    """Raw CSR input is validated before it can reach the device
    (detail/csr.hpp from_csr): malformed arrays -> InvalidArgument, column
    index out of range -> OutOfRange."""
    ok = dict(n_rows=2, n_cols=3, offsets=[0, 1, 2], cols=[0, 2], values=[1.0, 2.0],
              t_offsets=[0, 1, 1, 2], t_cols=[0, 1], t_values=[1.0, 2.0])
    bl.SparseMatrix(**ok)  # well formed
    for k, v in (("offsets", [0, 2, 1]), ("offsets", [1, 1, 2]), ("offsets", [0, 1]),
                 ("values", [1.0]), ("t_offsets", [0, 1, 1, 3]), ("offsets", [0, 1, 3]),
                 ("cols", [0, 2**33])):
        bad = dict(ok)
        bad[k] = v
        with pytest.raises(bl.InvalidArgument):
            bl.SparseMatrix(**bad)
    for k, v in (("cols", [0, 3]), ("cols", [-1, 2]), ("t_cols", [0, 2])):
        bad = dict(ok)
        bad[k] = v
        with pytest.raises(bl.OutOfRange):
            bl.SparseMatrix(**bad)
    with pytest.raises(bl.InvalidArgument):
        bl.SparseMatrix(-1, 3, [0], [], [], [0, 0, 0, 0], [], [])


def test_resolve_column_out_of_range_is_out_of_range():
    A = bl.SparseMatrix.from_triplets([(0, 0, 1.0)], 1, 1)
    p = bl.LpProblem(A, np.zeros(1), bl.Bounds(1), bl.Bounds(1))
    b = bl.BatchProblem(p, 2, bl.ObjectiveMode.kSharedObjective)
    with pytest.raises(bl.OutOfRange):
        bl.resolve_column(b, 2)
    with pytest.raises(bl.OutOfRange):
        bl.resolve_column(b, -1)
