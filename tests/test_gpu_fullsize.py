"""GPU parity at BASELINE.json's full problem sizes.

The reference CPU path cannot solve the big configurations in test time
(hours at C4), so parity there is checked through
  * size-independent properties of the products at C4 size (m = 100k,
    n = 200k): bitwise equality of sampled rows with the reference
    summation order, and the adjoint identity <A X, Y> = <X, A' Y>;
  * column slices of the real workloads against the compiled reference
    (oracle/_ref) on the full matrices: C3 capped at 128 iterations, C5
    solved to convergence (status identical, objective 1e-6 relative,
    iterations within 10 %).
"""
import numpy as np
import pytest

import paper_2601_21990_b200 as bl
from paper_2601_21990_b200 import instances as I

pytestmark = pytest.mark.gpu


def _csr_rows(A, rows, X, transpose):
    """Reference summation (csr_apply, sparse.hpp:176-183): per row, the
    stored nonzero order, separately rounded products and sums."""
    rp = A.t_row_offsets if transpose else A.row_offsets
    ci = A.t_col_indices if transpose else A.col_indices
    cv = A.t_values if transpose else A.values
    out = np.zeros((len(rows), X.shape[1]))
    for k, i in enumerate(rows):
        acc = np.zeros(X.shape[1])
        for q in range(rp[i], rp[i + 1]):
            acc = acc + cv[q] * X[ci[q]]
        out[k] = acc
    return out


@pytest.fixture(scope="module")
def c4_matrix():
    return I.config_problem("c4").A


@pytest.mark.parametrize("transpose", [False, True])
def test_c4_spmm_sampled_rows_bitwise(c4_matrix, transpose):
    A = c4_matrix
    rng = np.random.default_rng(3 + transpose)
    rin = A.n_rows() if transpose else A.n_cols()
    rout = A.n_cols() if transpose else A.n_rows()
    K = 40  # two column blocks, the second partly active
    X = rng.standard_normal((rin, K))
    out0 = rng.standard_normal((rout, K))
    got = bl.spmm(A, X, out0.copy(), transpose, 37)
    rows = np.sort(rng.choice(rout, 300, replace=False))
    want = _csr_rows(A, rows, X[:, :37], transpose)
    assert np.array_equal(got[rows, :37].view(np.int64), want.view(np.int64))
    assert np.array_equal(got[:, 37:], out0[:, 37:])


def test_c4_adjoint_identity(c4_matrix):
    A = c4_matrix
    rng = np.random.default_rng(11)
    X = rng.standard_normal((A.n_cols(), 8))
    Y = rng.standard_normal((A.n_rows(), 8))
    AX = bl.spmm(A, X)
    ATY = bl.spmm(A, Y, None, True)
    lhs = np.einsum("ij,ij->j", AX, Y)
    rhs = np.einsum("ij,ij->j", X, ATY)
    assert np.all(np.abs(lhs - rhs) <= 1e-10 * np.abs(lhs).max())


def _slice_batch(name, pairs):
    p = I.config_problem(name)
    x, frac = I.synthetic_branch_point(p, pairs)
    fb = bl.build_fsb_batch(bl.FsbRequest(p, x, frac))
    return p, fb


def _compare(got, want, rel_obj=1e-6):
    assert abs(got.iterations - want.iterations) <= 0.1 * max(want.iterations, 1)
    for g, w in zip(got.per_problem, want.per_problem):
        assert int(g.status) == w.status
        assert abs(g.iterations - w.iterations) <= 0.1 * max(w.iterations, 1)
        if np.isfinite(w.objective):
            assert abs(g.objective - w.objective) <= rel_obj * (1 + abs(w.objective))


def test_c3_slice_capped_matches_reference(ref):
    """C3 (m = 50k, n = 100k, 1M nonzeros): 4 branch pairs, 128 iterations."""
    p, fb = _slice_batch("c3", 4)
    cfg = bl.SolverConfig()
    cfg.max_iterations = 128
    got = bl.solve_batch(fb.batch, cfg, fb.presets, vectors=bl.Vectors.NONE)
    want = ref.solve_batch(p, fb.batch.batch_width(), 0, fb.batch.overrides(), cfg,
                           [(q.column, int(q.result.status), q.result.objective)
                            for q in fb.presets], vectors=False)
    _compare(got, want)


def test_c5_slice_converged_matches_reference(ref):
    """C5 (m = 20k, n = 40k): one branch pair solved to 1e-4 KKT."""
    p, fb = _slice_batch("c5", 1)
    cfg = bl.SolverConfig()
    got = bl.solve_batch(fb.batch, cfg, fb.presets, vectors=bl.Vectors.NONE)
    want = ref.solve_batch(p, fb.batch.batch_width(), 0, fb.batch.overrides(), cfg,
                           [(q.column, int(q.result.status), q.result.objective)
                            for q in fb.presets], vectors=False)
    _compare(got, want)
