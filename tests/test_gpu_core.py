"""GPU parity of the core kernels and solve_batch against the compiled
reference (oracle/_ref). Every call goes through the C-ABI."""
import math

import numpy as np
import pytest

import paper_2601_21990_b200 as bl
from paper_2601_21990_b200 import instances as I

pytestmark = pytest.mark.gpu


def random_sparse(rng, m, n, density):
    mask = rng.random((m, n)) < density
    r, c = np.nonzero(mask)
    v = rng.uniform(-1.0, 1.0, size=r.size)
    return bl.SparseMatrix.from_coo(r, c, v, m, n)


def as_problem(A):
    return bl.LpProblem(A, np.zeros(A.n_cols()), bl.Bounds(A.n_rows()), bl.Bounds(A.n_cols()))


@pytest.mark.parametrize("width,active", [(1, 1), (3, 3), (8, 5), (33, 33), (70, 41)])
@pytest.mark.parametrize("transpose", [False, True])
def test_spmm_bitwise_equals_reference(ref, width, active, transpose):
    """SpMM == reference csr_apply bit for bit, trailing columns untouched
    (test_sparse.cpp:109-135)."""
    rng = np.random.default_rng(width * 7 + active + transpose)
    A = random_sparse(rng, 300, 200, 0.05)
    rin = A.n_rows() if transpose else A.n_cols()
    rout = A.n_cols() if transpose else A.n_rows()
    X = rng.standard_normal((rin, width))
    out0 = rng.standard_normal((rout, width))
    got = bl.spmm(A, X, out0.copy(), transpose, active)
    want = ref.spmm(as_problem(A), X, transpose, active, out0.copy())
    assert np.array_equal(got.view(np.int64), want.view(np.int64))
    assert np.array_equal(got[:, active:], out0[:, active:])


def test_spectral_norm_known_values(ref):
    """test_sparse.cpp:159-185 KATs, and equality with the reference."""
    diag = bl.SparseMatrix.from_triplets([(0, 0, 3.0), (1, 1, 4.0)], 2, 2)
    assert bl.spectral_norm(diag) == pytest.approx(4.04, rel=1e-3)
    tri = bl.SparseMatrix.from_triplets([(0, 0, 1.0), (0, 1, 1.0), (1, 1, 1.0)], 2, 2)
    assert bl.spectral_norm(tri) / 1.01 == pytest.approx(1.618033988749895, rel=1e-3)
    u, v = [1.0, -2.0, 0.5], [3.0, 1.0]
    r1 = bl.SparseMatrix.from_triplets([(i, j, u[i] * v[j]) for i in range(3) for j in range(2)],
                                       3, 2)
    nu = sum(e * e for e in u)
    nv = sum(e * e for e in v)
    assert bl.spectral_norm(r1) / 1.01 == pytest.approx(math.sqrt(nu * nv), rel=1e-9)
    for A in (diag, tri, r1):
        assert bl.spectral_norm(A) == ref.spectral_norm(as_problem(A))
    with pytest.raises(bl.InvalidArgument):
        bl.spectral_norm(bl.SparseMatrix.from_triplets([], 3, 3))


def test_spectral_norm_c1_close_to_reference(ref):
    p = I.config_problem("c1")
    got = bl.spectral_norm(p.A)
    want = ref.spectral_norm(p)
    assert abs(got - want) <= 1e-12 * want


def _cfg(**kw):
    c = bl.SolverConfig()
    for k, v in kw.items():
        setattr(c, k, v)
    return c


@pytest.mark.parametrize("shape", [0, 1, 2])
def test_single_solve_matches_reference(ref, shape):
    """solve() on the seeded fixture families vs the reference solve: status
    identical, iterations within 10 %, objective within 1e-6 relative."""
    cfg = _cfg(eps_opt=1e-6)
    exact = 0
    for seed in range(1, 41):
        p = ref.test_lp(shape, seed)
        g = bl.solve(p, cfg)
        r = ref.solve(p, cfg).per_problem[0]
        assert int(g.status) == r.status, seed
        assert abs(g.iterations - r.iterations) <= 0.1 * max(r.iterations, 1), seed
        if r.status == 0:
            assert abs(g.objective - r.objective) <= 1e-6 * (1 + abs(r.objective)), seed
        exact += (g.iterations == r.iterations and g.objective == r.objective)
    assert exact >= 30  # ULP-level drift may only come from exp/log in weight updates


def test_c1_strong_branching_matches_reference(ref):
    p = I.config_problem("c1")
    root = ref.solve(p).per_problem[0]
    frac = I.pick_fractional(root.x, 16)
    req = bl.FsbRequest(p, root.x, frac)
    got = bl.run_fsb(req)
    want = ref.run_fsb(p, root.x, frac)
    for j, br in enumerate(got.branches):
        assert int(br.up_status) == want["up_status"][j]
        assert int(br.down_status) == want["down_status"][j]
        for g, w in ((br.up_objective, want["up_objective"][j]),
                     (br.down_objective, want["down_objective"][j])):
            assert abs(g - w) <= 1e-6 * (1 + abs(w))
        for g, w in ((br.up_iterations, want["up_iterations"][j]),
                     (br.down_iterations, want["down_iterations"][j])):
            assert abs(g - w) <= 0.1 * w
    assert abs(got.iterations - want["iterations"]) <= 0.1 * want["iterations"]


@pytest.mark.parametrize("loop", ["graph", "persistent", "cluster", "step"])
def test_loop_drivers_agree_with_reference_c1(ref, loop, monkeypatch):
    """Every loop driver (CUDA graph with conditional nodes, cooperative
    persistent grid, single thread-block cluster, host-stepped) runs the same
    device control logic: C1 strong branching matches the reference."""
    monkeypatch.setenv("BATCHLP_LOOP", loop)
    p = I.config_problem("c1")
    root = ref.solve(p).per_problem[0]
    frac = I.pick_fractional(root.x, 16)
    got = bl.run_fsb(bl.FsbRequest(p, root.x, frac))
    want = ref.run_fsb(p, root.x, frac)
    for j, br in enumerate(got.branches):
        assert int(br.up_status) == want["up_status"][j]
        assert int(br.down_status) == want["down_status"][j]
        assert abs(br.up_objective - want["up_objective"][j]) <= 1e-6 * (1 + abs(want["up_objective"][j]))
        assert abs(br.down_objective - want["down_objective"][j]) <= 1e-6 * (1 + abs(want["down_objective"][j]))
        assert abs(br.up_iterations - want["up_iterations"][j]) <= 0.1 * want["up_iterations"][j]
        assert abs(br.down_iterations - want["down_iterations"][j]) <= 0.1 * want["down_iterations"][j]
