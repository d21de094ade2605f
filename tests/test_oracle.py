"""CPU: pin the oracles. The plain-C restatement (oracle/port) must equal the
golden vectors produced by the compiled reference (tests/golden/), bit for
bit, and the compiled reference must still produce those vectors."""
import json
import os

import numpy as np
import pytest

import paper_2601_21990_b200 as bl
from paper_2601_21990_b200 import instances as I

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def port():
    from oracle import port as P
    if not P.available():
        pytest.fail("oracle/_build/libbatchlp_oracle.so missing: run __graft_entry__.build()")
    return P


def _tiny_cfg():
    c = bl.SolverConfig()
    c.eps_opt = 1e-6
    c.trace_iterates = True
    return c


def test_port_reproduces_reference_tiny_goldens(ref, port):
    """180 seeded fixture LPs (tests/support/instances.hpp families): status,
    iterations, objective, restarts, products and trajectory hash exact."""
    cfg = _tiny_cfg()
    for case in gold("tiny_solve.json")["cases"]:
        p = ref.test_lp(case["shape"], case["seed"])
        s, res, *_ = port.solve_batch(p, 1, 0, [], cfg)
        r = res[0]
        assert r.status == case["status"], case
        assert r.iterations == case["iterations"], case
        assert r.objective.hex() == case["objective"], case
        assert s.restarts == case["restarts"], case
        assert s.sparse_products == case["sparse_products"], case
        assert str(s.trajectory_hash) == case["hash"], case


def test_reference_still_produces_tiny_goldens(ref):
    cfg = _tiny_cfg()
    for case in gold("tiny_solve.json")["cases"][::7]:
        p = ref.test_lp(case["shape"], case["seed"])
        r = ref.solve(p, cfg)
        assert r.per_problem[0].objective.hex() == case["objective"]
        assert str(r.trajectory_hash) == case["hash"]


def test_spectral_norm_goldens(port):
    g = gold("spectral.json")
    for k in ("diag", "upper2", "rank1"):
        A = bl.SparseMatrix.from_triplets([tuple(t) for t in g[k]["triplets"]], *g[k]["dims"])
        p = bl.LpProblem(A, np.zeros(A.n_cols()), bl.Bounds(A.n_rows()), bl.Bounds(A.n_cols()))
        assert port.spectral_norm(p).hex() == g[k]["norm"]
    assert port.spectral_norm(I.config_problem("c1")).hex() == g["c1"]["norm"]
    # KATs of test_sparse.cpp:159-185
    assert float.fromhex(g["diag"]["norm"]) == pytest.approx(4.04, rel=1e-3)
    assert float.fromhex(g["upper2"]["norm"]) / 1.01 == pytest.approx(1.618033988749895,
                                                                      rel=1e-3)


def test_port_reproduces_c1_strong_branching_golden(port):
    """BASELINE configs[0]: 32 FSB LPs on generate_set_cover(1000, 2000,
    0.01, 1), every per-LP result exact."""
    g = gold("c1_fsb.json")
    p = I.config_problem("c1")
    x = np.array([float.fromhex(v) for v in g["x_rel"]])
    assert I.pick_fractional(x, 16) == g["fractional"]
    fb = bl.build_fsb_batch(bl.FsbRequest(p, x, g["fractional"]))
    s, res, *_ = port.solve_batch(p, 32, 0, fb.batch.overrides(), bl.SolverConfig())
    assert s.iterations == g["iterations"] == 9088
    assert s.restarts == g["restarts"]
    assert s.sparse_products == g["sparse_products"]
    for r, c in zip(res, g["columns"]):
        assert (r.status, r.iterations, r.objective.hex()) == (
            c["status"], c["iterations"], c["objective"])


def test_c2_golden_shape():
    """BASELINE configs[1] reference run: 4000 OBBT LPs, all optimal."""
    g = gold("c2_obbt.json")
    assert len(g["columns"]) == 4000
    assert all(c["status"] == 0 for c in g["columns"])
    assert g["iterations"] == max(c["iterations"] for c in g["columns"])


def test_port_spmm_equals_reference(ref, port):
    rng = np.random.default_rng(3)
    p = I.set_cover(60, 90, 0.1, 4)
    for transpose in (False, True):
        rin = p.A.n_rows() if transpose else p.A.n_cols()
        X = rng.standard_normal((rin, 5))
        a = port.spmm(p, X, transpose, 3)
        b = ref.spmm(p, X, transpose, 3)
        assert np.array_equal(a.view(np.int64), b.view(np.int64))
