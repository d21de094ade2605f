"""GPU parity beyond round 1's suites, against the compiled reference
(oracle/_ref) and the pinned C restatement (oracle/batchlp_oracle.c):

* C4 (the north-star shape, m = 100k, n = 200k, 2M nonzeros) and C3
  (m = 50k, n = 100k): a branch slice of the real strong-branching batch
  solved TO CONVERGENCE (1e-4 KKT) on the full matrix: status identical,
  objective within 1e-6 relative, per-LP iterations within 10 %.
* a wide batch (600 LPs, > 256 active for hundreds of iterations): pins the
  batch mean, which the device sums as a fixed tree once more than 256
  columns are active (reference: a sequential sum, batch_solver.hpp:209-222)
  -- the restart decisions it drives must land on the same iterations.
* run_obbt on C2 through the Python mirror: every tightened bound, change
  flag and status against the reference's run_obbt (obbt.hpp:156-223,
  tests/golden/c2_obbt_bounds.json).
* the broken-step-size branch (solver.hpp:250-263): with eta above 1/||A||
  the device raises DomainError exactly where the C restatement reports
  BL_ERR_DOMAIN (the reference cannot override eta; its own KAT of the rule,
  test_solver.cpp:139-145, runs in the C++ suites).
"""
import json
import os

import numpy as np
import pytest

import paper_2601_21990_b200 as bl
from paper_2601_21990_b200 import instances as I

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module", autouse=True)
def _threads():
    # the reference's own thread pool (sparse.hpp:198-206) on every host core
    old = os.environ.get("BATCHLP_THREADS")
    os.environ["BATCHLP_THREADS"] = str(os.cpu_count() or 1)
    yield
    if old is None:
        os.environ.pop("BATCHLP_THREADS", None)
    else:
        os.environ["BATCHLP_THREADS"] = old


def _presets(ps):
    return [(q.column, int(q.result.status), q.result.objective) for q in ps]


def _compare(got, want):
    assert len(got.per_problem) == len(want.per_problem)
    assert abs(got.iterations - want.iterations) <= 0.1 * max(want.iterations, 1)
    for j, (g, w) in enumerate(zip(got.per_problem, want.per_problem)):
        assert int(g.status) == w.status, j
        assert abs(g.iterations - w.iterations) <= 0.1 * max(w.iterations, 1), j
        if np.isfinite(w.objective):
            assert abs(g.objective - w.objective) <= 1e-6 * (1 + abs(w.objective)), j


def _fsb_slice(name, pairs):
    """The first `pairs` branch pairs of the config's strong-branching batch
    (x = 0.5 on the branched columns, acceptance.cpp:209-212)."""
    p = I.config_problem(name)
    x, frac = I.synthetic_branch_point(p, pairs)
    fb = bl.build_fsb_batch(bl.FsbRequest(p, x, frac))
    return p, fb


@pytest.mark.parametrize("name,pairs", [("c4", 4), ("c3", 4)])
def test_fsb_slice_converged_matches_reference(ref, name, pairs):
    p, fb = _fsb_slice(name, pairs)
    cfg = bl.SolverConfig()
    got = bl.solve_batch(fb.batch, cfg, fb.presets, vectors=bl.Vectors.NONE)
    want = ref.solve_batch(p, fb.batch.batch_width(), 0, fb.batch.overrides(), cfg,
                           _presets(fb.presets), vectors=False)
    assert fb.batch.batch_width() == 2 * pairs
    assert all(r.status != 3 for r in want.per_problem)  # converged, not capped
    _compare(got, want)


def test_wide_batch_tree_mean_matches_reference(ref):
    """600 OBBT LPs of C2 (min / max of the first 300 variables)."""
    import bench
    p = I.config_problem("c2")
    ob = bl.build_obbt_batch(p, bl.ObbtConfig())
    n = p.num_cols()
    cols = list(range(300)) + list(range(n, n + 300))
    lp, batch, presets = bench.subset_batch(bl, ob.batch, ob.presets, cols)
    cfg = bl.ObbtConfig().solver_config()
    got = bl.solve_batch(batch, cfg, presets, vectors=bl.Vectors.NONE)
    want = ref.solve_batch(lp, batch.batch_width(), 0, batch.overrides(), cfg,
                           _presets(presets), vectors=False)
    _compare(got, want)
    # the restarts the (tree-summed) mean triggered are the reference's
    assert got.restarts == want.restarts
    glog = [(e.at_iteration, int(e.reason)) for e in got.restart_log]
    wlog = [(e[0], e[1]) for e in want.restart_log]
    assert glog == wlog


def test_run_obbt_c2_bounds_match_reference_golden():
    with open(os.path.join(GOLDEN, "c2_obbt_bounds.json")) as f:
        g = json.load(f)
    o = bl.run_obbt(I.config_problem("c2"), bl.ObbtConfig())
    assert (o.changed_count, o.solved_count, o.limit_count) == (
        g["changed_count"], g["solved_count"], g["limit_count"])
    for i, v in enumerate(o.variables):
        assert (int(v.lower_changed), int(v.upper_changed)) == (
            g["lower_changed"][i], g["upper_changed"][i]), i
        assert (int(v.lower_status), int(v.upper_status)) == (
            g["lower_status"][i], g["upper_status"][i]), i
        for got, want in ((v.new_lower, g["new_lower"][i]), (v.new_upper, g["new_upper"][i])):
            w = float.fromhex(want)
            assert abs(got - w) <= 1e-6 * (1 + abs(w)), i


# LPs of testsupport::random_lp (shape, seed) and step-size factors k
# (eta = k / ||A||) for which the pinned C restatement reports BL_ERR_DOMAIN
DOMAIN_CASES = [(0, 3, 2.0), (0, 10, 2.0), (0, 12, 1.5), (0, 17, 3.0)]


@pytest.mark.parametrize("shape,seed,k", DOMAIN_CASES)
def test_broken_step_size_raises_domain_error(ref, shape, seed, k):
    from oracle import port
    from paper_2601_21990_b200.errors import DomainError
    p = ref.test_lp(shape, seed)
    eta = k / bl.spectral_norm(p.A)
    cfg = bl.SolverConfig()
    cfg.max_iterations = 300
    to_c = cfg.to_c

    def with_eta(*a, **kw):  # the C restatement reads bl_config.eta
        c = to_c(*a, **kw)
        c.eta = eta
        return c
    cfg.to_c = with_eta
    with pytest.raises(RuntimeError, match="code 3"):
        port.solve_batch(p, 1, cfg=cfg)
    cfg.to_c = to_c
    batch = bl.BatchProblem(p, 1, bl.ObjectiveMode.kSharedObjective)
    with pytest.raises(DomainError, match="step size exceeds"):
        bl.solve_batch(batch, cfg, (), vectors=bl.Vectors.NONE, eta=eta)
    # the same solve at the reference's own step size is fine
    bl.solve_batch(batch, cfg, (), vectors=bl.Vectors.NONE)


def _slices(width, g):
    base, extra = divmod(width, g)
    out, s = [], 0
    for r in range(g):
        e = s + base + (1 if r < extra else 0)
        out.append((s, e))
        s = e
    return out


def _sharded_case(kind):
    if kind == "fsb":  # C1 strong branching (the reference's root point)
        with open(os.path.join(GOLDEN, "c1_fsb.json")) as f:
            g = json.load(f)
        p = I.config_problem("c1")
        x = np.array([float.fromhex(v) for v in g["x_rel"]])
        fb = bl.build_fsb_batch(bl.FsbRequest(p, x, g["fractional"]))
        return fb.batch, fb.presets, bl.SolverConfig()
    p = I.boxed_feasible(300, 300, 10, 5)  # OBBT: a signed-unit batch of 600
    ob = bl.build_obbt_batch(p, bl.ObbtConfig())
    return ob.batch, ob.presets, bl.ObbtConfig().solver_config()


@pytest.mark.parametrize("kind", ["fsb", "obbt"])
def test_sharded_contexts_match_reference_slices(ref, kind):
    """Two contexts on one B200 (bl_solve_batch_sharded):
    every slice equals the reference's solve_batch on that slice, and is
    bit-identical to a single-context device solve of the same slice (a
    signed-unit slice is solved in place through the unit offset; the
    single-context run gets it rewritten as objective-entry overrides)."""
    import bench
    batch, presets, cfg = _sharded_case(kind)
    ws = [bl.BatchWorkspace(0), bl.BatchWorkspace(0)]
    got = bl.solve_batch_sharded(batch, cfg, presets, ws)
    assert len(got.per_problem) == batch.batch_width()
    for b, e in _slices(batch.batch_width(), 2):
        lp, sb, sp = bench.subset_batch(bl, batch, presets, list(range(b, e)))
        want = ref.solve_batch(lp, sb.batch_width(), 0, sb.overrides(), cfg, _presets(sp),
                               vectors=False)
        one = bl.solve_batch(sb, cfg, sp, vectors=bl.Vectors.NONE)
        sl = got.per_problem[b:e]
        for j, (g, w, o) in enumerate(zip(sl, want.per_problem, one.per_problem)):
            assert int(g.status) == w.status, (b, j)
            assert abs(g.iterations - w.iterations) <= 0.1 * max(w.iterations, 1), (b, j)
            if np.isfinite(w.objective):
                assert abs(g.objective - w.objective) <= 1e-6 * (1 + abs(w.objective)), (b, j)
            assert (int(g.status), g.iterations) == (int(o.status), o.iterations), (b, j)
            assert g.objective == o.objective or (np.isnan(g.objective) and np.isnan(o.objective))
