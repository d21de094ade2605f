"""Regenerates tests/golden/*.json from the compiled reference (oracle/_ref,
i.e. the unmodified reference headers). Run in the build container where
/root/reference exists:  python tests/golden/make_golden.py

Floats are stored as hex (float.hex) so comparisons are bit-exact.
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2601_21990_b200 as bl  # noqa: E402
from paper_2601_21990_b200 import instances as I  # noqa: E402
from oracle import ref  # noqa: E402


def hx(v):
    return float(v).hex()


def cols(summary):
    return [{"status": c.status, "iterations": c.iterations, "objective": hx(c.objective),
             "restarts": c.restarts} for c in summary.per_problem]


def write(name, obj):
    with open(os.path.join(HERE, name), "w") as f:
        json.dump(obj, f, separators=(",", ":"))
    print("wrote", name)


def tiny():
    cfg = bl.SolverConfig()
    cfg.eps_opt = 1e-6
    cfg.trace_iterates = True
    out = []
    for shape in (0, 1, 2):
        for seed in range(1, 61):
            p = ref.test_lp(shape, seed)
            r = ref.solve(p, cfg)
            c = r.per_problem[0]
            out.append({"shape": shape, "seed": seed, "status": c.status,
                        "iterations": c.iterations, "objective": hx(c.objective),
                        "restarts": r.restarts, "hash": str(r.trajectory_hash),
                        "sparse_products": r.sparse_products})
    write("tiny_solve.json", {"source": "reference solve(), eps_opt 1e-6, trace_iterates",
                              "fixtures": "testsupport::random_lp(shape, seed)",
                              "cases": out})


def spectral():
    mats = {
        "diag": [(0, 0, 3.0), (1, 1, 4.0)],
        "upper2": [(0, 0, 1.0), (0, 1, 1.0), (1, 1, 1.0)],
        "rank1": [(i, j, [1.0, -2.0, 0.5][i] * [3.0, 1.0][j]) for i in range(3) for j in range(2)],
    }
    dims = {"diag": (2, 2), "upper2": (2, 2), "rank1": (3, 2)}
    out = {}
    for k, t in mats.items():
        A = bl.SparseMatrix.from_triplets(t, *dims[k])
        p = bl.LpProblem(A, np.zeros(A.n_cols()), bl.Bounds(A.n_rows()), bl.Bounds(A.n_cols()))
        out[k] = {"triplets": t, "dims": dims[k], "norm": hx(ref.spectral_norm(p))}
    out["c1"] = {"norm": hx(ref.spectral_norm(I.config_problem("c1")))}
    write("spectral.json", out)


def c1():
    p = I.config_problem("c1")
    t = time.time()
    root = ref.solve(p)
    x = root.per_problem[0].x
    frac = I.pick_fractional(x, 16)
    fb = bl.build_fsb_batch(bl.FsbRequest(p, x, frac))
    s = ref.solve_batch(p, 32, 0, fb.batch.overrides(), bl.SolverConfig(), vectors=False)
    write("c1_fsb.json", {
        "source": "reference solve() root + solve_batch on build_fsb_batch, default config",
        "instance": "generate_set_cover(1000, 2000, 0.01, 1)",
        "root": {"iterations": root.iterations, "objective": hx(root.per_problem[0].objective)},
        "fractional": frac, "x_rel": [hx(v) for v in x],
        "iterations": s.iterations, "restarts": s.restarts,
        "sparse_products": s.sparse_products, "columns": cols(s),
        "seconds": time.time() - t})


def c2():
    p = I.config_problem("c2")
    ob = bl.build_obbt_batch(p, bl.ObbtConfig())
    cfg = bl.ObbtConfig().solver_config()
    t = time.time()
    s = ref.solve_batch(p, ob.batch.batch_width(), 1, [], cfg,
                        [(q.column, int(q.result.status), q.result.objective)
                         for q in ob.presets], vectors=False)
    write("c2_obbt.json", {
        "source": "reference solve_batch on build_obbt_batch (eps_opt 1e-4, eps_dual 1e-8)",
        "instance": "bl_gen_boxed_feasible(2000, 2000, 10, 11)",
        "iterations": s.iterations, "restarts": s.restarts,
        "sparse_products": s.sparse_products, "columns": cols(s),
        "seconds": time.time() - t, "threads": os.environ.get("BATCHLP_THREADS", "1")})


def c2_bounds():
    """The reference run_obbt (obbt.hpp:156-223) on C2: every tightened
    bound, its change flag, margin and status, and the counts."""
    p = I.config_problem("c2")
    t = time.time()
    o = ref.run_obbt(p)
    write("c2_obbt_bounds.json", {
        "source": "reference run_obbt, ObbtConfig{} (eps_opt 1e-4, eps_dual 1e-8, "
                  "min_improvement 1e-4)",
        "instance": "bl_gen_boxed_feasible(2000, 2000, 10, 11)",
        "changed_count": o["changed_count"], "solved_count": o["solved_count"],
        "limit_count": o["limit_count"], "iterations": o["iterations"],
        "mean_reduction_pct": hx(o["mean_reduction_pct"]),
        "new_lower": [hx(v) for v in o["new_lower"]],
        "new_upper": [hx(v) for v in o["new_upper"]],
        "lower_changed": o["lower_changed"].tolist(),
        "upper_changed": o["upper_changed"].tolist(),
        "lower_status": o["lower_status"].tolist(),
        "upper_status": o["upper_status"].tolist(),
        "seconds": time.time() - t, "threads": os.environ.get("BATCHLP_THREADS", "1")})


if __name__ == "__main__":
    os.environ.setdefault("BATCHLP_THREADS", str(os.cpu_count() or 1))
    which = sys.argv[1:] or ["tiny", "spectral", "c1", "c2"]
    for w in which:
        globals()[w]()
