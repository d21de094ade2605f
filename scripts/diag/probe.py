"""Diagnostics: GPU vs reference on tiny LPs and C1 (prints, never asserts)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2601_21990_b200 as bl
from paper_2601_21990_b200 import instances as I
from oracle import ref

def cfg(**kw):
    c = bl.SolverConfig()
    for k, v in kw.items(): setattr(c, k, v)
    return c

mode = os.environ.get("BATCHLP_STEP_MODE", "0")
print("step mode", mode, flush=True)
p = ref.test_lp(10, 0)
t = time.time(); g = bl.solve(p, cfg(eps_opt=1e-6)); r = ref.solve(p, cfg(eps_opt=1e-6))
print("two_var", g.status, g.iterations, g.objective, "| ref", r.per_problem[0].status, r.iterations, r.per_problem[0].objective, time.time()-t, flush=True)
for shape in (0, 1, 2):
    same = 0; bad = []
    for seed in range(1, 21):
        p = ref.test_lp(shape, seed)
        g = bl.solve(p, cfg(eps_opt=1e-6)); r = ref.solve(p, cfg(eps_opt=1e-6)); rr = r.per_problem[0]
        ok = int(g.status) == rr.status and g.iterations == rr.iterations and (g.objective == rr.objective or (np.isnan(g.objective) and np.isnan(rr.objective)))
        same += ok
        if not ok:
            bad.append((seed, int(g.status), rr.status, g.iterations, rr.iterations, g.objective, rr.objective, g.restarts, rr.restarts))
            b = bl.BatchProblem(p, 1, bl.ObjectiveMode.kSharedObjective, [])
            s = bl.solve_batch(b, cfg(eps_opt=1e-6))
            print("  eta", s.eta, r.eta, s.eta == r.eta)
            gl = [(e.at_iteration, int(e.reason), e.residual, e.anchor_residual) for e in s.restart_log]
            for k, (a, c) in enumerate(zip(gl, r.restart_log)):
                if a != c:
                    print("  first restart diff", k, a, c); break
            else:
                print("  restart logs equal", len(gl), len(r.restart_log))
    print("shape", shape, "exact", same, "/20", bad[:5], flush=True)
pc = I.config_problem("c1")
t = time.time(); rr = ref.solve(pc); print("ref root", time.time()-t, rr.iterations, flush=True)
t = time.time(); g = bl.solve(pc); el = time.time()-t
print("gpu root", el, g.status, g.iterations, g.objective, "ref", rr.per_problem[0].objective, rr.iterations, flush=True)
x = rr.per_problem[0].x
frac = I.pick_fractional(x, 16)
req = bl.FsbRequest(pc, x, frac)
for k in range(2):
    t = time.time(); o = bl.run_fsb(req); el = time.time() - t
    print("gpu fsb", el, o.iterations, flush=True)
w = ref.run_fsb(pc, x, frac)
print("ref fsb its", w["iterations"])
for j, b in enumerate(o.branches):
    print(j, int(b.up_status), w["up_status"][j], b.up_iterations, w["up_iterations"][j], b.up_objective - w["up_objective"][j], "|", int(b.down_status), w["down_status"][j], b.down_iterations, w["down_iterations"][j], b.down_objective - w["down_objective"][j])
