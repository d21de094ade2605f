import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2601_21990_b200 as bl
from paper_2601_21990_b200 import instances as I
from oracle import ref
pc = I.config_problem("c1")
rr = ref.solve(pc)
x = rr.per_problem[0].x
frac = I.pick_fractional(x, 16)
fb = bl.build_fsb_batch(bl.FsbRequest(pc, x, frac))
def run(K, cfg, cols=None):
    ovs = [o for o in fb.batch.overrides() if o.column < K]
    b = bl.BatchProblem(pc, K, bl.ObjectiveMode.kSharedObjective, ovs)
    g = bl.solve_batch(b, cfg, vectors=bl.Vectors.NONE)
    r = ref.solve_batch(pc, K, 0, ovs, cfg, vectors=False)
    print(f"K={K} its gpu {g.iterations} ref {r.iterations} restarts {g.restarts} {r.restarts}")
    print("  gpu", [(int(p.status), p.iterations) for p in g.per_problem])
    print("  ref", [(p.status, p.iterations) for p in r.per_problem])
    print("  objdiff", max(abs(a.objective - b.objective) / (1 + abs(b.objective)) for a, b in zip(g.per_problem, r.per_problem)))
c = bl.SolverConfig(); c.termination_check_period = 100000; c.max_iterations = 1500
run(32, c)
c = bl.SolverConfig()
for K in (3, 4, 8):
    run(K, c)
