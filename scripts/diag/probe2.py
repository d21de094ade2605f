"""Where does the batched trajectory leave the reference's? (prints only)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2601_21990_b200 as bl
from paper_2601_21990_b200 import instances as I
from oracle import ref

def logs(g, r, label):
    gl = [(e.at_iteration, int(e.reason), e.residual, e.anchor_residual) for e in g.restart_log]
    print(label, "gpu its", g.iterations, "restarts", g.restarts, "| ref its", r.iterations, r.restarts)
    for k, (a, c) in enumerate(zip(gl, r.restart_log)):
        if a != c:
            print("  first diff at restart", k, "gpu", a, "ref", c)
            print("  prev", gl[k-1] if k else None)
            return
    print("  logs equal over", min(len(gl), len(r.restart_log)))

pc = I.config_problem("c1")
rr = ref.solve(pc)
x = rr.per_problem[0].x
frac = I.pick_fractional(x, 16)
req = bl.FsbRequest(pc, x, frac)
fb = bl.build_fsb_batch(req)
cfg = bl.SolverConfig()
for K in (1, 2, 4, 32):
    b = bl.BatchProblem(pc, K, bl.ObjectiveMode.kSharedObjective, [])
    g = bl.solve_batch(b, cfg, vectors=bl.Vectors.NONE)
    r = ref.solve_batch(pc, K, 0, [], cfg, vectors=False)
    logs(g, r, f"copies K={K}")
    print("   per-col its", [p.iterations for p in g.per_problem][:4], [p.iterations for p in r.per_problem][:4])
for K in (1, 2, 32):
    ovs = [o for o in fb.batch.overrides() if o.column < K]
    b = bl.BatchProblem(pc, K, bl.ObjectiveMode.kSharedObjective, ovs)
    g = bl.solve_batch(b, cfg, vectors=bl.Vectors.NONE)
    r = ref.solve_batch(pc, K, 0, ovs, cfg, vectors=False)
    logs(g, r, f"fsb first K={K}")
    print("   per-col its", [p.iterations for p in g.per_problem][:8], [p.iterations for p in r.per_problem][:8])
