"""C1 FSB with a bounded iteration count (for ncu launch lists)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2601_21990_b200 as bl
from paper_2601_21990_b200 import instances as I
pc = I.config_problem("c1")
root = bl.solve(pc)
frac = I.pick_fractional(root.x, 16)
req = bl.FsbRequest(pc, root.x, frac)
cfg = bl.SolverConfig()
cfg.max_iterations = int(os.environ.get("MAXIT", "100000"))
for k in range(int(os.environ.get("REPS", "2"))):
    t = time.time(); o = bl.run_fsb(req, cfg); el = time.time() - t
    print("fsb", el, o.iterations, el / max(o.iterations, 1) * 1e6, "us/iter", flush=True)
