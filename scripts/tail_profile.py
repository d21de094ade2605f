"""Per-kind device time of the tail of a solve: runs the workload with an
iteration cap and uncapped, and prints (full - capped) per kernel kind per
loop pass (diagnostic; prints only).

  python scripts/tail_profile.py c2 1024
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2601_21990_b200 as bl  # noqa: E402
from paper_2601_21990_b200 import instances as I  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cap = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
p, batch, presets, cfg, spec = bench.build_workload(name, bl, I)
bl.solve_batch(batch, cfg, presets, vectors=bl.Vectors.NONE)  # warm
full = bl.solve_batch(batch, cfg, presets, vectors=bl.Vectors.NONE)
cfg.max_iterations = cap
part = bl.solve_batch(batch, cfg, presets, vectors=bl.Vectors.NONE)
passes = full.loop_passes - part.loop_passes
print(f"{name} loop={os.environ.get('BATCHLP_LOOP', 'auto')} tail after {cap} its: "
      f"{passes} passes, {full.device_ms - part.device_ms:.2f} ms, "
      f"{1e3 * (full.device_ms - part.device_ms) / max(passes, 1):.2f} us/pass")
for k in full.profile:
    lf, nf, _ = full.profile[k]
    lp, np_, _ = part.profile.get(k, (0, 0, 0))
    if lf - lp > 0:
        print(f"   {k:9s} launches={int(lf - lp):6d} avg={(nf - np_) / (lf - lp) / 1e3:8.2f}us "
              f"per-pass={(nf - np_) / max(passes, 1) / 1e3:8.2f}us")
