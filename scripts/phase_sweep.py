"""Where does a config's solve time go? Runs the workload with increasing
iteration caps and prints the device time of each iteration window, the
active width reached and the loop driver (diagnostic; prints only).

  python scripts/phase_sweep.py c2 [graph|persistent|auto]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2601_21990_b200 as bl  # noqa: E402
from paper_2601_21990_b200 import instances as I  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
if len(sys.argv) > 2 and sys.argv[2] != "auto":
    os.environ["BATCHLP_LOOP"] = sys.argv[2]
p, batch, presets, cfg, spec = bench.build_workload(name, bl, I)
caps = [64, 128, 256, 512, 1024, 2048, 4096, 8192, 16384, 100000]
prev_ms, prev_cap = 0.0, 0
s = bl.solve_batch(batch, cfg, presets, vectors=bl.Vectors.NONE)  # warm
full_its = s.iterations
print(f"{name} loop={os.environ.get('BATCHLP_LOOP', 'auto')} K={batch.batch_width()} "
      f"full: its={s.iterations} dev={s.device_ms:.2f}ms", flush=True)
for cap in caps:
    cfg.max_iterations = cap
    best = None
    for _ in range(2):
        s = bl.solve_batch(batch, cfg, presets, vectors=bl.Vectors.NONE)
        best = s.device_ms if best is None else min(best, s.device_ms)
    done = sum(1 for r in s.per_problem if int(r.status) != 3)
    win = max(min(cap, s.iterations) - prev_cap, 1)
    print(f"  cap={cap:6d} its={s.iterations:6d} dev={best:9.2f}ms finished={done:5d} "
          f"window={best - prev_ms:9.2f}ms  us/iter={1e3 * (best - prev_ms) / win:8.2f}",
          flush=True)
    prev_ms, prev_cap = best, min(cap, s.iterations)
    if cap >= full_its:
        break
