"""One solve of a config workload (for ncu captures / quick timing)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2601_21990_b200 as bl
from paper_2601_21990_b200 import instances as I
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
p, batch, presets, cfg, spec = bench.build_workload(name, bl, I)
if os.environ.get("MAXIT"):
    cfg.max_iterations = int(os.environ["MAXIT"])
for _ in range(reps):
    t = time.time()
    s = bl.solve_batch(batch, cfg, presets, vectors=bl.Vectors.NONE)
    el = time.time() - t
    print(f"{name}: K={batch.batch_width()} its={s.iterations} passes={s.loop_passes} "
          f"wall={el*1e3:.1f}ms dev={s.device_ms:.1f}ms us/pass={s.device_ms*1e3/max(s.loop_passes,1):.1f}",
          flush=True)
    for k, (l, ns, by) in s.profile.items():
        if l:
            print(f"   {k:9s} launches={int(l):6d} avg={ns/l/1e3:8.2f}us  total={ns/1e6:8.2f}ms  GB/s={by/ns if ns else 0:8.1f}")
