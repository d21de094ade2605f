"""Per-kind device time in iteration windows of a solve: runs the workload
with successive iteration caps and prints, per window, the time per loop
pass and per kernel kind (diagnostic; prints only).

  python scripts/window_profile.py c2 0,64,256,512,1024,100000
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2601_21990_b200 as bl  # noqa: E402
from paper_2601_21990_b200 import instances as I  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
caps = [int(c) for c in (sys.argv[2] if len(sys.argv) > 2 else "0,64,256,512,1024,100000").split(",")]
p, batch, presets, cfg, spec = bench.build_workload(name, bl, I)
bl.solve_batch(batch, cfg, presets, vectors=bl.Vectors.NONE)  # warm


def run(cap):
    if cap <= 0:
        return None
    cfg.max_iterations = cap
    return bl.solve_batch(batch, cfg, presets, vectors=bl.Vectors.NONE)


tag = " ".join(f"{k}={os.environ[k]}" for k in sorted(os.environ) if k.startswith("BATCHLP_"))
print(f"{name} K={batch.batch_width()} {tag}")
prev = None
for cap in caps:
    cur = run(cap)
    if cur is None:
        prev = None
        continue
    passes = cur.loop_passes - (prev.loop_passes if prev else 0)
    ms = cur.device_ms - (prev.device_ms if prev else 0.0)
    done = sum(1 for r in cur.per_problem if int(r.status) != 3)
    line = f"  ..{cap:6d}: {passes:6d} passes {ms:9.2f} ms {1e3 * ms / max(passes, 1):8.2f} us/pass finished={done}"
    parts = []
    for k in ("primal", "dual", "decide", "check", "cert", "compact", "snapshot",
              "tail_primal", "tail_dual", "tail_decide"):
        lf, nf, _ = cur.profile.get(k, (0, 0, 0))
        lp, np_, _ = prev.profile.get(k, (0, 0, 0)) if prev else (0, 0, 0)
        if lf - lp > 0:
            parts.append(f"{k}={(nf - np_) / max(passes, 1) / 1e3:.2f}")
    print(line + "  [us/pass " + " ".join(parts) + "]", flush=True)
    prev = cur
    if cur.iterations < cap:
        break
