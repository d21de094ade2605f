"""Where the end-to-end (host API) time of a C2 solve goes (run under gpurun)."""
import os, sys, time
import ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_2601_21990_b200 as bl
from paper_2601_21990_b200 import instances as I, _native as N
from paper_2601_21990_b200.solver import BatchWorkspace

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
p, batch, presets, cfg, spec = bench.build_workload(name, bl, I)
ws = BatchWorkspace()
for cache in (True, False, False, True):
    t0 = time.perf_counter()
    s = bl.solve_batch(batch, cfg, presets, ws, vectors=bl.Vectors.NONE, cache_problem=cache)
    t1 = time.perf_counter()
    print(f"cache={cache}: wall {1e3*(t1-t0):8.2f} ms  device {s.device_ms:8.2f} ms  its={s.iterations}")
# components
base = batch.base()
t0 = time.perf_counter(); dp = ws.resident(base, cache=False); t1 = time.perf_counter()
print(f"upload (resident, uncached): {1e3*(t1-t0):.2f} ms")
L = N.lib()
out = C.c_double()
t0 = time.perf_counter(); rc = L.bl_spectral_norm(ws.ctx.handle, dp.handle, C.byref(out)); t1 = time.perf_counter()
print(f"spectral norm: {1e3*(t1-t0):.2f} ms (rc={rc}, {out.value:.6g})")
t0 = time.perf_counter(); rc = L.bl_spectral_norm(ws.ctx.handle, dp.handle, C.byref(out)); t1 = time.perf_counter()
print(f"spectral norm (cached): {1e3*(t1-t0):.3f} ms")
import cProfile, pstats
pr = cProfile.Profile()
pr.enable()
s = bl.solve_batch(batch, cfg, presets, ws, vectors=bl.Vectors.NONE, cache_problem=False)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
