#!/usr/bin/env python3
"""Benchmark: LPs solved/sec to 1e-4 relative KKT (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2]
                  [--impl ours|reference]

One step = one batched solve of the whole workload (all LPs of the config to
their termination status). Default workload: BASELINE.json configs[1], OBBT
with 2n = 4000 LPs on a synthetic m = n = 2000 LP (fits one GPU). Under
torchrun (N > 1) the columns are sharded across ranks (no collective in the
iteration loop, one all_gather of per-LP scalars at the end); value = all LPs
/ max-over-ranks step time.

  value     device-resident solve: problem already in HBM, time from CUDA
            events recorded on the solver's own stream (max over ranks)
  e2e       the drop-in C-ABI (bl_problem_assign + bl_solve_batch, what the
            C++ headers call) from pinned host arrays: problem upload, step
            size, solve and per-LP result read-back inside the timed region
  roofline  dominant kernel (in-situ %globaltimer spans inside the graph)
            algorithmic bytes / time vs MEASURED_PEAKS.json hbm_gbs
  cpu_baseline  the reference CPU path (oracle/_ref) on a bounded sample
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "LPs solved/sec to 1e-4 rel. KKT at batch K; SpMM HBM GB/s vs peak"
UNIT = "LPs/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample", type=int, default=0,
                    help="variables (OBBT) / branch pairs (FSB) in the CPU sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------
def build_workload(name: str, bl, I):
    """(BatchProblem, presets, description dict) of a config."""
    spec = I.CONFIGS[name]
    p = I.config_problem(name)
    if spec.kind == "obbt":
        ob = bl.build_obbt_batch(p, bl.ObbtConfig())
        cfg = bl.ObbtConfig().solver_config()
        return p, ob.batch, ob.presets, cfg, spec
    # FSB: branch on the first K/2 fractional variables of the root relaxation
    # (C1: the reference recipe of SURVEY §8(d); large configs: x = 0.5 on
    # the first K/2 columns, acceptance.cpp:209-212).
    K = spec.K
    if name == "c1":
        root = bl.solve(p)
        x, frac = I.synthetic_branch_point(p, K // 2, root.x)
    else:
        x, frac = I.synthetic_branch_point(p, K // 2)
    fb = bl.build_fsb_batch(bl.FsbRequest(p, x, frac))
    return p, fb.batch, fb.presets, bl.SolverConfig(), spec


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(
                        ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                         "--format=csv,noheader,nounits"], capture_output=True, text=True,
                        timeout=5).stdout.strip()
                    if out:
                        self.samples.append([s.strip() for s in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4)
                          if len(s) > 3 + k and s[3 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def flush_l2(torch, dev):
    buf = getattr(flush_l2, "buf", None)
    if buf is None:
        buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB
        flush_l2.buf = buf
    buf.fill_(1.0)
    torch.cuda.synchronize(dev)


# ---------------------------------------------------------------------------
# CPU baseline: the reference (oracle/_ref) on a bounded sample
# ---------------------------------------------------------------------------
def cpu_sample(name, p, batch, presets, cfg, spec, sample):
    """Runs the compiled reference on a column sample of the workload;
    returns (LPs/s, description, threads)."""
    threads = os.cpu_count() or 1
    os.environ["BATCHLP_THREADS"] = str(threads)
    from oracle import ref
    from paper_2601_21990_b200 import distributed as D
    width = batch.batch_width()
    if spec.kind == "obbt":
        nv = sample or 600
        n = p.num_cols()
        cols = list(range(nv)) + list(range(n, n + nv))
    else:
        pairs = sample or min(width // 2, 16)
        half = width // 2
        cols = list(range(pairs)) + list(range(half, half + pairs))
    # rewrite the sample as a shared-objective batch (same LPs)
    from paper_2601_21990_b200.problem import ColumnOverride, LpProblem, OverrideKind
    colset = {c: i for i, c in enumerate(cols)}
    base = batch.base()
    ovs = []
    if batch.objective_mode() == 1:  # signed unit: zero base objective + entries
        n = base.num_cols()
        lp = LpProblem(base.A, np.zeros(n), base.row_bounds, base.var_bounds)
        for i, c in enumerate(cols):
            var, sign = (c, 1.0) if c < n else (c - n, -1.0)
            ovs.append(ColumnOverride(i, OverrideKind.kObjectiveEntry, var, sign))
    else:
        for o in batch.overrides():
            if o.column in colset:
                ovs.append(ColumnOverride(colset[o.column], o.kind, o.variable, o.value))
        lp = base
    pre = [(colset[q.column], int(q.result.status), q.result.objective) for q in presets
           if q.column in colset]
    t0 = time.perf_counter()
    r = ref.solve_batch(lp, len(cols), 0, ovs, cfg, pre, vectors=False)
    el = time.perf_counter() - t0
    desc = (f"reference solve_batch (oracle/_ref, g++ -O3) on {len(cols)} of {width} LPs "
            f"({'variables 0..' + str(nv - 1) + ' both directions' if spec.kind == 'obbt' else str(len(cols) // 2) + ' branch pairs'}), "
            f"full convergence, {r.iterations} batch iterations, {el:.2f} s, "
            f"BATCHLP_THREADS={threads}")
    return len(cols) / el, desc, threads, el


# ---------------------------------------------------------------------------
def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, world, rank)

    import torch
    import torch.distributed as dist
    import paper_2601_21990_b200 as bl
    from paper_2601_21990_b200 import instances as I
    from paper_2601_21990_b200 import distributed as D
    from paper_2601_21990_b200.solver import BatchWorkspace, DeviceProblem

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    p, batch, presets, cfg, spec = build_workload(args.config, bl, I)
    width = batch.batch_width()
    shard = D.shard_batch(batch, presets, rank, world) if world > 1 else None
    my_batch = shard.batch if shard else batch
    my_presets = shard.presets if shard else presets
    ws = BatchWorkspace(local)

    def step(cache=True):
        return bl.solve_batch(my_batch, cfg, my_presets, ws, vectors=bl.Vectors.NONE,
                              cache_problem=cache)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()

    # ---- value: device-resident -------------------------------------------
    for _ in range(max(args.warmup, 3)):
        s = step()
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    dev_ms, walls, launches, summaries = [], [], 0, []
    for _ in range(args.steps):
        flush_l2(torch, dev)
        barrier()
        t0 = time.perf_counter()
        s = step()
        walls.append(time.perf_counter() - t0)
        dev_ms.append(s.device_ms)
        launches += s.kernel_launches
        summaries.append(s)
    barrier()
    clk = clocks.stop()
    my_ms = sum(dev_ms) / args.steps
    if world > 1:
        t = torch.tensor([my_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
        # the one real exchange: per-LP scalars of every slice
        slices = D.column_slices(width, world)
        D.gather_results(D.pack(summaries[-1].per_problem), slices, dev)
    else:
        ms_step = my_ms
    value = width / (ms_step / 1e3)

    # ---- e2e: public API from pinned host buffers -------------------------
    A = my_batch.base().A
    pinned = {}
    for k, a in (("rp", A.row_offsets), ("ci", A.col_indices), ("cv", A.values),
                 ("trp", A.t_row_offsets), ("tci", A.t_col_indices), ("tcv", A.t_values)):
        t = torch.empty(a.shape, dtype=torch.from_numpy(a.copy()).dtype, pin_memory=True)
        t.numpy()[:] = a
        pinned[k] = t.numpy()
    base = my_batch.base()
    vecs = []
    for a in (base.objective, base.var_bounds.lower, base.var_bounds.upper,
              base.row_bounds.lower, base.row_bounds.upper):
        t = torch.empty(len(a), dtype=torch.float64, pin_memory=True)
        t.numpy()[:] = a
        vecs.append(t.numpy())
    h2d = sum(a.nbytes for a in pinned.values()) + sum(v.nbytes for v in vecs)
    from paper_2601_21990_b200.problem import Bounds, LpProblem, SparseMatrix
    e2e_prob = LpProblem(SparseMatrix(A.n_rows(), A.n_cols(), pinned["rp"], pinned["ci"],
                                      pinned["cv"], pinned["trp"], pinned["tci"],
                                      pinned["tcv"]),
                         vecs[0], Bounds.from_arrays(vecs[3], vecs[4]),
                         Bounds.from_arrays(vecs[1], vecs[2]))
    from paper_2601_21990_b200.problem import BatchProblem
    e2e_batch = BatchProblem(e2e_prob, my_batch.batch_width(), my_batch.objective_mode(),
                             my_batch.overrides())
    n_ov = len(my_batch.overrides())
    per_solve_h2d = n_ov * 24 + my_batch.batch_width() * (8 * 19 + 4 * 7 + 4 * 3) + 256
    per_solve_d2h = my_batch.batch_width() * (80 + 4) + 256
    # One long-lived workspace, as a solver process keeps its device context;
    # every step uploads the problem from pinned host memory into it
    # (bl_problem_assign), recomputes the step size (device power iteration)
    # and reads the per-LP results back into a host array (bl_solve_batch):
    # the calls the C++ drop-in headers make.
    import ctypes
    from paper_2601_21990_b200 import _native as NN
    e2e_walls = []
    wse = BatchWorkspace(local)
    dpe = wse.resident(e2e_prob, cache=False)  # device problem (warm-up upload)
    Lb = NN.lib()
    _, _, assign_args, keep = type(dpe)._arrays(e2e_prob)
    ovs = my_batch.overrides()
    ov_arr = (NN.bl_override * max(len(ovs), 1))()
    for k, o in enumerate(ovs):
        ov_arr[k].column, ov_arr[k].kind = o.column, int(o.kind)
        ov_arr[k].variable, ov_arr[k].value = o.variable, o.value
    pcols = np.array([q.column for q in my_presets], dtype=np.int32)
    ccfg = cfg.to_c(bl.Vectors.NONE, 0.0)
    summ = NN.bl_summary()
    res_h = (NN.bl_column_result * max(my_batch.batch_width(), 1))()

    def c_abi_solve():
        rc = Lb.bl_problem_assign(wse.ctx.handle, dpe.handle, *assign_args)
        if rc == 0:
            rc = Lb.bl_solve_batch(wse.ctx.handle, dpe.handle, my_batch.batch_width(),
                                   int(my_batch.objective_mode()), ov_arr, len(ovs),
                                   ctypes.byref(ccfg), NN.iptr(pcols) if len(pcols) else None,
                                   len(pcols), None, None, None, ctypes.byref(summ), res_h)
        if rc != 0:
            raise RuntimeError(f"bl_solve_batch failed: {rc} {Lb.bl_last_error(wse.ctx.handle)}")

    c_abi_solve()  # warm-up
    for _ in range(args.steps):
        flush_l2(torch, dev)
        barrier()
        t0 = time.perf_counter()
        c_abi_solve()
        e2e_walls.append(time.perf_counter() - t0)
    if summ.iterations != s.iterations:
        raise RuntimeError("e2e solve disagrees with the device-resident solve")
    del keep
    wse.ctx.close()
    e2e_s = sum(e2e_walls) / len(e2e_walls)
    if world > 1:
        t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = width / e2e_s

    # ---- roofline of the dominant kernel -----------------------------------
    prof = {}
    for s_ in summaries:
        for k, (lau, ns, by) in s_.profile.items():
            a = prof.setdefault(k, [0.0, 0.0, 0.0])
            a[0] += lau
            a[1] += ns
            a[2] += by
    row = {k: v for k, v in prof.items() if k in ("primal", "dual", "check") and v[1] > 0}
    dom = max(row, key=lambda k: row[k][1]) if row else None
    peak, peak_kind = peaks()
    roof = None
    if dom:
        ach = row[dom][2] / row[dom][1]  # bytes/ns == GB/s
        # DRAM traffic of one captured launch of this kernel (ncu --set full,
        # profiles/ncu_traffic.json), next to that launch's algorithmic bytes:
        # traffic/alg > 1 would mean wasted re-reads
        traffic, traffic_launch = None, None
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
                tj = json.load(f).get(args.config, {}).get(dom)
            if tj:
                traffic = tj["traffic"]
                traffic_launch = {"alg_bytes": tj["alg_bytes"],
                                  "traffic_over_alg": tj["traffic_over_alg"],
                                  "ncu_us": tj["ncu_us"], "launch": tj["launch"]}
        except Exception:
            pass
        total_ns = sum(v[1] for v in prof.values())
        roof = {"bound": "hbm", "kernel": f"k_{dom}", "achieved": round(ach, 1),
                "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                "frac": round(ach / peak, 4), "traffic": traffic,
                "traffic_launch": traffic_launch,
                "alg_bytes_per_launch": round(row[dom][2] / row[dom][0]),
                "avg_launch_us": round(row[dom][1] / row[dom][0] / 1e3, 3),
                "share_of_kernel_time": round(row[dom][1] / total_ns, 3) if total_ns else None,
                # the fast tail kernel (k_tail_fast: <= 32 LPs left, one
                # 16-CTA cluster) is latency-bound by construction; its
                # phases are timed on chip per pass
                "tail_kernel": ({
                    "kernel": "k_tail_fast", "bound": "latency",
                    "passes": int(prof["tail_decide"][0]),
                    "us_per_pass": round(sum(prof[k][1] for k in ("tail_primal", "tail_dual",
                                                                  "tail_decide"))
                                         / prof["tail_decide"][0] / 1e3, 3),
                    "share_of_kernel_time": round(sum(prof[k][1] for k in (
                        "tail_primal", "tail_dual", "tail_decide")) / total_ns, 3)}
                    if prof.get("tail_decide", [0])[0] else None),
                "kernels": {k: {"launches": int(v[0]), "ms": round(v[1] / 1e6, 3),
                                "GB/s": round(v[2] / v[1], 1) if v[1] and v[2] else None}
                            for k, v in sorted(prof.items()) if v[0]}}

    # ---- CPU baseline (rank 0, N = 1) --------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            v, desc, threads, _ = cpu_sample(args.config, p, batch, presets, cfg, spec,
                                             args.cpu_sample)
            cpu = {"value": round(v, 3), "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": desc}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        nnz = p.A.nnz()
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": round(ms_step, 3), "higher_is_better": True,
            "scaling": "weak" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, DESIGN.md §5)",
            "config": {"workload": f"{args.config}: {spec.description}", "K": width,
                       "m": p.num_rows(), "n": p.num_cols(), "nnz": nnz,
                       "eps_opt": cfg.eps_opt, "eps_dual": cfg.effective_eps_dual(),
                       "batch_iterations": summaries[-1].iterations,
                       "loop_passes": summaries[-1].loop_passes,
                       "l2": "flushed between steps (256 MiB write)",
                       "parallelism": f"columns sharded x{world}, A replicated"},
            "e2e": {"value": round(e2e, 3), "unit": UNIT,
                    "h2d_bytes_per_step": int(h2d + per_solve_h2d),
                    "d2h_bytes_per_step": int(per_solve_d2h)},
            "roofline": roof,
            "cpu_baseline": cpu,
            "clocks": clk,
            "gpu_launches": int(launches),
            "wall_ms_per_step": round(1e3 * sum(walls) / len(walls), 3),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_reference(args, world, rank):
    """--impl reference: the reference CPU path (oracle/_ref) on a bounded
    sample of the same workload, rank 0 only."""
    if rank != 0:
        return
    import paper_2601_21990_b200 as bl
    from paper_2601_21990_b200 import instances as I
    from oracle import ref
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    p, batch, presets, cfg, spec = build_workload_cpu(args.config, bl, I, ref)
    times, vals, desc, threads = [], [], "", 1
    # untimed warm-up steps on a small sample of the same workload (library
    # load, thread pool, page-in); the timed steps are full bounded samples
    warm = max(args.warmup, 3)
    for _ in range(warm):
        cpu_sample(args.config, p, batch, presets, cfg, spec, 8 if spec.kind == "obbt" else 1)
    for _ in range(max(args.steps, 1)):
        v, desc, threads, el = cpu_sample(args.config, p, batch, presets, cfg, spec,
                                          args.cpu_sample)
        vals.append(v)
        times.append(el)
    value = len(vals) / sum(1.0 / v for v in vals)
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": warm,
            "ms_per_step": round(1e3 * sum(times) / len(times), 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, DESIGN.md §5)",
            "config": {"workload": f"{args.config}: {spec.description}",
                       "K": batch.batch_width(), "m": p.num_rows(), "n": p.num_cols()},
            "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": threads,
                             "kind": "reference", "sample": desc},
            "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def build_workload_cpu(name, bl, I, ref):
    """Workload construction without a GPU (for the reference arm): the C1
    root relaxation comes from the reference solve."""
    spec = I.CONFIGS[name]
    p = I.config_problem(name)
    if spec.kind == "obbt":
        ob = bl.build_obbt_batch(p, bl.ObbtConfig())
        return p, ob.batch, ob.presets, bl.ObbtConfig().solver_config(), spec
    if name == "c1":
        x0 = ref.solve(p).per_problem[0].x
        x, frac = I.synthetic_branch_point(p, spec.K // 2, x0)
    else:
        x, frac = I.synthetic_branch_point(p, spec.K // 2)
    fb = bl.build_fsb_batch(bl.FsbRequest(p, x, frac))
    return p, fb.batch, fb.presets, bl.SolverConfig(), spec


if __name__ == "__main__":
    main()
