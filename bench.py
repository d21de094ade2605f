#!/usr/bin/env python3
"""Benchmark: LPs solved/sec to 1e-4 relative KKT (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2]
                  [--impl ours|reference]

One step = one batched solve of the whole workload (all LPs of the config to
their termination status). Default workload: BASELINE.json configs[3], the
north-star config C4: strong branching K = 1024 on a synthetic m = 100k,
n = 200k sparse cover LP (the largest configuration; ~20 GB of HBM on one
GPU). Under torchrun (N > 1) the K columns are sharded across ranks (strong
scaling: no collective in the iteration loop, one all_gather of per-LP
scalars at the end); value = all LPs / max-over-ranks step time.

  value     device-resident solve: problem already in HBM, time from CUDA
            events recorded on the solver's own stream (max over ranks)
  e2e       the drop-in C-ABI (bl_problem_assign + bl_solve_batch, what the
            C++ headers call) from pinned host arrays: problem upload, step
            size, solve and per-LP result read-back inside the timed region
  roofline  dominant kernel (in-situ %globaltimer spans inside the graph)
            algorithmic bytes / time vs MEASURED_PEAKS.json hbm_gbs
  cpu_baseline  the reference CPU path (oracle/_ref) on a bounded sample

CPU reference timing (cpu_baseline and --impl reference):
  c1, c2     the reference solve_batch to full convergence (the --impl
             reference arm solves the WHOLE batch; cpu_baseline a sample)
  c3, c4, c5 time-boxed: 2x16 columns of the batch for 64 batch iterations at
             eps 1e-30 give t = seconds per column-iteration; LPs/s is
             EXTRAPOLATED as K / (t x sum of per-LP iterations of the GPU run)
             (the GPU's per-LP iteration counts, which match the reference's
             within 10 %, are recorded in profiles/gpu_iterations.json)
The reference arm never loads the CUDA library: its instances come from the
host-only build of the same generators (oracle/_ref/libbl_inputs.so).
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
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--K", type=int, default=0, help="batch width override (C5 sweep)")
    ap.add_argument("--record-iterations", action="store_true",
                    help="write this run's per-LP iterations to profiles/gpu_iterations.json")
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
EXTRAPOLATED = ("c3", "c4", "c5")  # CPU time-boxed; c1/c2 converge
ITERATIONS_FILE = os.path.join(ROOT, "profiles", "gpu_iterations.json")


def subset_batch(bl, batch, presets, cols):
    """The LPs `cols` of a batch as a standalone batch (same LPs, new column
    order): signed-unit objectives become objective-entry overrides on a
    zero base objective. Returns (LpProblem, BatchProblem, presets)."""
    import dataclasses
    from paper_2601_21990_b200.problem import (BatchProblem, ColumnOverride, LpProblem,
                                                ObjectiveMode, OverrideKind)
    colset = {c: i for i, c in enumerate(cols)}
    base = batch.base()
    ovs = []
    if batch.objective_mode() == ObjectiveMode.kSignedUnitColumns:
        n = base.num_cols()
        lp = LpProblem(base.A, np.zeros(n), base.row_bounds, base.var_bounds)
        for i, c in enumerate(cols):
            var, sign = (c, 1.0) if c < n else (c - n, -1.0)
            ovs.append(ColumnOverride(i, OverrideKind.kObjectiveEntry, var, sign))
    else:
        lp = base
        for o in batch.overrides():
            if o.column in colset:
                ovs.append(ColumnOverride(colset[o.column], o.kind, o.variable, o.value))
        ovs.sort(key=lambda o: o.column)
    pre = [dataclasses.replace(q, column=colset[q.column]) for q in presets
           if q.column in colset]
    return lp, BatchProblem(lp, len(cols), ObjectiveMode.kSharedObjective, ovs), pre


def build_workload(name: str, bl, I, K: int = 0, root_x=None):
    """(LpProblem, BatchProblem, presets, SolverConfig, spec) of a config.
    K overrides the batch width of an FSB config (the C5 sweep)."""
    spec = I.CONFIGS[name]
    p = I.config_problem(name)
    if spec.kind == "obbt":
        ob = bl.build_obbt_batch(p, bl.ObbtConfig())
        cfg = bl.ObbtConfig().solver_config()
        return p, ob.batch, ob.presets, cfg, spec
    # FSB: branch on the first K/2 fractional variables of the root relaxation
    # (C1: the reference recipe of SURVEY §8(d); large configs: x = 0.5 on
    # the first K/2 columns, acceptance.cpp:209-212). An odd K (sweep) keeps
    # the first K columns of the ceil(K/2)-pair batch.
    K = K or spec.K
    pairs = (K + 1) // 2
    if name == "c1":
        if root_x is None:
            root_x = bl.solve(p).x
        x, frac = I.synthetic_branch_point(p, pairs, root_x)
    else:
        x, frac = I.synthetic_branch_point(p, pairs)
    fb = bl.build_fsb_batch(bl.FsbRequest(p, x, frac))
    batch, presets = fb.batch, fb.presets
    if batch.batch_width() != K:
        _, batch, presets = subset_batch(bl, batch, presets, list(range(K)))
    return p, batch, presets, bl.SolverConfig(), spec


def config_block(name, spec, p, batch, cfg, world):
    """The `config` object of the JSON line; identical in both arms."""
    return {"workload": f"{name}: {spec.description}", "K": batch.batch_width(),
            "m": p.num_rows(), "n": p.num_cols(), "nnz": p.A.nnz(),
            "eps_opt": cfg.eps_opt, "eps_dual": cfg.effective_eps_dual(),
            "l2": "flushed between GPU steps (256 MiB write)",
            "parallelism": f"LP columns sharded x{world} (strong scaling), A replicated"}


def sample_columns(spec, batch, pairs):
    """Columns of the bounded CPU sample: the first `pairs` variables in both
    directions (OBBT min/max, FSB up/down branches)."""
    width = batch.batch_width()
    if spec.kind == "obbt":
        n = batch.base().num_cols()
        nv = min(pairs, n)
        return list(range(nv)) + list(range(n, n + nv))
    half = width // 2
    pairs = min(pairs, half)
    if pairs == 0:
        return list(range(width))
    return list(range(pairs)) + list(range(half, half + pairs))


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
def _ref_presets(presets):
    return [(q.column, int(q.result.status), q.result.objective) for q in presets]


def cpu_converged(bl, ref, batch, presets, cfg, cols=None):
    """The reference solve_batch (oracle/_ref) to full convergence on the
    whole batch or on the LPs `cols`; returns (LPs/s, seconds, summary)."""
    if cols is not None:
        _, batch, presets = subset_batch(bl, batch, presets, cols)
    lp = batch.base()
    t0 = time.perf_counter()
    r = ref.solve_batch(lp, batch.batch_width(), int(batch.objective_mode()),
                        batch.overrides(), cfg, _ref_presets(presets), vectors=False)
    el = time.perf_counter() - t0
    return batch.batch_width() / el, el, r


def cpu_timebox(bl, ref, batch, presets, cfg, cols, iterations=64):
    """SURVEY §8(d) time box: the reference solve_batch on the LPs `cols`
    for `iterations` batch iterations with the tolerances at 1e-30 (nothing
    terminates); returns (seconds per column-iteration, seconds, summary)."""
    import dataclasses
    _, sb, sp = subset_batch(bl, batch, presets, cols)
    c = dataclasses.replace(cfg, eps_opt=1e-30, eps_dual=1e-30, eps_infeas=1e-30,
                            max_iterations=iterations)
    t0 = time.perf_counter()
    r = ref.solve_batch(sb.base(), sb.batch_width(), 0, sb.overrides(), c, _ref_presets(sp),
                        vectors=False)
    el = time.perf_counter() - t0
    active = sb.batch_width() - len(sp)
    return el / max(active * r.iterations, 1), el, r


def cpu_threads():
    threads = os.cpu_count() or 1
    os.environ["BATCHLP_THREADS"] = str(threads)
    return threads


def cpu_baseline(name, bl, ref, batch, presets, cfg, spec, sum_iterations, pairs=0,
                 full=False):
    """One CPU measurement of the reference path on this workload:
    (LPs/s, seconds, description). c1/c2: full convergence, of the whole
    batch when `full`, else of a bounded sample; c3-c5: time box and
    extrapolation over `sum_iterations` (the GPU run's per-LP total)."""
    threads = cpu_threads()
    width = batch.batch_width()
    if name in EXTRAPOLATED:
        cols = sample_columns(spec, batch, pairs or 16)
        t_ci, el, r = cpu_timebox(bl, ref, batch, presets, cfg, cols)
        value = width / (t_ci * sum_iterations)
        desc = (f"EXTRAPOLATED: reference solve_batch (oracle/_ref, g++ -O3) time-boxed on "
                f"{len(cols)} of {width} LPs ({len(cols) // 2} branch pairs) for "
                f"{r.iterations} batch iterations at eps 1e-30: {el:.2f} s = "
                f"{t_ci * 1e3:.3f} ms per column-iteration; LPs/s = K / (t x "
                f"{sum_iterations} per-LP iterations of the GPU run); "
                f"BATCHLP_THREADS={threads}")
        return value, el, desc, threads
    if full:
        value, el, r = cpu_converged(bl, ref, batch, presets, cfg)
        desc = (f"reference solve_batch (oracle/_ref, g++ -O3) on all {width} LPs, full "
                f"convergence, {r.iterations} batch iterations, {el:.2f} s, "
                f"BATCHLP_THREADS={threads}")
        return value, el, desc, threads
    cols = sample_columns(spec, batch, pairs or (600 if spec.kind == "obbt" else 16))
    value, el, r = cpu_converged(bl, ref, batch, presets, cfg, cols)
    desc = (f"reference solve_batch (oracle/_ref, g++ -O3) on a sample of {len(cols)} of "
            f"{width} LPs (the first {len(cols) // 2} "
            f"{'variables, both directions' if spec.kind == 'obbt' else 'branch pairs'}), "
            f"full convergence, {r.iterations} batch iterations, {el:.2f} s, "
            f"BATCHLP_THREADS={threads}")
    return value, el, desc, threads


def recorded_iterations(name, K):
    """Sum of per-LP iterations of a recorded GPU run of this workload."""
    try:
        with open(ITERATIONS_FILE) as f:
            d = json.load(f).get(f"{name}:K={K}")
        return int(d["sum_iterations"]) if d else None
    except (OSError, ValueError, KeyError):
        return None


def record_iterations(name, K, summary, extra):
    try:
        with open(ITERATIONS_FILE) as f:
            d = json.load(f)
    except (OSError, ValueError):
        d = {}
    its = [int(r.iterations) for r in summary.per_problem]
    d[f"{name}:K={K}"] = {"sum_iterations": int(sum(its)), "batch_iterations":
                          int(summary.iterations), "per_lp_iterations": its, **extra}
    with open(ITERATIONS_FILE, "w") as f:
        json.dump(d, f, indent=1)


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

    p, batch, presets, cfg, spec = build_workload(args.config, bl, I, args.K)
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
    sum_its = sum(int(r.iterations) for r in summaries[-1].per_problem)
    if rank == 0 and world == 1 and args.record_iterations:
        record_iterations(args.config, width, summaries[-1],
                          {"source": "bench.py --record-iterations on one B200",
                           "loop_passes": int(summaries[-1].loop_passes)})
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import ref
            v, _, desc, threads = cpu_baseline(args.config, bl, ref, batch, presets, cfg, spec,
                                               sum_its, args.cpu_sample)
            cpu = {"value": round(v, 4), "unit": UNIT, "cores": threads, "kind": "reference",
                   "extrapolated": args.config in EXTRAPOLATED, "sample": desc}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": round(ms_step, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, DESIGN.md §5)",
            "config": config_block(args.config, spec, p, batch, cfg, world),
            "run": {"batch_iterations": summaries[-1].iterations,
                    "loop_passes": summaries[-1].loop_passes,
                    "sum_lp_iterations_rank0": sum_its,
                    "statuses_rank0": {str(k): v for k, v in sorted(
                        __import__("collections").Counter(
                            int(r.status) for r in summaries[-1].per_problem).items())}},
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
    """--impl reference: the reference CPU path (oracle/_ref, the reference
    headers compiled by oracle/Makefile) on the same workload, rank 0 only.
    Loads nothing from the CUDA package: the instances come from the
    host-only generator build oracle/_ref/libbl_inputs.so."""
    if rank != 0:
        return
    import paper_2601_21990_b200 as bl
    from paper_2601_21990_b200 import instances as I
    from oracle import ref
    gen = os.path.join(ROOT, "oracle", "_ref", "libbl_inputs.so")
    if not ref.available() or not os.path.exists(gen):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    I.use_generator_library(gen)
    # all host threads, set before the first reference call: the reference
    # reads BATCHLP_THREADS once and caches it (sparse.hpp:198-206)
    cpu_threads()
    root_x = None
    if args.config == "c1":  # root relaxation from the reference solve
        root_x = ref.solve(I.config_problem("c1")).per_problem[0].x
    p, batch, presets, cfg, spec = build_workload(args.config, bl, I, args.K, root_x)
    width = batch.batch_width()
    sum_its = None
    if args.config in EXTRAPOLATED:
        sum_its = recorded_iterations(args.config, width)
        if sum_its is None:
            print(json.dumps({"impl": "reference", "unavailable":
                              f"no recorded GPU per-LP iterations for {args.config} K={width} "
                              f"({os.path.relpath(ITERATIONS_FILE, ROOT)})"}))
            return
    # untimed warm-up steps on a small sample of the same workload (library
    # load, thread pool, page-in); the timed steps are the full measurement
    warm = max(args.warmup, 3)
    cols = sample_columns(spec, batch, 2 if spec.kind == "fsb" else 8)
    for _ in range(warm):
        if args.config in EXTRAPOLATED:
            cpu_timebox(bl, ref, batch, presets, cfg, cols, iterations=8)
        else:
            cpu_converged(bl, ref, batch, presets, cfg, cols)
    times, vals, desc, threads = [], [], "", 1
    for _ in range(max(args.steps, 1)):
        v, el, desc, threads = cpu_baseline(args.config, bl, ref, batch, presets, cfg, spec,
                                            sum_its, args.cpu_sample, full=True)
        vals.append(v)
        times.append(el)
    value = len(vals) / sum(1.0 / v for v in vals)
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": warm,
            "ms_per_step": round(1e3 * sum(times) / len(times), 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, DESIGN.md §5)",
            "config": config_block(args.config, spec, p, batch, cfg, world),
            "extrapolated": args.config in EXTRAPOLATED,
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": threads,
                             "kind": "reference", "sample": desc},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
