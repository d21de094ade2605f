"""BASELINE configs[4] (C5): batch-size sweep K = 1 ... 4096 on the m = 20k,
n = 40k strong-branching LP -- LPs/s and SpMM GB/s vs K on one B200, with
the reference CPU path (oracle/_ref) beside it.

  python scripts/c5_sweep.py [--out DIR] [--max-k 4096] [--cpu-pairs 16]

Per K:
  * a warm-up solve, then two timed device-resident solves of the first K
    LPs of the C5 batch (bench.build_workload(..., K)); LPs/s = K / device
    time (CUDA events on the solver's stream, L2 flushed before each);
  * the dominant row kernel's algorithmic GB/s and its fraction of the
    measured HBM peak (in-situ %globaltimer spans);
  * SpMM GB/s: bl_measure_spmm (A X and A'Y at width K, 10 each), counting
    B_spmm = 12 nnz + 4 (rows_out + 1) + 8 K (cols_in + rows_out) per product;
  * CPU: the reference's per-column-iteration cost, time-boxed once on a
    16-pair sample, extrapolated to K / (t x the GPU run's
    summed per-LP iterations) -- labelled extrapolated.
Writes sweep.jsonl and sweep.md into --out.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2601_21990_b200 as bl  # noqa: E402
from paper_2601_21990_b200 import instances as I  # noqa: E402
from paper_2601_21990_b200.tuner import measure_spmm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/c5_sweep")
    ap.add_argument("--max-k", type=int, default=4096)
    ap.add_argument("--cpu-pairs", type=int, default=16)
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    import torch
    dev = torch.device("cuda", 0)
    peak, peak_kind = bench.peaks()
    ks = [1 << e for e in range(13) if (1 << e) <= args.max_k]
    rows = []
    p_full = None
    for K in ks:
        p, batch, presets, cfg, spec = bench.build_workload("c5", bl, I, K)
        p_full = p
        ws = bl.BatchWorkspace(0)
        bl.solve_batch(batch, cfg, presets, ws, vectors=bl.Vectors.NONE)  # warm
        ms, summ = [], None
        for _ in range(2):
            bench.flush_l2(torch, dev)
            summ = bl.solve_batch(batch, cfg, presets, ws, vectors=bl.Vectors.NONE)
            ms.append(summ.device_ms)
        dev_ms = min(ms)
        prof = summ.profile
        rk = {k: v for k, v in prof.items() if k in ("primal", "dual") and v[1] > 0}
        dom = max(rk, key=lambda k: rk[k][1]) if rk else None
        kern = None
        if dom:
            gbs = rk[dom][2] / rk[dom][1]
            kern = {"kernel": f"k_{dom}", "GB/s": round(gbs, 1), "frac": round(gbs / peak, 4)}
        # SpMM throughput at width K (both orientations, 10 products each)
        A = p.A
        total, _, _ = measure_spmm(A, K, 10, workspace=ws)
        m, n, nnz = A.n_rows(), A.n_cols(), A.nnz()
        b_ax = 12 * nnz + 4 * (m + 1) + 8 * K * (n + m)
        b_aty = 12 * nnz + 4 * (n + 1) + 8 * K * (m + n)
        spmm_gbs = 10 * (b_ax + b_aty) / total / 1e9 if total > 0 else None
        sum_its = sum(int(r.iterations) for r in summ.per_problem)
        row = {"K": K, "device_ms": round(dev_ms, 3), "lps_per_s": round(K / (dev_ms / 1e3), 3),
               "batch_iterations": int(summ.iterations), "sum_lp_iterations": sum_its,
               "loop_passes": int(summ.loop_passes), "dominant": kern,
               "spmm_gbs": round(spmm_gbs, 1) if spmm_gbs else None,
               "spmm_frac": round(spmm_gbs / peak, 4) if spmm_gbs else None}
        rows.append(row)
        print(json.dumps(row), flush=True)
        ws.ctx.close()
    # CPU: the reference's per-column-iteration cost, once (time box)
    cpu = None
    try:
        from oracle import ref
        if ref.available():
            threads = bench.cpu_threads()
            _, batch, presets, cfg, spec = bench.build_workload("c5", bl, I, 2 * args.cpu_pairs)
            cols = list(range(batch.batch_width()))
            t_ci, el, r = bench.cpu_timebox(bl, ref, batch, presets, cfg, cols)
            cpu = {"s_per_column_iteration": t_ci, "seconds": el, "threads": threads,
                   "sample": f"{len(cols)} LPs x {r.iterations} batch iterations at eps 1e-30"}
    except Exception as e:  # noqa: BLE001
        cpu = {"unavailable": str(e)}
    for row in rows:
        if cpu and "s_per_column_iteration" in cpu:
            row["cpu_lps_per_s_extrapolated"] = round(
                row["K"] / (cpu["s_per_column_iteration"] * row["sum_lp_iterations"]), 4)
    with open(os.path.join(args.out, "sweep.jsonl"), "w") as f:
        for row in rows:
            f.write(json.dumps(row) + "\n")
        f.write(json.dumps({"cpu": cpu, "peak_gbs": peak, "peak_kind": peak_kind,
                            "m": p_full.num_rows(), "n": p_full.num_cols(),
                            "nnz": p_full.A.nnz(), "when": time.ctime()}) + "\n")
    lines = ["| K | s per solve | LPs/s (GPU) | batch its | dominant kernel GB/s (frac) | "
             "SpMM GB/s (frac) | CPU LPs/s (extrap.) |", "|---|---|---|---|---|---|---|"]
    for r in rows:
        d = r["dominant"] or {}
        lines.append(f"| {r['K']} | {r['device_ms'] / 1e3:.3f} | {r['lps_per_s']:.1f} | "
                     f"{r['batch_iterations']} | {d.get('GB/s', '-')} ({d.get('frac', '-')}) | "
                     f"{r['spmm_gbs']} ({r['spmm_frac']}) | "
                     f"{r.get('cpu_lps_per_s_extrapolated', '-')} |")
    with open(os.path.join(args.out, "sweep.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
        f.write(f"\nCPU: {json.dumps(cpu)}\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
