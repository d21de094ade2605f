// bl_tma.cuh — TMA-gather variants of the plain primal / dual row kernels
// (column blocks of W = 32, bandwidth regime).
//
// The row kernels are latency bound (ncu: long-scoreboard stalls, L2 at
// 20-30 % of its throughput): a lane can keep only a few 16-byte gathers in
// registers. Here every warp owns one row at a time with lane j = slot j of
// the block, and keeps kTmaStages rows in flight in a shared-memory ring:
//   * the gathered operand rows of a CSR row arrive by TMA gather4
//     (cp.async.bulk.tensor.2d ... tile::gather4: four 256-byte rows of the
//     tiled [blocks * rows][32] fp64 tensor per instruction), the streamed
//     rows of the iterate / anchors by TMA 2-D tile loads, all completing on
//     one mbarrier per stage;
//   * the row pointers are prefetched two rows ahead and the column indices /
//     values one row ahead in registers, so issuing a row's TMA never waits
//     on a dependent load;
//   * the epilogue (projection, Halpern, per-column sums) is the one of
//     PrimalOp / DualOp, with one slot per lane (no shuffles), and the per-item
//     sums are folded deterministically like publish_item.
// Rows with more than kTmaCap nonzeros gather directly from global memory.
#pragma once

#include <cuda.h>

#include "bl_kernels.cuh"

namespace bl {

// Tensor maps of the tiled state, built on the host per solve
// (bl_solver.cu make_tma_maps): 2-D [32 slots][blocks * rows] fp64, 256-byte
// row pitch, box {32, 1}.
struct TmaMaps {
  CUtensorMap y[2];   // Y[cur]   (primal gather source, dual stream), nb * m rows
  CUtensorMap ax[2];  // AX[cur]  (dual stream),                        nb * m rows
  CUtensorMap x[2];   // X[cur]   (primal stream),                      nb * n rows
  CUtensorMap xt;     // XT       (dual gather source),                 nb * n rows
  CUtensorMap anx;    // anchor X,                                      nb * n rows
  CUtensorMap any;    // anchor Y,                                      nb * m rows
  CUtensorMap anax;   // anchor AX,                                     nb * m rows
};

constexpr int kTmaWarps = 4;
constexpr int kTmaThreads = 32 * kTmaWarps;
constexpr int kTmaStages = 2;
constexpr int kTmaCap = 24;  // staged nonzeros per row (multiple of 4)

struct alignas(128) TmaStage {
  double g[kTmaCap][32];  // gathered operand rows
  double s[4][32];        // streamed rows (x, anchor x | y, ax, anchor y, anchor ax)
  double v[kTmaCap];      // row values
  double rs[3];           // per-row scalars (c, xl, xu | rl, ru)
  int c[kTmaCap];         // row column indices
  int p, nnz;             // nonzero range of the row
  unsigned long long bar;
};
constexpr int kTmaSmem = kTmaWarps * kTmaStages * (int)sizeof(TmaStage);

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void tma_row(const CUtensorMap* map, double* dst, int row,
                                        unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(row), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_gather4(const CUtensorMap* map, double* dst, int r0, int r1,
                                            int r2, int r3, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
      "r"(smem_u32(bar))
      : "memory");
}

// Row metadata held in registers while it is prefetched.
struct TmaMeta {
  int p, e;          // nonzero range
  int c;             // this lane's column index (lane < nnz)
  double v;          // this lane's value
  double rs0, rs1, rs2;  // per-row scalars
};

// Deterministic reduction of per-lane (= per-slot) sums of a work item over
// the CTA's warps, then the item partials / last-CTA fold of publish_item.
template <int NS>
__device__ __forceinline__ void tma_publish(const double (&acc)[NS], int b, int r, int R,
                                            double* partials, int* counters, double* colsum,
                                            int s0, int Kp, double* red) {
  constexpr int W = 32;
  __shared__ int last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int s = 0; s < NS; ++s) red[(warp * NS + s) * W + lane] = acc[s];
  __syncthreads();
  for (int t = tid; t < NS * W; t += kTmaThreads) {
    const int s = t / W, jj = t - s * W;
    double sum = 0.0;
#pragma unroll
    for (int wp = 0; wp < kTmaWarps; ++wp) sum = __dadd_rn(sum, red[(wp * NS + s) * W + jj]);
    partials[((size_t)(b * R + r) * NS + s) * W + jj] = sum;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) last = (atomicAdd(&counters[b], 1) == R - 1);
  __syncthreads();
  if (last) {
    __threadfence();
    for (int t = tid; t < NS * W; t += kTmaThreads) {
      const int s = t / W, jj = t - s * W;
      const double* src = partials + ((size_t)b * R * NS + s) * W + jj;
      double sum = 0.0;
#pragma unroll 8
      for (int rr = 0; rr < R; ++rr) sum = __dadd_rn(sum, __ldcg(src + (size_t)rr * NS * W));
      colsum[(size_t)(s0 + s) * Kp + b * W + jj] = sum;
    }
    if (tid == 0) counters[b] = 0;
  }
  __syncthreads();
}

// Issues the TMA loads of one row into stage `st` (all lanes of the warp).
// NSTR streamed rows come from `smaps` at tiled row `srow`; the gathers from
// `gmap` at tiled rows gbase + column index.
template <int NSTR>
__device__ __forceinline__ void tma_issue(TmaStage* st, const TmaMeta& mt,
                                          const CUtensorMap* gmap, int gbase,
                                          const CUtensorMap* const (&smaps)[4], int srow,
                                          int lane) {
  const int nnz = mt.e - mt.p;
  const bool staged = nnz <= kTmaCap;
  const int groups = staged ? (nnz + 3) / 4 : 0;
  if (staged && lane < nnz) {
    st->c[lane] = mt.c;
    st->v[lane] = mt.v;
  }
  if (staged && nnz > 0 && lane >= nnz && lane < groups * 4) st->c[lane] = -1;  // pad marker
  if (lane == 0) {
    st->p = mt.p;
    st->nnz = nnz;
    st->rs[0] = mt.rs0;
    st->rs[1] = mt.rs1;
    st->rs[2] = mt.rs2;
  }
  // the stage was read by this warp (generic proxy) before the async writes
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    const unsigned bytes = (unsigned)(groups * 4 * 256 + NSTR * 256);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                     smem_u32(&st->bar)),
                 "r"(bytes)
                 : "memory");
  }
  __syncwarp();
  if (lane < groups) {
    int idx[4];
    const int last = st->c[nnz - 1];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c = st->c[4 * lane + k];
      idx[k] = gbase + (c >= 0 ? c : last);  // pad with a duplicate row
    }
    tma_gather4(gmap, &st->g[4 * lane][0], idx[0], idx[1], idx[2], idx[3], &st->bar);
  } else if (lane >= 28 && lane - 28 < NSTR) {
    const int k = lane - 28;
    tma_row(smaps[k], &st->s[k][0], srow, &st->bar);
  }
}

__device__ __forceinline__ void tma_wait(TmaStage* st, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred done;\n"
      "TMA_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n"
      "@!done bra TMA_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(&st->bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_meta(const int* __restrict__ rp,
                                              const int* __restrict__ ci,
                                              const double* __restrict__ cv, int row, int lane,
                                              TmaMeta& mt) {
  mt.p = __ldg(rp + row);
  mt.e = __ldg(rp + row + 1);
}
__device__ __forceinline__ void tma_load_vals(const int* __restrict__ ci,
                                              const double* __restrict__ cv, int lane,
                                              TmaMeta& mt, const double* s0, const double* s1,
                                              const double* s2, int row) {
  const int nnz = mt.e - mt.p;
  if (nnz <= kTmaCap && lane < nnz) {
    mt.c = __ldg(ci + mt.p + lane);
    mt.v = __ldg(cv + mt.p + lane);
  }
  mt.rs0 = s0 ? __ldg(s0 + row) : 0.0;
  mt.rs1 = __ldg(s1 + row);
  mt.rs2 = __ldg(s2 + row);
}

// Sequential dot of a staged (or, for long rows, global) row with this
// lane's slot: the reference csr_apply order, separately rounded.
__device__ __forceinline__ double tma_dot(const TmaStage* st, int nnz, int p,
                                          const int* __restrict__ ci,
                                          const double* __restrict__ cv,
                                          const double* gsrc, int lane) {
  double acc = 0.0;
  if (nnz <= kTmaCap) {
    for (int t = 0; t < nnz; ++t) acc = __dadd_rn(acc, __dmul_rn(st->v[t], st->g[t][lane]));
  } else {
    for (int q = p; q < p + nnz; ++q)
      acc = __dadd_rn(acc, __dmul_rn(__ldg(cv + q), __ldg(gsrc + (size_t)__ldg(ci + q) * 32 + lane)));
  }
  return acc;
}

// ---------------------------------------------------------------------------
// primal (plain pass): XT = proj(X - tau (c + A'Y)), X' = Halpern, sums
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kTmaThreads, 3) k_primal_tma(Params P,
                                                               const __grid_constant__ TmaMaps M) {
  extern __shared__ __align__(128) char tma_smem[];
  __shared__ double red[kTmaWarps * 2 * 32];
  const Ctrl C = *P.ctrl;
  if (C.done) return;
  prof_begin(P, K_PRIMAL);
  constexpr int W = 32;
  const int n = P.n, m = P.m;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  TmaStage* stages = reinterpret_cast<TmaStage*>(tma_smem) + warp * kTmaStages;
  if (lane < kTmaStages) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&stages[lane].bar))
                 : "memory");
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  unsigned phase = 0u;
  const int reset = C.anchor_reset;
  const double alpha = C.alpha, oma = 1.0 - alpha;
  const double* Ycur = P.Y[C.cur];
  double* Xnxt = P.X[C.cur ^ 1];
  const int nb = (C.active + W - 1) / W;
  const int R = C.Rp;
  const int items = nb * R;
  const int per = (n + R - 1) / R;
  const CUtensorMap* smaps[4] = {&M.x[C.cur], &M.anx, &M.anx, &M.anx};
  const int nstr = reset ? 1 : 2;
  const double* s0 = P.mode == BL_SHARED_OBJECTIVE ? P.c : nullptr;
  for (int w = blockIdx.x; w < items; w += gridDim.x) {
    const int b = w / R, r = w - b * R;
    const int r0 = min(n, r * per), r1 = min(n, r0 + per);
    const int j = b * W + lane;
    ColInfo col;
    load_col(P, j, C.active, false, col);
    double acc[2] = {0.0, 0.0};
    const int gbase = b * m;
    // this warp's rows: r0 + warp, r0 + warp + kTmaWarps, ...
    const int first = r0 + warp;
    const int count = first < r1 ? (r1 - first + kTmaWarps - 1) / kTmaWarps : 0;
    TmaMeta m0, m1, m2;  // rows k (issued next), k+1 (values), k+2 (pointers)
    auto rowk = [&](int k) { return first + k * kTmaWarps; };
    // prologue: issue rows 0 .. kTmaStages-1, prefetch the next two
    for (int k = 0; k < kTmaStages && k < count; ++k) {
      TmaMeta mt;
      tma_load_meta(P.trp, P.tci, P.tcv, rowk(k), lane, mt);
      tma_load_vals(P.tci, P.tcv, lane, mt, s0, P.xl, P.xu, rowk(k));
      if (nstr == 2) tma_issue<2>(&stages[k], mt, &M.y[C.cur], gbase, smaps, b * n + rowk(k), lane);
      else tma_issue<1>(&stages[k], mt, &M.y[C.cur], gbase, smaps, b * n + rowk(k), lane);
    }
    if (kTmaStages < count) {
      tma_load_meta(P.trp, P.tci, P.tcv, rowk(kTmaStages), lane, m1);
      tma_load_vals(P.tci, P.tcv, lane, m1, s0, P.xl, P.xu, rowk(kTmaStages));
    }
    if (kTmaStages + 1 < count) tma_load_meta(P.trp, P.tci, P.tcv, rowk(kTmaStages + 1), lane, m2);
    for (int k = 0; k < count; ++k) {
      const int sidx = k % kTmaStages;
      TmaStage* st = &stages[sidx];
      const int i = rowk(k);
      tma_wait(st, (phase >> sidx) & 1u);
      phase ^= 1u << sidx;
      const double bc = st->rs[0], bl = st->rs[1], bh = st->rs[2];
      const int pq = st->p, nnz = st->nnz;
      const double aty = tma_dot(st, nnz, pq, P.tci, P.tcv, Ycur + (size_t)gbase * W, lane);
      const double x = st->s[0][lane];
      const double ax = reset ? x : st->s[1][lane];
      double cc, lo, hi;
      col_vals(P, col, i, bc, bl, bh, cc, lo, hi);
      const double t = cc + aty;
      const double xt = project_box(x - col.step * t, lo, hi);
      const double dx = xt - x, da = x - ax;
      if (col.valid) {
        acc[0] += dx * dx;
        acc[1] += da * da;
      }
      const double xn = alpha * (2.0 * xt - x) + oma * ax;
      const size_t idx = ((size_t)b * n + i) * W + lane;
      P.XT[idx] = xt;
      __stcs(Xnxt + idx, xn);
      if (reset) __stcs(P.aX + idx, x);
      // refill this stage with row k + kTmaStages; advance the prefetches
      if (k + kTmaStages < count) {
        m0 = m1;
        if (nstr == 2)
          tma_issue<2>(st, m0, &M.y[C.cur], gbase, smaps, b * n + rowk(k + kTmaStages), lane);
        else
          tma_issue<1>(st, m0, &M.y[C.cur], gbase, smaps, b * n + rowk(k + kTmaStages), lane);
        m1 = m2;
        if (k + kTmaStages + 1 < count)
          tma_load_vals(P.tci, P.tcv, lane, m1, s0, P.xl, P.xu, rowk(k + kTmaStages + 1));
        if (k + kTmaStages + 2 < count)
          tma_load_meta(P.trp, P.tci, P.tcv, rowk(k + kTmaStages + 2), lane, m2);
      }
    }
    tma_publish<2>(acc, b, r, R, P.partials, P.counters, P.colsum, S_DX2, P.Kp, red);
  }
  prof_end(P, K_PRIMAL);
}

// ---------------------------------------------------------------------------
// dual (plain pass): AXT = A XT, YT = sigma (s - proj(s)), Y'/AX' = Halpern
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kTmaThreads, 3) k_dual_tma(Params P,
                                                             const __grid_constant__ TmaMaps M) {
  extern __shared__ __align__(128) char tma_smem[];
  __shared__ double red[kTmaWarps * 3 * 32];
  const Ctrl C = *P.ctrl;
  if (C.done) return;
  prof_begin(P, K_DUAL);
  constexpr int W = 32;
  const int n = P.n, m = P.m;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  TmaStage* stages = reinterpret_cast<TmaStage*>(tma_smem) + warp * kTmaStages;
  if (lane < kTmaStages) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&stages[lane].bar))
                 : "memory");
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  unsigned phase = 0u;
  const int reset = C.anchor_reset;
  const double alpha = C.alpha, oma = 1.0 - alpha;
  double* Ynxt = P.Y[C.cur ^ 1];
  double* AXnxt = P.AX[C.cur ^ 1];
  const int nb = (C.active + W - 1) / W;
  const int R = C.Rd;
  const int items = nb * R;
  const int per = (m + R - 1) / R;
  const CUtensorMap* smaps[4] = {&M.y[C.cur], &M.ax[C.cur], &M.any, &M.anax};
  const int nstr = reset ? 2 : 4;
  for (int w = blockIdx.x; w < items; w += gridDim.x) {
    const int b = w / R, r = w - b * R;
    const int r0 = min(m, r * per), r1 = min(m, r0 + per);
    const int j = b * W + lane;
    ColInfo col;
    load_col(P, j, C.active, true, col);
    double acc[3] = {0.0, 0.0, 0.0};
    const int gbase = b * n;
    const int first = r0 + warp;
    const int count = first < r1 ? (r1 - first + kTmaWarps - 1) / kTmaWarps : 0;
    TmaMeta m0, m1, m2;
    auto rowk = [&](int k) { return first + k * kTmaWarps; };
    for (int k = 0; k < kTmaStages && k < count; ++k) {
      TmaMeta mt;
      tma_load_meta(P.rp, P.ci, P.cv, rowk(k), lane, mt);
      tma_load_vals(P.ci, P.cv, lane, mt, nullptr, P.rl, P.ru, rowk(k));
      if (nstr == 4) tma_issue<4>(&stages[k], mt, &M.xt, gbase, smaps, b * m + rowk(k), lane);
      else tma_issue<2>(&stages[k], mt, &M.xt, gbase, smaps, b * m + rowk(k), lane);
    }
    if (kTmaStages < count) {
      tma_load_meta(P.rp, P.ci, P.cv, rowk(kTmaStages), lane, m1);
      tma_load_vals(P.ci, P.cv, lane, m1, nullptr, P.rl, P.ru, rowk(kTmaStages));
    }
    if (kTmaStages + 1 < count) tma_load_meta(P.rp, P.ci, P.cv, rowk(kTmaStages + 1), lane, m2);
    for (int k = 0; k < count; ++k) {
      const int sidx = k % kTmaStages;
      TmaStage* st = &stages[sidx];
      const int i = rowk(k);
      tma_wait(st, (phase >> sidx) & 1u);
      phase ^= 1u << sidx;
      const double lo = st->rs[1], hi = st->rs[2];
      const int pq = st->p, nnz = st->nnz;
      const double axt = tma_dot(st, nnz, pq, P.ci, P.cv, P.XT + (size_t)gbase * W, lane);
      const double y = st->s[0][lane], ax = st->s[1][lane];
      const double ay = reset ? y : st->s[2][lane];
      const double aax = reset ? ax : st->s[3][lane];
      const double sigma = col.step;
      // dual_step_element, solver.hpp:186-190
      const double vv = 2.0 * axt - ax;
      const double s = y / sigma + vv;
      const double yt = sigma * (s - project_box(s, lo, hi));
      const double dy = yt - y, da = y - ay;
      if (col.valid) {
        acc[0] += dy * dy;
        acc[1] += dy * (axt - ax);
        acc[2] += da * da;
      }
      const double yn = alpha * (2.0 * yt - y) + oma * ay;
      const double axn = alpha * (2.0 * axt - ax) + oma * aax;
      const size_t idx = ((size_t)b * m + i) * W + lane;
      __stcs(Ynxt + idx, yn);
      __stcs(AXnxt + idx, axn);
      if (reset) {
        __stcs(P.aY + idx, y);
        __stcs(P.aAX + idx, ax);
      }
      if (k + kTmaStages < count) {
        m0 = m1;
        if (nstr == 4)
          tma_issue<4>(st, m0, &M.xt, gbase, smaps, b * m + rowk(k + kTmaStages), lane);
        else
          tma_issue<2>(st, m0, &M.xt, gbase, smaps, b * m + rowk(k + kTmaStages), lane);
        m1 = m2;
        if (k + kTmaStages + 1 < count)
          tma_load_vals(P.ci, P.cv, lane, m1, nullptr, P.rl, P.ru, rowk(k + kTmaStages + 1));
        if (k + kTmaStages + 2 < count)
          tma_load_meta(P.rp, P.ci, P.cv, rowk(k + kTmaStages + 2), lane, m2);
      }
    }
    tma_publish<3>(acc, b, r, R, P.partials, P.counters, P.colsum, S_DY2, P.Kp, red);
  }
  prof_end(P, K_DUAL);
}

}  // namespace bl
