// bl_kernels.cuh — sm_100a device code of the batched PDHG hot path.
//
// Templates and device functions shared by the translation units: the
// per-width kernel instantiations (bl_w*.cu, built in parallel) and the
// width-independent kernels and launchers (bl_kernels.cu).
//
// One solver iteration (reference batch_solver.hpp:174-345) is three launches
// on plain iterations and up to seven on termination-check iterations:
//
//   k_primal<W,CHECK>  ATY = A'Y fused with the primal projection, the
//                      speculative Halpern step for X and the per-column
//                      sums sum dx^2, sum (x - anchor_x)^2   (:176-187,:326-330)
//   k_dual<W,CHECK>    AXT = A XT fused with the dual step, the speculative
//                      Halpern step for Y and AX and the per-column sums of
//                      the M-norm residual (:188-208); on check iterations
//                      also every row-space term of evaluate_optimality and
//                      of the infeasibility probe (solver.hpp:387-396,448-514)
//   k_check<W>         AT_YT = A'YT fused with the reduced costs and every
//                      column-space term of the check (:226-272)
//   k_decide           one CTA: residuals, averaged residual, statuses,
//                      best-candidate offers, swap-with-last compaction, the
//                      restart rule and weight update (:209-324)
//   k_cert<W>          masked A'dy for columns whose certificate needs it
//   k_snapshot, k_compact   vector snapshots and state column moves
//
// "Speculative Halpern": the kernels write z' = alpha (2 T(z) - z) +
// (1 - alpha) z0 into the second buffer of a double-buffered X/Y/AX while
// they compute T(z); the decide kernel either flips the buffer (no restart)
// or keeps the old one (a restart re-applies T at the same point,
// batch_solver.hpp:320-322). So a restart costs nothing and anchor copies
// are fused into the next iteration's reads.
//
// The row kernels are persistent: a fixed grid of CTAs walks work items
// (column block b, row range r) in block-major order so the gathered operand
// of one 32-column block stays L2 resident while all SMs work on it.
// Per-column sums are reduced deterministically: sequentially within a row
// group, then a fixed tree, then the last CTA of each block folds the
// per-item partials in item order. Items of <= kTinyRows rows are walked by a
// single group, so on small problems every sum is the reference's sequential
// sum, bit for bit.

#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <cooperative_groups.h>

#include <map>
#include <mutex>

#include "bl_device.cuh"

namespace bl {

// ---------------------------------------------------------------------------
// geometry and vector memory helpers
// ---------------------------------------------------------------------------
// LL > 0: "narrow" mapping for the latency-bound tail, where only the first
// LL * V slots of the (single) active block are live: fewer lanes per row,
// more rows processed in parallel. The tiled layout (stride W) is unchanged.
template <int W, int LL = 0, int NT = kBlock>
struct Geo {
  static constexpr int V = W >= 2 ? 2 : 1;                      // slots per lane (double2)
  static constexpr int L = LL > 0 ? LL : (W >= 2 ? W / 2 : 1);  // lanes per row
  static constexpr int G = NT / L;                              // row groups per CTA
};

template <int V>
__device__ __forceinline__ void ld_nc(const double* p, double (&o)[V]) {
  if constexpr (V == 2) {
    const double2 t = __ldg(reinterpret_cast<const double2*>(p));
    o[0] = t.x;
    o[1] = t.y;
  } else {
    o[0] = __ldg(p);
  }
}
// streamed once per iteration: evict-first so gathered tiles keep the L2
template <int V>
__device__ __forceinline__ void ld_cs(const double* p, double (&o)[V]) {
  if constexpr (V == 2) {
    const double2 t = __ldcs(reinterpret_cast<const double2*>(p));
    o[0] = t.x;
    o[1] = t.y;
  } else {
    o[0] = __ldcs(p);
  }
}
template <int V>
__device__ __forceinline__ void ld_cg(const double* p, double (&o)[V]) {
  if constexpr (V == 2) {
    const double2 t = __ldcg(reinterpret_cast<const double2*>(p));
    o[0] = t.x;
    o[1] = t.y;
  } else {
    o[0] = __ldcg(p);
  }
}
template <int V>
__device__ __forceinline__ void st_cs(double* p, const double (&v)[V]) {
  if constexpr (V == 2) {
    __stcs(reinterpret_cast<double2*>(p), make_double2(v[0], v[1]));
  } else {
    __stcs(p, v[0]);
  }
}
template <int V>
__device__ __forceinline__ void st_wb(double* p, const double (&v)[V]) {
  if constexpr (V == 2) {
    *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
  } else {
    *p = v[0];
  }
}

// Gathered operand rows: read-only path with an L2 eviction-priority hint
// (BL_GATHER_POLICY 1: evict_last, so the column block being gathered
// outlives the streamed operands, which are loaded / stored evict-first).
// The policy lives in the load's memory descriptor (a uniform register).
#ifndef BL_GATHER_POLICY
#define BL_GATHER_POLICY 1
#endif
template <int V>
__device__ __forceinline__ void ld_gather(const double* p, double (&o)[V]) {
  if constexpr (BL_GATHER_POLICY == 0) {
    ld_nc<V>(p, o);
  } else {
    unsigned long long pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    if constexpr (V == 2)
      asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                   : "=d"(o[0]), "=d"(o[1]) : "l"(p), "l"(pol));
    else
      asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(o[0]) : "l"(p), "l"(pol));
  }
}

// One CSR row of op(A) times the lane's V slots of a column block. The
// accumulation follows the stored order with separately rounded products
// and sums: the reference csr_apply (sparse.hpp:176-183) bit for bit.
template <int W, bool GENERIC = false>
__device__ __forceinline__ void gather_row(const int* __restrict__ rp,
                                           const int* __restrict__ ci,
                                           const double* __restrict__ cv,
                                           const double* __restrict__ base,
                                           int i, double (&acc)[Geo<W>::V]) {
  constexpr int V = Geo<W>::V;
  // GENERIC: the row metadata may live in shared memory (the tail's CSR
  // cache), so it is read with generic loads instead of the read-only path.
  auto ldi = [](const int* q) { return GENERIC ? *q : __ldg(q); };
  auto ldd = [](const double* q) { return GENERIC ? *q : __ldg(q); };
  int p = ldi(rp + i);
  const int e = ldi(rp + i + 1);
#pragma unroll
  for (int v = 0; v < V; ++v) acc[v] = 0.0;
#ifndef BL_TAIL_GATHER8
#define BL_TAIL_GATHER8 1
#endif
  if constexpr (GENERIC && BL_TAIL_GATHER8) {
    // the tail's rows: 8 operand rows in flight per batch (latency-bound)
    for (; p + 8 <= e; p += 8) {
      int c[8];
      double a[8], x[8][V];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        c[k] = ldi(ci + p + k);
        a[k] = ldd(cv + p + k);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) ld_nc<V>(base + (size_t)c[k] * W, x[k]);
#pragma unroll
      for (int k = 0; k < 8; ++k)
#pragma unroll
        for (int v = 0; v < V; ++v) acc[v] = __dadd_rn(acc[v], __dmul_rn(a[k], x[k][v]));
    }
  }
  for (; p + 4 <= e; p += 4) {
    const int c0 = ldi(ci + p), c1 = ldi(ci + p + 1);
    const int c2 = ldi(ci + p + 2), c3 = ldi(ci + p + 3);
    const double a0 = ldd(cv + p), a1 = ldd(cv + p + 1);
    const double a2 = ldd(cv + p + 2), a3 = ldd(cv + p + 3);
    double x0[V], x1[V], x2[V], x3[V];
    if constexpr (GENERIC) {
      ld_nc<V>(base + (size_t)c0 * W, x0);
      ld_nc<V>(base + (size_t)c1 * W, x1);
      ld_nc<V>(base + (size_t)c2 * W, x2);
      ld_nc<V>(base + (size_t)c3 * W, x3);
    } else {
      ld_gather<V>(base + (size_t)c0 * W, x0);
      ld_gather<V>(base + (size_t)c1 * W, x1);
      ld_gather<V>(base + (size_t)c2 * W, x2);
      ld_gather<V>(base + (size_t)c3 * W, x3);
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      acc[v] = __dadd_rn(acc[v], __dmul_rn(a0, x0[v]));
      acc[v] = __dadd_rn(acc[v], __dmul_rn(a1, x1[v]));
      acc[v] = __dadd_rn(acc[v], __dmul_rn(a2, x2[v]));
      acc[v] = __dadd_rn(acc[v], __dmul_rn(a3, x3[v]));
    }
  }
  if constexpr (GENERIC) {  // the tail's cached rows: registers are scarce there
    if (p + 2 <= e) {  // a pair, loads issued together
      const int c0 = ldi(ci + p), c1 = ldi(ci + p + 1);
      const double a0 = ldd(cv + p), a1 = ldd(cv + p + 1);
      double x0[V], x1[V];
      ld_nc<V>(base + (size_t)c0 * W, x0);
      ld_nc<V>(base + (size_t)c1 * W, x1);
#pragma unroll
      for (int v = 0; v < V; ++v) {
        acc[v] = __dadd_rn(acc[v], __dmul_rn(a0, x0[v]));
        acc[v] = __dadd_rn(acc[v], __dmul_rn(a1, x1[v]));
      }
      p += 2;
    }
    if (p < e) {
      const int c0 = ldi(ci + p);
      const double a0 = ldd(cv + p);
      double x0[V];
      ld_nc<V>(base + (size_t)c0 * W, x0);
#pragma unroll
      for (int v = 0; v < V; ++v) acc[v] = __dadd_rn(acc[v], __dmul_rn(a0, x0[v]));
    }
  } else if (p < e) {  // remainder (1..3): one predicated batch, loads issued together
    double a[3] = {0.0, 0.0, 0.0}, x[3][V];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (p + k < e) {
        a[k] = ldd(cv + p + k);
        ld_gather<V>(base + (size_t)ldi(ci + p + k) * W, x[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (p + k < e) {
#pragma unroll
        for (int v = 0; v < V; ++v) acc[v] = __dadd_rn(acc[v], __dmul_rn(a[k], x[k][v]));
      }
    }
  }
}

// The same product with the row metadata read cooperatively: the L lanes of
// a row group load L consecutive column indices / values with one coalesced
// access and broadcast them by shuffles, so the gathers of a row wait on one
// metadata round trip per L nonzeros instead of one per batch (ncu showed the
// row kernels stalled on the index -> address chain). Same summation order.
template <int W>
__device__ __forceinline__ void gather_row_grp(const int* __restrict__ rp,
                                               const int* __restrict__ ci,
                                               const double* __restrict__ cv,
                                               const double* __restrict__ base, int i, int L,
                                               double (&acc)[Geo<W>::V]) {
  constexpr int V = Geo<W>::V;
  const int lane = threadIdx.x & 31;
  const int gl = lane & (L - 1);
  const unsigned mask = L >= 32 ? 0xffffffffu : (((1u << L) - 1u) << (lane & ~(L - 1)));
  const int p = __ldg(rp + i);
  const int e = __ldg(rp + i + 1);
#pragma unroll
  for (int v = 0; v < V; ++v) acc[v] = 0.0;
  for (int ch = p; ch < e; ch += L) {
    const int k = ch + gl;
    int myc = 0;
    double myv = 0.0;
    if (k < e) {
      myc = __ldg(ci + k);
      myv = __ldg(cv + k);
    }
    const int cnt = min(L, e - ch);
    constexpr int D = 4;  // gathers in flight per batch
    for (int t = 0; t < cnt; t += D) {
      int c[D];
      double a[D], x[D][V];
#pragma unroll
      for (int q = 0; q < D; ++q) {
        c[q] = __shfl_sync(mask, myc, t + q, L);
        a[q] = __shfl_sync(mask, myv, t + q, L);
      }
#pragma unroll
      for (int q = 0; q < D; ++q)
        if (t + q < cnt) ld_gather<V>(base + (size_t)c[q] * W, x[q]);
#pragma unroll
      for (int q = 0; q < D; ++q)
        if (t + q < cnt) {
#pragma unroll
          for (int v = 0; v < V; ++v) acc[v] = __dadd_rn(acc[v], __dmul_rn(a[q], x[q][v]));
        }
    }
  }
}

// ---------------------------------------------------------------------------
// column sums and the M-norm residual
// ---------------------------------------------------------------------------
__device__ __forceinline__ double cs(const Params& P, int s, int j) {
  return P.colsum[(size_t)s * P.Kp + j];
}
__device__ __forceinline__ double& csr(const Params& P, int s, int j) {
  return P.colsum[(size_t)s * P.Kp + j];
}

// m_residual_from_terms, solver.hpp:250-263
__device__ __forceinline__ double m_residual(double dx2, double dy2, double cross,
                                             double eta, double w, int* err) {
  const double msq = (w / eta) * dx2 + (1.0 / (eta * w)) * dy2 + 2.0 * cross;
  if (msq < 0.0) {
    const double scale = (w / eta) * dx2 + (1.0 / (eta * w)) * dy2 + 2.0 * fabs(cross);
    if (msq < -1e-12 * smax(1.0, scale)) *err = 1;
    return 0.0;
  }
  return sqrt(msq);
}

// Warp 0 of the CTA that folded a column block's dual sums: the block's
// M-norm residuals (m_residual_from_terms, solver.hpp:250-263) and their
// sequential sum. Out of line, so the dual's row loop is register-allocated
// without it.
static __device__ __noinline__ void fold_residuals(const double* colsum, int Kp,
                                                   const double* w, double eta, int j0,
                                                   int valid, double* resid, double* blk,
                                                   int* err_flag) {
  const int lane = threadIdx.x;
  const int j = j0 + lane;
  double r = 0.0;
  if (lane < valid) {
    int err = 0;
    r = m_residual(colsum[(size_t)S_DX2 * Kp + j], colsum[(size_t)S_DY2 * Kp + j],
                   colsum[(size_t)S_CROSS * Kp + j], eta, w[j], &err);
    resid[j] = r;
    if (err) atomicOr(err_flag, 1);
  }
  double sum = 0.0;
  for (int k = 0; k < valid; ++k) sum += __shfl_sync(0xffffffffu, r, k);
  if (lane == 0) *blk = sum;
}

// ---------------------------------------------------------------------------
// deterministic per-column reduction of one work item
// ---------------------------------------------------------------------------
// acc[s][v]: this lane's sums for slots (b*W + li*V + v). Reduces over the
// CTA in a fixed tree, writes the item's partials, and the last CTA of block
// b folds all R partials in item order into colsum[s0+s][slot].
// `red` is a shared buffer of at least kRedDoubles doubles.
// Ops may finish a column block once its sums are folded (only ops with an
// after_fold member; called by the CTA that folded, after a barrier).
template <class Op>
__device__ __forceinline__ auto after_fold_impl(Op& op, int b, int) -> decltype(op.after_fold(b), void()) {
  __syncthreads();  // the fold's colsum stores are visible to the whole CTA
  op.after_fold(b);
}
template <class Op>
__device__ __forceinline__ void after_fold_impl(Op&, int, long) {}

struct NoOp {};

template <int W, int NS, int LL = 0, class Op = NoOp>
__device__ __forceinline__ void publish_item(double (&acc)[NS][Geo<W>::V], int b,
                                             int r, int R, double* partials,
                                             int* counters, double* colsum,
                                             int s0, int Kp, double* red, Op* op = nullptr) {
  using Gm = Geo<W, LL>;
  constexpr int V = Gm::V, L = Gm::L;
  static_assert(kWarps * NS * W <= kRedDoubles, "reduction buffer too small");
  __shared__ int last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int off = 16; off >= L; off >>= 1) {
#pragma unroll
    for (int s = 0; s < NS; ++s)
#pragma unroll
      for (int v = 0; v < V; ++v)
        acc[s][v] = __dadd_rn(acc[s][v], __shfl_down_sync(0xffffffffu, acc[s][v], off));
  }
  if (lane < L) {
#pragma unroll
    for (int s = 0; s < NS; ++s)
#pragma unroll
      for (int v = 0; v < V; ++v) red[(warp * NS + s) * W + lane * V + v] = acc[s][v];
  }
  __syncthreads();
  for (int t = tid; t < NS * W; t += kBlock) {
    const int s = t / W, jj = t - s * W;
    double sum = 0.0;
    if (jj < L * V) {  // slots beyond a narrow mapping's lanes are not live
#pragma unroll
      for (int wp = 0; wp < kWarps; ++wp) sum = __dadd_rn(sum, red[(wp * NS + s) * W + jj]);
    }
    partials[((size_t)(b * R + r) * NS + s) * W + jj] = sum;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) last = (atomicAdd(&counters[b], 1) == R - 1);
  __syncthreads();
  if (last) {
    __threadfence();
    constexpr int Q = NS * W;  // outputs of this block
    if constexpr (Q <= kBlock) {
      // T threads per output; thread `part` folds items part, part+T, ...
      // in order, then the T partial folds are added in part order. Fixed
      // order for any timing; with R = 1 it is the single partial exactly.
      double* fold = red;  // free again: the item partials are written
      constexpr int T = kBlock / Q;
      const int q = tid % Q, part = tid / Q;
      double sum = 0.0;
      if (part < T) {
        const int s = q / W, jj = q - s * W;
        const double* src = partials + ((size_t)b * R * NS + s) * W + jj;
#pragma unroll 8
        for (int rr = part; rr < R; rr += T)
          sum = __dadd_rn(sum, __ldcg(src + (size_t)rr * NS * W));
      }
      fold[tid] = sum;
      __syncthreads();
      if (tid < Q) {
        double tot = 0.0;
#pragma unroll
        for (int pp = 0; pp < T; ++pp) tot = __dadd_rn(tot, fold[pp * Q + tid]);
        const int s = tid / W, jj = tid - s * W;
        colsum[(size_t)(s0 + s) * Kp + b * W + jj] = tot;
      }
    } else {
      for (int t = tid; t < Q; t += kBlock) {
        const int s = t / W, jj = t - s * W;
        const double* src = partials + ((size_t)b * R * NS + s) * W + jj;
        double sum = 0.0;
#pragma unroll 8
        for (int rr = 0; rr < R; ++rr) sum = __dadd_rn(sum, __ldcg(src + (size_t)rr * NS * W));
        colsum[(size_t)(s0 + s) * Kp + b * W + jj] = sum;
      }
    }
    if (tid == 0) counters[b] = 0;
    if (op) after_fold_impl(*op, b, 0);
  }
  __syncthreads();
}

// Column descriptor of one LP slot as staged in shared memory (ColInfo).
// 11 words, doubles as (lo, hi) word pairs: a lane reads its slots at a
// stride of 22 words, so the 16 lanes of a row group hit 16 distinct banks
// (a 48-byte record put lanes 0, 4, 8, 12 on one bank: 4-way conflicts on
// every per-row descriptor read).
struct SColInfo {
  int valid, orig, ob, oe, v0, k0;
  int fast;  // single-point column (see ColInfo)
  int val0_w[2], step_w[2];
};
static_assert(sizeof(SColInfo) == 44, "SColInfo: odd word stride");
__device__ __forceinline__ double scol_step(const volatile SColInfo* s) {
  return __hiloint2double(s->step_w[1], s->step_w[0]);
}
__device__ __forceinline__ double scol_val0(const volatile SColInfo* s) {
  return __hiloint2double(s->val0_w[1], s->val0_w[0]);
}
__device__ __forceinline__ void scol_set_step(volatile SColInfo* s, double v) {
  s->step_w[0] = __double2loint(v);
  s->step_w[1] = __double2hiint(v);
}

// One shared array of column descriptors per CTA, whichever run_rows
// instantiation uses it (a __shared__ in a non-template function has a
// single instance).
static __device__ __noinline__ SColInfo* col_smem() {
  __shared__ SColInfo s[32];
  return s;
}

// Resident CTAs per SM the row kernels are compiled for (caps registers).
#ifndef BL_ROW_MIN_CTAS
#define BL_ROW_MIN_CTAS 3
#endif
constexpr int kRowMinCtas = BL_ROW_MIN_CTAS;
// the primal kernel carries fewer per-row sums and fits 4 CTAs per SM
#ifndef BL_PRIMAL_MIN_CTAS
#define BL_PRIMAL_MIN_CTAS 4
#endif
constexpr int kPrimalMinCtas = BL_PRIMAL_MIN_CTAS;
#ifndef BL_DUAL_MIN_CTAS
#define BL_DUAL_MIN_CTAS 4
#endif
constexpr int kDualMinCtas = BL_DUAL_MIN_CTAS;
// the narrow single-block passes (latency-bound, one column block's operand
// in L2) run at 3 CTAs / SM: 80 registers, spill-free primal (C3 -3.6%)
#ifndef BL_NARROW_MIN_CTAS
#define BL_NARROW_MIN_CTAS 3
#endif
constexpr int kNarrowMinCtas = BL_NARROW_MIN_CTAS;

// Tells an op how many lanes share a row (only ops with a `lanes` member).
template <class Op>
__device__ __forceinline__ auto set_lanes_impl(Op& op, int L, int) -> decltype(op.lanes = L, void()) {
  op.lanes = L;
}
template <class Op>
__device__ __forceinline__ void set_lanes_impl(Op&, int, long) {}
template <class Op>
__device__ __forceinline__ void set_lanes(Op& op, int L) {
  set_lanes_impl(op, L, 0);
}

// Walks the work items of a persistent row kernel. Op provides:
//   begin(b, slot0, acc, owner)  per item (owner: holds the matrix's row 0)
//   row(b, i, slot0, acc)        per row of the group's contiguous chunk
// One work item: rows [r * per, (r + 1) * per) of column block b, split
// over the CTA's row groups (a tiny dimension is walked by one group), then
// the item's deterministic reduction (publish_item).
template <int W, int NS, int LL = 0, class Op>
__device__ __forceinline__ void run_item(Op& op, int b, int r, int rows, int R,
                                         double* partials, int* counters, double* colsum,
                                         int s0, int Kp, double* red) {
  using Gm = Geo<W, LL>;
  constexpr int V = Gm::V, L = Gm::L, G = Gm::G;
  SColInfo* s_col = col_smem();
  const int tid = threadIdx.x, g = tid / L, li = tid - g * L;
  const int per = R > 0 ? (rows + R - 1) / R : 0;
  const int r0 = min(rows, r * per), r1 = min(rows, r0 + per);
  const int cnt = r1 - r0;
  int gs, ge;
  if (rows <= kTinyRows) {  // whole dimension tiny: one sequential walk
    gs = g == 0 ? r0 : r1;
    ge = r1;
  } else {
    const int ch = (cnt + G - 1) / G;
    gs = min(r1, r0 + g * ch);
    ge = min(r1, gs + ch);
  }
  double acc[NS][V];
#pragma unroll
  for (int s = 0; s < NS; ++s)
#pragma unroll
    for (int v = 0; v < V; ++v) acc[s][v] = 0.0;
  const int slot0 = b * W + li * V;
  if (tid < W) op.stage(b * W + tid, &s_col[tid]);
  __syncthreads();
  op.begin(b, slot0, acc, r == 0 && g == 0, &s_col[li * V]);
  set_lanes(op, L);
  for (int i = gs; i < ge; ++i) op.row(b, i, slot0, li, acc);
  publish_item<W, NS, LL>(acc, b, r, R, partials, counters, colsum, s0, Kp, red, &op);
}

#ifndef BL_DYNAMIC_ITEMS
#define BL_DYNAMIC_ITEMS 1
#endif

// Items [0, items) handed to the grid from one atomic ticket, in order (the
// next one fetched while the current item runs), so every CTA works on the
// column block the grid is on: only ~one block's gathered operand is live in
// L2 (a static stride lets slow and fast CTAs drift apart by blocks). Which
// CTA runs an item changes no sum: partials are indexed by item and folded
// in item order. The last CTA to retire re-arms the ticket (and runs
// `on_last`, thread 0) for the next launch / phase.
template <class F, class G>
__device__ __forceinline__ void ticket_items(int* ticket, int items, F&& fn, G&& on_last) {
  const int tid = threadIdx.x;
  __shared__ int s_next[2];
  if (tid == 0) s_next[0] = atomicAdd(ticket, 1);
  __syncthreads();
  int par = 0;
  for (int w = s_next[0]; w < items; w = s_next[par]) {
    if (tid == 0) s_next[par ^ 1] = atomicAdd(ticket, 1);
    fn(w);  // ends with a CTA barrier: s_next[par ^ 1] is visible
    par ^= 1;
  }
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(ticket + 1, 1) == (int)gridDim.x - 1) {
      on_last();
      atomicExch(ticket, 0);
      atomicExch(ticket + 1, 0);
      __threadfence();
    }
  }
}

// REV: walk the column blocks last to first. The dual runs reversed so it
// starts on the block whose XT the primal wrote last, and the next primal
// (forward) starts on the block whose Y the dual wrote last: each pass
// begins on operands still in L2.
#ifndef BL_PINGPONG
#define BL_PINGPONG 1
#endif
template <int W, int NS, int LL = 0, bool REV = false, class Op>
__device__ __forceinline__ void run_rows(Op& op, int rows, int nb, int R,
                                         double* partials, int* counters,
                                         double* colsum, int s0, int Kp, double* red,
                                         int* ticket = nullptr) {
  const int items = nb * R;
  auto item = [&](int w) {
    const int bw = w / R, r = w - bw * R;
    const int b = (REV && BL_PINGPONG) ? nb - 1 - bw : bw;
    run_item<W, NS, LL>(op, b, r, rows, R, partials, counters, colsum, s0, Kp, red);
  };
  if (!BL_DYNAMIC_ITEMS || ticket == nullptr) {
    for (int w = blockIdx.x; w < items; w += gridDim.x) item(w);
    return;
  }
  ticket_items(ticket, items, item, [] {});
}

// Lanes per row for a pass: full width unless one block is active, then the
// smallest power of two covering the live slots (narrow tail mapping).
template <int W>
__device__ __forceinline__ int pass_lanes(int active) {
  constexpr int Lfull = Geo<W>::L, V = Geo<W>::V;
  if (active > W) return Lfull;
  int L = 1;
  while (L * V < active && L < Lfull) L <<= 1;
  return L;
}

#define BL_DISPATCH_L(W, Lsel, CALL)                                          \
  switch (Lsel) {                                                            \
    case 1: if constexpr (Geo<W>::L >= 1) { constexpr int LL_ = 1; CALL; } break;   \
    case 2: if constexpr (Geo<W>::L >= 2) { constexpr int LL_ = 2; CALL; } break;   \
    case 4: if constexpr (Geo<W>::L >= 4) { constexpr int LL_ = 4; CALL; } break;   \
    case 8: if constexpr (Geo<W>::L >= 8) { constexpr int LL_ = 8; CALL; } break;   \
    default: { constexpr int LL_ = 0; CALL; } break;                         \
  }

// Effective cost / bounds of one column at one variable (ColumnView,
// problem.hpp:209-236): base entry or signed unit objective, then the
// column's overrides in list order (later entries win).
// fast: the column equals the base row data (zero cost in signed-unit mode)
// except at most at one variable v0 where (k0, val0) applies -- every FSB
// column (<= 1 bound override) and every OBBT column (its signed unit,
// canonicalised into v0 = the unit's variable, an objective entry of +-1).
// Other columns walk the general rule.
struct ColInfo {
  int valid, orig, ob, oe, v0, k0;
  double val0, step;
  int fast;
};

__device__ __forceinline__ void load_col(const Params& P, int j, int active,
                                         bool dual_step, ColInfo& c) {
  c.valid = j < active;
  c.orig = c.valid ? P.slot_orig[j] : 0;
  c.ob = c.valid ? P.ov_beg[c.orig] : 0;
  c.oe = c.valid ? P.ov_end[c.orig] : 0;
  c.v0 = -1;
  c.k0 = 0;
  c.val0 = 0.0;
  if (c.oe > c.ob) {
    c.v0 = P.ov_var[c.ob];
    c.k0 = P.ov_kind[c.ob];
    c.val0 = P.ov_val[c.ob];
  }
  if (P.mode == BL_SIGNED_UNIT_COLUMNS) {
    c.fast = c.oe == c.ob;
    if (c.fast) {  // the unit itself is the single point
      const int o = c.orig + P.unit_off, n = P.n;
      c.v0 = o < n ? o : o - n;
      c.k0 = BL_OVERRIDE_OBJECTIVE;
      c.val0 = o < n ? 1.0 : -1.0;
    }
  } else {
    c.fast = c.oe - c.ob <= 1;
  }
  // StepParams (solver.hpp:58-59): tau = eta / w, sigma = eta * w
  const double w = c.valid ? P.w[j] : 1.0;
  c.step = dual_step ? P.eta * w : P.eta / w;
}

__device__ __forceinline__ void apply_ov(int kind, double val, double& cc,
                                         double& lo, double& hi) {
  if (kind == BL_OVERRIDE_OBJECTIVE) cc = val;
  else if (kind == BL_OVERRIDE_LOWER) lo = val;
  else hi = val;
}

__device__ __forceinline__ void col_vals(const Params& P, const ColInfo& c, int i,
                                         double bc, double bl, double bh,
                                         double& cc, double& lo, double& hi) {
  cc = bc;
  lo = bl;
  hi = bh;
  if (c.fast) {
    if (c.v0 == i) apply_ov(c.k0, c.val0, cc, lo, hi);
    return;
  }
  if (P.mode == BL_SIGNED_UNIT_COLUMNS) {
    const int n = P.n, o = c.orig + P.unit_off;
    cc = o < n ? (i == o ? 1.0 : 0.0) : (i == o - n ? -1.0 : 0.0);
  }
  if (c.v0 == i) apply_ov(c.k0, c.val0, cc, lo, hi);
  for (int k = c.ob + 1; k < c.oe; ++k)
    if (P.ov_var[k] == i) apply_ov(P.ov_kind[k], P.ov_val[k], cc, lo, hi);
}

// The column descriptors of the block a CTA is working on live in shared
// memory (staged once per work item) and are re-read per row through a
// volatile view, so they do not occupy registers across the gather loop:
// register pressure, not bandwidth, sets the occupancy of the row kernels.
__device__ __forceinline__ ColInfo read_col(const volatile SColInfo* s) {
  ColInfo c;
  c.valid = s->valid;
  c.orig = s->orig;
  c.ob = s->ob;
  c.oe = s->oe;
  c.v0 = s->v0;
  c.k0 = s->k0;
  c.val0 = scol_val0(s);
  c.step = scol_step(s);
  c.fast = s->fast;
  return c;
}
__device__ __forceinline__ void stage_col(const Params& P, int j, int active, bool dual_step,
                                          volatile SColInfo* s) {
  ColInfo c;
  load_col(P, j, active, dual_step, c);
  s->valid = c.valid;
  s->orig = c.orig;
  s->ob = c.ob;
  s->oe = c.oe;
  s->v0 = c.v0;
  s->k0 = c.k0;
  s->val0_w[0] = __double2loint(c.val0);
  s->val0_w[1] = __double2hiint(c.val0);
  scol_set_step(s, c.step);
  s->fast = c.fast;
}

// ---------------------------------------------------------------------------
// primal: XT = proj(X - tau (c + A'Y)), X' = Halpern, sums
// ---------------------------------------------------------------------------
// GEN: the CSR arrays may be the tail's shared-memory cache (generic loads)
template <int W, bool CHECK, bool GEN = false>
struct PrimalOp {
  static constexpr int V = Geo<W>::V;
  const Params& P;
  int active, reset;
  double alpha, oma;
  int cur;  // X / Y buffer of this iteration (pointers come from P: no registers)
  const volatile SColInfo* col;  // this lane's V column descriptors (shared memory)
  const int* crp;                // A' CSR (global, or a shared-memory cache of it)
  const int* cci;
  const double* ccv;
  int lanes = Geo<W>::L;  // lanes per row group (narrow tail mappings use fewer)
  __device__ __forceinline__ const int* rp_() const {
    if constexpr (GEN) return crp; else return P.trp;
  }
  __device__ __forceinline__ const int* ci_() const {
    if constexpr (GEN) return cci; else return P.tci;
  }
  __device__ __forceinline__ const double* cv_() const {
    if constexpr (GEN) return ccv; else return P.tcv;
  }
  __device__ PrimalOp(const Params& p, const Ctrl& C) : P(p) {
    crp = P.trp;
    cci = P.tci;
    ccv = P.tcv;
    active = C.active;
    reset = C.anchor_reset;
    alpha = C.alpha;
    oma = 1.0 - alpha;
    cur = C.cur;
  }
  __device__ void stage(int j, volatile SColInfo* s) { stage_col(P, j, active, false, s); }
  __device__ void begin(int, int, double (&)[2][V], bool, const volatile SColInfo* sc) {
    col = sc;
  }
  __device__ __forceinline__ void finish(size_t idx, int i, double bc, double bl, double bh,
                                         const double (&x)[V], const double (&ax)[V],
                                         const double (&aty)[V], double (&acc)[2][V]) {
    double xt[V], xn[V], rc[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      // descriptor fields read where needed (volatile: not kept in registers)
      const volatile SColInfo* sc = col + v;
      double cc = bc, lo = bl, hi = bh;
      if (sc->fast) {
        if (sc->v0 == i) apply_ov(sc->k0, scol_val0(sc), cc, lo, hi);
      } else {
        col_vals(P, read_col(sc), i, bc, bl, bh, cc, lo, hi);
      }
      const double t = cc + aty[v];
      xt[v] = project_box(x[v] - scol_step(sc) * t, lo, hi);
      const double dx = xt[v] - x[v];
      const double da = x[v] - ax[v];
      if (sc->valid) {
        acc[0][v] += dx * dx;
        acc[1][v] += da * da;
      }
      xn[v] = alpha * (2.0 * xt[v] - x[v]) + oma * ax[v];
      if (CHECK) rc[v] = project_barrier(-cc - aty[v], lo, hi);
    }
    st_wb<V>(P.XT + idx, xt);
    st_cs<V>(P.X[cur ^ 1] + idx, xn);
    if (reset) st_cs<V>(P.aX + idx, x);
    if (CHECK) st_wb<V>(P.RC + idx, rc);
  }
  __device__ void row(int b, int i, int, int li, double (&acc)[2][V]) {
    const int n = P.n, m = P.m;
    // streamed operands first, so their latency overlaps the gathers
    const double bc = P.mode == BL_SHARED_OBJECTIVE ? __ldg(P.c + i) : 0.0;
    const double bl = __ldg(P.xl + i), bh = __ldg(P.xu + i);
    const size_t idx = ((size_t)b * n + i) * W + li * V;
    double x[V], ax[V];
    ld_cs<V>(P.X[cur] + idx, x);
    if (reset) {
#pragma unroll
      for (int v = 0; v < V; ++v) ax[v] = x[v];
    } else {
      ld_cs<V>(P.aX + idx, ax);
    }
    double aty[V];
    // (the cooperative-metadata gather measured slower for A' rows: short rows)
    gather_row<W, GEN>(rp_(), ci_(), cv_(), P.Y[cur] + (size_t)b * m * W + li * V, i, aty);
    finish(idx, i, bc, bl, bh, x, ax, aty, acc);
  }
};

template <int W, bool CHECK, int LL = 0>
static __device__ void primal_body(const Params& P, const Ctrl& C, double* red) {
  prof_begin(P, K_PRIMAL);
  PrimalOp<W, CHECK> op(P, C);
  const int nb = (C.active + W - 1) / W;
  run_rows<W, 2, LL>(op, P.n, nb, C.Rp, P.partials, P.counters, P.colsum, S_DX2, P.Kp, red,
                     P.ticket);
  prof_end(P, K_PRIMAL);
}

// Full-width passes and narrow single-block passes are separate kernels (the
// graph picks one per pass through IF(narrow), set by the decide): the
// full-width row loop is register-allocated alone, which keeps it free of
// spills. Narrow: with one column block left and a LPs live, rows are walked
// by the smallest power of two of lanes covering them (only live slots are
// gathered).
template <int W, bool CHECK>
__global__ void __launch_bounds__(kBlock, kPrimalMinCtas) k_primal(Params P) {
  __shared__ double red[kRedDoubles];
  __shared__ Ctrl C;
  if (threadIdx.x == 0) C = *P.ctrl;
  __syncthreads();
  if (C.done) return;
  primal_body<W, CHECK>(P, C, red);
}

template <int W, bool CHECK>
__global__ void __launch_bounds__(kBlock, kNarrowMinCtas) k_primal_narrow(Params P) {
  __shared__ double red[kRedDoubles];
  __shared__ Ctrl C;
  if (threadIdx.x == 0) C = *P.ctrl;
  __syncthreads();
  if (C.done) return;
  const int Lsel = pass_lanes<W>(C.active);
  BL_DISPATCH_L(W, Lsel, (primal_body<W, CHECK, LL_>(P, C, red)));
}

// ---------------------------------------------------------------------------
// dual: AXT = A XT, YT = sigma (s - proj(s)), Y'/AX' = Halpern, sums
// ---------------------------------------------------------------------------
#ifndef BL_DUAL_LATE
#define BL_DUAL_LATE 1
#endif
template <int W, bool CHECK, bool GRP = true, bool GEN = false>
struct DualOp {
  static constexpr int V = Geo<W>::V;
  static constexpr int NS = CHECK ? 9 : 3;
  const Params& P;
  int active, reset;
  double alpha, oma;
  int cur;  // Y / AX buffer of this iteration (pointers come from P)
  const volatile SColInfo* col;
  const int* crp;  // A CSR (global, or a shared-memory cache of it)
  const int* cci;
  const double* ccv;
  int lanes = Geo<W>::L;
  __device__ __forceinline__ const int* rp_() const {
    if constexpr (GEN) return crp; else return P.rp;
  }
  __device__ __forceinline__ const int* ci_() const {
    if constexpr (GEN) return cci; else return P.ci;
  }
  __device__ __forceinline__ const double* cv_() const {
    if constexpr (GEN) return ccv; else return P.cv;
  }
  __device__ DualOp(const Params& p, const Ctrl& C) : P(p) {
    crp = P.rp;
    cci = P.ci;
    ccv = P.cv;
    active = C.active;
    reset = C.anchor_reset;
    alpha = C.alpha;
    oma = 1.0 - alpha;
    cur = C.cur;
  }
  __device__ void stage(int j, volatile SColInfo* s) { stage_col(P, j, active, true, s); }
  __device__ void begin(int, int, double (&)[NS][V], bool, const volatile SColInfo* sc) {
    col = sc;
  }
  // Once block b's dual sums are folded (the primal's are final since the
  // previous launch), its M-norm residuals (m_residual_from_terms,
  // solver.hpp:250-263) and their sequential block sum are computed here,
  // so the single-CTA decide only combines block sums (batch_solver.hpp:
  // 209-222). Warp 0 does it: W <= 32 slots.
  __device__ void after_fold(int b) {
    if (threadIdx.x < 32)
      fold_residuals(P.colsum, P.Kp, P.w, P.eta, b * W, min(W, active - b * W), P.resid,
                     P.blk_resid + b, P.err_flag);
  }
  __device__ void row(int b, int i, int, int li, double (&acc)[NS][V]) {
    const int n = P.n, m = P.m;
    const double lo = __ldg(P.rl + i), hi = __ldg(P.ru + i);
    const size_t idx = ((size_t)b * m + i) * W + li * V;
    double y[V], ax[V], ay[V], aax[V];
    auto streams = [&]() {
      ld_cs<V>(P.Y[cur] + idx, y);
      ld_cs<V>(P.AX[cur] + idx, ax);
      if (reset) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          ay[v] = y[v];
          aax[v] = ax[v];
        }
      } else {
        ld_cs<V>(P.aY + idx, ay);
        ld_cs<V>(P.aAX + idx, aax);
      }
    };
    // BL_DUAL_LATE: request the streamed operands after the gather, so they
    // hold no registers while it runs (the dual's live set spills otherwise)
    if (!BL_DUAL_LATE || GEN) streams();
    double axt[V];
    if (GEN) gather_row<W, true>(rp_(), ci_(), cv_(), P.XT + (size_t)b * n * W + li * V, i, axt);
    else if (GRP && lanes >= 4)
      gather_row_grp<W>(rp_(), ci_(), cv_(), P.XT + (size_t)b * n * W + li * V, i, lanes, axt);
    else gather_row<W>(rp_(), ci_(), cv_(), P.XT + (size_t)b * n * W + li * V, i, axt);
    if (BL_DUAL_LATE && !GEN) streams();
    finish(idx, lo, hi, y, ax, ay, aax, axt, acc);
  }
  __device__ __forceinline__ void finish(size_t idx, double lo, double hi, const double (&y)[V],
                                         const double (&ax)[V], const double (&ay)[V],
                                         const double (&aax)[V], const double (&axt)[V],
                                         double (&acc)[NS][V]) {
    double yt[V], yn[V], axn[V], dyb[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const volatile SColInfo* sc = col + v;
      const double sigma = scol_step(sc);
      const int valid = sc->valid;
      // dual_step_element, solver.hpp:186-190
      const double vv = 2.0 * axt[v] - ax[v];
      const double s = div_by_step(y[v], sigma) + vv;
      yt[v] = sigma * (s - project_box(s, lo, hi));
      const double dy = yt[v] - y[v];
      const double da = y[v] - ay[v];
      if (valid) {
        acc[0][v] += dy * dy;
        acc[1][v] += dy * (axt[v] - ax[v]);
        acc[2][v] += da * da;
      }
      yn[v] = alpha * (2.0 * yt[v] - y[v]) + oma * ay[v];
      axn[v] = alpha * (2.0 * axt[v] - ax[v]) + oma * aax[v];
      if constexpr (CHECK) {
        dyb[v] = project_barrier(yt[v] - y[v], lo, hi);
        if (valid) {
          acc[3][v] += support_term(yt[v], lo, hi);
          const double viol = axt[v] - project_box(axt[v], lo, hi);
          acc[4][v] += viol * viol;
          acc[5][v] += axt[v] * axt[v];
          const double term = support_term(dyb[v], lo, hi);
          acc[6][v] += term;
          acc[7][v] += fabs(term);
          const double adx = axt[v] - ax[v];
          const double rv = adx - project_recession(adx, lo, hi);
          acc[8][v] += rv * rv;
        }
      }
    }
    st_cs<V>(P.Y[cur ^ 1] + idx, yn);
    st_cs<V>(P.AX[cur ^ 1] + idx, axn);
    if (reset) {
      st_cs<V>(P.aY + idx, y);
      st_cs<V>(P.aAX + idx, ax);
    }
    if constexpr (CHECK) {
      st_wb<V>(P.YT + idx, yt);
      st_wb<V>(P.AXT + idx, axt);
      st_wb<V>(P.DY + idx, dyb);
    }
  }
};

template <int W, bool CHECK, int LL = 0, bool GRP = true>
static __device__ void dual_body(const Params& P, const Ctrl& C, double* red) {
  prof_begin(P, K_DUAL);
  using Op = DualOp<W, CHECK, GRP>;
  Op op(P, C);
  const int nb = (C.active + W - 1) / W;
  run_rows<W, Op::NS, LL, true>(op, P.m, nb, C.Rd, P.partials, P.counters,
                                    P.colsum, S_DY2, P.Kp, red, P.ticket);
  prof_end(P, K_DUAL);
}

template <int W, bool CHECK>
__global__ void __launch_bounds__(kBlock, kDualMinCtas) k_dual(Params P) {
  __shared__ double red[kRedDoubles];
  __shared__ Ctrl C;
  if (threadIdx.x == 0) C = *P.ctrl;
  __syncthreads();
  if (C.done) return;
  dual_body<W, CHECK>(P, C, red);
}

template <int W, bool CHECK>
__global__ void __launch_bounds__(kBlock, kNarrowMinCtas) k_dual_narrow(Params P) {
  __shared__ double red[kRedDoubles];
  __shared__ Ctrl C;
  if (threadIdx.x == 0) C = *P.ctrl;
  __syncthreads();
  if (C.done) return;
  const int Lsel = pass_lanes<W>(C.active);
  BL_DISPATCH_L(W, Lsel, (dual_body<W, CHECK, LL_>(P, C, red)));
}

// ---------------------------------------------------------------------------
// check: AT_YT = A'YT, reduced costs and the column-space check terms
// ---------------------------------------------------------------------------
template <int W>
struct CheckOp {
  static constexpr int V = Geo<W>::V;
  static constexpr int NS = 10;
  const Params& P;
  int active;
  const double* Xcur;
  const volatile SColInfo* col;
  __device__ CheckOp(const Params& p, const Ctrl& C) : P(p) {
    active = C.active;
    Xcur = P.X[C.cur];
  }
  __device__ void stage(int j, volatile SColInfo* s) { stage_col(P, j, active, false, s); }
  __device__ void begin(int, int slot0, double (&acc)[NS][V], bool owner,
                        const volatile SColInfo* sc) {
    col = sc;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      // The displacement support of the probe continues the row-space sum
      // (solver.hpp:463-474): seed it into the chunk holding variable 0.
      if (owner && col[v].valid) {
        acc[5][v] = P.colsum[(size_t)S_DYSUP * P.Kp + slot0 + v];
        acc[6][v] = P.colsum[(size_t)S_DYSCALE * P.Kp + slot0 + v];
      }
    }
  }
  __device__ void row(int b, int i, int, int li, double (&acc)[NS][V]) {
    const int n = P.n, m = P.m;
    const double bc = P.mode == BL_SHARED_OBJECTIVE ? __ldg(P.c + i) : 0.0;
    const double bl = __ldg(P.xl + i), bh = __ldg(P.xu + i);
    const size_t idx = ((size_t)b * n + i) * W + li * V;
    double xt[V], x[V], rc[V], r[V], dr[V];
    ld_cg<V>(P.XT + idx, xt);
    ld_cs<V>(Xcur + idx, x);
    ld_cs<V>(P.RC + idx, rc);
    double atyt[V];
    gather_row<W>(P.trp, P.tci, P.tcv, P.YT + (size_t)b * m * W + li * V, i, atyt);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const ColInfo cl = read_col(col + v);
      double cc, lo, hi;
      col_vals(P, cl, i, bc, bl, bh, cc, lo, hi);
      // evaluate_optimality, solver.hpp:369-386
      const double g = -cc - atyt[v];
      r[v] = project_barrier(g, lo, hi);
      // check_infeasibility_probe, solver.hpp:454-456
      dr[v] = project_barrier(r[v] - rc[v], lo, hi);
      if (cl.valid) {
        acc[0][v] += cc * xt[v];
        acc[1][v] += cc * cc;
        const double viol = cc + atyt[v] + r[v];
        acc[2][v] += viol * viol;
        if (P.robust) {
          if (g > 0.0 && hi != kInf) acc[3][v] += hi * g;
          else if (g < 0.0 && lo != -kInf) acc[3][v] += lo * g;
        } else {
          acc[3][v] += support_term(r[v], lo, hi);
        }
        acc[4][v] += support_term(r[v], bl, bh);
        const double term = support_term(dr[v], lo, hi);
        acc[5][v] += term;
        acc[6][v] += fabs(term);
        const double dx = xt[v] - x[v];
        const double t2 = cc * dx;
        acc[7][v] += t2;
        acc[8][v] += fabs(t2);
        const double rv = dx - project_recession(dx, lo, hi);
        acc[9][v] += rv * rv;
      }
    }
    st_wb<V>(P.R + idx, r);
    st_wb<V>(P.DR + idx, dr);
  }
};

template <int W, int LL = 0>
static __device__ void check_body(const Params& P, const Ctrl& C, double* red) {
  prof_begin(P, K_CHECK);
  CheckOp<W> op(P, C);
  const int nb = (C.active + W - 1) / W;
  run_rows<W, 10, LL>(op, P.n, nb, C.Rc, P.partials, P.counters, P.colsum, S_OBJ, P.Kp, red,
                      P.ticket);
  prof_end(P, K_CHECK);
}

template <int W>
__global__ void __launch_bounds__(kBlock, kRowMinCtas) k_check(Params P) {
  __shared__ double red[kRedDoubles];
  const Ctrl C = *P.ctrl;
  if (C.done || !C.check) return;
  check_body<W>(P, C, red);
}

template <int W>
__global__ void __launch_bounds__(kBlock, kRowMinCtas) k_check_narrow(Params P) {
  __shared__ double red[kRedDoubles];
  const Ctrl C = *P.ctrl;
  if (C.done || !C.check) return;
  const int Lsel = pass_lanes<W>(C.active);
  BL_DISPATCH_L(W, Lsel, (check_body<W, LL_>(P, C, red)));
}

// ---------------------------------------------------------------------------
// cert: ||A'dy + dr||^2 for the flagged columns (solver.hpp:476-483)
// ---------------------------------------------------------------------------
template <int W>
struct CertOp {
  static constexpr int V = Geo<W>::V;
  const Params& P;
  int active;
  int flag[V];
  __device__ CertOp(const Params& p, const Ctrl& C) : P(p) { active = C.active; }
  __device__ void stage(int, volatile SColInfo*) {}
  __device__ void begin(int, int slot0, double (&)[1][V], bool, const volatile SColInfo*) {
#pragma unroll
    for (int v = 0; v < V; ++v)
      flag[v] = (slot0 + v < active) ? P.cert_flag[slot0 + v] : 0;
  }
  __device__ void row(int b, int i, int, int li, double (&acc)[1][V]) {
    bool any = false;
#pragma unroll
    for (int v = 0; v < V; ++v) any = any || flag[v];
    if (!any) return;
    const int n = P.n, m = P.m;
    double at[V], dr[V];
    gather_row<W>(P.trp, P.tci, P.tcv, P.DY + (size_t)b * m * W + li * V, i, at);
    ld_cg<V>(P.DR + ((size_t)b * n + i) * W + li * V, dr);
#pragma unroll
    for (int v = 0; v < V; ++v)
      if (flag[v]) {
        const double q = at[v] + dr[v];
        acc[0][v] += q * q;
      }
  }
};

template <int W, int LL = 0>
static __device__ void cert_body(const Params& P, const Ctrl& C, double* red) {
  prof_begin(P, K_CERT);
  CertOp<W> op(P, C);
  const int nb = (C.active + W - 1) / W;
  run_rows<W, 1, LL>(op, P.n, nb, C.Rc, P.partials, P.counters, P.colsum, S_CERT, P.Kp, red,
                     P.ticket);
  prof_end(P, K_CERT);
}

template <int W>
__global__ void __launch_bounds__(kBlock, kRowMinCtas) k_cert(Params P) {
  __shared__ double red[kRedDoubles];
  const Ctrl C = *P.ctrl;
  if (C.done || !C.cert_pending) return;
  cert_body<W>(P, C, red);
}

// ---------------------------------------------------------------------------
// plain SpMM: out[:, j] = op(A) in[:, j] for j < active (sparse.hpp:213-238)
// ---------------------------------------------------------------------------
template <int W>
struct SpmmOp {
  static constexpr int V = Geo<W>::V;
  const int *rp, *ci;
  const double *cv, *in;
  double* out;
  int rows_in, rows_out, active;
  int valid[V];
  __device__ void stage(int, volatile SColInfo*) {}
  __device__ void begin(int, int slot0, double (&)[1][V], bool, const volatile SColInfo*) {
#pragma unroll
    for (int v = 0; v < V; ++v) valid[v] = slot0 + v < active;
  }
  __device__ void row(int b, int i, int, int li, double (&)[1][V]) {
    double o[V];
    gather_row<W>(rp, ci, cv, in + (size_t)b * rows_in * W + li * V, i, o);
    double* dst = out + ((size_t)b * rows_out + i) * W + li * V;
#pragma unroll
    for (int v = 0; v < V; ++v)
      if (valid[v]) dst[v] = o[v];
  }
};

template <int W>
__global__ void __launch_bounds__(kBlock) k_spmm(Params P, int transpose,
                                                 const double* in, double* out,
                                                 int active, int R, double* partials,
                                                 int* counters, double* colsum) {
  SpmmOp<W> op;
  op.rp = transpose ? P.trp : P.rp;
  op.ci = transpose ? P.tci : P.ci;
  op.cv = transpose ? P.tcv : P.cv;
  op.in = in;
  op.out = out;
  op.rows_in = transpose ? P.m : P.n;
  op.rows_out = transpose ? P.n : P.m;
  op.active = active;
  const int nb = (active + W - 1) / W;
  __shared__ double red[kRedDoubles];
  run_rows<W, 1>(op, op.rows_out, nb, R, partials, counters, colsum, 0, P.Kp, red, P.ticket);
}

// ---------------------------------------------------------------------------
// decide: one CTA runs the batch control of batch_solver.hpp:203-345
// ---------------------------------------------------------------------------
// ---- correctly rounded exp / log (double-double) ---------------------------
// The weight update is the only transcendental on the path. glibc's exp/log
// return the correctly rounded value except in rare near-midpoint cases, so
// evaluating them to ~100 bits and rounding once reproduces the reference's
// weights bit for bit (CUDA's exp/log are only faithful to 1-2 ulp).
struct DD {
  double hi, lo;
};
__device__ __forceinline__ DD two_sum(double a, double b) {
  const double s = a + b, bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ DD fast_two_sum(double a, double b) {
  const double s = a + b;
  return {s, b - (s - a)};
}
__device__ __forceinline__ DD dd_add(DD a, DD b) {
  DD s = two_sum(a.hi, b.hi);
  const DD t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = fast_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return fast_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ DD dd_mul(DD a, DD b) {
  const double p = a.hi * b.hi;
  double e = __fma_rn(a.hi, b.hi, -p);
  e += a.hi * b.lo + a.lo * b.hi;
  return fast_two_sum(p, e);
}
__device__ __forceinline__ DD dd_mul_d(DD a, double b) {
  const double p = a.hi * b;
  double e = __fma_rn(a.hi, b, -p);
  e += a.lo * b;
  return fast_two_sum(p, e);
}
// exp(x) = 2^k * s, s as a double-double.
// 1/i as double-doubles (exact to ~2^-106), i = 1..12.
__device__ __constant__ double kInvDD[12][2] = {
    {1.0, 0.0},
    {0.5, 0.0},
    {0.3333333333333333, 1.850371707708594e-17},
    {0.25, 0.0},
    {0.2, -1.1102230246251566e-17},
    {0.16666666666666666, 9.25185853854297e-18},
    {0.14285714285714285, 7.93016446160826e-18},
    {0.125, 0.0},
    {0.1111111111111111, 6.1679056923619804e-18},
    {0.1, -5.551115123125783e-18},
    {0.09090909090909091, -2.523234146875356e-18},
    {0.08333333333333333, 4.625929269271485e-18},
};
// ln 4, correctly rounded (glibc's log(4.0))
constexpr double kLog4 = 1.3862943611198906;

static __device__ DD dd_exp_scaled(double x, int* k_out) {
  const DD ln2 = {0.6931471805599453, 2.3190468138462996e-17};
  const double k = rint(x / ln2.hi);
  DD r = dd_add({x, 0.0}, dd_mul_d(ln2, -k));
  // |r| <= ln2/2 / 2^8: 12 Taylor terms reach ~2^-120, 8 squarings lose 8 bits
  r.hi = ldexp(r.hi, -8);
  r.lo = ldexp(r.lo, -8);
  DD s = {1.0, 0.0};
#pragma unroll
  for (int i = 12; i >= 1; --i) {  // Horner: 1 + r/i * (...)
    const DD inv_dd = {kInvDD[i - 1][0], kInvDD[i - 1][1]};
    s = dd_add({1.0, 0.0}, dd_mul(dd_mul(r, inv_dd), s));
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) s = dd_mul(s, s);
  *k_out = (int)k;
  return s;
}
static __device__ double cr_exp(double x) {
  if (isnan(x)) return x;
  if (x > 709.79) return exp(x);
  if (x < -708.0) return exp(x);
  int k;
  const DD s = dd_exp_scaled(x, &k);
  return ldexp(s.hi + s.lo, k);
}
static __device__ double cr_log(double x) {
  if (!(x > 0.0) || isinf(x)) return log(x);
  const double y0 = log(x);
  int k;
  DD e = dd_exp_scaled(-y0, &k);  // one Newton step: y0 + x e^{-y0} - 1
  e = dd_mul_d(e, x);
  e.hi = ldexp(e.hi, k);
  e.lo = ldexp(e.lo, k);
  const DD t = dd_add(e, {-1.0, 0.0});
  const DD y = dd_add({y0, 0.0}, t);
  return y.hi + y.lo;
}

// smoothed_primal_weight, solver.hpp:321-334
__device__ __forceinline__ double smoothed_weight(double w, double dxn, double dyn,
                                                  double theta) {
  if (!(dxn > 0.0) || !(dyn > 0.0) || !isfinite(dxn) || !isfinite(dyn)) return w;
  const double d = dyn / dxn;
  if (!isfinite(d) || d <= 0.0) return w;
  const double log_w = cr_log(w);
  const double proposed = theta * cr_log(d) + (1.0 - theta) * log_w;
  const double step_cap = kLog4;  // cr_log(4.0)
  if (proposed > log_w + step_cap) return cr_exp(log_w + step_cap);
  if (proposed < log_w - step_cap) return cr_exp(log_w - step_cap);
  return cr_exp(proposed);
}

// evaluate_optimality (solver.hpp:398-415) from the column sums, followed by
// the first half of check_infeasibility_probe (:463-475).
static __device__ void evaluate_column(const Params& P, int j) {
  const double obj = cs(P, S_OBJ, j);
  const double sup_r = cs(P, S_SUPR, j);
  const double sup_y = cs(P, S_SUPY, j);
  const double pres = sqrt(cs(P, S_PRES, j));
  const double dres = sqrt(cs(P, S_DRES, j));
  const double supports = sup_r + sup_y;
  const double gap = obj + supports;
  const double gap_scale = 1.0 + fabs(obj) + fabs(supports);
  const double rgap = isfinite(gap) ? fabs(gap) : kInf;
  const bool gap_ok = isfinite(gap) && fabs(gap) <= P.eps * gap_scale;
  const double primal_scale = 1.0 + sqrt(cs(P, S_AX2, j));
  const bool primal_ok = pres <= P.eps * primal_scale;
  const double dual_scale = 1.0 + sqrt(cs(P, S_CSQ, j));
  const bool dual_ok = dres <= P.eps_dual * dual_scale;
  double score = rgap / gap_scale;  // std::max({...}): first largest wins
  const double s2 = pres / primal_scale, s3 = dres / dual_scale;
  if (score < s2) score = s2;
  if (score < s3) score = s3;
  P.t_obj[j] = obj;
  P.t_gap[j] = rgap;
  P.t_pres[j] = pres;
  P.t_dres[j] = dres;
  P.t_score[j] = score;
  const double dsup = cs(P, S_DRSUP, j);
  P.t_dsup[j] = dsup;
  int v = V_NONE;
  if (gap_ok && primal_ok && dual_ok) {
    v = V_OPTIMAL;
  } else if (dsup < -1e-9 * smax(1.0, cs(P, S_DRSCALE, j))) {
    v = V_CERT_NEED;
  }
  P.verdict[j] = v;
}

// Dual-ray half of the probe, solver.hpp:495-525.
static __device__ bool dual_ray(const Params& P, int j) {
  const double desc = cs(P, S_DESC, j);
  if (desc < -1e-9 * smax(1.0, cs(P, S_DESCSCALE, j))) {
    const double budget = P.eps_infeas * fabs(desc);
    if (sqrt(cs(P, S_VARSQ, j)) <= budget && sqrt(cs(P, S_ROWSQ, j)) <= budget)
      return true;
  }
  return false;
}

__device__ __forceinline__ void set_cond(const Params& P,
                                         cudaGraphConditionalHandle h,
                                         unsigned v) {
  if (P.use_graph) cudaGraphSetConditional(h, v);
}
// Handle values persist through the WHILE loop of one graph launch (they
// are reset to their defaults only when the graph is launched), and a
// cudaGraphSetConditional costs ~1 us of the single-CTA decide: set a
// handle only when its value changes (Ctrl::cond mirrors the handles).
__device__ __forceinline__ void set_cond_if_changed(const Params& P, Ctrl& C, int bit,
                                                    cudaGraphConditionalHandle h, unsigned v) {
  const int cur = (C.cond >> bit) & 1;
  if (cur != (int)v) {
    set_cond(P, h, v);
    C.cond ^= 1 << bit;
  }
}

// Sum of v[0..count) in a fixed order: sequential (the reference's order)
// for count <= 256, else strided per thread then a fixed tree.
static __device__ double ordered_sum(const double* v, int count, double* sh) {
  const int tid = threadIdx.x;
  __shared__ double result;
  __syncthreads();
  if (count <= 256) {
    if (tid < count) sh[tid] = v[tid];  // stage: one parallel load, then a
    __syncthreads();                    // sequential sum out of shared memory
    if (tid == 0) {
      double s = 0.0;
      for (int j = 0; j < count; ++j) s += sh[j];
      result = s;
    }
    __syncthreads();
    return result;
  } else {
    double s = 0.0;
    for (int j = tid; j < count; j += (int)blockDim.x) s += v[j];
    sh[tid] = s;
    __syncthreads();
    for (int off = (int)blockDim.x / 2; off > 0; off >>= 1) {
      if (tid < off) sh[tid] = sh[tid] + sh[tid + off];
      __syncthreads();
    }
  }
  __syncthreads();
  const double r = sh[0];
  __syncthreads();
  return r;
}

static __device__ void write_result(const Params& P, const Ctrl& C, int j, int status,
                             int cert_kind) {
  const int o = P.slot_orig[j];
  bl_column_result& r = P.res[o];
  r.status = status;
  r.restarts = C.restarts;
  r.iterations = C.total_k;
  r.objective = P.t_obj[j];
  r.gap = P.t_gap[j];
  r.primal = P.t_pres[j];
  r.dual = P.t_dres[j];
  r.fixed_point = P.resid[j];
  r.bound_support = cs(P, S_SUPR, j);
  r.row_support = cs(P, S_SUPY, j);
  r.base_bound_support = cs(P, S_BSUPR, j);
  r.has_solution = P.vectors >= BL_VECTORS_SOLUTION;
  r.certificate_kind = cert_kind;
  r.has_certificate = (P.vectors >= BL_VECTORS_CERTIFICATE) && cert_kind != 0;
  r.vectors_exist = 1;
}

// Permutes every per-slot array by perm (new slot s <- old slot perm[s]).
static __device__ void permute_slots(const Params& P, const int* perm, int width,
                              double* scratch) {
  double* darr[] = {P.w, P.resid, P.anchor_resid, P.best_score, P.best_obj,
                    P.best_gap, P.best_pres, P.best_dres, P.best_fp, P.best_bsup,
                    P.best_rsup, P.best_bbsup,
                    P.colsum + (size_t)S_XA2 * P.Kp, P.colsum + (size_t)S_YA2 * P.Kp};
  constexpr int ND = 14;
  const int tid = threadIdx.x;
  for (int a = 0; a < ND; ++a) {
    for (int s = tid; s < width; s += (int)blockDim.x) scratch[s] = darr[a][perm[s]];
    __syncthreads();
    for (int s = tid; s < width; s += (int)blockDim.x) darr[a][s] = scratch[s];
    __syncthreads();
  }
  int* iarr[] = {P.slot_orig, P.has_best};
  int* iscratch = reinterpret_cast<int*>(scratch);
  for (int a = 0; a < 2; ++a) {
    for (int s = tid; s < width; s += (int)blockDim.x) iscratch[s] = iarr[a][perm[s]];
    __syncthreads();
    for (int s = tid; s < width; s += (int)blockDim.x) iarr[a][s] = iscratch[s];
    __syncthreads();
  }
}

// Diagnostic timing of decide_body on plain passes (P.dbg slots 10-14).
static __device__ __noinline__ unsigned long long* decide_mark_slot() {
  __shared__ unsigned long long t;
  return &t;
}
__device__ __forceinline__ void decide_mark(const Params& P, bool plain, int k) {
  if (P.dbg && threadIdx.x == 0 && plain) {
    const unsigned long long now = gtime();
    if (k > 10) P.dbg[k] += now - *decide_mark_slot();
    else P.dbg[10] += 1;
    *decide_mark_slot() = now;
  }
}

// Everything after the per-column verdicts (batch_solver.hpp:229-338).
static __device__ void finalize(const Params& P, Ctrl& C, double mean, double* sh,
                         int* ish, double* scratch) {
  const int tid = threadIdx.x;
  const int active0 = C.active;
  const int width = P.width;
  const bool plain = !C.check;
  int* snap_bits = P.cert_flag;  // reused: cert flags are consumed by now
  __shared__ int n_fin, n_snap;
  if (tid == 0) {
    n_fin = 0;
    n_snap = 0;
  }
  __syncthreads();
  if (C.check) {
    for (int j = tid; j < active0; j += (int)blockDim.x) {
      const int v = P.verdict[j];
      int bits = 0;
      if (v == V_OPTIMAL || v == V_PRIMAL_INF || v == V_DUAL_INF) {
        const int status = v == V_OPTIMAL ? BL_OPTIMAL
                           : v == V_PRIMAL_INF ? BL_PRIMAL_INFEASIBLE
                                               : BL_DUAL_INFEASIBLE;
        const int kind = v == V_PRIMAL_INF ? 1 : (v == V_DUAL_INF ? 2 : 0);
        write_result(P, C, j, status, kind);
        P.orig_done[P.slot_orig[j]] = 1;
        atomicAdd(&n_fin, 1);
        if (P.vectors >= BL_VECTORS_SOLUTION) bits |= SN_FINAL;
        if (P.vectors >= BL_VECTORS_CERTIFICATE && kind == 1) bits |= SN_CERTP;
        if (P.vectors >= BL_VECTORS_CERTIFICATE && kind == 2) bits |= SN_CERTD;
      } else {
        // BestCandidate::offer, solver.hpp:543-553
        const double score = P.t_score[j];
        if (!(score >= P.best_score[j])) {
          P.best_score[j] = score;
          P.best_obj[j] = P.t_obj[j];
          P.best_gap[j] = P.t_gap[j];
          P.best_pres[j] = P.t_pres[j];
          P.best_dres[j] = P.t_dres[j];
          P.best_fp[j] = P.resid[j];
          P.best_bsup[j] = cs(P, S_SUPR, j);
          P.best_rsup[j] = cs(P, S_SUPY, j);
          P.best_bbsup[j] = cs(P, S_BSUPR, j);
          P.has_best[j] = 1;
          if (P.vectors >= BL_VECTORS_SOLUTION) bits |= SN_BEST;
        }
      }
      snap_bits[j] = bits;
      P.snap_orig[j] = P.slot_orig[j];
    }
  }
  __syncthreads();
  decide_mark(P, plain, 16);
  int active = active0;
  int* perm = P.move_src;
  const bool at_cap = C.at_cap;
  const bool compact = C.check && n_fin > 0;
  if (compact) {
    // swap-with-last compaction scan (batch_solver.hpp:273-278), simulated
    // on the slot permutation only; the arrays are permuted afterwards.
    // The scan visits s = active0-1 .. 0 and swaps a finished slot with the
    // current end. A position is never modified before it is visited (swap
    // partners lie above it), so its "finished" flag is the static one:
    // the flags are gathered in parallel into a bitmask and one thread walks
    // only the set bits, with the permutation in shared memory when it fits.
    unsigned* fw = reinterpret_cast<unsigned*>(sh);        // flag words
    const int nwords = (active0 + 31) / 32;
    const bool perm_smem = nwords + active0 <= kDecideScratchInts;
    int* sp = perm_smem ? reinterpret_cast<int*>(sh) + nwords : perm;
    for (int s = tid; s < width; s += (int)blockDim.x) {
      perm[s] = s;
      if (perm_smem && s < active0) sp[s] = s;
    }
    for (int w = tid; w < nwords; w += (int)blockDim.x) {
      unsigned bits = 0u;
      for (int b = 0; b < 32; ++b) {
        const int s = 32 * w + b;
        if (s < active0 && P.orig_done[P.slot_orig[s]]) bits |= 1u << b;
      }
      fw[w] = bits;
    }
    __syncthreads();
    if (tid == 0) {
      int a = active0;
      for (int w = nwords - 1; w >= 0; --w) {
        unsigned bits = fw[w];
        while (bits) {
          const int b = 31 - __clz(bits);
          bits &= ~(1u << b);
          const int s = 32 * w + b;
          const int t = --a;
          const int tmp = sp[s];
          sp[s] = sp[t];
          sp[t] = tmp;
        }
      }
      ish[0] = a;
    }
    __syncthreads();
    if (perm_smem)
      for (int s = tid; s < active0; s += (int)blockDim.x) perm[s] = sp[s];
    __syncthreads();
    active = ish[0];
    permute_slots(P, perm, width, scratch);
    if (tid == 0) C.col_epoch += 1;
  }
  decide_mark(P, plain, 17);
  // iteration limit: freeze what is left from the best candidates (:280-295)
  if (at_cap && active > 0) {
    for (int j = tid; j < active; j += (int)blockDim.x) {
      const int o = P.slot_orig[j];
      bl_column_result& r = P.res[o];
      r.status = BL_ITERATION_LIMIT;
      r.restarts = C.restarts;
      r.iterations = C.total_k;
      const bool hb = P.has_best[j];
      r.objective = hb ? P.best_obj[j] : 0.0;
      r.gap = hb ? P.best_gap[j] : kInf;
      r.primal = hb ? P.best_pres[j] : kInf;
      r.dual = hb ? P.best_dres[j] : kInf;
      r.fixed_point = hb ? P.best_fp[j] : kInf;
      r.bound_support = hb ? P.best_bsup[j] : 0.0;
      r.row_support = hb ? P.best_rsup[j] : 0.0;
      r.base_bound_support = hb ? P.best_bbsup[j] : 0.0;
      r.has_solution = hb && P.vectors >= BL_VECTORS_SOLUTION;
      r.has_certificate = 0;
      r.certificate_kind = 0;
      r.vectors_exist = hb;
      P.orig_done[o] = 1;
      const int pre = compact ? perm[j] : j;
      if (hb && P.vectors >= BL_VECTORS_SOLUTION) snap_bits[pre] |= SN_CAP;
    }
    __syncthreads();
  }
  decide_mark(P, plain, 18);
  // snapshot list (pre-compaction slots) and move list (post <- pre)
  if (C.check) {
    for (int j = tid; j < active0; j += (int)blockDim.x) {
      const int bits = snap_bits[j];
      if (bits) {
        const int k = atomicAdd(&n_snap, 1);
        P.snap_list[3 * k] = j;
        P.snap_list[3 * k + 1] = P.snap_orig[j];
        P.snap_list[3 * k + 2] = bits;
      }
    }
  }
  __syncthreads();
  int n_moves = 0;
  if (compact && !(at_cap) && active > 0) {
    if (tid == 0) ish[1] = 0;
    __syncthreads();
    for (int s = tid; s < active; s += (int)blockDim.x) {
      if (perm[s] != s) {
        const int k = atomicAdd(&ish[1], 1);
        P.moves[2 * k] = s;
        P.moves[2 * k + 1] = perm[s];
      }
    }
    __syncthreads();
    n_moves = ish[1];
  }
  __syncthreads();
  decide_mark(P, plain, 19);

  if (tid == 0) {
    C.n_snap = n_snap;
    C.n_moves = n_moves;
    C.snap_cur = C.cur;
    C.active = active;
    C.n_finished = n_fin;
    if (active == 0 || at_cap) C.done = 1;
    ish[2] = 0;  // restart
    if (!C.done && C.inner_k >= 1) {
      // restart_reason, solver.hpp:299-311
      int reason = -1;
      if (mean <= P.beta_s * C.mean_anchor) reason = BL_RESTART_SUFFICIENT;
      else if (mean <= P.beta_n * C.mean_anchor && mean > C.mean_prev)
        reason = BL_RESTART_NECESSARY;
      else if ((double)C.inner_k > P.beta_a * (double)C.total_k)
        reason = BL_RESTART_ARTIFICIAL;
      if (reason >= 0) {
        if (C.log_count < P.log_cap) {
          bl_restart_event& e = P.log[C.log_count];
          e.at_iteration = C.total_k;
          e.reason = reason;
          e.reserved = 0;
          e.residual = mean;
          e.anchor_residual = C.mean_anchor;
        }
        C.log_count += 1;
        ish[2] = 1;
      }
    }
  }
  __syncthreads();
  decide_mark(P, plain, 20);
  const bool restart = ish[2] != 0;
  if (restart) {
    // gated weight update on the post-compaction active columns (:303-319)
    for (int j = tid; j < active; j += (int)blockDim.x) {
      if (P.resid[j] <= P.anchor_resid[j]) {
        const double dxn = sqrt(cs(P, S_XA2, j));
        const double dyn = sqrt(cs(P, S_YA2, j));
        P.w[j] = smoothed_weight(P.w[j], dxn, dyn, P.theta);
      }
    }
  }
  __syncthreads();
  decide_mark(P, plain, 21);
  if (tid == 0) {
    C.hash_pending = 0;
    if (!C.done) {
      if (restart) {
        C.anchor_reset = 1;
        C.inner_k = 0;
        C.restarts += 1;
        C.col_epoch += 1;  // weights changed
      } else {
        C.alpha_used = C.alpha;
        C.cur ^= 1;
        C.anchor_reset = 0;
        C.mean_prev = mean;
        C.inner_k += 1;
        C.total_k += 1;
        C.hash_pending = P.trace;
      }
      C.alpha = (double)(C.inner_k + 1) / (double)(C.inner_k + 2);
      C.at_cap = C.total_k >= P.max_it;
      C.check = (C.total_k % P.period == 0) || C.at_cap;
      const int nba = (C.active + P.W - 1) / P.W;
      if (P.r_tab) {  // the same rule, tabulated per active block count on the host
        C.Rp = P.r_tab[nba];
        C.Rd = P.r_tab[P.Kp / P.W + 1 + nba];
      } else {
        C.Rp = rounds_adjust(items_per_block(P.n, P.m, P.W, P.grid, nba, P.l2_budget), nba,
                             P.grid_run);
        C.Rd = rounds_adjust(items_per_block(P.m, P.n, P.W, P.grid, nba, P.l2_budget), nba,
                             P.grid_run);
      }
      C.Rc = C.Rp;
    }
    C.cert_pending = 0;
    // The graph loop hands the tail over to the persistent kernel once an
    // iteration's streamed state is small enough to be latency-bound.
    const double state_bytes =
        8.0 * (double)((C.active + P.W - 1) / P.W) * P.W * (double)(P.n + P.m);
    const bool handover = P.handover_bytes > 0.0 && state_bytes < P.handover_bytes;
    set_cond_if_changed(P, C, CB_LOOP, P.h_loop, (C.done || handover) ? 0u : 1u);
    set_cond_if_changed(P, C, CB_CHECK, P.h_check, (!C.done && C.check) ? 1u : 0u);
    set_cond_if_changed(P, C, CB_SNAP, P.h_snap, (C.n_snap > 0 || C.n_moves > 0) ? 1u : 0u);
    if (P.trace) set_cond_if_changed(P, C, CB_TRACE, P.h_trace, C.hash_pending ? 1u : 0u);
    // narrow row kernels once a single block with <= W/2 live LPs is left
    if (P.narrow_ok) {
      const unsigned nw = C.active <= P.W / 2 ? 1u : 0u;
      if (((C.cond >> CB_NARROW) & 1) != (int)nw) set_cond(P, P.h_narrow2, nw);
      set_cond_if_changed(P, C, CB_NARROW, P.h_narrow, nw);
    }
  }
  decide_mark(P, plain, 22);
}

// Folds the finished launches' entry/exit stamps into the accumulators and
// credits this iteration's row kernels with their algorithmic bytes
// (compulsory traffic, gathers counted once).
// Called by the first K_KINDS threads (one kind each).
static __device__ void prof_fold(const Params& P, const Ctrl& C, int k, unsigned long long now) {
  if (!P.prof || k >= K_KINDS) return;
  const unsigned long long s = P.prof[2 * k], e = P.prof[2 * k + 1];
  if (e != 0ull && s != ~0ull && e >= s) {
    P.prof_acc[3 * k] += (double)(e - s);
    P.prof_acc[3 * k + 1] += 1.0;
  }
  P.prof[2 * k] = k == K_DECIDE ? now : ~0ull;
  P.prof[2 * k + 1] = 0ull;
  if (k != 0) return;
  const double n = P.n, m = P.m, nnz = (double)P.nnz, K = C.active;
  const double chk = C.check ? 1.0 : 0.0;
  P.prof_acc[3 * K_PRIMAL + 2] += 12.0 * nnz + 4.0 * (n + 1) + 24.0 * n + 8.0 * K * (m + 4.0 * n + chk * n);
  P.prof_acc[3 * K_DUAL + 2] += 12.0 * nnz + 4.0 * (m + 1) + 16.0 * m + 8.0 * K * (n + 6.0 * m + chk * 3.0 * m);
  if (C.check)
    P.prof_acc[3 * K_CHECK + 2] += 12.0 * nnz + 4.0 * (n + 1) + 24.0 * n + 8.0 * K * (m + 5.0 * n);
}

static __device__ void decide_body(const Params& P, int phase) {
  double* scratch = P.scratch;
  __shared__ double sh[kDecideScratchInts / 2];
  __shared__ int ish[4];
  __shared__ Ctrl C;
  const int tid = threadIdx.x;
  if (tid == 0) C = *P.ctrl;
  __syncthreads();
  if (C.done) return;
  if (phase == 1 && !C.cert_pending) return;
  const int active = C.active;
  double mean;
  const bool plain_pass = !C.check;
  if (phase == 0) decide_mark(P, plain_pass, 10);
  if (phase == 0) {
    if (tid < 32) {
      unsigned long long now = 0;
      if (tid == 0) now = gtime();
      now = __shfl_sync(0xffffffffu, now, 0);
      prof_fold(P, C, tid, now);
    }
    if (tid == 0) {
      ish[3] = 0;
      C.launches += 3 + (C.check ? 1 : 0);
      C.passes += 1;
      // a loop pass either advances total_k or is the single re-application
      // after a restart, so this bound is never reached by a correct run
      if (C.passes > 2 * P.max_it + 1024) ish[3] = 2;
    }
    __syncthreads();
    // The residuals were computed by the dual kernel's per-block folds
    // (DualOp::after_fold); a broken metric raised err_flag there.
    const int count = P.avg_all ? P.width : active;
    if (tid == 0 && *reinterpret_cast<volatile int*>(P.err_flag)) ish[3] = 1;
    __syncthreads();
    if (ish[3]) {
      if (tid == 0) {
        C.error = ish[3] == 2 ? BL_ERR_LOGIC : BL_ERR_DOMAIN;
        if (P.prof) atomicMax(&P.prof[2 * K_DECIDE + 1], gtime());
        C.done = 1;
        set_cond_if_changed(P, C, CB_LOOP, P.h_loop, 0u);
        set_cond_if_changed(P, C, CB_CHECK, P.h_check, 0u);
        set_cond_if_changed(P, C, CB_CERT, P.h_cert, 0u);
        set_cond_if_changed(P, C, CB_SNAP, P.h_snap, 0u);
        if (P.trace) set_cond_if_changed(P, C, CB_TRACE, P.h_trace, 0u);
        *P.ctrl = C;
      }
      return;
    }
    // Averaged residual (batch_solver.hpp:209-222): up to 256 terms, the
    // reference's sequential sum in slot order; a wider batch adds the
    // column blocks' sequential sums in block order.
    if (count <= 256 || P.avg_all) {
      mean = ordered_sum(P.resid, count, sh) / (double)count;
    } else {
      mean = ordered_sum(P.blk_resid, (active + P.W - 1) / P.W, sh) / (double)count;
    }
    decide_mark(P, plain_pass, 11);
    if (C.inner_k == 0) {
      for (int j = tid; j < active; j += (int)blockDim.x) P.anchor_resid[j] = P.resid[j];
    }
    if (tid == 0) {
      if (C.inner_k == 0) C.mean_anchor = mean;
      C.mean = mean;
      C.sparse_products += 2;
      if (C.check) C.sparse_products += 1;
      ish[0] = 0;
    }
    __syncthreads();
    if (C.check) {
      for (int j = tid; j < active; j += (int)blockDim.x) {
        evaluate_column(P, j);
        int need = P.verdict[j] == V_CERT_NEED;
        if (!need && P.verdict[j] == V_NONE && dual_ray(P, j)) P.verdict[j] = V_DUAL_INF;
        P.cert_flag[j] = need;
        if (need) atomicAdd(&ish[0], 1);
      }
      __syncthreads();
      if (ish[0] > 0) {
        if (tid == 0) {
          C.sparse_products += ish[0];
          C.cert_pending = 1;
          C.launches += 2;
          set_cond_if_changed(P, C, CB_CERT, P.h_cert, 1u);
          *P.ctrl = C;
          if (P.prof) atomicMax(&P.prof[2 * K_DECIDE + 1], gtime());
        }
        return;
      }
    }
    if (tid == 0) set_cond_if_changed(P, C, CB_CERT, P.h_cert, 0u);
  } else {
    mean = C.mean;
    for (int j = tid; j < active; j += (int)blockDim.x) {
      if (P.verdict[j] != V_CERT_NEED) continue;
      const double res = sqrt(cs(P, S_CERT, j));
      if (res <= P.eps_infeas * fabs(P.t_dsup[j])) P.verdict[j] = V_PRIMAL_INF;
      else P.verdict[j] = dual_ray(P, j) ? V_DUAL_INF : V_NONE;
    }
    __syncthreads();
  }
  if (phase == 0) decide_mark(P, plain_pass, 12);
  finalize(P, C, mean, sh, ish, scratch);
  __syncthreads();
  if (phase == 0) decide_mark(P, plain_pass, 13);
  if (tid == 0) {
    if (C.n_snap > 0 || C.n_moves > 0) C.launches += 2;
    if (C.hash_pending) C.launches += 1;
    *P.ctrl = C;
    if (P.prof) atomicMax(&P.prof[2 * K_DECIDE + 1], gtime());
  }
}

// ---------------------------------------------------------------------------
// snapshots (vectors of finished / best / capped columns) and compaction
// ---------------------------------------------------------------------------
static __device__ void snapshot_body(const Params& P, const Ctrl& C) {
  const int ns = C.n_snap;
  if (ns == 0) return;
  prof_begin(P, K_SNAPSHOT);
  const int n = P.n, m = P.m, W = P.W;
  const double* Xold = P.X[C.snap_cur];
  const long long total = (long long)ns * (n + m);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(t / (n + m));
    const int i0 = (int)(t - (long long)k * (n + m));
    const int j = P.snap_list[3 * k], o = P.snap_list[3 * k + 1];
    const int bits = P.snap_list[3 * k + 2];
    if (i0 < n) {
      const int i = i0;
      const size_t e = tidx(n, W, i, j);
      const size_t ro = (size_t)o * n + i;
      if (bits & SN_BEST) {
        P.BX[e] = P.XT[e];
        P.BR[e] = P.R[e];
      }
      if (bits & SN_FINAL) {
        P.RX[ro] = P.XT[e];
        P.RR[ro] = P.R[e];
      }
      if (bits & (SN_CERTP | SN_CERTD)) P.RDX[ro] = P.XT[e] - Xold[e];
      if (bits & SN_CERTP) P.RDR[ro] = P.DR[e];
      if (bits & SN_CAP) {
        P.RX[ro] = P.BX[e];
        P.RR[ro] = P.BR[e];
      }
    } else {
      const int i = i0 - n;
      const size_t e = tidx(m, W, i, j);
      const size_t ro = (size_t)o * m + i;
      if (bits & SN_BEST) P.BY[e] = P.YT[e];
      if (bits & SN_FINAL) P.RY[ro] = P.YT[e];
      if (bits & SN_CERTP) P.RDY[ro] = P.DY[e];
      if (bits & SN_CAP) P.RY[ro] = P.BY[e];
    }
  }
  prof_end(P, K_SNAPSHOT);
}

// Column moves of the swap-with-last compaction (batch_solver.hpp:143-156,
// 273-278). The reference swaps X/Y/AX/anchors but not the operator outputs
// XT/YT/AXT, and applies the Halpern step after compaction (:326-335): a
// column moved into a hole is combined with the T-output that the finished
// column left in that slot. Reproduced here for parity: on a Halpern
// iteration the moved column's next iterate is recomputed from XT/YT/AXT of
// the destination slot and its own pre-step iterate and anchor. On a
// restart iteration (no Halpern) the current iterate is moved as is.
static __device__ void compact_body(const Params& P, const Ctrl& C) {
  const int nm = C.n_moves;
  if (nm == 0) return;
  prof_begin(P, K_COMPACT);
  const int n = P.n, m = P.m, W = P.W;
  const bool halpern = !C.anchor_reset;
  const double a = C.alpha_used, oma = 1.0 - a;
  const int cn = C.cur, co = C.cur ^ 1;
  const bool best = P.vectors >= BL_VECTORS_SOLUTION;
  const long long total = (long long)nm * (n + m);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(t / (n + m));
    const int i0 = (int)(t - (long long)k * (n + m));
    const int dst = P.moves[2 * k], src = P.moves[2 * k + 1];
    if (i0 < n) {
      const size_t d = tidx(n, W, i0, dst), s = tidx(n, W, i0, src);
      if (halpern) {
        const double ax = P.aX[s];
        P.X[cn][d] = a * (2.0 * P.XT[d] - P.X[co][s]) + oma * ax;
        P.aX[d] = ax;
      } else {
        P.X[cn][d] = P.X[cn][s];
      }
      if (best) {
        P.BX[d] = P.BX[s];
        P.BR[d] = P.BR[s];
      }
    } else {
      const int i = i0 - n;
      const size_t d = tidx(m, W, i, dst), s = tidx(m, W, i, src);
      if (halpern) {
        const double ay = P.aY[s], aax = P.aAX[s];
        P.Y[cn][d] = a * (2.0 * P.YT[d] - P.Y[co][s]) + oma * ay;
        P.AX[cn][d] = a * (2.0 * P.AXT[d] - P.AX[co][s]) + oma * aax;
        P.aY[d] = ay;
        P.aAX[d] = aax;
      } else {
        P.Y[cn][d] = P.Y[cn][s];
        P.AX[cn][d] = P.AX[cn][s];
      }
      if (best) P.BY[d] = P.BY[s];
    }
  }
  prof_end(P, K_COMPACT);
}

// FNV-1a over the bytes of X[:,0] then Y[:,0] (solver.hpp:170-177,
// batch_solver.hpp:339-344). Sequential by definition: one thread.
static __device__ void trace_body(const Params& P) {
  Ctrl* C = P.ctrl;
  if (!C->hash_pending) return;
  uint64_t h = C->hash;
  const double* x = P.X[C->cur];
  const double* y = P.Y[C->cur];
  for (int i = 0; i < P.n; ++i) {
    const uint64_t bits = (uint64_t)__double_as_longlong(x[(size_t)i * P.W]);
    for (int k = 0; k < 8; ++k) {
      h ^= (bits >> (8 * k)) & 0xffu;
      h *= 1099511628211ull;
    }
  }
  for (int i = 0; i < P.m; ++i) {
    const uint64_t bits = (uint64_t)__double_as_longlong(y[(size_t)i * P.W]);
    for (int k = 0; k < 8; ++k) {
      h ^= (bits >> (8 * k)) & 0xffu;
      h *= 1099511628211ull;
    }
  }
  C->hash = h;
  C->hash_pending = 0;
}






// ---------------------------------------------------------------------------
// persistent loop: the whole solve in ONE cooperative launch
// ---------------------------------------------------------------------------
// All CTAs are co-resident (cooperative launch); phases are separated by a
// grid barrier instead of kernel boundaries, CTA 0 runs the decide phase.
// The gpu-scope fences of the barrier also invalidate L1, so gathers of data
// written earlier in the launch see the new values.
__device__ __forceinline__ void grid_sync(unsigned long long* bar, unsigned long long& target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1ull);
    unsigned long long v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
      if (v >= target) break;
      __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ Ctrl load_ctrl(const Ctrl* c) {
  static_assert(sizeof(Ctrl) % 8 == 0, "Ctrl must be 8-byte sized");
  Ctrl out;
  const unsigned long long* src = reinterpret_cast<const unsigned long long*>(c);
  unsigned long long* dst = reinterpret_cast<unsigned long long*>(&out);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(Ctrl) / 8); ++i) dst[i] = __ldcg(src + i);
  return out;
}

// One thread-block cluster: phases separated by the hardware cluster
// barrier (release/acquire at cluster scope; it also invalidates L1, so the
// gathers see data other CTAs of the cluster wrote in the previous phase).
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// The row phases of one loop pass with LL lanes per row (0: full width).
template <int W, int LL, class Sync>
__device__ __forceinline__ void loop_rows(const Params& P, const Ctrl& C, double* red, Sync& sync) {
  if (C.check) {
    primal_body<W, true, LL>(P, C, red);
    sync();
    dual_body<W, true, LL, false>(P, C, red);
    sync();
    check_body<W, LL>(P, C, red);
    sync();
  } else {
    primal_body<W, false, LL>(P, C, red);
    sync();
    dual_body<W, false, LL, false>(P, C, red);
    sync();
  }
}

// ---------------------------------------------------------------------------
// fast tail passes: one cluster, one active column block, plain iteration
// ---------------------------------------------------------------------------
// In the tail an iteration is a few microseconds of work, so latency chains
// decide its cost. A plain pass (no termination check, no certificate, no
// compaction) therefore runs a lean schedule that computes exactly what the
// generic phases + decide_body compute for such a pass:
//  * each CTA of the cluster owns fixed row ranges of A' (primal) and A
//    (dual) for the whole launch, with their CSR metadata cached in shared
//    memory (loaded once per launch);
//  * column descriptors are cached in shared memory and restaged only when
//    the slot weights / permutation change (Ctrl::col_epoch);
//  * per-CTA partial sums go to P.tail_part without fences or atomics; the
//    cluster barrier publishes them and warp 0 of CTA 0 folds them in CTA
//    order inside a warp-synchronous decide.
struct TailRows {
  unsigned long long mark;  // last tail timing mark (CTA 0, BATCHLP_TAIL_TRACE)
  int pr0, pr1, dr0, dr1;  // A' rows (primal) and A rows (dual) of this CTA
  int pcached, dcached;    // metadata in shared memory?
  const int *prp, *pci, *drp, *dci;
  const double *pcv, *dcv;
  int epoch;
  // in-kernel profile of the fast passes (CTA 0, thread 0): phase start and
  // [primal, dual, decide] x [ns, passes, algorithmic bytes], flushed to
  // P.prof_acc once at exit instead of per-pass global stamps and atomics
  int prof_on;
  int npass;  // fast passes run by this launch
  unsigned long long pt;
  double pacc[3][3];
  double* part;  // the double-buffered partials (dynamic shared memory)
};
// Per-slot state of the fast decide kept in CTA 0's shared memory during the
// launch and written back at exit: the five column sums and the residual of
// the last pass ([6][32]), and the anchor residuals.
static __device__ __noinline__ double* tail_sums() {
  __shared__ double t[6 * 32];
  return t;
}
static __device__ __noinline__ double* tail_ar() {
  __shared__ double t[32];
  return t;
}
static __device__ __noinline__ double* tail_w() {
  __shared__ double w[32];  // slot weights (staged with the column descriptors)
  return w;
}
static __device__ __noinline__ SColInfo* tail_cols(int which) {
  __shared__ SColInfo s[2][32];  // [0] primal steps (tau), [1] dual steps (sigma)
  return s[which];
}
static __device__ __noinline__ TailRows* tail_rows() {
  __shared__ TailRows t;
  return &t;
}
// Diagnostic timing of the fast tail schedule (P.dbg, BATCHLP_TAIL_TRACE):
// CTA 0 accumulates the %globaltimer time spent between marks k-1 and k.
__device__ __forceinline__ void tail_mark(const Params& P, int k) {
  if (P.dbg && blockIdx.x == 0 && threadIdx.x == 0) {
    TailRows* t = tail_rows();
    const unsigned long long now = gtime();
    if (k > 0) P.dbg[k] += now - t->mark;
    else P.dbg[0] += 1;
    t->mark = now;
  }
}

// Closes fast-pass phase k (0 primal, 1 dual, 2 decide) on CTA 0.
__device__ __forceinline__ void tail_phase(int k) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    TailRows* t = tail_rows();
    if (t->prof_on) {
      const unsigned long long now = gtime();
      t->pacc[k][0] += (double)(now - t->pt);
      t->pacc[k][1] += 1.0;
      t->pt = now;
    }
  }
}

// [pass parity][cluster CTA][5 sums][32 slots]: the partials of a fast tail
// pass. Every CTA keeps a full copy in its dynamic shared memory; each CTA
// pushes its own partials into all copies through distributed shared memory,
// so every CTA can run the (deterministic) decide itself. Double-buffered by
// pass parity: a CTA can be one phase ahead of another, never more.
constexpr int kTailPartDoubles = 2 * 16 * 5 * 32;
__device__ __forceinline__ double* tail_part_smem(int parity) {
  return tail_rows()->part + parity * (16 * 5 * 32);
}
static __device__ __noinline__ Ctrl* tail_ctrl() {
  __shared__ Ctrl c;
  return &c;
}
// Every CTA's copy of the control block during fast tail passes: CTA 0's
// decide writes the new state into all of them through distributed shared
// memory, so a pass starts without a global-memory round trip.
static __device__ __noinline__ Ctrl* tail_ctrl_in() {
  __shared__ Ctrl c;
  return &c;
}

// Publishes the decided control block to this CTA's next pass (called by
// the 32 lanes of warp 0; every CTA decides for itself).
static __device__ void tail_commit_ctrl(int lane) {
  constexpr int kWords = (int)(sizeof(Ctrl) / 8);
  const unsigned long long* src = reinterpret_cast<const unsigned long long*>(tail_ctrl());
  unsigned long long* dst = reinterpret_cast<unsigned long long*>(tail_ctrl_in());
  __syncwarp();
  for (int k = lane; k < kWords; k += 32) dst[k] = src[k];
}

// Copies rows [r0, r1) of a CSR into shared memory at *cursor; returns
// pointers offset so that they can be indexed with global row / nonzero
// indices. Falls back to the global arrays when the cache is too small.
static __device__ void tail_cache_rows(const int* rp, const int* ci, const double* cv, int r0, int r1,
                                char*& cursor, char* end, const int*& orp, const int*& oci,
                                const double*& ocv) {
  const int q0 = rp[r0], q1 = rp[r1];
  const size_t need = 4 * (size_t)(r1 - r0 + 1) + 4 * (size_t)(q1 - q0) + 8 * (size_t)(q1 - q0) + 16;
  orp = rp;
  oci = ci;
  ocv = cv;
  if (cursor == nullptr || cursor + need > end) return;
  int* srp = reinterpret_cast<int*>(cursor);
  int* sci = srp + (r1 - r0 + 1);
  double* scv = reinterpret_cast<double*>(
      (reinterpret_cast<uintptr_t>(sci + (q1 - q0)) + 7) & ~uintptr_t(7));
  for (int k = threadIdx.x; k <= r1 - r0; k += blockDim.x) srp[k] = rp[r0 + k];
  for (int k = threadIdx.x; k < q1 - q0; k += blockDim.x) {
    sci[k] = ci[q0 + k];
    scv[k] = cv[q0 + k];
  }
  cursor = reinterpret_cast<char*>(scv + (q1 - q0));
  orp = srp - r0;
  oci = sci - q0;
  ocv = scv - q0;
}

static __device__ void tail_setup(const Params& P, char* dyn, int dyn_bytes) {
  TailRows* t = tail_rows();
  const int c = blockIdx.x, cl = gridDim.x;
  if (threadIdx.x == 0) {
    // a tiny dimension is one sequential walk by CTA 0 (reference order)
    const bool tn = P.n <= kTinyRows, tm = P.m <= kTinyRows;
    t->pr0 = tn ? 0 : (int)((long long)P.n * c / cl);
    t->pr1 = tn ? (c == 0 ? P.n : 0) : (int)((long long)P.n * (c + 1) / cl);
    t->dr0 = tm ? 0 : (int)((long long)P.m * c / cl);
    t->dr1 = tm ? (c == 0 ? P.m : 0) : (int)((long long)P.m * (c + 1) / cl);
    t->epoch = -1;
  }
  __syncthreads();
  char* cur = dyn_bytes > 0 ? dyn : nullptr;
  char* end = dyn + dyn_bytes;
  const int *prp, *pci, *drp, *dci;
  const double *pcv, *dcv;
  tail_cache_rows(P.trp, P.tci, P.tcv, t->pr0, t->pr1, cur, end, prp, pci, pcv);
  tail_cache_rows(P.rp, P.ci, P.cv, t->dr0, t->dr1, cur, end, drp, dci, dcv);
  if (threadIdx.x == 0) {
    t->pcached = prp != P.trp;
    t->dcached = drp != P.rp;
    t->prp = prp;
    t->pci = pci;
    t->pcv = pcv;
    t->drp = drp;
    t->dci = dci;
    t->dcv = dcv;
  }
  __syncthreads();
}

// Sums of this CTA's rows for NS columns-sums, reduced over the CTA in a
// fixed tree and stored to P.tail_part[cta][k0 + s][jj].
template <int W, int NS, int LL, int NT>
__device__ __forceinline__ void tail_publish(const Params& P, const Ctrl& C,
                                             double (&acc)[NS][Geo<W>::V], int k0, double* red) {
  using Gm = Geo<W, LL, NT>;
  constexpr int NW = NT / 32;
  auto cluster = cooperative_groups::this_cluster();
  const int cl = (int)cluster.num_blocks();
  double* part = tail_part_smem((int)(C.passes & 1));
  constexpr int V = Gm::V, L = Gm::L;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int off = 16; off >= L; off >>= 1)
#pragma unroll
    for (int s = 0; s < NS; ++s)
#pragma unroll
      for (int v = 0; v < V; ++v)
        acc[s][v] = __dadd_rn(acc[s][v], __shfl_down_sync(0xffffffffu, acc[s][v], off));
  if (lane < L) {
#pragma unroll
    for (int s = 0; s < NS; ++s)
#pragma unroll
      for (int v = 0; v < V; ++v) red[(warp * NS + s) * W + lane * V + v] = acc[s][v];
  }
  __syncthreads();
  // this CTA's sums for the live slots, then one copy into every CTA
  for (int t = tid; t < NS * W; t += NT) {
    const int s = t / W, jj = t - s * W;
    double sum = 0.0;
    if (jj < L * V) {
#pragma unroll
      for (int wp = 0; wp < NW; ++wp) sum = __dadd_rn(sum, red[(wp * NS + s) * W + jj]);
    }
    red[NW * NS * W + t] = sum;
  }
  __syncthreads();
  for (int t = tid; t < cl * NS * W; t += NT) {
    const int rank = t / (NS * W), u = t - rank * (NS * W);
    const int s = u / W, jj = u - s * W;
    double* dst = cluster.map_shared_rank(part, rank);
    dst[(blockIdx.x * 5 + k0 + s) * 32 + jj] = red[NW * NS * W + u];
  }
  __syncthreads();
}

template <int W, int LL, int NT>
static __device__ void tail_rows_pass(const Params& P, const Ctrl& C, double* red) {
  using Gm = Geo<W, LL, NT>;
  constexpr int V = Gm::V, L = Gm::L, G = Gm::G;
  const TailRows* t = tail_rows();
  const int tid = threadIdx.x, g = tid / L, li = tid - g * L;
  const bool tiny_n = P.n <= kTinyRows, tiny_m = P.m <= kTinyRows;
  {
    PrimalOp<W, false, true> op(P, C);
    op.col = tail_cols(0) + li * V;
    op.crp = t->prp;
    op.cci = t->pci;
    op.ccv = t->pcv;
    op.lanes = L;
    double acc[2][V];
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int v = 0; v < V; ++v) acc[s][v] = 0.0;
    const int r0 = t->pr0, r1 = t->pr1;
    if (tiny_n) {
      if (g == 0)
        for (int i = r0; i < r1; ++i) op.row(0, i, 0, li, acc);
    } else {
      for (int i = r0 + g; i < r1; i += G) op.row(0, i, 0, li, acc);
    }
    tail_mark(P, 2);
    tail_publish<W, 2, LL, NT>(P, C, acc, 0, red);
    tail_mark(P, 3);
  }
  cluster_sync_all();
  tail_phase(0);
  tail_mark(P, 4);
  {
    DualOp<W, false, false, true> op(P, C);
    op.col = tail_cols(1) + li * V;
    op.crp = t->drp;
    op.cci = t->dci;
    op.ccv = t->dcv;
    op.lanes = L;
    double acc[3][V];
#pragma unroll
    for (int s = 0; s < 3; ++s)
#pragma unroll
      for (int v = 0; v < V; ++v) acc[s][v] = 0.0;
    const int r0 = t->dr0, r1 = t->dr1;
    if (tiny_m) {
      if (g == 0)
        for (int i = r0; i < r1; ++i) op.row(0, i, 0, li, acc);
    } else {
      for (int i = r0 + g; i < r1; i += G) op.row(0, i, 0, li, acc);
    }
    tail_mark(P, 5);
    tail_publish<W, 3, LL, NT>(P, C, acc, 2, red);
    tail_mark(P, 6);
  }
  cluster_sync_all();
  tail_phase(1);
  tail_mark(P, 7);
}

// decide_body's logic for a plain pass (no check) with active <= 32, run
// by warp 0 of EVERY CTA on its own copy of the partials (the computation is
// deterministic, so all CTAs reach the same control block without a
// broadcast or a cluster barrier): lane j owns slot j. Global side effects
// (weights, restart log) are CTA 0's; a weight change is applied to every
// CTA's shared descriptors here, so no CTA re-reads P.w in the loop.
static __device__ void tail_decide(const Params& P) {
  const int lane = threadIdx.x;
  Ctrl& C = *tail_ctrl();
  unsigned long long tdbg = 0;
  const bool trace = P.dbg && blockIdx.x == 0 && lane == 0;
  if (trace) tdbg = gtime();
  if (lane == 0) C = *tail_ctrl_in();
  __syncwarp();
  const int active = C.active;
  const int cl = gridDim.x;
  double dx2 = 0.0, xa2 = 0.0, dy2 = 0.0, cross = 0.0, ya2 = 0.0, r = 0.0, w = 1.0;
  int err = 0;
  if (lane < active) {
    // fold the CTA partials in CTA order (sequential, fixed)
    const double* part = tail_part_smem((int)(C.passes & 1));
    for (int c = 0; c < cl; ++c) {
      const double* tp = part + c * 5 * 32 + lane;
      dx2 = __dadd_rn(dx2, tp[0]);
      xa2 = __dadd_rn(xa2, tp[32]);
      dy2 = __dadd_rn(dy2, tp[64]);
      cross = __dadd_rn(cross, tp[96]);
      ya2 = __dadd_rn(ya2, tp[128]);
    }
    double* ts = tail_sums();
    ts[0 * 32 + lane] = dx2;
    ts[1 * 32 + lane] = xa2;
    ts[2 * 32 + lane] = dy2;
    ts[3 * 32 + lane] = cross;
    ts[4 * 32 + lane] = ya2;
    w = tail_w()[lane];
    r = m_residual(dx2, dy2, cross, P.eta, w, &err);
    ts[5 * 32 + lane] = r;
  }
  const bool bad = __any_sync(0xffffffffu, err != 0);
  if (trace) {  // diagnostic split of the fast decide (BATCHLP_TAIL_TRACE)
    const unsigned long long now = gtime();
    P.dbg[14] += now - tdbg;
    tdbg = now;
  }
  int loop_err = 0;
  if (lane == 0) {
    C.launches += 3;
    C.passes += 1;
    if (C.passes > 2 * P.max_it + 1024) loop_err = 1;
  }
  loop_err = __shfl_sync(0xffffffffu, loop_err, 0);
  if (bad || loop_err) {
    if (lane == 0) {
      C.error = loop_err ? BL_ERR_LOGIC : BL_ERR_DOMAIN;
      C.done = 1;
    }
    tail_commit_ctrl(lane);
    return;
  }
  // averaged residual: sequential sum in slot order (ordered_sum, count <= 256);
  // the terms are staged in shared memory so their loads issue back to back
  __shared__ double rs[32];
  rs[lane] = r;
  __syncwarp();
  double sum = 0.0;
#pragma unroll
  for (int j = 0; j < 32; ++j)
    if (j < active) sum += rs[j];
  const double mean = sum / (double)active;
  const bool first = C.inner_k == 0;
  if (first && lane < active) tail_ar()[lane] = r;
  // restart rule (solver.hpp:299-311) on the pre-step state
  int reason = -1;
  if (C.inner_k >= 1) {
    if (mean <= P.beta_s * C.mean_anchor) reason = BL_RESTART_SUFFICIENT;
    else if (mean <= P.beta_n * C.mean_anchor && mean > C.mean_prev)
      reason = BL_RESTART_NECESSARY;
    else if ((double)C.inner_k > P.beta_a * (double)C.total_k)
      reason = BL_RESTART_ARTIFICIAL;
  }
  if (reason >= 0 && lane < active) {
    const double ar = first ? r : tail_ar()[lane];
    if (r <= ar) {
      const double nw = smoothed_weight(w, sqrt(xa2), sqrt(ya2), P.theta);
      if (blockIdx.x == 0) P.w[lane] = nw;
      // StepParams (solver.hpp:58-59), as load_col computes them
      tail_w()[lane] = nw;
      scol_set_step(tail_cols(0) + lane, P.eta / nw);
      scol_set_step(tail_cols(1) + lane, P.eta * nw);
    }
  }
  __syncwarp();  // every lane has read the control block
  if (trace) P.dbg[15] += gtime() - tdbg;
  if (lane == 0) {
    if (first) C.mean_anchor = mean;
    C.mean = mean;
    C.sparse_products += 2;
    C.n_snap = 0;
    C.n_moves = 0;
    C.snap_cur = C.cur;
    C.n_finished = 0;
    C.hash_pending = 0;
    if (reason >= 0) {
      if (blockIdx.x == 0 && C.log_count < P.log_cap) {
        bl_restart_event& e = P.log[C.log_count];
        e.at_iteration = C.total_k;
        e.reason = reason;
        e.reserved = 0;
        e.residual = mean;
        e.anchor_residual = C.mean_anchor;
      }
      C.log_count += 1;
      C.anchor_reset = 1;
      C.inner_k = 0;
      C.restarts += 1;
      C.col_epoch += 1;
      tail_rows()->epoch = C.col_epoch;  // the descriptors were updated above
    } else {
      C.alpha_used = C.alpha;
      C.cur ^= 1;
      C.anchor_reset = 0;
      C.mean_prev = mean;
      C.inner_k += 1;
      C.total_k += 1;
    }
    C.alpha = (double)(C.inner_k + 1) / (double)(C.inner_k + 2);
    C.at_cap = C.total_k >= P.max_it;
    C.check = (C.total_k % P.period == 0) || C.at_cap;
    C.cert_pending = 0;
  }
  tail_commit_ctrl(lane);
}

// One fast tail pass on the cluster (all CTAs of NT threads).
template <int W, int NT = kBlock>
static __device__ void tail_pass(const Params& P, const Ctrl& C, double* red) {
  TailRows* t = tail_rows();
  if (t->epoch != C.col_epoch) {  // uniform across the CTA
    const int tid = threadIdx.x;
    if (tid < W) {
      stage_col(P, tid, C.active, false, tail_cols(0) + tid);
      stage_col(P, tid, C.active, true, tail_cols(1) + tid);
    }
    if (tid < 32) tail_w()[tid] = tid < C.active ? P.w[tid] : 1.0;
    __syncthreads();
    if (tid == 0) t->epoch = C.col_epoch;
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && t->prof_on) {
    // algorithmic bytes of the pass (prof_fold's model, plain pass)
    const double n = P.n, m = P.m, nnz = (double)P.nnz, K = C.active;
    t->pacc[0][2] += 12.0 * nnz + 4.0 * (n + 1) + 24.0 * n + 8.0 * K * (m + 4.0 * n);
    t->pacc[1][2] += 12.0 * nnz + 4.0 * (m + 1) + 16.0 * m + 8.0 * K * (n + 6.0 * m);
  }
  const int Lsel = pass_lanes<W>(C.active);
  tail_mark(P, 1);
  BL_DISPATCH_L(W, Lsel, (tail_rows_pass<W, LL_, NT>(P, C, red)));
  if (threadIdx.x < 32) tail_decide(P);
  tail_mark(P, 8);
  __syncthreads();  // this CTA's next pass sees its decided control block
  tail_phase(2);
  tail_mark(P, 9);
}

// Whether the next pass can take the fast tail schedule.
__device__ __forceinline__ bool tail_fast_ok(const Params& P, const Ctrl& C, int W) {
  return (C.active + W - 1) / W == 1 && C.active <= 32 && !C.check && !P.trace && !P.avg_all &&
         P.tail_part != nullptr;
}

// Dedicated fast-tail kernel: one cluster of kTailThreads-thread CTAs runs
// plain tail passes until a pass needs the generic schedule (termination
// check, certificate, compaction) or the solve is done; the generic cluster
// kernel then runs that one pass (single-pass mode) and the tail graph loops
// (bl_solver.cu). More threads per CTA than the generic kernel: more row
// groups, so fewer rows per group in a pass.
// (threads per CTA of the fast tail kernel; its reduction scratch is
// kTailRedBytes of dynamic shared memory)
#ifndef BL_TAIL_THREADS
#define BL_TAIL_THREADS 512
#endif
constexpr int kTailThreads = BL_TAIL_THREADS;
// per-warp sums plus one row of CTA sums
constexpr int kTailRedBytes = (kTailThreads / 32 + 1) * 3 * 32 * 8;
constexpr int kTailPartBytes = kTailPartDoubles * 8;
template <int W>
__global__ void __launch_bounds__(kTailThreads, 1) k_tail_fast(Params P, int tail_smem) {
  // dynamic shared memory: the per-warp reduction scratch, then the CSR cache
  extern __shared__ __align__(16) char tail_dyn[];
  double* red = reinterpret_cast<double*>(tail_dyn);
  if (threadIdx.x == 0) tail_rows()->part = reinterpret_cast<double*>(tail_dyn + kTailRedBytes);
  tail_setup(P, tail_dyn + kTailRedBytes + kTailPartBytes, tail_smem);
  if (threadIdx.x == 0) *tail_ctrl_in() = load_ctrl(P.ctrl);
  __syncthreads();
  // Profiling: fold the stamps a generic pass left (CTA 0), then time the
  // fast passes locally (tail_phase); the fast passes write no global stamps.
  TailRows* tr = tail_rows();
  if (threadIdx.x == 0) {
    tr->prof_on = blockIdx.x == 0 && P.prof != nullptr;
    for (int k = 0; k < 3; ++k) tr->pacc[k][0] = tr->pacc[k][1] = tr->pacc[k][2] = 0.0;
  }
  __syncthreads();
  if (tr->prof_on && threadIdx.x < 32) {
    const Ctrl C0 = *tail_ctrl_in();
    prof_fold(P, C0, threadIdx.x, gtime());
  }
  if (threadIdx.x < W) tail_ar()[threadIdx.x] = P.anchor_resid[threadIdx.x];
  if (threadIdx.x == 0) tr->npass = 0;
  // every CTA of the cluster has started before any pushes into its shared
  // memory (distributed shared memory rule)
  cluster_sync_all();
  for (;;) {
    tail_mark(P, 0);
    const Ctrl C = *tail_ctrl_in();
    if (C.done || !tail_fast_ok(P, C, W)) break;
    if (tr->prof_on && threadIdx.x == 0) tr->pt = gtime();
    tail_pass<W, kTailThreads>(P, C, red);
    if (threadIdx.x == 0) tr->npass += 1;
  }
  // write back the decide state the fast passes kept on chip (CTA 0)
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const Ctrl& C = *tail_ctrl_in();
    if (tr->npass > 0) {
      if (lane < W) P.anchor_resid[lane] = tail_ar()[lane];
      if (lane < C.active) {
        const double* ts = tail_sums();
        csr(P, S_DX2, lane) = ts[0 * 32 + lane];
        csr(P, S_XA2, lane) = ts[1 * 32 + lane];
        csr(P, S_DY2, lane) = ts[2 * 32 + lane];
        csr(P, S_CROSS, lane) = ts[3 * 32 + lane];
        csr(P, S_YA2, lane) = ts[4 * 32 + lane];
        P.resid[lane] = ts[5 * 32 + lane];
      }
      if (lane == 0) *P.ctrl = C;
    }
  }
  if (tr->prof_on && threadIdx.x == 0) {
    const int kinds[3] = {K_TAIL_PRIMAL, K_TAIL_DUAL, K_TAIL_DECIDE};
    for (int k = 0; k < 3; ++k)
      for (int f = 0; f < 3; ++f) P.prof_acc[3 * kinds[k] + f] += tr->pacc[k][f];
    // the next generic decide starts a fresh decide interval
    P.prof[2 * K_DECIDE] = ~0ull;
    P.prof[2 * K_DECIDE + 1] = 0ull;
  }
}

// CL = false: cooperative grid over all SMs (grid barriers); it hands over
// (returns) once at most P.tail_blocks column blocks are active.
// CL = true: ONE cluster of P.grid CTAs for the latency-bound tail, where an
// iteration is a few microseconds of work and a grid-wide barrier would cost
// more than the work itself; rows are walked with the narrow mapping.
template <int W, bool CL>
__global__ void __launch_bounds__(kBlock) k_loop(Params P, int tail_smem) {
  __shared__ double red[kRedDoubles];
  extern __shared__ __align__(16) char tail_dyn[];
  unsigned long long target = 0;
  (void)tail_dyn;
  (void)tail_smem;
  auto sync = [&]() {
    if constexpr (CL) cluster_sync_all();
    else grid_sync(P.barrier, target);
  };
  const int grid = gridDim.x;
  for (;;) {
    Ctrl C = load_ctrl(P.ctrl);
    if (C.done) break;
    const int nba = (C.active + W - 1) / W;
    if (!CL && P.tail_blocks > 0 && nba <= P.tail_blocks) break;

    // work decomposition for THIS launch's grid (the control block may have
    // been written by a driver with another grid)
    C.Rp = items_per_block(P.n, P.m, W, grid, nba, P.l2_budget);
    C.Rd = items_per_block(P.m, P.n, W, grid, nba, P.l2_budget);
#ifndef BL_LOOP_ROUNDS
#define BL_LOOP_ROUNDS 1
#endif
    if (!CL && BL_LOOP_ROUNDS) {  // the grid-stride walk runs in rounds of this grid
      C.Rp = rounds_adjust(C.Rp, nba, grid);
      C.Rd = rounds_adjust(C.Rd, nba, grid);
    }
    C.Rc = C.Rp;
    const int Lsel = CL ? pass_lanes<W>(C.active) : Geo<W>::L;
    BL_DISPATCH_L(W, Lsel, (loop_rows<W, LL_>(P, C, red, sync)));
    if (blockIdx.x == 0) decide_body(P, 0);
    sync();
    C = load_ctrl(P.ctrl);
    if (C.cert_pending) {
      C.Rc = items_per_block(P.n, P.m, W, grid, (C.active + W - 1) / W, P.l2_budget);
      const int Lc = CL ? pass_lanes<W>(C.active) : Geo<W>::L;
      BL_DISPATCH_L(W, Lc, (cert_body<W, LL_>(P, C, red)));
      sync();
      if (blockIdx.x == 0) decide_body(P, 1);
      sync();
      C = load_ctrl(P.ctrl);
    }
    if (C.n_snap > 0 || C.n_moves > 0) {
      snapshot_body(P, C);
      sync();
      compact_body(P, C);
      sync();
    }
    if (C.hash_pending) {
      if (blockIdx.x == 0 && threadIdx.x == 0) trace_body(P);
      sync();
    }
    if constexpr (CL) {
      if (P.tail_single) break;  // one generic pass between fast-tail launches
    }
  }
  if constexpr (CL) {
    // tail graph: loop again (fast tail kernel, then this kernel) unless done
    if (P.tail_single && blockIdx.x == 0 && threadIdx.x == 0) {
      const Ctrl Cf = load_ctrl(P.ctrl);
      cudaGraphSetConditional(P.h_tail, Cf.done ? 0u : 1u);
    }
  }
}

// ---------------------------------------------------------------------------
// init (batch_solver.hpp:130-136; warm start solver.hpp:590-597)
// ---------------------------------------------------------------------------


// column-major host layout <-> column-block tiled layout



// ---------------------------------------------------------------------------
// power iteration (sparse.hpp:249-287), two start vectors as a W=2 batch
// ---------------------------------------------------------------------------
struct PiOp {
  static constexpr int V = 2;
  const int *rp, *ci;
  const double *cv, *in;
  double* out;
  int rows_in, rows_out;
  int valid[2];
  __device__ void stage(int, volatile SColInfo*) {}
  __device__ void begin(int, int, double (&)[1][2], bool, const volatile SColInfo*) {}
  __device__ void row(int, int i, int, int, double (&acc)[1][2]) {
    double o[2];
    gather_row<2>(rp, ci, cv, in, i, o);
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      if (valid[v]) {
        out[(size_t)i * 2 + v] = o[v];
        acc[0][v] += o[v] * o[v];
      }
    }
  }
};



// stage 0 (after u = A v): null-space test; stage 1 (after w = A'u):
// estimate, stagnation and the normalisation v = w / ||w||. One thread per
// start vector updates the state; k_pi_fill then rewrites v.




// iteration counter bump (end of one power-iteration step)

// ---------------------------------------------------------------------------
// per-width launchers: defined (and explicitly instantiated) only in the
// bl_w<W>.cu translation units, called through the dispatchers in
// bl_kernels.cu
// ---------------------------------------------------------------------------
template <int W>
struct WLaunch {
  static void iteration_check(const Params& P, cudaStream_t s);
  static void iteration_plain(const Params& P, cudaStream_t s);
  static void iteration_check_narrow(const Params& P, cudaStream_t s);
  static void iteration_plain_narrow(const Params& P, cudaStream_t s);
  static void spmm(const Params& P, cudaStream_t s, bool transpose, const double* in,
                   double* out, int active, int R);
  static void cert(const Params& P, cudaStream_t s);
  static int loop_ctas_per_sm();
  static cudaError_t loop(const Params& P, cudaStream_t s);
  static cudaError_t loop_cluster(const Params& P, cudaStream_t s, int tail_smem);
  static int max_tail_cluster();
  static int row_ctas_per_sm();
  static int plain_ctas_per_sm();
  static cudaError_t tail_fast(const Params& P, cudaStream_t s, int tail_smem);
};

// Each row kernel is launched with SMs x (its own max resident CTAs, <= 4):
// the grid-stride item loop does not depend on the grid size.
inline int grid_of(const void* fn) {
  static std::mutex mu;
  static std::map<const void*, int> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(fn);
  if (it != cache.end()) return it->second;
  int dev = 0, sms = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kBlock, 0);
  if (occ < 1) occ = 1;
  if (occ > 4) occ = 4;
  return cache[fn] = sms * occ;
}

#ifdef BL_WLAUNCH_DEFINE
}  // namespace bl
namespace bl {

template <int W>
void WLaunch<W>::iteration_check(const Params& P, cudaStream_t s) {
  k_primal<W, true><<<grid_of((const void*)k_primal<W, true>), kBlock, 0, s>>>(P);
  k_dual<W, true><<<grid_of((const void*)k_dual<W, true>), kBlock, 0, s>>>(P);
  k_check<W><<<grid_of((const void*)k_check<W>), kBlock, 0, s>>>(P);
}

template <int W>
void WLaunch<W>::iteration_plain(const Params& P, cudaStream_t s) {
  k_primal<W, false><<<grid_of((const void*)k_primal<W, false>), kBlock, 0, s>>>(P);
  k_dual<W, false><<<grid_of((const void*)k_dual<W, false>), kBlock, 0, s>>>(P);
}

template <int W>
void WLaunch<W>::iteration_check_narrow(const Params& P, cudaStream_t s) {
  k_primal_narrow<W, true><<<grid_of((const void*)k_primal_narrow<W, true>), kBlock, 0, s>>>(P);
  k_dual_narrow<W, true><<<grid_of((const void*)k_dual_narrow<W, true>), kBlock, 0, s>>>(P);
  k_check_narrow<W><<<grid_of((const void*)k_check_narrow<W>), kBlock, 0, s>>>(P);
}

template <int W>
void WLaunch<W>::iteration_plain_narrow(const Params& P, cudaStream_t s) {
  k_primal_narrow<W, false><<<grid_of((const void*)k_primal_narrow<W, false>), kBlock, 0, s>>>(P);
  k_dual_narrow<W, false><<<grid_of((const void*)k_dual_narrow<W, false>), kBlock, 0, s>>>(P);
}

template <int W>
void WLaunch<W>::spmm(const Params& P, cudaStream_t s, bool transpose, const double* in,
                      double* out, int active, int R) {
  k_spmm<W><<<P.grid, kBlock, 0, s>>>(P, transpose ? 1 : 0, in, out, active, R, P.partials,
                                       P.counters, P.colsum);
}

template <int W>
void WLaunch<W>::cert(const Params& P, cudaStream_t s) {
  k_cert<W><<<P.grid, kBlock, 0, s>>>(P);
}

// CTAs per SM the persistent loop kernel can keep co-resident.
template <int W>
int WLaunch<W>::loop_ctas_per_sm() {
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_loop<W, false>, kBlock, 0);
  return occ < 1 ? 1 : occ;
}

// The whole solve (or its remainder) as one cooperative launch of P.grid
// co-resident CTAs.
template <int W>
cudaError_t WLaunch<W>::loop(const Params& P, cudaStream_t s) {
  Params Q = P;
  int no_tail_smem = 0;
  void* args[] = {&Q, &no_tail_smem};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(&k_loop<W, false>),
                                     dim3(P.grid), dim3(kBlock), args, 0, s);
}

// The tail as ONE thread-block cluster of P.grid CTAs (<= 16; sizes above
// 8 need the non-portable-cluster opt-in).
template <int W>
cudaError_t WLaunch<W>::loop_cluster(const Params& P, cudaStream_t s, int tail_smem) {
  cudaError_t e = cudaSuccess;
  auto fn = k_loop<W, true>;
  if (P.grid > 8) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  if (tail_smem > 0) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, tail_smem);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P.grid);
  cfg.blockDim = dim3(kBlock);
  cfg.dynamicSmemBytes = tail_smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = P.grid;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fn, P, tail_smem);
}

// Largest cluster (<= 16) of the tail kernel the device can place.
template <int W>
int WLaunch<W>::max_tail_cluster() {
  int best = 8;
  auto fn = k_loop<W, true>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
      cudaSuccess) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16);
    cfg.blockDim = dim3(kBlock);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 16;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&clusters, fn, &cfg) == cudaSuccess && clusters > 0)
      best = 16;
  }
  cudaGetLastError();
  return best;
}

// The fast-tail kernel as one cluster of P.grid CTAs of kTailThreads threads.
template <int W>
cudaError_t WLaunch<W>::tail_fast(const Params& P, cudaStream_t s, int tail_smem) {
  cudaError_t e = cudaSuccess;
  auto fn = k_tail_fast<W>;
  if (P.grid > 8) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  const int dyn = tail_smem + kTailRedBytes + kTailPartBytes;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P.grid);
  cfg.blockDim = dim3(kTailThreads);
  cfg.dynamicSmemBytes = dyn;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = P.grid;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fn, P, tail_smem);
}

// Resident CTAs per SM of the plain-pass row kernels (their launch grid, grid_of).
template <int W>
int WLaunch<W>::plain_ctas_per_sm() {
  int a = 1, b = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_primal<W, false>, kBlock, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_dual<W, false>, kBlock, 0);
  int occ = a < b ? a : b;
  if (occ > 4) occ = 4;
  return occ < 1 ? 1 : occ;
}

// Resident CTAs per SM of the widest row kernels (grid of the plain kernels).
template <int W>
int WLaunch<W>::row_ctas_per_sm() {
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dual<W, true>, kBlock, 0);
  int occ2 = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, k_check<W>, kBlock, 0);
  if (occ2 < occ) occ = occ2;
  return occ < 1 ? 1 : occ;
}
#endif  // BL_WLAUNCH_DEFINE

}  // namespace bl
