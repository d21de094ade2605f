// bl_slice.cuh — slice-staged primal / dual row kernels (W = 32, plain
// passes, small gather operands).
//
// The register-gather row kernels are bound by L2 gather traffic: every
// nonzero re-reads a 256-byte row segment of the gathered operand (Y for the
// primal, XT for the dual), ~7x the compulsory bytes on the benchmark
// matrices. When the operand has few rows (rows_in <=
// kSliceMaxRows, e.g. the C1/C2 problems with m, n <= 2560), an 8-slot
// sub-slice of a column block — rows_in x 8 doubles, strided in the tiled
// layout — fits in shared memory. A work item is (column block b, 8-slot
// group q, row range):
//  * the CTA copies the sub-slice once (16-byte cp.async per thread), then
//    every gather of the item reads shared memory;
//  * the rows are processed in chunks of `ch` rows through a `stages`-deep
//    mbarrier pipeline: each chunk's streamed operands (X, aX — or Y, AX, aY,
//    aAX: cp.async) and its CSR nonzeros (1-D bulk copies of the aligned
//    superset of [rp[c0], rp[c1])) land in shared memory while the previous
//    chunks are computed, so no thread waits on a dependent global load;
//  * 4 lanes per CSR row (2 slots each), one row per 4-thread group.
// Global traffic per item: the sub-slice once, the streamed rows once, the
// CSR once. Same arithmetic and summation order as PrimalOp / DualOp; the
// per-item sums are folded deterministically per (b, q).
//
// Measured on B200 (C2, K = 4000; profiles/r01_slice): correct, but slower
// than the register-gather kernels (primal 145-159 us vs 121 us per pass):
// the ~210 KB of shared memory per CTA leaves one CTA of 256-384 threads per
// SM, 2-3 warps per scheduler, and the kernel stalls on fixed-latency and
// shared-memory dependencies at IPC ~1.5. Opt-in with BATCHLP_SLICE=1.
#pragma once

#include <cuda.h>

#include "bl_kernels.cuh"

namespace bl {

constexpr int kSliceLanes = kSliceCols / 2;
constexpr int kSliceMaxThreads = 512;
constexpr int kSliceMaxWarps = kSliceMaxThreads / 32;

// Work items per (block, group): minimise rounds x (1/R + slice-load share).
__device__ __forceinline__ int slice_items(int rows, int nvb, int grid) {
  int best = 1;
  float best_cost = 3.0e38f;
  for (int R = 1; R <= kSliceRMax; ++R) {
    if (R > 1 && rows / R < 64) break;
    const int rounds = (nvb * R + grid - 1) / grid;
    const float cost = rounds * (1.0f / R + 0.15f);
    if (cost < best_cost) {
      best_cost = cost;
      best = R;
    }
  }
  return best;
}

__device__ __forceinline__ unsigned slice_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void slice_expect(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(slice_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void slice_cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(slice_u32(dst)), "l"(src)
               : "memory");
}
// arrives on `bar` once this thread's earlier cp.async copies have landed
__device__ __forceinline__ void slice_arrive_cp(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(slice_u32(bar))
               : "memory");
}
// rows [r0, r0 + nrows) of slots [8q, 8q + 8) of tiled block b (`rows` rows
// per block) -> dst[nrows][8]; every thread copies its share
__device__ __forceinline__ void slice_rows(double* dst, const double* src, int b, int q, int rows,
                                           int r0, int nrows) {
  const double* base = src + ((size_t)b * rows + r0) * 32 + q * kSliceCols;
  for (int t = threadIdx.x; t < nrows * kSliceLanes; t += blockDim.x) {
    const int row = t / kSliceLanes, part = t - row * kSliceLanes;
    slice_cp16(dst + row * kSliceCols + part * 2, base + (size_t)row * 32 + part * 2);
  }
}
__device__ __forceinline__ void slice_bulk(void* dst, const void* src, unsigned bytes,
                                           unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          slice_u32(dst)),
      "l"(src), "r"(bytes), "r"(slice_u32(bar))
      : "memory");
}
__device__ __forceinline__ void slice_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred done;\n"
      "SLICE_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n"
      "@!done bra SLICE_WAIT_%=;\n"
      "}\n" ::"r"(slice_u32(bar)),
      "r"(parity)
      : "memory");
}

// Per-item sums -> partials of virtual block vb = 4 b + q -> last CTA folds
// the R partials in item order into colsum[s0 + s][32 b + 8 q + jj].
template <int NS>
__device__ __forceinline__ void slice_publish(double (&acc)[NS][2], int vb, int r, int R,
                                              double* partials, int* counters, double* colsum,
                                              int s0, int Kp, double* red) {
  __shared__ int last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = blockDim.x >> 5;
#pragma unroll
  for (int off = 16; off >= kSliceLanes; off >>= 1)
#pragma unroll
    for (int s = 0; s < NS; ++s)
#pragma unroll
      for (int v = 0; v < 2; ++v)
        acc[s][v] = __dadd_rn(acc[s][v], __shfl_down_sync(0xffffffffu, acc[s][v], off));
  if (lane < kSliceLanes) {
#pragma unroll
    for (int s = 0; s < NS; ++s)
#pragma unroll
      for (int v = 0; v < 2; ++v) red[(warp * NS + s) * kSliceCols + lane * 2 + v] = acc[s][v];
  }
  __syncthreads();
  if (tid < NS * kSliceCols) {
    const int s = tid / kSliceCols, jj = tid - s * kSliceCols;
    double sum = 0.0;
    for (int wp = 0; wp < nw; ++wp) sum = __dadd_rn(sum, red[(wp * NS + s) * kSliceCols + jj]);
    partials[((size_t)(vb * R + r) * NS + s) * kSliceCols + jj] = sum;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) last = (atomicAdd(&counters[vb], 1) == R - 1);
  __syncthreads();
  if (last) {
    __threadfence();
    if (tid < NS * kSliceCols) {
      const int s = tid / kSliceCols, jj = tid - s * kSliceCols;
      const double* src = partials + ((size_t)vb * R * NS + s) * kSliceCols + jj;
      double sum = 0.0;
      for (int rr = 0; rr < R; ++rr)
        sum = __dadd_rn(sum, __ldcg(src + (size_t)rr * NS * kSliceCols));
      colsum[(size_t)(s0 + s) * Kp + (vb >> 2) * 32 + (vb & 3) * kSliceCols + jj] = sum;
    }
    if (tid == 0) counters[vb] = 0;
  }
  __syncthreads();
}

// DUAL = false: XT = proj(X - tau (c + A'Y)), X' = Halpern; sums dx2, xa2.
// DUAL = true:  AXT = A XT, YT = sigma (s - proj(s)), Y'/AX' = Halpern;
//               sums dy2, cross, ya2.
template <bool DUAL>
__global__ void __launch_bounds__(kSliceMaxThreads, 1)
    k_slice(Params P) {
  constexpr int W = 32;
  constexpr int NS = DUAL ? 3 : 2;  // sums
  constexpr int NA = DUAL ? 4 : 2;  // streamed arrays
  extern __shared__ __align__(128) char slice_smem[];
  __shared__ double red[kSliceMaxWarps * NS * kSliceCols];
  __shared__ SColInfo scol[kSliceCols];
  __shared__ __align__(8) unsigned long long bar[1 + kSliceMaxStages];
  const Ctrl C = *P.ctrl;
  if (C.done) return;
  prof_begin(P, DUAL ? K_DUAL : K_PRIMAL);
  const SliceGeo G = DUAL ? P.slice_d : P.slice_p;
  const int rows = DUAL ? P.m : P.n, rows_in = DUAL ? P.n : P.m;
  const int* __restrict__ rp = DUAL ? P.rp : P.trp;
  const int* ci = DUAL ? P.ci : P.tci;
  const double* cv = DUAL ? P.cv : P.tcv;
  const int tid = threadIdx.x, g = tid / kSliceLanes, li = tid - g * kSliceLanes;
  const int ch = G.ch, S = G.stages;
  double* sl = reinterpret_cast<double*>(slice_smem);
  int* rps = reinterpret_cast<int*>(slice_smem + slice_bytes(rows_in));
  char* stage0 = slice_smem + slice_bytes(rows_in) + slice_rp_bytes(rows);
  const int stage_bytes = slice_stage_bytes(NA, ch, G.nz);
  const size_t arr_bytes = (size_t)ch * kSliceCols * 8;
  if (tid == 0) {
    // bar[0]: the sub-slice, one cp.async arrival per thread; bar[1 + st]:
    // stage st, one per thread plus the elected thread's expect_tx (CSR bulk)
    const unsigned nt = blockDim.x;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(slice_u32(&bar[0])), "r"(nt)
                 : "memory");
    for (int k = 1; k <= S; ++k)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(slice_u32(&bar[k])), "r"(nt + 1)
                   : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned ph = 0u;  // bit k: parity of bar[k]'s next completion
  const int reset = C.anchor_reset;
  const double alpha = C.alpha, oma = 1.0 - alpha;
  const int cur = C.cur;
  // streamed arrays of the pass; the anchors are not read on a reset pass
  const int na_load = reset ? NA / 2 : NA;
  const double* gsrc = DUAL ? P.XT : P.Y[cur];
  const double* asrc[NA];
  if constexpr (DUAL) {
    asrc[0] = P.Y[cur];
    asrc[1] = P.AX[cur];
    asrc[2] = P.aY;
    asrc[3] = P.aAX;
  } else {
    asrc[0] = P.X[cur];
    asrc[1] = P.aX;
  }
  const int nvb = (C.active + kSliceCols - 1) / kSliceCols;
  const int R = slice_items(rows, nvb, gridDim.x);
  const int items = nvb * R;
  const int per = (rows + R - 1) / R;
  for (int w = blockIdx.x; w < items; w += gridDim.x) {
    const int vb = w / R, r = w - vb * R;
    const int b = vb >> 2, q = vb & 3;
    const int r0 = min(rows, r * per), r1 = min(rows, r0 + per);
    for (int t = tid; t <= r1 - r0; t += blockDim.x) rps[t] = __ldg(rp + r0 + t);
    if (tid < kSliceCols) stage_col(P, b * W + q * kSliceCols + tid, C.active, DUAL, &scol[tid]);
    __syncthreads();
    const int nch = (r1 - r0 + ch - 1) / ch;
    // chunk k -> stage k % S: streamed rows (all threads, cp.async) + CSR
    // supersets (elected thread, bulk copies), completing on one mbarrier
    auto issue = [&](int k) {
      const int st = k % S;
      char* sb = stage0 + (size_t)st * stage_bytes;
      const int c0 = r0 + k * ch, c1 = min(r1, c0 + ch);
      unsigned long long* br = &bar[1 + st];
      for (int a = 0; a < na_load; ++a)
        slice_rows(reinterpret_cast<double*>(sb + a * arr_bytes), asrc[a], b, q, rows, c0, c1 - c0);
      if (tid == 0) {
        const int p0 = rps[c0 - r0], p1 = rps[c1 - r0];
        const int a0 = p0 & ~3, a1 = (p1 + 3) & ~3;
        const int e0 = p0 & ~1, e1 = (p1 + 1) & ~1;
        slice_expect(br, (unsigned)((a1 - a0) * 4 + (e1 - e0) * 8));
        char* cvb = sb + NA * arr_bytes;
        if (e1 > e0) slice_bulk(cvb, cv + e0, (unsigned)(e1 - e0) * 8, br);
        if (a1 > a0) slice_bulk(cvb + (size_t)(G.nz + 2) * 8, ci + a0, (unsigned)(a1 - a0) * 4, br);
      }
      slice_arrive_cp(br);
    };
    // the previous item's generic reads of the buffers precede the bulk writes
    if (tid == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    slice_rows(sl, gsrc, b, q, rows_in, 0, rows_in);
    slice_arrive_cp(&bar[0]);
    for (int k = 0; k < S && k < nch; ++k) issue(k);
    double acc[NS][2];
#pragma unroll
    for (int s = 0; s < NS; ++s) acc[s][0] = acc[s][1] = 0.0;
    for (int k = 0; k < nch; ++k) {
      const int st = k % S;
      slice_wait(&bar[1 + st], (ph >> (1 + st)) & 1u);
      ph ^= 1u << (1 + st);
      if (k == 0) {
        slice_wait(&bar[0], ph & 1u);
        ph ^= 1u;
      }
      const char* sb = stage0 + (size_t)st * stage_bytes;
      const int c0 = r0 + k * ch, c1 = min(r1, c0 + ch);
      const int i = c0 + g;
      if (g < ch && i < c1) {
        const int pc = rps[c0 - r0];
        const double* cvs = reinterpret_cast<const double*>(sb + NA * arr_bytes) - (pc & ~1);
        const int* cis =
            reinterpret_cast<const int*>(sb + NA * arr_bytes + (size_t)(G.nz + 2) * 8) - (pc & ~3);
        const double* arr = reinterpret_cast<const double*>(sb) + g * kSliceCols + li * 2;
        const size_t astride = (size_t)ch * kSliceCols;
        // bounds first: their (L2) latency overlaps the gather
        double bc = 0.0, lo, hi;
        if constexpr (DUAL) {
          lo = __ldg(P.rl + i);
          hi = __ldg(P.ru + i);
        } else {
          if (P.mode == BL_SHARED_OBJECTIVE) bc = __ldg(P.c + i);
          lo = __ldg(P.xl + i);
          hi = __ldg(P.xu + i);
        }
        // one CSR row times this lane's two slots: stored order, separately
        // rounded (csr_apply, sparse.hpp:176-183)
        double gs[2] = {0.0, 0.0};
        {
          int p = rps[i - r0];
          const int e = rps[i - r0 + 1];
          const double* slo = sl + li * 2;
          for (; p + 2 <= e; p += 2) {
            const int j0 = cis[p], j1 = cis[p + 1];
            const double v0 = cvs[p], v1 = cvs[p + 1];
            const double2 x0 = *reinterpret_cast<const double2*>(slo + (size_t)j0 * kSliceCols);
            const double2 x1 = *reinterpret_cast<const double2*>(slo + (size_t)j1 * kSliceCols);
            gs[0] = __dadd_rn(gs[0], __dmul_rn(v0, x0.x));
            gs[1] = __dadd_rn(gs[1], __dmul_rn(v0, x0.y));
            gs[0] = __dadd_rn(gs[0], __dmul_rn(v1, x1.x));
            gs[1] = __dadd_rn(gs[1], __dmul_rn(v1, x1.y));
          }
          if (p < e) {
            const double v0 = cvs[p];
            const double2 x0 = *reinterpret_cast<const double2*>(slo + (size_t)cis[p] * kSliceCols);
            gs[0] = __dadd_rn(gs[0], __dmul_rn(v0, x0.x));
            gs[1] = __dadd_rn(gs[1], __dmul_rn(v0, x0.y));
          }
        }
        const size_t idx = ((size_t)b * rows + i) * W + q * kSliceCols + li * 2;
        if constexpr (DUAL) {
          const double2 yv = *reinterpret_cast<const double2*>(arr);
          const double2 xv = *reinterpret_cast<const double2*>(arr + astride);
          const double y[2] = {yv.x, yv.y}, ax[2] = {xv.x, xv.y};
          double ay[2], aax[2];
          if (reset) {
            ay[0] = y[0];
            ay[1] = y[1];
            aax[0] = ax[0];
            aax[1] = ax[1];
          } else {
            const double2 a1 = *reinterpret_cast<const double2*>(arr + 2 * astride);
            const double2 a2 = *reinterpret_cast<const double2*>(arr + 3 * astride);
            ay[0] = a1.x;
            ay[1] = a1.y;
            aax[0] = a2.x;
            aax[1] = a2.y;
          }
          double yn[2], axn[2];
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const ColInfo cl = read_col(&scol[li * 2 + v]);
            const double sigma = cl.step;
            // dual_step_element, solver.hpp:186-190
            const double vv = 2.0 * gs[v] - ax[v];
            const double s = y[v] / sigma + vv;
            const double yt = sigma * (s - project_box(s, lo, hi));
            const double dy = yt - y[v];
            const double da = y[v] - ay[v];
            if (cl.valid) {
              acc[0][v] += dy * dy;
              acc[1][v] += dy * (gs[v] - ax[v]);
              acc[NS - 1][v] += da * da;
            }
            yn[v] = alpha * (2.0 * yt - y[v]) + oma * ay[v];
            axn[v] = alpha * (2.0 * gs[v] - ax[v]) + oma * aax[v];
          }
          __stcs(reinterpret_cast<double2*>(P.Y[cur ^ 1] + idx), make_double2(yn[0], yn[1]));
          __stcs(reinterpret_cast<double2*>(P.AX[cur ^ 1] + idx), make_double2(axn[0], axn[1]));
          if (reset) {
            __stcs(reinterpret_cast<double2*>(P.aY + idx), make_double2(y[0], y[1]));
            __stcs(reinterpret_cast<double2*>(P.aAX + idx), make_double2(ax[0], ax[1]));
          }
        } else {
          const double2 xv = *reinterpret_cast<const double2*>(arr);
          const double x[2] = {xv.x, xv.y};
          double ax[2];
          if (reset) {
            ax[0] = x[0];
            ax[1] = x[1];
          } else {
            const double2 av = *reinterpret_cast<const double2*>(arr + astride);
            ax[0] = av.x;
            ax[1] = av.y;
          }
          double xt[2], xn[2];
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const ColInfo cl = read_col(&scol[li * 2 + v]);
            double cc, l2, h2;
            col_vals(P, cl, i, bc, lo, hi, cc, l2, h2);
            const double t = cc + gs[v];
            xt[v] = project_box(x[v] - cl.step * t, l2, h2);
            const double dx = xt[v] - x[v];
            const double da = x[v] - ax[v];
            if (cl.valid) {
              acc[0][v] += dx * dx;
              acc[1][v] += da * da;
            }
            xn[v] = alpha * (2.0 * xt[v] - x[v]) + oma * ax[v];
          }
          *reinterpret_cast<double2*>(P.XT + idx) = make_double2(xt[0], xt[1]);
          __stcs(reinterpret_cast<double2*>(P.X[cur ^ 1] + idx), make_double2(xn[0], xn[1]));
          if (reset) __stcs(reinterpret_cast<double2*>(P.aX + idx), make_double2(x[0], x[1]));
        }
      }
      __syncthreads();  // stage st is free
      if (k + S < nch) {
        if (tid == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(k + S);
      }
    }
    slice_publish<NS>(acc, vb, r, R, P.slice_part, P.slice_cnt, P.colsum, DUAL ? S_DY2 : S_DX2,
                      P.Kp, red);
  }
  prof_end(P, DUAL ? K_DUAL : K_PRIMAL);
}

// Direct variant (SliceGeo.stages == 0): only the sub-slice and the item's
// row pointers are staged; the streamed rows and the CSR are read from global
// memory by 1024 threads (32 warps per SM, the register-gather kernels'
// occupancy). A row then costs one L2 round trip per batch of 4 nonzeros
// (ci/cv; the operand rows come from shared memory) instead of two.
constexpr int kSliceDirectThreads = 1024;

template <bool DUAL>
__global__ void __launch_bounds__(kSliceDirectThreads, 1) k_slice_direct(Params P) {
  constexpr int W = 32;
  constexpr int NS = DUAL ? 3 : 2;
  extern __shared__ __align__(128) char slice_smem[];
  __shared__ double red[(kSliceDirectThreads / 32) * NS * kSliceCols];
  __shared__ SColInfo scol[kSliceCols];
  const Ctrl C = *P.ctrl;
  if (C.done) return;
  prof_begin(P, DUAL ? K_DUAL : K_PRIMAL);
  const int rows = DUAL ? P.m : P.n, rows_in = DUAL ? P.n : P.m;
  const int* __restrict__ rp = DUAL ? P.rp : P.trp;
  const int* __restrict__ ci = DUAL ? P.ci : P.tci;
  const double* __restrict__ cv = DUAL ? P.cv : P.tcv;
  const int tid = threadIdx.x, g = tid / kSliceLanes, li = tid - g * kSliceLanes;
  const int groups = blockDim.x / kSliceLanes;
  double* sl = reinterpret_cast<double*>(slice_smem);
  int* rps = reinterpret_cast<int*>(slice_smem + slice_bytes(rows_in));
  const int reset = C.anchor_reset;
  const double alpha = C.alpha, oma = 1.0 - alpha;
  const int cur = C.cur;
  const double* gsrc = DUAL ? P.XT : P.Y[cur];
  const int nvb = (C.active + kSliceCols - 1) / kSliceCols;
  const int R = slice_items(rows, nvb, gridDim.x);
  const int items = nvb * R;
  const int per = (rows + R - 1) / R;
  for (int w = blockIdx.x; w < items; w += gridDim.x) {
    const int vb = w / R, r = w - vb * R;
    const int b = vb >> 2, q = vb & 3;
    const int r0 = min(rows, r * per), r1 = min(rows, r0 + per);
    slice_rows(sl, gsrc, b, q, rows_in, 0, rows_in);
    for (int t = tid; t <= r1 - r0; t += blockDim.x) rps[t] = __ldg(rp + r0 + t);
    if (tid < kSliceCols) stage_col(P, b * W + q * kSliceCols + tid, C.active, DUAL, &scol[tid]);
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    double acc[NS][2];
#pragma unroll
    for (int s = 0; s < NS; ++s) acc[s][0] = acc[s][1] = 0.0;
    const double* slo = sl + li * 2;
    for (int i = r0 + g; i < r1; i += groups) {
      const size_t idx = ((size_t)b * rows + i) * W + q * kSliceCols + li * 2;
      // streamed operands and bounds first: their latency overlaps the gather
      double2 s0, s1, s2 = make_double2(0.0, 0.0), s3 = make_double2(0.0, 0.0);
      double bc = 0.0, lo, hi;
      if constexpr (DUAL) {
        lo = __ldg(P.rl + i);
        hi = __ldg(P.ru + i);
        s0 = __ldcs(reinterpret_cast<const double2*>(P.Y[cur] + idx));
        s1 = __ldcs(reinterpret_cast<const double2*>(P.AX[cur] + idx));
        if (!reset) {
          s2 = __ldcs(reinterpret_cast<const double2*>(P.aY + idx));
          s3 = __ldcs(reinterpret_cast<const double2*>(P.aAX + idx));
        }
      } else {
        if (P.mode == BL_SHARED_OBJECTIVE) bc = __ldg(P.c + i);
        lo = __ldg(P.xl + i);
        hi = __ldg(P.xu + i);
        s0 = __ldcs(reinterpret_cast<const double2*>(P.X[cur] + idx));
        if (!reset) s1 = __ldcs(reinterpret_cast<const double2*>(P.aX + idx));
      }
      // one CSR row times this lane's two slots: stored order, separately
      // rounded (csr_apply, sparse.hpp:176-183)
      double gs[2] = {0.0, 0.0};
      {
        int p = rps[i - r0];
        const int e = rps[i - r0 + 1];
        for (; p < e; p += 4) {
          int c[4];
          double a[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const bool in = p + k < e;
            c[k] = in ? __ldg(ci + p + k) : 0;
            a[k] = in ? __ldg(cv + p + k) : 0.0;
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (p + k < e) {
              const double2 x = *reinterpret_cast<const double2*>(slo + (size_t)c[k] * kSliceCols);
              gs[0] = __dadd_rn(gs[0], __dmul_rn(a[k], x.x));
              gs[1] = __dadd_rn(gs[1], __dmul_rn(a[k], x.y));
            }
          }
        }
      }
      if constexpr (DUAL) {
        const double y[2] = {s0.x, s0.y}, ax[2] = {s1.x, s1.y};
        const double ay[2] = {reset ? y[0] : s2.x, reset ? y[1] : s2.y};
        const double aax[2] = {reset ? ax[0] : s3.x, reset ? ax[1] : s3.y};
        double yn[2], axn[2];
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const ColInfo cl = read_col(&scol[li * 2 + v]);
          const double sigma = cl.step;
          // dual_step_element, solver.hpp:186-190
          const double vv = 2.0 * gs[v] - ax[v];
          const double sv = y[v] / sigma + vv;
          const double yt = sigma * (sv - project_box(sv, lo, hi));
          const double dy = yt - y[v];
          const double da = y[v] - ay[v];
          if (cl.valid) {
            acc[0][v] += dy * dy;
            acc[1][v] += dy * (gs[v] - ax[v]);
            acc[NS - 1][v] += da * da;
          }
          yn[v] = alpha * (2.0 * yt - y[v]) + oma * ay[v];
          axn[v] = alpha * (2.0 * gs[v] - ax[v]) + oma * aax[v];
        }
        __stcs(reinterpret_cast<double2*>(P.Y[cur ^ 1] + idx), make_double2(yn[0], yn[1]));
        __stcs(reinterpret_cast<double2*>(P.AX[cur ^ 1] + idx), make_double2(axn[0], axn[1]));
        if (reset) {
          __stcs(reinterpret_cast<double2*>(P.aY + idx), s0);
          __stcs(reinterpret_cast<double2*>(P.aAX + idx), s1);
        }
      } else {
        const double x[2] = {s0.x, s0.y};
        const double ax[2] = {reset ? x[0] : s1.x, reset ? x[1] : s1.y};
        double xt[2], xn[2];
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const ColInfo cl = read_col(&scol[li * 2 + v]);
          double cc, l2, h2;
          col_vals(P, cl, i, bc, lo, hi, cc, l2, h2);
          const double t = cc + gs[v];
          xt[v] = project_box(x[v] - cl.step * t, l2, h2);
          const double dx = xt[v] - x[v];
          const double da = x[v] - ax[v];
          if (cl.valid) {
            acc[0][v] += dx * dx;
            acc[1][v] += da * da;
          }
          xn[v] = alpha * (2.0 * xt[v] - x[v]) + oma * ax[v];
        }
        *reinterpret_cast<double2*>(P.XT + idx) = make_double2(xt[0], xt[1]);
        __stcs(reinterpret_cast<double2*>(P.X[cur ^ 1] + idx), make_double2(xn[0], xn[1]));
        if (reset) __stcs(reinterpret_cast<double2*>(P.aX + idx), s0);
      }
    }
    slice_publish<NS>(acc, vb, r, R, P.slice_part, P.slice_cnt, P.colsum, DUAL ? S_DY2 : S_DX2,
                      P.Kp, red);
  }
  prof_end(P, DUAL ? K_DUAL : K_PRIMAL);
}

}  // namespace bl
