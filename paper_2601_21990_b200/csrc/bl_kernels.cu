// bl_kernels.cu — width-independent kernels of the batched PDHG hot path
// (decide, snapshots, compaction, trace, init, layout conversion, power
// iteration) and the host launchers, which dispatch the width-templated
// kernels to the bl_w<W>.cu translation units. The device code itself is in
// bl_kernels.cuh (see its header comment for the iteration structure).

#include "bl_kernels.cuh"

namespace bl {

extern template struct WLaunch<1>;
extern template struct WLaunch<2>;
extern template struct WLaunch<4>;
extern template struct WLaunch<8>;
extern template struct WLaunch<16>;
extern template struct WLaunch<32>;

__global__ void __launch_bounds__(kDecideThreads) k_decide(Params P, int phase) {
  decide_body(P, phase);
}

__global__ void k_snapshot(Params P) {
  const Ctrl C = *P.ctrl;
  snapshot_body(P, C);
}

__global__ void k_compact(Params P) {
  const Ctrl C = *P.ctrl;
  compact_body(P, C);
}

__global__ void k_trace(Params P) { trace_body(P); }

__global__ void k_init(Params P, const double* warm_x, const double* warm_y) {
  const int n = P.n, m = P.m, W = P.W, width = P.width;
  const long long tx = (long long)width * n, total = tx + (long long)width * m;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    if (t < tx) {
      const int s = (int)(t / n), i = (int)(t - (long long)s * n);
      const int o = P.slot_orig[s];
      ColInfo c;
      load_col(P, s, P.width, false, c);
      double cc, lo, hi;
      col_vals(P, c, i, 0.0, P.xl[i], P.xu[i], cc, lo, hi);
      const double x0 = warm_x ? warm_x[(size_t)o * n + i] : 0.0;
      P.X[0][tidx(n, W, i, s)] = project_box(x0, lo, hi);
    } else {
      const long long u = t - tx;
      const int s = (int)(u / m), i = (int)(u - (long long)s * m);
      const int o = P.slot_orig[s];
      P.Y[0][tidx(m, W, i, s)] = warm_y ? warm_y[(size_t)o * m + i] : 0.0;
    }
  }
}

__global__ void k_to_tiled(const double* src, double* dst, int rows, int width,
                           int W, int active) {
  const long long total = (long long)rows * active;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(t / rows), i = (int)(t - (long long)j * rows);
    dst[tidx(rows, W, i, j)] = src[(size_t)j * rows + i];
  }
}

__global__ void k_from_tiled(const double* src, double* dst, int rows, int width,
                             int W, int active) {
  const long long total = (long long)rows * active;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(t / rows), i = (int)(t - (long long)j * rows);
    dst[(size_t)j * rows + i] = src[tidx(rows, W, i, j)];
  }
}

__global__ void __launch_bounds__(kBlock) k_pi_spmv(Params P, int transpose,
                                                   const double* in, double* out,
                                                   PiState* st, int stage, int R,
                                                   double* partials, int* counters,
                                                   double* colsum) {
  PiOp op;
  op.rp = transpose ? P.trp : P.rp;
  op.ci = transpose ? P.tci : P.ci;
  op.cv = transpose ? P.tcv : P.cv;
  op.in = in;
  op.out = out;
  op.rows_in = transpose ? P.m : P.n;
  op.rows_out = transpose ? P.n : P.m;
  bool any = false;
  for (int v = 0; v < 2; ++v) {
    op.valid[v] = !st[v].done && (stage == 0 || !st[v].reset);
    any = any || op.valid[v];
  }
  if (!any) return;
  __shared__ double red[kRedDoubles];
  run_rows<2, 1>(op, op.rows_out, 1, R, partials, counters, colsum, 0, 2, red);
}

__global__ void k_pi_state(PiState* st, const double* colsum, int stage) {
  if (threadIdx.x >= 2) return;
  PiState& s = st[threadIdx.x];
  s.fill = 0;
  if (s.done) return;
  if (stage == 0) {
    s.unorm = sqrt(colsum[threadIdx.x]);
    s.reset = s.unorm == 0.0;
    if (s.reset) {
      // start vector fell into the null space (sparse.hpp:261-268)
      s.estimate = 0.0;
      s.stagnant = 0;
      s.fill = 1;
    }
  } else if (!s.reset) {
    s.wnorm = sqrt(colsum[threadIdx.x]);
    const double prev = s.estimate;
    s.estimate = s.unorm;
    if (prev > 0.0 && fabs(s.estimate - prev) <= 1e-4 * s.estimate) {
      if (++s.stagnant >= 10) s.done = 1;
    } else {
      s.stagnant = 0;
    }
    if (!s.done && s.wnorm == 0.0) s.done = 1;
    if (!s.done) s.fill = 2;
  }
}

__global__ void k_pi_fill(int n, double* Vv, const double* Wv, const PiState* st) {
  for (int v = 0; v < 2; ++v) {
    const int f = st[v].fill;
    if (f == 1) {
      const int hot = st[v].iter % n;
      for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        Vv[(size_t)i * 2 + v] = i == hot ? 1.0 : 0.0;
    } else if (f == 2) {
      const double wn = st[v].wnorm;
      for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        Vv[(size_t)i * 2 + v] = Wv[(size_t)i * 2 + v] / wn;
    }
  }
}

__global__ void k_pi_tick(PiState* st) {
  if (threadIdx.x < 2) {
    PiState& s = st[threadIdx.x];
    if (!s.done) {
      s.iter += 1;
      if (s.iter >= 5000) s.done = 1;
    }
  }
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
#define BL_DISPATCH_W(Wv, ...)                            \
  switch (Wv) {                                           \
    case 1: { constexpr int W_ = 1; __VA_ARGS__; } break;   \
    case 2: { constexpr int W_ = 2; __VA_ARGS__; } break;   \
    case 4: { constexpr int W_ = 4; __VA_ARGS__; } break;   \
    case 8: { constexpr int W_ = 8; __VA_ARGS__; } break;   \
    case 16: { constexpr int W_ = 16; __VA_ARGS__; } break; \
    default: { constexpr int W_ = 32; __VA_ARGS__; } break; \
  }

// The context's grid (the work-item basis of every row kernel, and the size of
// the partial buffers) follows the plain passes' occupancy: they carry almost
// all the time, and items per block = their launch grid is what keeps one
// column block in flight (C4 -5.5% against the check kernel's 3 CTAs / SM).
// Kernels at lower occupancy walk the same items in more rounds.
int max_ctas_per_sm() { return WLaunch<32>::plain_ctas_per_sm(); }
int plain_ctas_per_sm(int W) {
  int r = 1;
  BL_DISPATCH_W(W, r = WLaunch<W_>::plain_ctas_per_sm());
  return r;
}

static int fill_grid(long long work) {
  long long g = (work + 255) / 256;
  if (g < 1) g = 1;
  if (g > 148 * 16) g = 148 * 16;
  return (int)g;
}

void launch_init(const Params& P, cudaStream_t s, const double* warm_x,
                 const double* warm_y) {
  k_init<<<fill_grid((long long)P.width * (P.n + P.m)), 256, 0, s>>>(P, warm_x, warm_y);
}

void launch_spmm(const Params& P, cudaStream_t s, bool transpose, const double* in,
                 double* out, int active) {
  const int rows = transpose ? P.n : P.m, rows_in = transpose ? P.m : P.n;
  BL_DISPATCH_W(P.W, {
    constexpr int G = Geo<W_>::G;
    int R;
    if (P.l2_budget > 0) {  // the row kernels' L2-aware decomposition
      R = items_per_block(rows, rows_in, W_, P.grid, (active + W_ - 1) / W_, P.l2_budget);
    } else {
      R = rows <= kTinyRows ? 1 : (rows + 2 * G - 1) / (2 * G);
      if (R > P.grid) R = P.grid;
    }
    if (R < 1) R = 1;
    WLaunch<W_>::spmm(P, s, transpose, in, out, active, R);
  });
}

void launch_iteration_check(const Params& P, cudaStream_t s) {
  BL_DISPATCH_W(P.W, WLaunch<W_>::iteration_check(P, s));
}

void launch_iteration_plain(const Params& P, cudaStream_t s) {
  BL_DISPATCH_W(P.W, WLaunch<W_>::iteration_plain(P, s));
}

void launch_iteration_check_narrow(const Params& P, cudaStream_t s) {
  BL_DISPATCH_W(P.W, WLaunch<W_>::iteration_check_narrow(P, s));
}

void launch_iteration_plain_narrow(const Params& P, cudaStream_t s) {
  BL_DISPATCH_W(P.W, WLaunch<W_>::iteration_plain_narrow(P, s));
}

int loop_ctas_per_sm(int W) {
  int occ = 1;
  BL_DISPATCH_W(W, occ = WLaunch<W_>::loop_ctas_per_sm());
  return occ;
}

cudaError_t launch_loop(const Params& P, cudaStream_t s) {
  cudaError_t e = cudaSuccess;
  BL_DISPATCH_W(P.W, e = WLaunch<W_>::loop(P, s));
  return e;
}

cudaError_t launch_loop_cluster(const Params& P, cudaStream_t s, int tail_smem) {
  cudaError_t e = cudaSuccess;
  BL_DISPATCH_W(P.W, e = WLaunch<W_>::loop_cluster(P, s, tail_smem));
  return e;
}

cudaError_t launch_tail_fast(const Params& P, cudaStream_t s, int tail_smem) {
  cudaError_t e = cudaSuccess;
  BL_DISPATCH_W(P.W, e = WLaunch<W_>::tail_fast(P, s, tail_smem));
  return e;
}

// Largest cluster (<= 16) of the tail kernel the device can place (cached).
int max_tail_cluster(int W) {
  static std::mutex mu;
  static std::map<int, int> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(W);
  if (it != cache.end()) return it->second;
  int best = 8;
  BL_DISPATCH_W(W, best = WLaunch<W_>::max_tail_cluster());
  cache[W] = best;
  return best;
}

void launch_decide(const Params& P, cudaStream_t s, int phase) {
  k_decide<<<1, kDecideThreads, 0, s>>>(P, phase);
}

void launch_cert(const Params& P, cudaStream_t s) {
  BL_DISPATCH_W(P.W, WLaunch<W_>::cert(P, s));
}

void launch_snap_compact(const Params& P, cudaStream_t s) {
  k_snapshot<<<P.grid, 256, 0, s>>>(P);
  k_compact<<<P.grid, 256, 0, s>>>(P);
}

void launch_trace(const Params& P, cudaStream_t s) { k_trace<<<1, 1, 0, s>>>(P); }

void launch_to_tiled(cudaStream_t s, const double* src, double* dst, int rows,
                     int width, int W, int active) {
  k_to_tiled<<<fill_grid((long long)rows * active), 256, 0, s>>>(src, dst, rows, width,
                                                                 W, active);
}
void launch_from_tiled(cudaStream_t s, const double* src, double* dst, int rows,
                       int width, int W, int active) {
  k_from_tiled<<<fill_grid((long long)rows * active), 256, 0, s>>>(src, dst, rows,
                                                                   width, W, active);
}

// One power-iteration step for both start vectors (V, U, Wv tiled W=2).
void launch_pi_step(const Params& P, cudaStream_t s, double* Vv, double* U,
                    double* Wv, PiState* st) {
  constexpr int G = Geo<2>::G;
  int Ra = P.m <= kTinyRows ? 1 : (P.m + 2 * G - 1) / (2 * G);
  int Rt = P.n <= kTinyRows ? 1 : (P.n + 2 * G - 1) / (2 * G);
  if (Ra > P.grid) Ra = P.grid;
  if (Rt > P.grid) Rt = P.grid;
  if (Ra < 1) Ra = 1;
  if (Rt < 1) Rt = 1;
  k_pi_spmv<<<P.grid, kBlock, 0, s>>>(P, 0, Vv, U, st, 0, Ra, P.partials, P.counters,
                                      P.colsum);
  k_pi_state<<<1, 32, 0, s>>>(st, P.colsum, 0);
  k_pi_fill<<<fill_grid(P.n), 256, 0, s>>>(P.n, Vv, Wv, st);
  k_pi_spmv<<<P.grid, kBlock, 0, s>>>(P, 1, U, Wv, st, 1, Rt, P.partials, P.counters,
                                      P.colsum);
  k_pi_state<<<1, 32, 0, s>>>(st, P.colsum, 1);
  k_pi_fill<<<fill_grid(P.n), 256, 0, s>>>(P.n, Vv, Wv, st);
  k_pi_tick<<<1, 32, 0, s>>>(st);
}

}  // namespace bl
