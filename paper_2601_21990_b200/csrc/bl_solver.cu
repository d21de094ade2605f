// bl_solver.cu — C-ABI (include/batchlp_cuda.h) and host orchestration of
// the device-resident batched PDHG loop.
//
// solve_batch (reference batch_solver.hpp:78-355) runs as
//   validation (BatchProblem ctor problem.hpp:146-167, cfg.check()
//   solver.hpp:90-102, presets :93-99) -> eta (device power iteration,
//   cached per problem) -> slot permutation parking the presets (:157-160)
//   -> init kernels (X = proj(0), Y = 0, AX = A X) -> ONE CUDA graph launch:
//   a WHILE conditional node whose body is one solver iteration, with IF
//   nodes for the check, certificate and snapshot/compaction branches. The
//   host is not consulted between iterations; it reads the control block
//   once at the end.

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "batchlp_cuda.h"
#include "bl_device.cuh"


namespace {

struct BlError {
  int code;
  std::string msg;
};

[[noreturn]] void raise(int code, const std::string& msg) { throw BlError{code, msg}; }

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    raise(BL_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Grow-only device buffer (BatchWorkspace semantics, batch_solver.hpp:59-67).
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  void* ensure(size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (bytes > cap) {
      if (p) cudaFree(p);
      p = nullptr;
      cap = 0;
      ck(cudaMalloc(&p, bytes), "cudaMalloc");
      cap = bytes;
    }
    return p;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

std::string g_create_error;

}  // namespace

struct bl_problem {
  bl_ctx* ctx = nullptr;
  int m = 0, n = 0;
  int64_t nnz = 0;
  DevBuf rp, ci, cv, trp, tci, tcv, c, xl, xu, rl, ru;
  bool norm_valid = false;
  double norm = 0.0;
  std::vector<double> h_xl, h_xu;  // for override validation
  std::vector<int> h_rp, h_trp;    // row pointers (tail shared-memory cache sizing)
};

struct bl_ctx {
  int device = 0;
  cudaStream_t stream = nullptr, side = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int grid = 148;
  int sms = 148;
  long long l2_bytes = 126ll << 20;
  std::string err;
  // workspace
  enum {
    B_X0, B_X1, B_Y0, B_Y1, B_AX0, B_AX1, B_aX, B_aY, B_aAX, B_XT, B_YT, B_DY,
    B_RC, B_R, B_DR, B_AXT, B_BX, B_BY, B_BR, B_RX, B_RY, B_RR, B_RDX, B_RDY, B_RDR,
    B_SLOTD, B_SLOTI, B_ORIGI, B_RES, B_COLSUM, B_PART, B_CNT, B_SNAP, B_MOVES,
    B_LOG, B_CTRL, B_PROF, B_PROFACC, B_BAR, B_OV, B_OVD, B_WARMX, B_WARMY, B_PI, B_TMP0, B_TMP1,
    B_TUNE0, B_TUNE1, B_TUNE2, B_TUNE3,
    B_TAIL, B_DBG, B_RTAB, B_COUNT
  };
  DevBuf buf[B_COUNT];
  // last solve
  bool last_valid = false;
  int last_width = 0, last_n = 0, last_m = 0, last_vectors = 0;
  std::vector<bl_column_result> last_res;
  int last_log = 0;
  std::vector<bl_kernel_stat> last_prof;
  // graph cache
  cudaGraphExec_t exec = nullptr;
  cudaGraph_t graph = nullptr;
  bl::Params exec_params{};
  int exec_trace = -1;
  bl::Ctrl* h_ctrl = nullptr;  // pinned
  // tail graph cache
  cudaGraphExec_t tail_exec = nullptr;
  cudaGraph_t tail_graph = nullptr;
  bl::Params tail_params{};
  int tail_smem = -1;
  // power-iteration graph cache (16 steps), keyed by its parameters
  cudaGraphExec_t pi_exec = nullptr;
  bl::Params pi_params{};
  const void* pi_ptrs[4] = {nullptr, nullptr, nullptr, nullptr};
  // transient one-orientation CSR of bl_csr_apply
  bl_problem csr_scratch;
};

namespace {

template <class F>
int guarded(bl_ctx* ctx, F&& f) {
  try {
    f();
    return BL_OK;
  } catch (const BlError& e) {
    if (ctx) ctx->err = e.msg;
    else g_create_error = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    if (ctx) ctx->err = e.what();
    else g_create_error = e.what();
    return BL_ERR_CUDA;
  }
}

void check_config(const bl_config& c) {
  // SolverConfig::check, solver.hpp:90-102 (same messages)
  if (!(c.beta_sufficient > 0.0 && c.beta_sufficient < c.beta_necessary &&
        c.beta_necessary < 1.0))
    raise(BL_ERR_INVALID_ARGUMENT, "config: need 0 < beta_s < beta_n < 1");
  if (!(c.theta > 0.0 && c.theta <= 1.0))
    raise(BL_ERR_INVALID_ARGUMENT, "config: need 0 < theta <= 1");
  if (c.termination_check_period < 1)
    raise(BL_ERR_INVALID_ARGUMENT, "config: check period must be >= 1");
  if (c.max_iterations < 0)
    raise(BL_ERR_INVALID_ARGUMENT, "config: negative iteration limit");
  if (!(c.eps_opt > 0.0) || !(c.eps_infeas > 0.0))
    raise(BL_ERR_INVALID_ARGUMENT, "config: tolerances must be positive");
}

bool interval_valid(double lo, double hi) {  // Interval::valid, bounds.hpp:35-38
  return !std::isnan(lo) && !std::isnan(hi) && lo < HUGE_VAL && hi > -HUGE_VAL &&
         lo <= hi;
}

// Column-block width: the batch width rounded up to a power of two, at most
// 32 (BATCHLP_MAX_W lowers the cap for tuning sweeps).
int pow2_width(int width) {
  static int cap = [] {
    const char* e = std::getenv("BATCHLP_MAX_W");
    const int v = e ? std::atoi(e) : 32;
    return (v == 1 || v == 2 || v == 4 || v == 8 || v == 16) ? v : 32;
  }();
  int W = 1;
  while (W < width && W < cap) W <<= 1;
  return W;
}

int groups_for(int W) {
  const int L = W >= 2 ? W / 2 : 1;
  return bl::kBlock / L;
}

int items_for(int rows, int W, int grid) {
  if (rows <= bl::kTinyRows) return 1;
  const int G = groups_for(W);
  int R = (rows + 2 * G - 1) / (2 * G);
  if (R > grid) R = grid;
  if (R < 1) R = 1;
  return R;
}

template <class T>
void upload(DevBuf& b, const T* src, size_t count, cudaStream_t s) {
  b.ensure(count * sizeof(T) + 16);
  if (count) ck(cudaMemcpyAsync(b.p, src, count * sizeof(T), cudaMemcpyHostToDevice, s),
                "upload");
}

// Device power iteration, sparse.hpp:249-319.
double device_spectral_norm(bl_ctx* ctx, bl_problem* p) {
  if (p->nnz == 0) raise(BL_ERR_INVALID_ARGUMENT, "spectral_norm: zero matrix");
  if (p->norm_valid) return p->norm;
  const int n = p->n, m = p->m;
  cudaStream_t s = ctx->stream;
  // start vectors, computed on the host exactly as the reference does
  std::vector<double> v0((size_t)2 * n);
  const double one = 1.0 / std::sqrt(static_cast<double>(n));
  std::vector<double> mixed(n);
  std::uint64_t state = 0x9e3779b97f4a7c15ull;
  double norm_sq = 0.0;
  for (int i = 0; i < n; ++i) {
    state ^= state << 13;
    state ^= state >> 7;
    state ^= state << 17;
    mixed[i] = (state >> 11) * 0x1.0p-53 * 2.0 - 1.0;
    norm_sq += mixed[i] * mixed[i];
  }
  const double inv = 1.0 / std::sqrt(norm_sq);
  for (double& e : mixed) e *= inv;
  for (int i = 0; i < n; ++i) {
    v0[(size_t)i * 2] = one;
    v0[(size_t)i * 2 + 1] = mixed[i];
  }
  // workspace: V (n x 2), U (m x 2), Wv (n x 2), state, partials, counters
  const size_t vbytes = sizeof(double) * 2 * ((size_t)n + n + m);
  double* V = static_cast<double*>(ctx->buf[bl_ctx::B_PI].ensure(vbytes));
  double* U = V + (size_t)2 * n;
  double* Wv = U + (size_t)2 * m;
  bl::PiState st0[2] = {};
  bl::PiState* st = static_cast<bl::PiState*>(ctx->buf[bl_ctx::B_TMP0].ensure(sizeof(st0)));
  ck(cudaMemcpyAsync(V, v0.data(), sizeof(double) * 2 * n, cudaMemcpyHostToDevice, s), "pi v0");
  ck(cudaMemcpyAsync(st, st0, sizeof(st0), cudaMemcpyHostToDevice, s), "pi state");
  bl::Params P{};
  P.m = m;
  P.n = n;
  P.rp = p->rp.as<int>();
  P.ci = p->ci.as<int>();
  P.cv = p->cv.as<double>();
  P.trp = p->trp.as<int>();
  P.tci = p->tci.as<int>();
  P.tcv = p->tcv.as<double>();
  P.grid = ctx->grid;
  const int Rmax = std::max(items_for(m, 2, ctx->grid), items_for(n, 2, ctx->grid));
  P.partials = static_cast<double*>(
      ctx->buf[bl_ctx::B_PART].ensure(sizeof(double) * 2 * (size_t)std::max(Rmax, 1)));
  P.counters = static_cast<int*>(ctx->buf[bl_ctx::B_CNT].ensure(sizeof(int) * 64));
  ck(cudaMemsetAsync(P.counters, 0, sizeof(int) * 64, s), "memset counters");
  P.colsum = static_cast<double*>(ctx->buf[bl_ctx::B_TMP1].ensure(sizeof(double) * 2));
  P.Kp = 2;
  // 16 steps (7 kernels each) per host check, replayed from a CUDA graph:
  // one launch instead of 112; rebuilt only when the buffers or the problem
  // change (bl_problem_assign keeps them)
  const void* ptrs[4] = {V, U, Wv, st};
  if (!ctx->pi_exec || std::memcmp(&ctx->pi_params, &P, sizeof(P)) != 0 ||
      std::memcmp(ctx->pi_ptrs, ptrs, sizeof(ptrs)) != 0) {
    if (ctx->pi_exec) cudaGraphExecDestroy(ctx->pi_exec);
    ctx->pi_exec = nullptr;
    cudaGraph_t g;
    ck(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "pi capture");
    for (int k = 0; k < 16; ++k) bl::launch_pi_step(P, s, V, U, Wv, st);
    ck(cudaStreamEndCapture(s, &g), "pi capture end");
    const cudaError_t e = cudaGraphInstantiate(&ctx->pi_exec, g, 0);
    cudaGraphDestroy(g);
    ck(e, "pi graph instantiate");
    ctx->pi_params = P;
    std::memcpy(ctx->pi_ptrs, ptrs, sizeof(ptrs));
  }
  bl::PiState hst[2];
  for (int it = 0; it < 5000; it += 16) {
    ck(cudaGraphLaunch(ctx->pi_exec, s), "pi graph launch");
    ck(cudaMemcpyAsync(hst, st, sizeof(hst), cudaMemcpyDeviceToHost, s), "pi read");
    ck(cudaStreamSynchronize(s), "pi sync");
    if (hst[0].done && hst[1].done) break;
  }
  ck(cudaGetLastError(), "power iteration");
  const double a = hst[0].estimate, b = hst[1].estimate;
  p->norm = ((a < b) ? b : a) * 1.01;
  p->norm_valid = true;
  return p->norm;
}

// Shared memory for the tail cluster's CSR cache: the largest per-CTA slice
// (rows + 1 pointers, indices, values, alignment) of A' and A together;
// 0 (read from global memory) when it would not fit next to the static
// shared memory of the loop kernel.
int tail_smem_bytes(const bl_problem* p, int cl) {
  size_t worst = 0;
  for (int c = 0; c < cl; ++c) {
    size_t bytes = 32;
    for (int pass = 0; pass < 2; ++pass) {
      const std::vector<int>& rp = pass == 0 ? p->h_trp : p->h_rp;
      const int rows = (int)rp.size() - 1;
      const int r0 = (int)((long long)rows * c / cl), r1 = (int)((long long)rows * (c + 1) / cl);
      const size_t nz = (size_t)(rp[r1] - rp[r0]);
      bytes += 4 * (size_t)(r1 - r0 + 1) + 12 * nz + 16;
    }
    worst = std::max(worst, bytes);
  }
  return worst <= (size_t)160 * 1024 ? (int)((worst + 15) / 16 * 16) : 0;
}

void free_graph(bl_ctx* ctx) {
  if (ctx->exec) cudaGraphExecDestroy(ctx->exec);
  if (ctx->graph) cudaGraphDestroy(ctx->graph);
  ctx->exec = nullptr;
  ctx->graph = nullptr;
  ctx->exec_trace = -1;
}

// Adds a conditional node to `g` with dependencies; returns its body graphs.
cudaGraphNode_t add_cond(cudaGraph_t g, const cudaGraphNode_t* deps, size_t ndeps,
                         cudaGraphConditionalHandle h, cudaGraphConditionalNodeType type,
                         unsigned size, cudaGraph_t* bodies) {
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = h;
  np.conditional.type = type;
  np.conditional.size = size;
  cudaGraphNode_t node;
  ck(cudaGraphAddNode(&node, g, deps, ndeps, &np), "cudaGraphAddNode(conditional)");
  for (unsigned i = 0; i < size; ++i) bodies[i] = np.conditional.phGraph_out[i];
  return node;
}

template <class F>
void capture_into(cudaStream_t s, cudaGraph_t g, F&& f) {
  ck(cudaStreamBeginCaptureToGraph(s, g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed),
     "begin capture");
  f();
  cudaGraph_t out;
  ck(cudaStreamEndCapture(s, &out), "end capture");
}

// Builds the whole-solve graph:
//   WHILE(loop) { IF(check){primal+dual+check} ELSE {primal+dual};
//                 decide0; IF(cert){cert; decide1}; IF(snap){snapshot;
//                 compact}; [IF(trace){trace}] }
void build_graph(bl_ctx* ctx, bl::Params P) {
  free_graph(ctx);
  cudaGraph_t g;
  ck(cudaGraphCreate(&g, 0), "cudaGraphCreate");
  cudaGraphConditionalHandle hl, hc, hcert, hs, ht;
  ck(cudaGraphConditionalHandleCreate(&hl, g, 1, cudaGraphCondAssignDefault), "handle");
  ck(cudaGraphConditionalHandleCreate(&hc, g, 1, cudaGraphCondAssignDefault), "handle");
  ck(cudaGraphConditionalHandleCreate(&hcert, g, 0, cudaGraphCondAssignDefault), "handle");
  ck(cudaGraphConditionalHandleCreate(&hs, g, 0, cudaGraphCondAssignDefault), "handle");
  ht = 0;
  if (P.trace)  // an unused handle makes instantiation fail
    ck(cudaGraphConditionalHandleCreate(&ht, g, 0, cudaGraphCondAssignDefault), "handle");
  // one handle per conditional node: the check and the plain branch each get one
  cudaGraphConditionalHandle hn = 0, hn2 = 0;
  if (P.narrow_ok) {
    ck(cudaGraphConditionalHandleCreate(&hn, g, 0, cudaGraphCondAssignDefault), "handle");
    ck(cudaGraphConditionalHandleCreate(&hn2, g, 0, cudaGraphCondAssignDefault), "handle");
  }
  P.h_narrow = hn;
  P.h_narrow2 = hn2;

  P.use_graph = 1;
  P.h_loop = hl;
  P.h_check = hc;
  P.h_cert = hcert;
  P.h_snap = hs;
  P.h_trace = ht;
  cudaGraph_t wbody;
  add_cond(g, nullptr, 0, hl, cudaGraphCondTypeWhile, 1, &wbody);
  cudaGraph_t ifb[2];
  cudaGraphNode_t n_it = add_cond(wbody, nullptr, 0, hc, cudaGraphCondTypeIf, 2, ifb);
  cudaStream_t s2 = ctx->side;
  if (P.narrow_ok) {
    // each branch: IF(narrow) { single-block narrow kernels } ELSE { full width }
    cudaGraph_t cb[2], pb[2];
    add_cond(ifb[0], nullptr, 0, hn, cudaGraphCondTypeIf, 2, cb);
    add_cond(ifb[1], nullptr, 0, hn2, cudaGraphCondTypeIf, 2, pb);
    capture_into(s2, cb[0], [&] { bl::launch_iteration_check_narrow(P, s2); });
    capture_into(s2, cb[1], [&] { bl::launch_iteration_check(P, s2); });
    capture_into(s2, pb[0], [&] { bl::launch_iteration_plain_narrow(P, s2); });
    capture_into(s2, pb[1], [&] { bl::launch_iteration_plain(P, s2); });
  } else {
    capture_into(s2, ifb[0], [&] { bl::launch_iteration_check(P, s2); });
    capture_into(s2, ifb[1], [&] { bl::launch_iteration_plain(P, s2); });
  }
  // decide (phase 0) then the conditional tails, captured into the body
  cudaStream_t s = s2;
  ck(cudaStreamBeginCaptureToGraph(s, wbody, &n_it, nullptr, 1, cudaStreamCaptureModeRelaxed),
     "begin capture body");
  bl::launch_decide(P, s, 0);
  auto append_cond = [&](cudaGraphConditionalHandle h, cudaGraph_t* body) {
    cudaStreamCaptureStatus st;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    cudaGraph_t cg;
    ck(cudaStreamGetCaptureInfo(s, &st, nullptr, &cg, &deps, &nd), "capture info");
    cudaGraphNode_t node = add_cond(cg, deps, nd, h, cudaGraphCondTypeIf, 1, body);
    ck(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies),
       "update deps");
  };
  cudaGraph_t bcert, bsnap, btrace;
  append_cond(hcert, &bcert);
  append_cond(hs, &bsnap);
  if (P.trace) append_cond(ht, &btrace);
  cudaGraph_t outg;
  ck(cudaStreamEndCapture(s, &outg), "end capture body");
  capture_into(s2, bcert, [&] {
    bl::launch_cert(P, s2);
    bl::launch_decide(P, s2, 1);
  });
  capture_into(s2, bsnap, [&] { bl::launch_snap_compact(P, s2); });
  if (P.trace) capture_into(s2, btrace, [&] { bl::launch_trace(P, s2); });
  ck(cudaGraphInstantiate(&ctx->exec, g, 0), "cudaGraphInstantiate");
  ctx->graph = g;
  ctx->exec_params = P;
  ctx->exec_trace = P.trace;
}

bool same_params(const bl::Params& a, const bl::Params& b) {
  bl::Params x = a, y = b;
  x.use_graph = y.use_graph = 0;
  x.h_loop = y.h_loop = x.h_check = y.h_check = x.h_cert = y.h_cert = 0;
  x.h_snap = y.h_snap = x.h_trace = y.h_trace = 0;
  x.h_tail = y.h_tail = 0;
  return std::memcmp(&x, &y, sizeof(bl::Params)) == 0;
}

void free_tail_graph(bl_ctx* ctx) {
  if (ctx->tail_exec) cudaGraphExecDestroy(ctx->tail_exec);
  if (ctx->tail_graph) cudaGraphDestroy(ctx->tail_graph);
  ctx->tail_exec = nullptr;
  ctx->tail_graph = nullptr;
  ctx->tail_smem = -1;
}

// The tail as a device-driven loop: WHILE(not done) { fast-tail cluster
// kernel (plain passes); generic cluster kernel (exactly one pass: check,
// certificate, compaction, restart bookkeeping) } — the generic kernel sets
// the WHILE condition, so the host is not consulted between iterations.
void run_tail_graph(bl_ctx* ctx, const bl::Params& Q, int smem) {
  if (!ctx->tail_exec || ctx->tail_smem != smem || !same_params(ctx->tail_params, Q)) {
    free_tail_graph(ctx);
    cudaGraph_t g;
    ck(cudaGraphCreate(&g, 0), "cudaGraphCreate(tail)");
    cudaGraphConditionalHandle h;
    ck(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault), "tail handle");
    cudaGraph_t body;
    add_cond(g, nullptr, 0, h, cudaGraphCondTypeWhile, 1, &body);
    cudaStream_t s2 = ctx->side;
    bl::Params F = Q, G = Q;
    F.tail_single = 0;
    F.h_tail = h;
    G.tail_single = 1;
    G.h_tail = h;
    capture_into(s2, body, [&] {
      ck(bl::launch_tail_fast(F, s2, smem), "tail fast launch");
      ck(bl::launch_loop_cluster(G, s2, smem), "tail generic launch");
    });
    ck(cudaGraphInstantiate(&ctx->tail_exec, g, 0), "cudaGraphInstantiate(tail)");
    ctx->tail_graph = g;
    ctx->tail_params = Q;
    ctx->tail_smem = smem;
  }
  ck(cudaGraphLaunch(ctx->tail_exec, ctx->stream), "cudaGraphLaunch(tail)");
}

void run_loop_graph(bl_ctx* ctx, const bl::Params& P) {
  if (!ctx->exec || !same_params(ctx->exec_params, P) || ctx->exec_trace != P.trace)
    build_graph(ctx, P);
  ck(cudaGraphLaunch(ctx->exec, ctx->stream), "cudaGraphLaunch");
}

// Debug path: same kernels, host reads the control block every iteration.
void run_loop_steps(bl_ctx* ctx, bl::Params P) {
  P.use_graph = 0;
  cudaStream_t s = ctx->stream;
  bl::Ctrl* h = ctx->h_ctrl;
  for (;;) {
    ck(cudaMemcpyAsync(h, P.ctrl, sizeof(bl::Ctrl), cudaMemcpyDeviceToHost, s), "ctrl");
    ck(cudaStreamSynchronize(s), "step sync");
    if (h->done) break;
    const bool narrow = P.narrow_ok && h->active <= P.W / 2;
    if (h->check) {
      if (narrow) bl::launch_iteration_check_narrow(P, s);
      else bl::launch_iteration_check(P, s);
    } else {
      if (narrow) bl::launch_iteration_plain_narrow(P, s);
      else bl::launch_iteration_plain(P, s);
    }
    bl::launch_decide(P, s, 0);
    bl::launch_cert(P, s);
    bl::launch_decide(P, s, 1);
    bl::launch_snap_compact(P, s);
    if (P.trace) bl::launch_trace(P, s);
    ck(cudaGetLastError(), "step launch");
  }
}

bl_config config_or_default(const bl_config* cfg) {
  bl_config c;
  bl_config_default(&c);
  if (cfg) c = *cfg;
  return c;
}

void solve_batch_impl(bl_ctx* ctx, bl_problem* p, int32_t width, int32_t mode,
                      const bl_override* ov, int32_t n_ov, const bl_config* cfg_in,
                      const int32_t* presets, int32_t n_presets, const double* w0,
                      const double* warm_x, const double* warm_y, bl_summary* summary,
                      bl_column_result* results, int unit_off = -1) {
  const bl_config cfg = config_or_default(cfg_in);
  const int n = p->n, m = p->m;
  // BatchProblem constructor checks (problem.hpp:146-167); a shard of a
  // signed-unit batch (unit_off >= 0) was checked as a whole by the caller
  if (width < 0) raise(BL_ERR_INVALID_ARGUMENT, "batch: negative width");
  if (mode == BL_SIGNED_UNIT_COLUMNS && unit_off < 0 && width != 2 * n)
    raise(BL_ERR_INVALID_ARGUMENT, "batch: signed unit columns require width 2n");
  for (int k = 0; k < n_ov; ++k) {
    const bl_override& o = ov[k];
    if (o.column < 0 || o.column >= width)
      raise(BL_ERR_OUT_OF_RANGE, "batch: override column out of range");
    if (o.variable < 0 || o.variable >= n)
      raise(BL_ERR_OUT_OF_RANGE, "batch: override variable out of range");
    double lo = p->h_xl[o.variable], hi = p->h_xu[o.variable];
    if (o.kind == BL_OVERRIDE_LOWER) lo = o.value;
    if (o.kind == BL_OVERRIDE_UPPER) hi = o.value;
    if (o.kind != BL_OVERRIDE_OBJECTIVE && !interval_valid(lo, hi))
      raise(BL_ERR_INVALID_ARGUMENT,
            "batch: override inverts the bound interval of variable " +
                std::to_string(o.variable));
  }
  // solve_batch (batch_solver.hpp:83-100)
  check_config(cfg);
  std::vector<int> frozen(width > 0 ? width : 0, 0);
  for (int k = 0; k < n_presets; ++k) {
    const int c = presets[k];
    if (c < 0 || c >= width)
      raise(BL_ERR_OUT_OF_RANGE, "solve_batch: preset column out of range");
    if (frozen[c]) raise(BL_ERR_INVALID_ARGUMENT, "solve_batch: duplicate preset column");
    frozen[c] = 1;
  }
  bl_summary sum{};
  sum.trajectory_hash = 1469598103934665603ull;
  ctx->last_valid = false;
  if (width == 0) {
    if (summary) *summary = sum;
    return;
  }
  cudaStream_t s = ctx->stream;
  ck(cudaEventRecord(ctx->ev0, s), "event");

  // step size (solver.hpp:62-64)
  double eta = cfg.eta;
  if (!(eta > 0.0)) eta = 0.998 / (p->nnz == 0 ? 1.0 : device_spectral_norm(ctx, p));
  const double eps_dual = cfg.eps_dual < 0.0 ? cfg.eps_opt : cfg.eps_dual;

  const int W = pow2_width(width);
  const int Kp = (width + W - 1) / W * W;
  const int nb = Kp / W;
  const int vec = cfg.vectors;

  // slot permutation with presets parked (batch_solver.hpp:157-160)
  std::vector<int> slot(width);
  for (int j = 0; j < width; ++j) slot[j] = j;
  std::vector<double> wts(width, cfg.w_init);
  if (w0)
    for (int j = 0; j < width; ++j) wts[j] = w0[j];
  int active = width;
  for (int sidx = active - 1; sidx >= 0; --sidx) {
    if (frozen[slot[sidx]]) {
      const int t = --active;
      std::swap(slot[sidx], slot[t]);
      std::swap(wts[sidx], wts[t]);
    }
  }

  // overrides sorted by column (stable, problem.hpp:168-176)
  std::vector<bl_override> ovs(ov, ov + n_ov);
  std::stable_sort(ovs.begin(), ovs.end(),
                   [](const bl_override& a, const bl_override& b) { return a.column < b.column; });
  std::vector<int> ob(width, 0), oe(width, 0);
  {
    std::vector<int> off(width + 1, 0);
    for (const auto& o : ovs) ++off[o.column + 1];
    for (int j = 0; j < width; ++j) off[j + 1] += off[j];
    for (int j = 0; j < width; ++j) {
      ob[j] = off[j];
      oe[j] = off[j + 1];
    }
  }

  // ---- workspace ----
  auto dmat = [&](int which, size_t rows) {
    return static_cast<double*>(ctx->buf[which].ensure(sizeof(double) * rows * (size_t)Kp));
  };
  bl::Params P{};
  P.m = m;
  P.n = n;
  P.rp = p->rp.as<int>();
  P.ci = p->ci.as<int>();
  P.cv = p->cv.as<double>();
  P.trp = p->trp.as<int>();
  P.tci = p->tci.as<int>();
  P.tcv = p->tcv.as<double>();
  P.c = p->c.as<double>();
  P.xl = p->xl.as<double>();
  P.xu = p->xu.as<double>();
  P.rl = p->rl.as<double>();
  P.ru = p->ru.as<double>();
  P.width = width;
  P.Kp = Kp;
  P.mode = mode;
  P.unit_off = unit_off > 0 ? unit_off : 0;
  P.W = W;
  P.X[0] = dmat(bl_ctx::B_X0, n);
  P.X[1] = dmat(bl_ctx::B_X1, n);
  P.Y[0] = dmat(bl_ctx::B_Y0, m);
  P.Y[1] = dmat(bl_ctx::B_Y1, m);
  P.AX[0] = dmat(bl_ctx::B_AX0, m);
  P.AX[1] = dmat(bl_ctx::B_AX1, m);
  P.aX = dmat(bl_ctx::B_aX, n);
  P.aY = dmat(bl_ctx::B_aY, m);
  P.aAX = dmat(bl_ctx::B_aAX, m);
  P.XT = dmat(bl_ctx::B_XT, n);
  P.YT = dmat(bl_ctx::B_YT, m);
  P.DY = dmat(bl_ctx::B_DY, m);
  P.AXT = dmat(bl_ctx::B_AXT, m);
  P.RC = dmat(bl_ctx::B_RC, n);
  P.R = dmat(bl_ctx::B_R, n);
  P.DR = dmat(bl_ctx::B_DR, n);
  if (vec >= BL_VECTORS_SOLUTION) {
    P.BX = dmat(bl_ctx::B_BX, n);
    P.BY = dmat(bl_ctx::B_BY, m);
    P.BR = dmat(bl_ctx::B_BR, n);
    P.RX = static_cast<double*>(ctx->buf[bl_ctx::B_RX].ensure(sizeof(double) * (size_t)width * n));
    P.RY = static_cast<double*>(ctx->buf[bl_ctx::B_RY].ensure(sizeof(double) * (size_t)width * m));
    P.RR = static_cast<double*>(ctx->buf[bl_ctx::B_RR].ensure(sizeof(double) * (size_t)width * n));
  }
  if (vec >= BL_VECTORS_CERTIFICATE) {
    P.RDX = static_cast<double*>(ctx->buf[bl_ctx::B_RDX].ensure(sizeof(double) * (size_t)width * n));
    P.RDY = static_cast<double*>(ctx->buf[bl_ctx::B_RDY].ensure(sizeof(double) * (size_t)width * m));
    P.RDR = static_cast<double*>(ctx->buf[bl_ctx::B_RDR].ensure(sizeof(double) * (size_t)width * n));
  }
  // per-slot doubles: w resid anchor best*9 t*6 scratch blk_resid = 20 arrays
  constexpr int kSlotD = 20;
  double* sd = static_cast<double*>(ctx->buf[bl_ctx::B_SLOTD].ensure(sizeof(double) * kSlotD * (size_t)Kp));
  P.w = sd;
  P.resid = sd + 1 * (size_t)Kp;
  P.anchor_resid = sd + 2 * (size_t)Kp;
  P.best_score = sd + 3 * (size_t)Kp;
  P.best_obj = sd + 4 * (size_t)Kp;
  P.best_gap = sd + 5 * (size_t)Kp;
  P.best_pres = sd + 6 * (size_t)Kp;
  P.best_dres = sd + 7 * (size_t)Kp;
  P.best_fp = sd + 8 * (size_t)Kp;
  P.best_bsup = sd + 9 * (size_t)Kp;
  P.best_rsup = sd + 10 * (size_t)Kp;
  P.best_bbsup = sd + 11 * (size_t)Kp;
  P.t_obj = sd + 12 * (size_t)Kp;
  P.t_gap = sd + 13 * (size_t)Kp;
  P.t_pres = sd + 14 * (size_t)Kp;
  P.t_dres = sd + 15 * (size_t)Kp;
  P.t_score = sd + 16 * (size_t)Kp;
  P.t_dsup = sd + 17 * (size_t)Kp;
  P.scratch = sd + 18 * (size_t)Kp;
  P.blk_resid = sd + 19 * (size_t)Kp;  // one per column block (<= Kp)
  constexpr int kSlotI = 7;
  int* si = static_cast<int*>(ctx->buf[bl_ctx::B_SLOTI].ensure(sizeof(int) * kSlotI * (size_t)Kp));
  P.slot_orig = si;
  P.has_best = si + 1 * (size_t)Kp;
  P.verdict = si + 2 * (size_t)Kp;
  P.cert_flag = si + 3 * (size_t)Kp;
  P.move_src = si + 4 * (size_t)Kp;
  P.snap_orig = si + 5 * (size_t)Kp;
  P.err_flag = si + 6 * (size_t)Kp;
  ck(cudaMemsetAsync(P.err_flag, 0, sizeof(int), s), "err flag");
  int* oi = static_cast<int*>(ctx->buf[bl_ctx::B_ORIGI].ensure(sizeof(int) * 3 * (size_t)width));
  P.orig_done = oi;
  P.ov_beg = oi + width;
  P.ov_end = oi + 2 * (size_t)width;
  P.res = static_cast<bl_column_result*>(
      ctx->buf[bl_ctx::B_RES].ensure(sizeof(bl_column_result) * (size_t)width));
  P.colsum = static_cast<double*>(ctx->buf[bl_ctx::B_COLSUM].ensure(sizeof(double) * bl::S_COUNT * (size_t)Kp));
  // loop driver: one cooperative persistent launch (default), the CUDA
  // graph with conditional nodes, or host-stepped kernels (debugging)
  // 0 auto: the graph loop while an iteration streams more than
  //   kHandoverBytes of state (bandwidth-bound; separately compiled kernels
  //   run at higher occupancy), then the persistent kernel for the
  //   latency-bound rest, then (<= tail_blocks active column blocks) one
  //   thread-block cluster for the last few LPs; 1 graph only;
  //   2 host-stepped; 3 persistent grid + cluster; 4 cluster only.
  double kHandoverBytes = 16.0 * (1 << 20);
  if (const char* e = std::getenv("BATCHLP_HANDOVER_MB")) kHandoverBytes = std::atof(e) * (1 << 20);
  int mode_loop = 0;
  if (const char* e = std::getenv("BATCHLP_LOOP")) {
    if (std::strcmp(e, "graph") == 0) mode_loop = 1;
    else if (std::strcmp(e, "step") == 0) mode_loop = 2;
    else if (std::strcmp(e, "persistent") == 0) mode_loop = 3;
    else if (std::strcmp(e, "cluster") == 0) mode_loop = 4;
  }
  int tail_blocks = 1;
  if (const char* e = std::getenv("BATCHLP_TAIL_BLOCKS")) tail_blocks = std::atoi(e);
  int tail_cluster = bl::max_tail_cluster(W);
  if (const char* e = std::getenv("BATCHLP_TAIL_CLUSTER")) tail_cluster = std::atoi(e);
  if (tail_cluster < 1) tail_cluster = 1;
  if (tail_cluster > 16) tail_cluster = 16;
  if (const char* e = std::getenv("BATCHLP_STEP_MODE"))
    if (e[0] == '1') mode_loop = 2;
  const int grid = ctx->grid;
  int occ_loop = bl::loop_ctas_per_sm(W);
  if (occ_loop > 4) occ_loop = 4;
  const int grid_loop = ctx->sms * occ_loop;
  const double state0 = 8.0 * (double)nb * W * (double)(n + m);
  const bool use_graph = mode_loop == 1 || mode_loop == 2 ||
                         (mode_loop == 0 && state0 >= kHandoverBytes);
  const bool use_loop = mode_loop == 3 || mode_loop == 0;
  const bool use_cluster = (mode_loop == 0 || mode_loop == 3) ? tail_blocks > 0 : mode_loop == 4;
  // Gathered-operand bytes kept in flight (tuned on B200:
  // fewer blocks in flight raise the L2 hit rate of the gathers);
  // overridable for tuning sweeps.
  long long l2_budget = 16ll << 20;
  if (const char* e = std::getenv("BATCHLP_L2_BUDGET_MB")) l2_budget = std::atoll(e) << 20;
  // partials: the largest (active blocks x items per block) any iteration
  // uses, under either driver's grid
  size_t max_items = 1;
  for (int g : {grid, grid_loop, tail_cluster}) {
    for (int nba = 1; nba <= nb; ++nba) {
      const size_t a = (size_t)nba * bl::items_per_block(n, m, W, g, nba, l2_budget);
      const size_t b = (size_t)nba * bl::items_per_block(m, n, W, g, nba, l2_budget);
      max_items = std::max(max_items, std::max(a, b));
    }
  }
  // the initial AX = A X (launch_spmm) picks its own item count per block
  max_items = std::max(max_items, (size_t)nb * std::max(items_for(m, W, grid),
                                                       items_for(n, W, grid)));
  P.partials = static_cast<double*>(
      ctx->buf[bl_ctx::B_PART].ensure(sizeof(double) * max_items * 10 * W));
  // per-block fold counters, then the row kernels' work-item ticket
  const int cbank = std::max(nb, 64);
  P.counters = static_cast<int*>(
      ctx->buf[bl_ctx::B_CNT].ensure(sizeof(int) * ((size_t)cbank + 2)));
  // Block-major dynamic work items pay off once one column block's gathered
  // operand is a sizeable share of L2 (C4: -21% per row pass, measured); on
  // small problems the per-item atomics cost more than the drift they
  // prevent (C2: +15%), so they use the static stride.
  {
    static const double min_bytes = [] {
      const char* e = std::getenv("BATCHLP_TICKET_MIN_BYTES");
      return e ? std::atof(e) : 4.0 * (1 << 20);
    }();
    const double block_operand = 8.0 * W * (double)std::max(m, n);
    P.ticket = block_operand >= min_bytes ? P.counters + cbank : nullptr;
  }
  // narrow single-block row kernels in the graph / step drivers: only large
  // problems reach a single block there (small ones hand over to the
  // persistent / cluster kernels first), so only they carry the IF(narrow)
  // branches (two extra conditional nodes per pass)
  P.narrow_ok = (W >= 16 && P.ticket != nullptr) ? 1 : 0;
  P.snap_list = static_cast<int*>(ctx->buf[bl_ctx::B_SNAP].ensure(sizeof(int) * 3 * (size_t)Kp));
  P.moves = static_cast<int*>(ctx->buf[bl_ctx::B_MOVES].ensure(sizeof(int) * 2 * (size_t)Kp));
  P.log_cap = 1 << 16;
  P.log = static_cast<bl_restart_event*>(
      ctx->buf[bl_ctx::B_LOG].ensure(sizeof(bl_restart_event) * (size_t)P.log_cap));
  P.ctrl = static_cast<bl::Ctrl*>(ctx->buf[bl_ctx::B_CTRL].ensure(sizeof(bl::Ctrl)));
  P.prof = static_cast<unsigned long long*>(
      ctx->buf[bl_ctx::B_PROF].ensure(sizeof(unsigned long long) * 2 * bl::K_KINDS));
  P.prof_acc = static_cast<double*>(
      ctx->buf[bl_ctx::B_PROFACC].ensure(sizeof(double) * 3 * bl::K_KINDS));
  P.nnz = p->nnz;
  {
    unsigned long long hp[2 * bl::K_KINDS];
    for (int k = 0; k < bl::K_KINDS; ++k) {
      hp[2 * k] = ~0ull;
      hp[2 * k + 1] = 0ull;
    }
    ck(cudaMemcpyAsync(P.prof, hp, sizeof(hp), cudaMemcpyHostToDevice, s), "prof");
    ck(cudaMemsetAsync(P.prof_acc, 0, sizeof(double) * 3 * bl::K_KINDS, s), "prof acc");
  }
  {
    const size_t nov = std::max<size_t>(ovs.size(), 1);
    int* ovi = static_cast<int*>(ctx->buf[bl_ctx::B_OV].ensure(sizeof(int) * 2 * nov));
    double* ovd = static_cast<double*>(ctx->buf[bl_ctx::B_OVD].ensure(sizeof(double) * nov));
    std::vector<int> hv(2 * nov, 0);
    std::vector<double> hd(nov, 0.0);
    for (size_t k = 0; k < ovs.size(); ++k) {
      hv[k] = ovs[k].variable;
      hv[nov + k] = ovs[k].kind;
      hd[k] = ovs[k].value;
    }
    ck(cudaMemcpyAsync(ovi, hv.data(), sizeof(int) * 2 * nov, cudaMemcpyHostToDevice, s), "ov");
    ck(cudaMemcpyAsync(ovd, hd.data(), sizeof(double) * nov, cudaMemcpyHostToDevice, s), "ov");
    P.ov_var = ovi;
    P.ov_kind = ovi + nov;
    P.ov_val = ovd;
  }
  P.eta = eta;
  P.eps = cfg.eps_opt;
  P.eps_dual = eps_dual;
  P.eps_infeas = cfg.eps_infeas;
  P.theta = cfg.theta;
  P.beta_s = cfg.beta_sufficient;
  P.beta_n = cfg.beta_necessary;
  P.beta_a = cfg.beta_artificial;
  P.max_it = cfg.max_iterations;
  P.period = cfg.termination_check_period;
  P.robust = cfg.robust_bound_contribution != 0;
  P.avg_all = cfg.average_over_all_columns != 0;
  P.trace = cfg.trace_iterates != 0;
  P.vectors = vec;
  P.grid = use_graph ? grid : grid_loop;
  // the graph / step drivers' plain row kernels launch at their own occupancy
  P.grid_run = use_graph ? ctx->sms * bl::plain_ctas_per_sm(W) : 0;
  if (std::getenv("BATCHLP_NO_ROUNDS")) P.grid_run = 0;
  P.l2_budget = l2_budget;
  {  // the decide kernel's work-item geometry per active block count
    std::vector<int> tab(2 * ((size_t)nb + 1));
    for (int nba = 0; nba <= nb; ++nba) {
      tab[nba] = bl::rounds_adjust(bl::items_per_block(n, m, W, P.grid, nba, l2_budget), nba,
                                   P.grid_run);
      tab[nb + 1 + nba] = bl::rounds_adjust(bl::items_per_block(m, n, W, P.grid, nba, l2_budget),
                                            nba, P.grid_run);
    }
    int* dtab = static_cast<int*>(ctx->buf[bl_ctx::B_RTAB].ensure(sizeof(int) * tab.size()));
    ck(cudaMemcpyAsync(dtab, tab.data(), sizeof(int) * tab.size(), cudaMemcpyHostToDevice, s),
       "geometry table");
    P.r_tab = dtab;
  }
  P.handover_bytes = (mode_loop == 0) ? kHandoverBytes : 0.0;
  P.tail_part = static_cast<double*>(
      ctx->buf[bl_ctx::B_TAIL].ensure(sizeof(double) * 16 * 5 * 32));
  if (std::getenv("BATCHLP_NO_FAST_TAIL")) P.tail_part = nullptr;
  P.dbg = nullptr;
  if (std::getenv("BATCHLP_TAIL_TRACE")) {
    P.dbg = static_cast<unsigned long long*>(
        ctx->buf[bl_ctx::B_DBG].ensure(sizeof(unsigned long long) * 32));
    ck(cudaMemsetAsync(P.dbg, 0, sizeof(unsigned long long) * 32, s), "dbg");
  }
  P.barrier = static_cast<unsigned long long*>(
      ctx->buf[bl_ctx::B_BAR].ensure(sizeof(unsigned long long)));
  ck(cudaMemsetAsync(P.barrier, 0, sizeof(unsigned long long), s), "barrier");

  // ---- host-side initial state ----
  {
    std::vector<double> hsd((size_t)kSlotD * Kp, 0.0);
    for (int j = 0; j < width; ++j) hsd[j] = wts[j];
    for (int j = 0; j < Kp; ++j) hsd[3 * (size_t)Kp + j] = HUGE_VAL;  // best_score
    ck(cudaMemcpyAsync(sd, hsd.data(), sizeof(double) * hsd.size(), cudaMemcpyHostToDevice, s), "slotd");
    std::vector<int> hsi((size_t)kSlotI * Kp, 0);
    for (int j = 0; j < width; ++j) hsi[j] = slot[j];
    for (int j = width; j < Kp; ++j) hsi[j] = 0;
    ck(cudaMemcpyAsync(si, hsi.data(), sizeof(int) * hsi.size(), cudaMemcpyHostToDevice, s), "sloti");
    std::vector<int> hoi((size_t)3 * width);
    for (int j = 0; j < width; ++j) {
      hoi[j] = frozen[j];
      hoi[width + j] = ob[j];
      hoi[2 * (size_t)width + j] = oe[j];
    }
    ck(cudaMemcpyAsync(oi, hoi.data(), sizeof(int) * hoi.size(), cudaMemcpyHostToDevice, s), "origi");
    ck(cudaMemsetAsync(P.counters, 0, sizeof(int) * ((size_t)std::max(nb, 64) + 2), s), "counters");
    ck(cudaMemsetAsync(P.res, 0, sizeof(bl_column_result) * (size_t)width, s), "res");
    ck(cudaMemsetAsync(P.colsum, 0, sizeof(double) * bl::S_COUNT * (size_t)Kp, s), "colsum");
  }
  const double* dwx = nullptr;
  const double* dwy = nullptr;
  if (warm_x && warm_y) {
    upload(ctx->buf[bl_ctx::B_WARMX], warm_x, (size_t)width * n, s);
    upload(ctx->buf[bl_ctx::B_WARMY], warm_y, (size_t)width * m, s);
    dwx = ctx->buf[bl_ctx::B_WARMX].as<double>();
    dwy = ctx->buf[bl_ctx::B_WARMY].as<double>();
  }
  bl::launch_init(P, s, dwx, dwy);
  bl::launch_spmm(P, s, false, P.X[0], P.AX[0], width);  // AX = A X (:137)
  ck(cudaGetLastError(), "init launch");

  bl::Ctrl c0{};
  c0.inner_k = 0;
  c0.total_k = 0;
  c0.sparse_products = 1;
  c0.hash = 1469598103934665603ull;
  c0.alpha = 0.5;
  c0.active = active;
  c0.cur = 0;
  c0.done = active == 0;
  c0.at_cap = 0 >= cfg.max_iterations;
  c0.check = 1;
  c0.anchor_reset = 1;
  c0.cond = bl::kCondDefaults;  // the graph handles' defaults at launch
  {
    const int nba = (active + W - 1) / W;
    c0.Rp = bl::rounds_adjust(bl::items_per_block(n, m, W, P.grid, nba, l2_budget), nba,
                              P.grid_run);
    c0.Rd = bl::rounds_adjust(bl::items_per_block(m, n, W, P.grid, nba, l2_budget), nba,
                              P.grid_run);
    c0.Rc = c0.Rp;
  }
  *ctx->h_ctrl = c0;
  ck(cudaMemcpyAsync(P.ctrl, ctx->h_ctrl, sizeof(bl::Ctrl), cudaMemcpyHostToDevice, s), "ctrl");

  if (active > 0) {
    if (mode_loop == 2) {
      run_loop_steps(ctx, P);
    } else {
      if (use_graph) run_loop_graph(ctx, P);
      if (use_loop) {
        // continues from the control block wherever the graph stopped (a
        // no-op launch when the graph already finished the batch)
        bl::Params Q = P;
        Q.grid = grid_loop;
        Q.grid_run = 0;
        Q.handover_bytes = 0.0;
        Q.use_graph = 0;
        Q.tail_blocks = use_cluster ? tail_blocks : 0;
        ck(bl::launch_loop(Q, s), "cooperative loop launch");
      }
      if (use_cluster) {
        // the last few LPs: one cluster, hardware barriers (no-op when the
        // batch is already finished)
        bl::Params Q = P;
        Q.grid = tail_cluster;
        Q.grid_run = 0;
        Q.handover_bytes = 0.0;
        Q.use_graph = 0;
        Q.tail_blocks = 0;
        Q.tail_single = 0;
        const int smem = tail_smem_bytes(p, tail_cluster);
        const bool fast_tail = P.tail_part && !P.trace && !P.avg_all && W <= 32 &&
                               !std::getenv("BATCHLP_NO_TAIL_GRAPH");
        if (fast_tail) run_tail_graph(ctx, Q, smem);
        else ck(bl::launch_loop_cluster(Q, s, smem), "cluster loop launch");
      }
    }
  }
  ck(cudaGetLastError(), "loop launch");
  ck(cudaMemcpyAsync(ctx->h_ctrl, P.ctrl, sizeof(bl::Ctrl), cudaMemcpyDeviceToHost, s), "ctrl");
  std::vector<bl_column_result> dres(width);
  ck(cudaMemcpyAsync(dres.data(), P.res, sizeof(bl_column_result) * width, cudaMemcpyDeviceToHost, s),
     "results");
  std::vector<int> done(width);
  ck(cudaMemcpyAsync(done.data(), P.orig_done, sizeof(int) * width, cudaMemcpyDeviceToHost, s), "done");
  unsigned long long hprof[2 * bl::K_KINDS];
  double hacc[3 * bl::K_KINDS];
  ck(cudaMemcpyAsync(hprof, P.prof, sizeof(hprof), cudaMemcpyDeviceToHost, s), "prof");
  ck(cudaMemcpyAsync(hacc, P.prof_acc, sizeof(hacc), cudaMemcpyDeviceToHost, s), "prof acc");
  ck(cudaEventRecord(ctx->ev1, s), "event");
  ck(cudaStreamSynchronize(s), "solve sync");
  if (P.dbg) {
    unsigned long long d[32];
    cudaMemcpy(d, P.dbg, sizeof(d), cudaMemcpyDeviceToHost);
    const double passes = d[0] > 0 ? (double)d[0] : 1.0;
    static const char* what[] = {"", "top->rows", "primal rows", "primal publish", "primal sync",
                                 "dual rows", "dual publish", "dual sync", "decide", "final sync"};
    std::fprintf(stderr, "[tail trace] %llu loop tops\n", (unsigned long long)d[0]);
    for (int k = 1; k < 10; ++k)
      std::fprintf(stderr, "[tail trace] %-16s %8.3f us/pass\n", what[k], d[k] / passes / 1e3);
    const double dp = d[10] > 0 ? (double)d[10] : 1.0;
    static const char* dwhat[] = {"resid+mean", "check block", "finalize"};
    std::fprintf(stderr, "[decide trace] %llu plain passes\n", (unsigned long long)d[10]);
    for (int k = 11; k < 14; ++k)
      std::fprintf(stderr, "[decide trace] %-16s %8.3f us/pass\n", dwhat[k - 11], d[k] / dp / 1e3);
    static const char* fwhat[] = {"fin: verdicts", "fin: compaction", "fin: cap", "fin: lists",
                                  "fin: rule+geometry", "fin: weights", "fin: conds"};
    for (int k = 16; k < 23; ++k)
      std::fprintf(stderr, "[decide trace] %-18s %8.3f us/pass\n", fwhat[k - 16], d[k] / dp / 1e3);
    std::fprintf(stderr, "[fast decide] ctrl+fold+resid %8.3f us/pass\n", d[14] / passes / 1e3);
    std::fprintf(stderr, "[fast decide] mean+rule       %8.3f us/pass\n", d[15] / passes / 1e3);
  }
  const bl::Ctrl C = *ctx->h_ctrl;
  if (C.error == BL_ERR_DOMAIN)
    raise(BL_ERR_DOMAIN,
          "residual metric is not positive semidefinite; step size exceeds 1/||A||");
  if (C.error == BL_ERR_LOGIC)
    raise(BL_ERR_LOGIC, "solve_batch: loop pass bound exceeded (internal error)");
  for (int j = 0; j < width; ++j)
    if (!done[j]) raise(BL_ERR_LOGIC, "solve_batch: column finished without a result");
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
  sum.iterations = C.total_k;
  sum.restarts = C.restarts;
  sum.restart_log_size = std::min(C.log_count, P.log_cap);
  sum.sparse_products = C.sparse_products;
  sum.trajectory_hash = C.hash;
  sum.eta = eta;
  sum.device_ms = ms;
  sum.kernel_launches = C.launches + 2;  // + init and AX = A X
  sum.loop_passes = C.passes;
  {
    static const char* names[bl::K_KINDS] = {"primal",      "dual",      "check",
                                             "decide",      "cert",      "snapshot",
                                             "compact",     "trace",     "tail_primal",
                                             "tail_dual",   "tail_decide"};
    ctx->last_prof.assign(bl::K_KINDS, bl_kernel_stat{});
    for (int k = 0; k < bl::K_KINDS; ++k) {
      bl_kernel_stat& st = ctx->last_prof[k];
      std::snprintf(st.name, sizeof(st.name), "%s", names[k]);
      st.total_ns = hacc[3 * k];
      st.launches = hacc[3 * k + 1];
      st.alg_bytes = hacc[3 * k + 2];
      const unsigned long long b = hprof[2 * k], e = hprof[2 * k + 1];
      if (e != 0ull && b != ~0ull && e >= b) {  // launches after the last fold
        st.total_ns += (double)(e - b);
        st.launches += 1.0;
      }
    }
  }
  if (summary) *summary = sum;
  ctx->last_res = dres;
  for (int j = 0; j < width; ++j)
    if (!frozen[j] && results) results[j] = dres[j];
  ctx->last_valid = true;
  ctx->last_width = width;
  ctx->last_n = n;
  ctx->last_m = m;
  ctx->last_vectors = vec;
  ctx->last_log = sum.restart_log_size;
  for (int j = 0; j < width; ++j)
    if (frozen[j]) ctx->last_res[j].has_solution = ctx->last_res[j].has_certificate = 0;
}

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================
namespace {
// Work decomposition of a standalone SpMM (bl_spmm, bl_csr_apply, the
// tuner): the row kernels' L2-aware items per block and, when one column
// block's operand is large, block-major dynamic work items (as in a solve);
// partials sized for either orientation.
void spmm_geometry(bl_ctx* ctx, bl::Params& P, int nb, int rows, int rows_in, int W,
                   cudaStream_t s) {
  P.l2_budget = 16ll << 20;
  size_t R = (size_t)std::max(items_for(rows, W, ctx->grid), items_for(rows_in, W, ctx->grid));
  R = std::max(R, (size_t)bl::items_per_block(rows, rows_in, W, ctx->grid, nb, P.l2_budget));
  R = std::max(R, (size_t)bl::items_per_block(rows_in, rows, W, ctx->grid, nb, P.l2_budget));
  P.partials = static_cast<double*>(
      ctx->buf[bl_ctx::B_PART].ensure(sizeof(double) * (size_t)nb * R * 10 * W));
  const size_t nc = (size_t)std::max(nb, 64) + 2;
  P.counters = static_cast<int*>(ctx->buf[bl_ctx::B_CNT].ensure(sizeof(int) * nc));
  ck(cudaMemsetAsync(P.counters, 0, sizeof(int) * nc, s), "counters");
  const double block_operand = 8.0 * W * (double)std::max(rows, rows_in);
  P.ticket = block_operand >= 4.0 * (1 << 20) ? P.counters + std::max(nb, 64) : nullptr;
}

// op(A) x for the first `active` of `width` column-major host columns:
// tiles them, runs the SpMM kernel, untiles, copies back (bl_spmm,
// bl_csr_apply).
void device_spmm(bl_ctx* ctx, const bl_problem* p, bool transpose, int width, int active,
                 const double* x, double* out) {
  if (active < 0) active = width;
  if (active > width) raise(BL_ERR_INVALID_ARGUMENT, "spmm: active width too large");
  if (active == 0) return;
  const int rin = transpose ? p->m : p->n, rout = transpose ? p->n : p->m;
  const int W = pow2_width(width);
  const int Kp = (width + W - 1) / W * W;
  cudaStream_t s = ctx->stream;
  double* tin = static_cast<double*>(ctx->buf[bl_ctx::B_TMP0].ensure(sizeof(double) * ((size_t)rin * Kp + 1)));
  double* tout = static_cast<double*>(ctx->buf[bl_ctx::B_TMP1].ensure(sizeof(double) * ((size_t)rout * Kp + 1)));
  double* raw = static_cast<double*>(ctx->buf[bl_ctx::B_WARMX].ensure(
      sizeof(double) * ((size_t)std::max(rin, rout) * width + 1)));
  ck(cudaMemcpyAsync(raw, x, sizeof(double) * (size_t)rin * active, cudaMemcpyHostToDevice, s), "x");
  bl::launch_to_tiled(s, raw, tin, rin, width, W, active);
  bl::Params P{};
  P.m = p->m;
  P.n = p->n;
  P.rp = p->rp.as<int>();
  P.ci = p->ci.as<int>();
  P.cv = p->cv.as<double>();
  P.trp = p->trp.as<int>();
  P.tci = p->tci.as<int>();
  P.tcv = p->tcv.as<double>();
  P.W = W;
  P.Kp = Kp;
  P.grid = ctx->grid;
  const int nb = Kp / W;
  spmm_geometry(ctx, P, nb, rout, rin, W, s);
  P.colsum = static_cast<double*>(ctx->buf[bl_ctx::B_COLSUM].ensure(sizeof(double) * bl::S_COUNT * (size_t)Kp));
  bl::launch_spmm(P, s, transpose, tin, tout, active);
  bl::launch_from_tiled(s, tout, raw, rout, width, W, active);
  ck(cudaMemcpyAsync(out, raw, sizeof(double) * (size_t)rout * active, cudaMemcpyDeviceToHost, s), "out");
  ck(cudaStreamSynchronize(s), "spmm sync");
  ck(cudaGetLastError(), "spmm");
}
}  // namespace

extern "C" {

void bl_config_default(bl_config* c) {
  // SolverConfig defaults, solver.hpp:67-86
  c->eps_opt = 1e-4;
  c->eps_infeas = 1e-8;
  c->eps_dual = -1.0;
  c->theta = 0.5;
  c->beta_sufficient = 0.2;
  c->beta_necessary = 0.8;
  c->beta_artificial = 0.36;
  c->max_iterations = 100000;
  c->termination_check_period = 64;
  c->w_init = 1.0;
  c->robust_bound_contribution = 0;
  c->average_over_all_columns = 0;
  c->trace_iterates = 0;
  c->vectors = BL_VECTORS_SOLUTION;
  c->eta = 0.0;
}

int bl_abi_version(void) { return BL_ABI_VERSION; }

int bl_ctx_create(int device, bl_ctx** out) {
  *out = nullptr;
  bl_ctx* ctx = new bl_ctx();
  const int rc = guarded(nullptr, [&] {
    ck(cudaSetDevice(device), "cudaSetDevice");
    ctx->device = device;
    ck(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking), "stream");
    ck(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreate(&ctx->ev0), "event");
    ck(cudaEventCreate(&ctx->ev1), "event");
    ck(cudaMallocHost(&ctx->h_ctrl, sizeof(bl::Ctrl)), "pinned ctrl");
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    int occ = bl::max_ctas_per_sm();
    if (occ > 4) occ = 4;
    ctx->grid = sms * occ;
    ctx->sms = sms;
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device);
    if (l2 > 0) ctx->l2_bytes = l2;
  });
  if (rc != BL_OK) {
    delete ctx;
    return rc;
  }
  *out = ctx;
  return BL_OK;
}

void bl_ctx_destroy(bl_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  free_graph(ctx);
  free_tail_graph(ctx);
  if (ctx->pi_exec) cudaGraphExecDestroy(ctx->pi_exec);
  for (auto& b : ctx->buf) b.release();
  for (DevBuf* b : {&ctx->csr_scratch.rp, &ctx->csr_scratch.ci, &ctx->csr_scratch.cv}) b->release();
  if (ctx->h_ctrl) cudaFreeHost(ctx->h_ctrl);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  delete ctx;
}

const char* bl_last_error(const bl_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_create_error.c_str();
}

namespace {
// Fills `p` (grow-only buffers: a re-upload of a problem of the same size
// keeps every device address, so captured CUDA graphs stay valid).
void fill_problem(bl_ctx* ctx, bl_problem* p, int32_t m, int32_t n, int64_t nnz,
                  const int32_t* rowptr, const int32_t* col, const double* val,
                  const int32_t* t_rowptr, const int32_t* t_col, const double* t_val,
                  const double* objective, const double* var_lower, const double* var_upper,
                  const double* row_lower, const double* row_upper) {
    if (m < 0 || n < 0 || nnz < 0) raise(BL_ERR_INVALID_ARGUMENT, "sparse: negative dimension");
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    cudaStream_t s = ctx->stream;
    p->ctx = ctx;
    p->m = m;
    p->n = n;
    p->nnz = nnz;
    upload(p->rp, rowptr, (size_t)m + 1, s);
    upload(p->ci, col, (size_t)nnz, s);
    upload(p->cv, val, (size_t)nnz, s);
    upload(p->trp, t_rowptr, (size_t)n + 1, s);
    upload(p->tci, t_col, (size_t)nnz, s);
    upload(p->tcv, t_val, (size_t)nnz, s);
    upload(p->c, objective, (size_t)n, s);
    upload(p->xl, var_lower, (size_t)n, s);
    upload(p->xu, var_upper, (size_t)n, s);
    upload(p->rl, row_lower, (size_t)m, s);
    upload(p->ru, row_upper, (size_t)m, s);
    p->h_xl.assign(var_lower, var_lower + n);
    p->h_rp.assign(rowptr, rowptr + m + 1);
    p->h_trp.assign(t_rowptr, t_rowptr + n + 1);
    p->h_xu.assign(var_upper, var_upper + n);
    p->norm_valid = false;
    ck(cudaStreamSynchronize(s), "upload sync");
}
}  // namespace

int bl_problem_upload(bl_ctx* ctx, int32_t m, int32_t n, int64_t nnz,
                      const int32_t* rowptr, const int32_t* col, const double* val,
                      const int32_t* t_rowptr, const int32_t* t_col,
                      const double* t_val, const double* objective,
                      const double* var_lower, const double* var_upper,
                      const double* row_lower, const double* row_upper,
                      bl_problem** out) {
  *out = nullptr;
  bl_problem* p = new bl_problem();
  const int rc = guarded(ctx, [&] {
    fill_problem(ctx, p, m, n, nnz, rowptr, col, val, t_rowptr, t_col, t_val, objective,
                 var_lower, var_upper, row_lower, row_upper);
  });
  if (rc != BL_OK) {
    bl_problem_free(p);
    return rc;
  }
  *out = p;
  return BL_OK;
}

int bl_problem_assign(bl_ctx* ctx, bl_problem* p, int32_t m, int32_t n, int64_t nnz,
                      const int32_t* rowptr, const int32_t* col, const double* val,
                      const int32_t* t_rowptr, const int32_t* t_col,
                      const double* t_val, const double* objective,
                      const double* var_lower, const double* var_upper,
                      const double* row_lower, const double* row_upper) {
  return guarded(ctx, [&] {
    if (!p || p->ctx != ctx) raise(BL_ERR_INVALID_ARGUMENT, "assign: problem of another context");
    fill_problem(ctx, p, m, n, nnz, rowptr, col, val, t_rowptr, t_col, t_val, objective,
                 var_lower, var_upper, row_lower, row_upper);
  });
}

void bl_problem_free(bl_problem* p) {
  if (!p) return;
  for (DevBuf* b : {&p->rp, &p->ci, &p->cv, &p->trp, &p->tci, &p->tcv, &p->c, &p->xl,
                    &p->xu, &p->rl, &p->ru})
    b->release();
  delete p;
}

int bl_spectral_norm(bl_ctx* ctx, bl_problem* p, double* out) {
  return guarded(ctx, [&] {
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    *out = device_spectral_norm(ctx, p);
  });
}

int bl_spmm(bl_ctx* ctx, const bl_problem* p, int transpose, int32_t width,
            int32_t active, const double* x, double* out) {
  return guarded(ctx, [&] {
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    device_spmm(ctx, p, transpose != 0, width, active, x, out);
  });
}

int bl_csr_apply(bl_ctx* ctx, int32_t rows, int32_t cols, int64_t nnz, const int32_t* rowptr,
                 const int32_t* col, const double* val, const double* x, double* out) {
  return guarded(ctx, [&] {
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (rows < 0 || cols < 0 || nnz < 0) raise(BL_ERR_INVALID_ARGUMENT, "csr_apply: negative dimension");
    if (nnz > INT32_MAX) raise(BL_ERR_INVALID_ARGUMENT, "csr_apply: too many nonzeros");
    if (rows == 0) return;
    if (rowptr[0] != 0 || rowptr[rows] != nnz)
      raise(BL_ERR_INVALID_ARGUMENT, "csr_apply: malformed row offsets");
    for (int32_t i = 0; i < rows; ++i)
      if (rowptr[i + 1] < rowptr[i]) raise(BL_ERR_INVALID_ARGUMENT, "csr_apply: malformed row offsets");
    for (int64_t q = 0; q < nnz; ++q)
      if (col[q] < 0 || col[q] >= cols) raise(BL_ERR_OUT_OF_RANGE, "csr_apply: column index out of range");
    // a transient one-orientation problem (grow-only buffers of the context)
    bl_problem& t = ctx->csr_scratch;
    cudaStream_t s = ctx->stream;
    t.ctx = ctx;
    t.m = rows;
    t.n = cols;
    t.nnz = nnz;
    upload(t.rp, rowptr, (size_t)rows + 1, s);
    upload(t.ci, col, (size_t)nnz, s);
    upload(t.cv, val, (size_t)nnz, s);
    t.norm_valid = false;
    device_spmm(ctx, &t, false, 1, 1, x, out);
  });
}

int bl_measure_spmm(bl_ctx* ctx, const bl_problem* p, int32_t width, int32_t repetitions,
                    double* total_s, double* per_column_s, int32_t* clamped) {
  return guarded(ctx, [&] {
    if (width < 1) raise(BL_ERR_INVALID_ARGUMENT, "tuner: width must be >= 1");
    if (repetitions < 3) raise(BL_ERR_INVALID_ARGUMENT, "tuner: need >= 3 repetitions");
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    const int n = p->n, m = p->m;
    // the reference's seeded blocks (tuner.hpp:79-82), column-major
    std::mt19937_64 rng(0x5eedu);
    std::vector<double> hx((size_t)n * width), hy((size_t)m * width);
    for (double& v : hx) v = (double)(rng() >> 11) * 0x1.0p-53 * 2.0 - 1.0;
    for (double& v : hy) v = (double)(rng() >> 11) * 0x1.0p-53 * 2.0 - 1.0;
    const int W = pow2_width(width);
    const int Kp = (width + W - 1) / W * W;
    cudaStream_t s = ctx->stream;
    auto dbuf = [&](int which, size_t rows) {
      return static_cast<double*>(ctx->buf[which].ensure(sizeof(double) * (rows * Kp + 1)));
    };
    double* x = dbuf(bl_ctx::B_TUNE0, n);
    double* y = dbuf(bl_ctx::B_TUNE1, m);
    double* ax = dbuf(bl_ctx::B_TUNE2, m);
    double* aty = dbuf(bl_ctx::B_TUNE3, n);
    double* raw = static_cast<double*>(ctx->buf[bl_ctx::B_WARMX].ensure(
        sizeof(double) * ((size_t)std::max(n, m) * width + 1)));
    ck(cudaMemcpyAsync(raw, hx.data(), sizeof(double) * hx.size(), cudaMemcpyHostToDevice, s), "x");
    bl::launch_to_tiled(s, raw, x, n, width, W, width);
    ck(cudaMemcpyAsync(raw, hy.data(), sizeof(double) * hy.size(), cudaMemcpyHostToDevice, s), "y");
    bl::launch_to_tiled(s, raw, y, m, width, W, width);
    bl::Params P{};
    P.m = m;
    P.n = n;
    P.rp = p->rp.as<int>();
    P.ci = p->ci.as<int>();
    P.cv = p->cv.as<double>();
    P.trp = p->trp.as<int>();
    P.tci = p->tci.as<int>();
    P.tcv = p->tcv.as<double>();
    P.W = W;
    P.Kp = Kp;
    P.grid = ctx->grid;
    const int nb = Kp / W;
    spmm_geometry(ctx, P, nb, m, n, W, s);
    P.colsum = static_cast<double*>(
        ctx->buf[bl_ctx::B_COLSUM].ensure(sizeof(double) * bl::S_COUNT * (size_t)Kp));
    for (int warm = 0; warm < 2; ++warm) {
      bl::launch_spmm(P, s, false, x, ax, width);
      bl::launch_spmm(P, s, true, y, aty, width);
    }
    ck(cudaEventRecord(ctx->ev0, s), "event");
    for (int r = 0; r < repetitions; ++r) bl::launch_spmm(P, s, false, x, ax, width);
    for (int r = 0; r < repetitions; ++r) bl::launch_spmm(P, s, true, y, aty, width);
    ck(cudaEventRecord(ctx->ev1, s), "event");
    ck(cudaEventSynchronize(ctx->ev1), "tuner sync");
    ck(cudaGetLastError(), "tuner spmm");
    float ms = 0.f, oms = 0.f;
    ck(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1), "elapsed");
    // the measurement's own overhead: an empty event interval
    ck(cudaEventRecord(ctx->ev0, s), "event");
    ck(cudaEventRecord(ctx->ev1, s), "event");
    ck(cudaEventSynchronize(ctx->ev1), "tuner sync");
    ck(cudaEventElapsedTime(&oms, ctx->ev0, ctx->ev1), "elapsed");
    double total = ((double)ms - (double)oms) * 1e-3;
    int cl = 0;
    if (total < 0.0) {
      total = 0.0;
      cl = 1;
    }
    if (total_s) *total_s = total;
    if (per_column_s) *per_column_s = total / width;
    if (clamped) *clamped = cl;
  });
}

int bl_solve_batch(bl_ctx* ctx, bl_problem* p, int32_t width, int32_t mode,
                   const bl_override* overrides, int32_t n_overrides,
                   const bl_config* cfg, const int32_t* preset_columns,
                   int32_t n_presets, const double* initial_weights,
                   const double* warm_x, const double* warm_y, bl_summary* summary,
                   bl_column_result* results) {
  return guarded(ctx, [&] {
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    solve_batch_impl(ctx, p, width, mode, overrides, n_overrides, cfg, preset_columns,
                     n_presets, initial_weights, warm_x, warm_y, summary, results);
  });
}

int bl_solve_batch_sharded(bl_ctx* const* ctxs, bl_problem* const* probs, int32_t n_shards,
                           int32_t width, int32_t mode, const bl_override* overrides,
                           int32_t n_overrides, const bl_config* cfg,
                           const int32_t* preset_columns, int32_t n_presets,
                           const double* initial_weights, bl_summary* summaries,
                           bl_column_result* results) {
  if (n_shards < 1 || ctxs == nullptr || probs == nullptr) {
    g_create_error = "solve_batch_sharded: need at least one (context, problem) pair";
    return BL_ERR_INVALID_ARGUMENT;
  }
  bl_ctx* lead = ctxs[0];
  return guarded(lead, [&] {
    for (int s = 0; s < n_shards; ++s) {
      if (!ctxs[s] || !probs[s] || probs[s]->ctx != ctxs[s])
        raise(BL_ERR_INVALID_ARGUMENT, "solve_batch_sharded: problem of another context");
      for (int t = 0; t < s; ++t)
        if (ctxs[t] == ctxs[s])
          raise(BL_ERR_INVALID_ARGUMENT, "solve_batch_sharded: a context appears twice");
      if (probs[s]->m != probs[0]->m || probs[s]->n != probs[0]->n ||
          probs[s]->nnz != probs[0]->nnz)
        raise(BL_ERR_INVALID_ARGUMENT, "solve_batch_sharded: replicas of different problems");
    }
    const int n = probs[0]->n;
    // the whole batch's checks, in the single-device order (problem.hpp:146-167,
    // solver.hpp:90-102, batch_solver.hpp:93-99); each shard re-checks its part
    if (width < 0) raise(BL_ERR_INVALID_ARGUMENT, "batch: negative width");
    if (mode == BL_SIGNED_UNIT_COLUMNS && width != 2 * n)
      raise(BL_ERR_INVALID_ARGUMENT, "batch: signed unit columns require width 2n");
    for (int k = 0; k < n_overrides; ++k)
      if (overrides[k].column < 0 || overrides[k].column >= width)
        raise(BL_ERR_OUT_OF_RANGE, "batch: override column out of range");
    check_config(config_or_default(cfg));
    std::vector<char> seen(width > 0 ? width : 0, 0);
    for (int k = 0; k < n_presets; ++k) {
      const int c = preset_columns[k];
      if (c < 0 || c >= width) raise(BL_ERR_OUT_OF_RANGE, "solve_batch: preset column out of range");
      if (seen[c]) raise(BL_ERR_INVALID_ARGUMENT, "solve_batch: duplicate preset column");
      seen[c] = 1;
    }
    // contiguous near-equal column slices (distributed.py column_slices)
    std::vector<int> beg(n_shards + 1, 0);
    for (int s = 0, at = 0; s < n_shards; ++s) {
      beg[s] = at;
      at += width / n_shards + (s < width % n_shards ? 1 : 0);
      beg[s + 1] = at;
    }
    struct Part {
      std::vector<bl_override> ov;
      std::vector<int32_t> presets;
      std::vector<double> w0;
      int code = BL_OK;
      std::string msg;
    };
    std::vector<Part> parts(n_shards);
    for (int k = 0; k < n_overrides; ++k) {  // overrides keep their list order
      const int c = overrides[k].column;
      const int s = int(std::upper_bound(beg.begin(), beg.end() - 1, c) - beg.begin()) - 1;
      bl_override o = overrides[k];
      o.column = c - beg[s];
      parts[s].ov.push_back(o);
    }
    for (int k = 0; k < n_presets; ++k) {
      const int c = preset_columns[k];
      const int s = int(std::upper_bound(beg.begin(), beg.end() - 1, c) - beg.begin()) - 1;
      parts[s].presets.push_back(c - beg[s]);
    }
    // one host thread per shard, each on its own context / device; every
    // shard writes its per-LP records straight into its slice of `results`
    auto run = [&](int s) {
      Part& pt = parts[s];
      bl_ctx* c = ctxs[s];
      const int w = beg[s + 1] - beg[s];
      const int rc = guarded(c, [&] {
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        solve_batch_impl(c, probs[s], w, mode, pt.ov.data(), (int32_t)pt.ov.size(), cfg,
                         pt.presets.empty() ? nullptr : pt.presets.data(),
                         (int32_t)pt.presets.size(),
                         initial_weights ? initial_weights + beg[s] : nullptr, nullptr, nullptr,
                         summaries ? &summaries[s] : nullptr, results + beg[s],
                         mode == BL_SIGNED_UNIT_COLUMNS ? beg[s] : -1);
      });
      if (rc != BL_OK) {
        pt.code = rc;
        pt.msg = c->err;
      }
    };
    std::vector<std::thread> threads;
    for (int s = 1; s < n_shards; ++s) threads.emplace_back(run, s);
    run(0);
    for (std::thread& t : threads) t.join();
    for (int s = 0; s < n_shards; ++s)
      if (parts[s].code != BL_OK)
        raise(parts[s].code, "shard " + std::to_string(s) + ": " + parts[s].msg);
  });
}

int bl_fetch_solution(bl_ctx* ctx, int32_t column, double* x, double* y,
                      double* reduced) {
  return guarded(ctx, [&] {
    if (!ctx->last_valid) raise(BL_ERR_LOGIC, "fetch: no solve on this context");
    if (column < 0 || column >= ctx->last_width)
      raise(BL_ERR_OUT_OF_RANGE, "fetch: column out of range");
    if (!ctx->last_res[column].has_solution)
      raise(BL_ERR_INVALID_ARGUMENT, "fetch: column has no solution vectors");
    const int n = ctx->last_n, m = ctx->last_m;
    cudaStream_t s = ctx->stream;
    if (x) ck(cudaMemcpyAsync(x, ctx->buf[bl_ctx::B_RX].as<double>() + (size_t)column * n,
                              sizeof(double) * n, cudaMemcpyDeviceToHost, s), "fetch x");
    if (y) ck(cudaMemcpyAsync(y, ctx->buf[bl_ctx::B_RY].as<double>() + (size_t)column * m,
                              sizeof(double) * m, cudaMemcpyDeviceToHost, s), "fetch y");
    if (reduced)
      ck(cudaMemcpyAsync(reduced, ctx->buf[bl_ctx::B_RR].as<double>() + (size_t)column * n,
                         sizeof(double) * n, cudaMemcpyDeviceToHost, s), "fetch r");
    ck(cudaStreamSynchronize(s), "fetch sync");
  });
}

int bl_fetch_certificate(bl_ctx* ctx, int32_t column, double* dx, double* dy,
                         double* dr) {
  return guarded(ctx, [&] {
    if (!ctx->last_valid) raise(BL_ERR_LOGIC, "fetch: no solve on this context");
    if (column < 0 || column >= ctx->last_width)
      raise(BL_ERR_OUT_OF_RANGE, "fetch: column out of range");
    const bl_column_result& r = ctx->last_res[column];
    if (!r.has_certificate) raise(BL_ERR_INVALID_ARGUMENT, "fetch: column has no certificate");
    const int n = ctx->last_n, m = ctx->last_m;
    cudaStream_t s = ctx->stream;
    if (dx) ck(cudaMemcpyAsync(dx, ctx->buf[bl_ctx::B_RDX].as<double>() + (size_t)column * n,
                               sizeof(double) * n, cudaMemcpyDeviceToHost, s), "fetch dx");
    if (r.certificate_kind == 1) {
      if (dy) ck(cudaMemcpyAsync(dy, ctx->buf[bl_ctx::B_RDY].as<double>() + (size_t)column * m,
                                 sizeof(double) * m, cudaMemcpyDeviceToHost, s), "fetch dy");
      if (dr) ck(cudaMemcpyAsync(dr, ctx->buf[bl_ctx::B_RDR].as<double>() + (size_t)column * n,
                                 sizeof(double) * n, cudaMemcpyDeviceToHost, s), "fetch dr");
    }
    ck(cudaStreamSynchronize(s), "fetch sync");
  });
}

int bl_fetch_profile(bl_ctx* ctx, bl_kernel_stat* out, int32_t cap, int32_t* n_out) {
  return guarded(ctx, [&] {
    const int k = std::min<int>(cap, (int)ctx->last_prof.size());
    for (int i = 0; i < k; ++i) out[i] = ctx->last_prof[i];
    if (n_out) *n_out = k;
  });
}

int bl_fetch_restart_log(bl_ctx* ctx, bl_restart_event* out, int32_t cap, int32_t* n_out) {
  return guarded(ctx, [&] {
    if (!ctx->last_valid) raise(BL_ERR_LOGIC, "fetch: no solve on this context");
    const int k = std::min(cap, ctx->last_log);
    if (k > 0)
      ck(cudaMemcpy(out, ctx->buf[bl_ctx::B_LOG].p, sizeof(bl_restart_event) * k,
                    cudaMemcpyDeviceToHost), "fetch log");
    if (n_out) *n_out = k;
  });
}

}  // extern "C"
