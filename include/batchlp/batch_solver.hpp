// batchlp/batch_solver.hpp — THE hot path of the B200 drop-in.
//
// batchlp::solve_batch with the reference's signature and semantics
// (reference proj/include/batchlp/batch_solver.hpp:45-82, 83-355): K LPs
// sharing A iterate together as column-block tiles in HBM, restarts are
// synchronised on the batch-averaged residual, finished columns are
// compacted out with the reference's swap-with-last order, and results come
// back in original column order. The whole loop is device resident
// (csrc/bl_solver.cu: CUDA graph with conditional nodes, then a persistent
// cooperative kernel for the latency-bound tail); the host waits once.
//
// BatchWorkspace keeps the reference's role — caller-owned, grow-only state
// reused across rounds (batch_solver.hpp:59-67, strong_branching.hpp:129-179)
// — but what it owns is a device context: a CUDA stream, the HBM buffers of
// the last solve and the residency cache of uploaded problems.
#ifndef BATCHLP_B200_BATCH_SOLVER_HPP
#define BATCHLP_B200_BATCH_SOLVER_HPP

#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <vector>

#include "batchlp/device.hpp"
#include "batchlp/problem.hpp"
#include "batchlp/solver.hpp"
#include "batchlp/sparse.hpp"

namespace batchlp {

struct PresetColumn {
  int column = 0;
  SolveResult result;
};

struct BatchSolveSummary {
  std::vector<SolveResult> per_problem;  // original column order
  std::int64_t iterations = 0;
  int restarts = 0;
  std::int64_t sparse_products = 0;
  std::vector<RestartEvent> restart_log;
  std::uint64_t trajectory_hash = 1469598103934665603ull;
};

class BatchWorkspace {
 public:
  BatchWorkspace() = default;
  explicit BatchWorkspace(int device) : device_(device) {}
  cuda::Context& context() {
    if (!ctx_) ctx_ = std::make_unique<cuda::Context>(device_);
    return *ctx_;
  }

 private:
  int device_ = cuda::Context::default_device();
  std::unique_ptr<cuda::Context> ctx_;
};

// What a solve copies back per LP (extension; the reference always returns
// x / y / reduced costs and the certificate vectors by value).
enum class VectorMode {
  kNone = BL_VECTORS_NONE,                // status, objective, residuals, supports
  kSolution = BL_VECTORS_SOLUTION,        // + x, y, reduced costs
  kCertificate = BL_VECTORS_CERTIFICATE,  // + infeasibility certificates (reference default)
};

struct BatchOptions {
  VectorMode vectors = VectorMode::kCertificate;
  // Multi-GPU (extension): two or more device ordinals shard
  // the batch into contiguous column slices, one per listed device (a device
  // listed twice gets two contexts); A is replicated, nothing is exchanged
  // while iterating, and each slice restarts on its own averaged residual
  // -- the result equals the reference's solve_batch run slice by slice.
  // Empty or one entry: the workspace's (or this thread's) context.
  std::vector<int> devices;
};

inline BatchSolveSummary solve_batch(const BatchProblem& batch, const SolverConfig& cfg = {},
                                     std::span<const PresetColumn> presets = {},
                                     BatchWorkspace* external_ws = nullptr,
                                     std::span<const double> initial_weights = {},
                                     const BatchOptions& options = {}) {
  // validation order of the reference (batch_solver.hpp:83-100, 115-118)
  cfg.check();
  const int width = batch.batch_width();
  std::vector<int> cols;
  cols.reserve(presets.size());
  {
    std::vector<char> seen(static_cast<std::size_t>(width > 0 ? width : 0), 0);
    for (const PresetColumn& pc : presets) {
      if (pc.column < 0 || pc.column >= width)
        throw std::out_of_range("solve_batch: preset column out of range");
      if (seen[pc.column]) throw std::invalid_argument("solve_batch: duplicate preset column");
      seen[pc.column] = 1;
      cols.push_back(pc.column);
    }
  }
  BatchSolveSummary summary;
  if (width == 0) return summary;
  if (!initial_weights.empty() && static_cast<int>(initial_weights.size()) != width)
    throw std::invalid_argument("solve_batch: initial weight count mismatch");

  detail::DeviceRun run;
  if (options.devices.size() > 1) {
    std::vector<cuda::Context*> ctxs;
    for (std::size_t k = 0; k < options.devices.size(); ++k) {
      int seen = 0;
      for (std::size_t q = 0; q < k; ++q) seen += options.devices[q] == options.devices[k];
      ctxs.push_back(&cuda::shard_context(options.devices[k], seen));
    }
    run = detail::run_sharded(ctxs, batch, cfg, cols, initial_weights,
                              static_cast<int>(options.vectors));
  } else {
    cuda::Context& ctx = external_ws           ? external_ws->context()
                         : options.devices.empty() ? cuda::thread_context()
                                                   : cuda::shard_context(options.devices[0], 0);
    run = detail::run_on_device(ctx, batch, cfg, cols, initial_weights, nullptr,
                                static_cast<int>(options.vectors));
  }
  summary.iterations = run.summary.iterations;
  summary.restarts = run.summary.restarts;
  summary.sparse_products = run.summary.sparse_products;
  summary.trajectory_hash = run.summary.trajectory_hash;
  summary.restart_log = std::move(run.restart_log);
  summary.per_problem = std::move(run.results);
  for (const PresetColumn& pc : presets) summary.per_problem[pc.column] = pc.result;
  return summary;
}

}  // namespace batchlp

#endif  // BATCHLP_B200_BATCH_SOLVER_HPP
