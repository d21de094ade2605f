// batchlp/solver.hpp — solver configuration, results and the single-LP solve
// of the B200 drop-in.
//
// Source-compatible with the public surface of the reference's solver.hpp
// (reference proj/include/batchlp/solver.hpp:51-145, 299-334, 529-531,
// 569-703): the value types field for field, the scalar control rules
// (restart_reason, smoothed_primal_weight, step_size_for) as host helpers,
// and solve(), which runs as a width-1 batch on the GPU — the reference's
// width-1 batch is bit-identical to its single solve (batch_solver.hpp:22-24,
// test_batch_solver.cpp:33-54), so this is the same trajectory.
//
// The vector-level operator primitives of the reference (apply_T,
// m_norm_residual, halpern_combine, evaluate_optimality,
// check_infeasibility_probe) exist here only fused inside the sm_100a
// kernels (csrc/bl_kernels.cu); INTEGRATION.md lists them as not exported.
#ifndef BATCHLP_B200_SOLVER_HPP
#define BATCHLP_B200_SOLVER_HPP

#include <cmath>
#include <cstdint>
#include <limits>
#include <optional>
#include <stdexcept>
#include <vector>

#include "batchlp/bounds.hpp"
#include "batchlp/problem.hpp"
#include "batchlp/sparse.hpp"

namespace batchlp {

// tau = eta / w, sigma = eta * w (reference solver.hpp:51-60).
struct StepParams {
  double eta = 0.0;
  double w = 1.0;
  double tau = 0.0;
  double sigma = 0.0;

  StepParams() = default;
  StepParams(double eta_in, double w_in)
      : eta(eta_in), w(w_in), tau(eta_in / w_in), sigma(eta_in * w_in) {}
};

// 0.998 / ||A||_2 (reference solver.hpp:62-64); the norm comes from the
// device power iteration.
inline double step_size_for(const SparseMatrix& a) {
  return 0.998 / (a.nnz() == 0 ? 1.0 : spectral_norm(a));
}

// Reference solver.hpp:66-103, same fields, defaults and checks.
struct SolverConfig {
  double eps_opt = 1e-4;
  double eps_infeas = 1e-8;
  double eps_dual = -1.0;  // < 0: eps_opt
  double theta = 0.5;
  double beta_sufficient = 0.2;
  double beta_necessary = 0.8;
  double beta_artificial = 0.36;
  std::int64_t max_iterations = 100000;
  std::int64_t termination_check_period = 64;
  double w_init = 1.0;
  bool robust_bound_contribution = false;
  bool average_over_all_columns = false;
  bool trace_iterates = false;

  double effective_eps_dual() const { return eps_dual < 0.0 ? eps_opt : eps_dual; }

  void check() const {
    const bool betas = beta_sufficient > 0.0 && beta_sufficient < beta_necessary &&
                       beta_necessary < 1.0;
    if (!betas) throw std::invalid_argument("config: need 0 < beta_s < beta_n < 1");
    if (!(theta > 0.0 && theta <= 1.0))
      throw std::invalid_argument("config: need 0 < theta <= 1");
    if (termination_check_period < 1)
      throw std::invalid_argument("config: check period must be >= 1");
    if (max_iterations < 0) throw std::invalid_argument("config: negative iteration limit");
    if (!(eps_opt > 0.0) || !(eps_infeas > 0.0))
      throw std::invalid_argument("config: tolerances must be positive");
  }
};

// Enumerator order equals the C-ABI's (bl_status, bl_restart_reason).
enum class SolveStatus { kOptimal, kPrimalInfeasible, kDualInfeasible, kIterationLimit };
enum class RestartReason { kSufficientDecay, kNecessaryNoProgress, kArtificial };

struct RestartEvent {
  std::int64_t at_iteration = 0;
  RestartReason reason = RestartReason::kSufficientDecay;
  double residual = 0.0;
  double anchor_residual = 0.0;
};

struct InfeasibilityProbe {
  std::vector<double> delta_x, delta_y, delta_r;
};

struct Residuals {
  double gap = kInf;
  double primal = kInf;
  double dual = kInf;
  double fixed_point = kInf;
};

// Reference solver.hpp:134-145, plus `device`: scalars the GPU computed for
// the returned triple, so callers such as OBBT's safety margin
// (obbt.hpp:121-137) need not copy x / y / r back.
struct SolveResult {
  SolveStatus status = SolveStatus::kIterationLimit;
  double objective = std::numeric_limits<double>::quiet_NaN();
  std::vector<double> x, y, reduced_costs;
  Residuals residuals;
  std::int64_t iterations = 0;
  int restarts = 0;
  InfeasibilityProbe certificate;
  std::vector<RestartEvent> restart_log;
  std::uint64_t trajectory_hash = 1469598103934665603ull;
  std::int64_t sparse_products = 0;

  struct DeviceScalars {
    bool valid = false;               // filled by a device solve
    bool vectors_exist = false;       // the reference would return x / y / r
    double bound_support = 0.0;       // phi over the column's variable box of r
    double row_support = 0.0;         // phi over the row box of y
    double base_bound_support = 0.0;  // phi over the BASE variable box of r
  } device;
};

struct WarmStart {
  std::vector<double> x, y;
};

// Restart rule on the averaged residual (reference solver.hpp:299-311).
inline std::optional<RestartReason> restart_reason(double r, double r_anchor, double r_prev,
                                                   std::int64_t inner_k, std::int64_t total_k,
                                                   const SolverConfig& cfg) {
  if (r <= cfg.beta_sufficient * r_anchor) return RestartReason::kSufficientDecay;
  const bool stalled = r > r_prev;
  if (stalled && r <= cfg.beta_necessary * r_anchor) return RestartReason::kNecessaryNoProgress;
  if (static_cast<double>(inner_k) > cfg.beta_artificial * static_cast<double>(total_k))
    return RestartReason::kArtificial;
  return std::nullopt;
}

// log-space smoothing of the primal weight towards ||dy|| / ||dx||, each
// update capped at a factor of 4 (reference solver.hpp:321-334). The device
// decide kernel evaluates the same formula with correctly rounded exp/log.
inline double smoothed_primal_weight(double w, double dx_norm, double dy_norm, double theta) {
  const bool usable = dx_norm > 0.0 && dy_norm > 0.0 && std::isfinite(dx_norm) &&
                      std::isfinite(dy_norm);
  if (!usable) return w;
  const double ratio = dy_norm / dx_norm;
  if (!std::isfinite(ratio) || !(ratio > 0.0)) return w;
  const double lw = std::log(w);
  const double target = theta * std::log(ratio) + (1.0 - theta) * lw;
  const double cap = std::log(4.0);
  if (target > lw + cap) return std::exp(lw + cap);
  if (target < lw - cap) return std::exp(lw - cap);
  return std::exp(target);
}

}  // namespace batchlp

#include "batchlp/detail/device_solve.hpp"

namespace batchlp {

// One LP (reference solver.hpp:569-703) as a width-1 device batch.
inline SolveResult solve(const LpProblem& p, const SolverConfig& cfg = {},
                         const WarmStart* warm = nullptr) {
  cfg.check();
  const std::size_t n = static_cast<std::size_t>(p.num_cols());
  const std::size_t m = static_cast<std::size_t>(p.num_rows());
  if (p.objective.size() != n || p.row_bounds.size() != m || p.var_bounds.size() != n)
    throw std::invalid_argument("solve: inconsistent problem dimensions");
  if (warm != nullptr && (warm->x.size() != n || warm->y.size() != m))
    throw std::invalid_argument("solve: warm start dimension mismatch");
  BatchProblem one(p, 1, ObjectiveMode::kSharedObjective, {});
  detail::DeviceRun run = detail::run_on_device(cuda::thread_context(), one, cfg, {}, {},
                                                warm, BL_VECTORS_CERTIFICATE);
  SolveResult r = std::move(run.results[0]);
  r.restart_log = std::move(run.restart_log);
  r.trajectory_hash = run.summary.trajectory_hash;
  r.sparse_products = run.summary.sparse_products;
  return r;
}

}  // namespace batchlp

#endif  // BATCHLP_B200_SOLVER_HPP
