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
// The vector-level operator primitives of the reference (solver.hpp:147-297,
// 336-565: apply_operator, apply_T, m_norm_squared / m_norm_residual,
// halpern_combine, evaluate_optimality, check_infeasibility_probe, the
// best-candidate snapshot) are exported for single host vectors, the way the
// reference's tests and callers use them: their sparse products run on the
// device (csr_apply / spmv -> bl_csr_apply / bl_spmm, bit-identical to the
// reference's stored-order sums), the elementwise terms are the same
// expressions the fused epilogues evaluate per LP column inside the batch
// kernels (csrc/bl_kernels.cuh), evaluated here in the reference's order.
#ifndef BATCHLP_B200_SOLVER_HPP
#define BATCHLP_B200_SOLVER_HPP

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <optional>
#include <span>
#include <stdexcept>
#include <utility>
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

namespace detail {

// Plain sequential reductions (reference solver.hpp:149-177).
inline double dot(std::span<const double> a, std::span<const double> b) {
  double acc = 0.0;
  const std::size_t n = a.size();
  for (std::size_t k = 0; k < n; ++k) acc += a[k] * b[k];
  return acc;
}
inline double norm(std::span<const double> a) { return std::sqrt(dot(a, a)); }
inline double distance(std::span<const double> a, std::span<const double> b) {
  double acc = 0.0;
  const std::size_t n = a.size();
  for (std::size_t k = 0; k < n; ++k) {
    const double diff = a[k] - b[k];
    acc += diff * diff;
  }
  return std::sqrt(acc);
}
// FNV-1a over the bytes of v (the trajectory hash, solver.hpp:170-177).
inline std::uint64_t fold_hash(std::uint64_t h, std::span<const double> v) {
  const auto* p = reinterpret_cast<const unsigned char*>(v.data());
  const std::size_t bytes = v.size() * sizeof(double);
  for (std::size_t k = 0; k < bytes; ++k) h = (h ^ p[k]) * 1099511628211ull;
  return h;
}

}  // namespace detail

// sigma (s - proj(s)), s = y / sigma + v (reference solver.hpp:181-190); the
// dual epilogue of k_dual evaluates the same expression per LP column.
inline double dual_step_element(double y, double v, double sigma, double lo, double hi) {
  const double s = y / sigma + v;
  return sigma * (s - project_box(s, lo, hi));
}

// One operator application on one column (reference solver.hpp:192-213):
// aty = A'y, xt = proj(x - tau (c + aty)), axt = A xt, yt = dual step of
// 2 axt - ax. Both products run on the device.
inline void apply_operator(const ColumnView& col, const CsrView& a, const CsrView& at,
                           const StepParams& sp, const double* x, const double* y,
                           const double* ax, double* aty, double* xt, double* axt,
                           double* yt) {
  const int n = a.n_cols, m = a.n_rows;
  csr_apply(at, y, aty);
  for (int j = 0; j < n; ++j) {
    const double moved = x[j] - sp.tau * (col.cost(j) + aty[j]);
    xt[j] = project_box(moved, col.lower(j), col.upper(j));
  }
  csr_apply(a, xt, axt);
  const Bounds& rows = col.problem().row_bounds;
  for (int i = 0; i < m; ++i)
    yt[i] = dual_step_element(y[i], 2.0 * axt[i] - ax[i], sp.sigma, rows.lower[i],
                              rows.upper[i]);
}

// T(x, y) from scratch (reference solver.hpp:215-230): A x first, then the
// operator.
inline std::pair<std::vector<double>, std::vector<double>> apply_T(const LpProblem& p,
                                                                   const StepParams& sp,
                                                                   std::span<const double> x,
                                                                   std::span<const double> y) {
  const std::size_t n = static_cast<std::size_t>(p.num_cols());
  const std::size_t m = static_cast<std::size_t>(p.num_rows());
  if (x.size() != n || y.size() != m) throw std::invalid_argument("apply_T: dimension mismatch");
  std::vector<double> ax(m), aty(n), xt(n), axt(m), yt(m);
  spmv(p.A, x, ax);
  apply_operator(ColumnView(p), p.A.view(), p.A.transpose_view(), sp, x.data(), y.data(),
                 ax.data(), aty.data(), xt.data(), axt.data(), yt.data());
  return {std::move(xt), std::move(yt)};
}

// (w/eta)|dx|^2 + |dy|^2/(eta w) + 2 dy.(A dx) (reference solver.hpp:232-246).
inline double m_norm_squared(std::span<const double> dx, std::span<const double> dy,
                             std::span<const double> a_dx, double eta, double w) {
  double sx = 0.0;
  for (const double d : dx) sx += d * d;
  double sy = 0.0, cr = 0.0;
  for (std::size_t i = 0; i < dy.size(); ++i) {
    sy += dy[i] * dy[i];
    cr += dy[i] * a_dx[i];
  }
  return (w / eta) * sx + (1.0 / (eta * w)) * sy + 2.0 * cr;
}

namespace detail {

// sqrt of the metric; a negative form beyond 1e-12 of its scale means the
// step size broke the metric (reference solver.hpp:250-263). The device
// decide kernel applies the same rule and reports BL_ERR_DOMAIN.
inline double m_residual_from_terms(double dx_sq, double dy_sq, double cross, double eta,
                                    double w) {
  const double px = (w / eta) * dx_sq, py = (1.0 / (eta * w)) * dy_sq;
  const double msq = px + py + 2.0 * cross;
  if (!(msq < 0.0)) return std::sqrt(msq);
  const double scale = px + py + 2.0 * std::abs(cross);
  if (msq < -1e-12 * std::max(1.0, scale))
    throw std::domain_error(
        "residual metric is not positive semidefinite; step size exceeds 1/||A||");
  return 0.0;
}

}  // namespace detail

// ||T(z) - z||_M from the carried products (reference solver.hpp:267-289).
inline double m_norm_residual(std::span<const double> x, std::span<const double> y,
                              std::span<const double> xt, std::span<const double> yt,
                              std::span<const double> ax, std::span<const double> axt,
                              double eta, double w) {
  double sx = 0.0;
  for (std::size_t j = 0; j < x.size(); ++j) {
    const double d = xt[j] - x[j];
    sx += d * d;
  }
  double sy = 0.0, cr = 0.0;
  for (std::size_t i = 0; i < y.size(); ++i) {
    const double d = yt[i] - y[i];
    sy += d * d;
    cr += d * (axt[i] - ax[i]);
  }
  return detail::m_residual_from_terms(sx, sy, cr, eta, w);
}

// z <- alpha (2 t - z) + (1 - alpha) anchor (reference solver.hpp:291-297;
// fused into k_primal / k_dual as the speculative Halpern buffer).
inline void halpern_combine(double alpha, std::span<const double> t_out,
                            std::span<const double> anchor, std::span<double> z) {
  const double keep = 1.0 - alpha;
  for (std::size_t k = 0; k < z.size(); ++k)
    z[k] = alpha * (2.0 * t_out[k] - z[k]) + keep * anchor[k];
}

// Reference solver.hpp:336-354.
struct OptimalityReport {
  double objective = 0.0;
  double bound_support = 0.0;
  double row_support = 0.0;
  double gap = kInf;
  double primal_residual = kInf;
  double dual_residual = kInf;
  bool gap_ok = false;
  bool primal_ok = false;
  bool dual_ok = false;
  double score = kInf;

  bool optimal() const { return gap_ok && primal_ok && dual_ok; }
  double dual_objective() const { return -(bound_support + row_support); }
};

// The three optimality tests at a candidate (reference solver.hpp:356-416);
// k_check (column space) and k_dual<CHECK> (row space) accumulate the same
// sums per LP column. at_yt = A'yt is an input, as in the reference.
inline OptimalityReport evaluate_optimality(const ColumnView& col, std::span<const double> xt,
                                            std::span<const double> yt,
                                            std::span<const double> axt,
                                            std::span<const double> at_yt,
                                            std::span<double> reduced_out, double eps,
                                            double eps_dual, bool robust_bound_contribution) {
  const LpProblem& p = col.problem();
  const int n = p.num_cols(), m = p.num_rows();
  double obj = 0.0, cc_sum = 0.0, dviol = 0.0, sup_r = 0.0;
  for (int j = 0; j < n; ++j) {
    const double c = col.cost(j), lo = col.lower(j), hi = col.upper(j);
    obj += c * xt[j];
    cc_sum += c * c;
    const double g = -c - at_yt[j];
    const double r = project_barrier_cone(g, lo, hi);
    reduced_out[j] = r;
    const double v = c + at_yt[j] + r;
    dviol += v * v;
    if (!robust_bound_contribution) {
      sup_r += support_term(r, lo, hi);
    } else if (g > 0.0 && hi != kInf) {
      sup_r += hi * g;
    } else if (g < 0.0 && lo != -kInf) {
      sup_r += lo * g;
    }
  }
  double sup_y = 0.0, pviol = 0.0, ax_sq = 0.0;
  for (int i = 0; i < m; ++i) {
    const double lo = p.row_bounds.lower[i], hi = p.row_bounds.upper[i];
    sup_y += support_term(yt[i], lo, hi);
    const double v = axt[i] - project_box(axt[i], lo, hi);
    pviol += v * v;
    ax_sq += axt[i] * axt[i];
  }
  OptimalityReport rep;
  rep.objective = obj;
  rep.bound_support = sup_r;
  rep.row_support = sup_y;
  rep.primal_residual = std::sqrt(pviol);
  rep.dual_residual = std::sqrt(dviol);
  const double supports = sup_r + sup_y;
  const double gap = obj + supports;
  const double gap_scale = 1.0 + std::abs(obj) + std::abs(supports);
  const double primal_scale = 1.0 + std::sqrt(ax_sq);
  const double dual_scale = 1.0 + std::sqrt(cc_sum);
  const bool finite_gap = std::isfinite(gap);
  rep.gap = finite_gap ? std::abs(gap) : kInf;
  rep.gap_ok = finite_gap && std::abs(gap) <= eps * gap_scale;
  rep.primal_ok = rep.primal_residual <= eps * primal_scale;
  rep.dual_ok = rep.dual_residual <= eps_dual * dual_scale;
  rep.score = std::max({rep.gap / gap_scale, rep.primal_residual / primal_scale,
                        rep.dual_residual / dual_scale});
  return rep;
}

enum class CertificateKind { kNone, kPrimal, kDual };

// Scratch of check_infeasibility_probe (reference solver.hpp:420-423).
struct CertificateWorkspace {
  std::vector<double> reduced_current, delta_r, delta_y, at_delta_y;
};

// Primal certificate from the displacement (dy, dr), then the dual ray from
// dx (reference solver.hpp:425-527); the conditional A'dy runs on the device
// (k_cert does the same for the flagged columns of a batch).
inline CertificateKind check_infeasibility_probe(
    const ColumnView& col, const CsrView& at, std::span<const double> x,
    std::span<const double> y, std::span<const double> xt, std::span<const double> yt,
    std::span<const double> aty, std::span<const double> ax, std::span<const double> axt,
    std::span<const double> reduced_candidate, double eps, CertificateWorkspace& ws,
    InfeasibilityProbe* out, std::int64_t* product_count) {
  const LpProblem& p = col.problem();
  const int n = p.num_cols(), m = p.num_rows();
  const Bounds& rows = p.row_bounds;
  ws.reduced_current.resize(n);
  ws.delta_r.resize(n);
  ws.delta_y.resize(m);
  for (int i = 0; i < m; ++i)
    ws.delta_y[i] = project_barrier_cone(yt[i] - y[i], rows.lower[i], rows.upper[i]);
  for (int j = 0; j < n; ++j) {
    const double lo = col.lower(j), hi = col.upper(j);
    const double cur = project_barrier_cone(-col.cost(j) - aty[j], lo, hi);
    ws.reduced_current[j] = cur;
    ws.delta_r[j] = project_barrier_cone(reduced_candidate[j] - cur, lo, hi);
  }
  auto record = [&](bool primal) {
    if (out == nullptr) return;
    out->delta_x.assign(n, 0.0);
    for (int j = 0; j < n; ++j) out->delta_x[j] = xt[j] - x[j];
    if (primal) {
      out->delta_y = ws.delta_y;
      out->delta_r = ws.delta_r;
    } else {
      out->delta_y.clear();
      out->delta_r.clear();
    }
  };

  // support sum of the displacement, tested against its own cancellation
  // scale (a raw sign test would certify rounding noise)
  double sup = 0.0, sup_scale = 0.0;
  for (int i = 0; i < m; ++i) {
    const double t = support_term(ws.delta_y[i], rows.lower[i], rows.upper[i]);
    sup += t;
    sup_scale += std::abs(t);
  }
  for (int j = 0; j < n; ++j) {
    const double t = support_term(ws.delta_r[j], col.lower(j), col.upper(j));
    sup += t;
    sup_scale += std::abs(t);
  }
  if (sup < -1e-9 * std::max(1.0, sup_scale)) {
    ws.at_delta_y.resize(n);
    csr_apply(at, ws.delta_y.data(), ws.at_delta_y.data());
    if (product_count != nullptr) ++*product_count;
    double res = 0.0;
    for (int j = 0; j < n; ++j) {
      const double v = ws.at_delta_y[j] + ws.delta_r[j];
      res += v * v;
    }
    if (std::sqrt(res) <= eps * std::abs(sup)) {
      record(true);
      return CertificateKind::kPrimal;
    }
  }

  double descent = 0.0, descent_scale = 0.0;
  for (int j = 0; j < n; ++j) {
    const double t = col.cost(j) * (xt[j] - x[j]);
    descent += t;
    descent_scale += std::abs(t);
  }
  if (!(descent < -1e-9 * std::max(1.0, descent_scale))) return CertificateKind::kNone;
  double var_res = 0.0;
  for (int j = 0; j < n; ++j) {
    const double dx = xt[j] - x[j];
    const double v = dx - project_recession_cone(dx, col.lower(j), col.upper(j));
    var_res += v * v;
  }
  double row_res = 0.0;
  for (int i = 0; i < m; ++i) {
    const double adx = axt[i] - ax[i];
    const double v = adx - project_recession_cone(adx, rows.lower[i], rows.upper[i]);
    row_res += v * v;
  }
  const double budget = eps * std::abs(descent);
  if (std::sqrt(var_res) <= budget && std::sqrt(row_res) <= budget) {
    record(false);
    return CertificateKind::kDual;
  }
  return CertificateKind::kNone;
}

namespace detail {

// Lowest-score candidate so far (reference solver.hpp:535-554); the batch
// kernels keep the same snapshot per LP column on the device.
struct BestCandidate {
  double score = kInf;
  std::vector<double> x, y, reduced;
  OptimalityReport report;
  double fixed_point = kInf;

  void offer(const OptimalityReport& rep, double fixed_point_residual,
             std::span<const double> xt, std::span<const double> yt,
             std::span<const double> r) {
    if (!(rep.score < score)) return;
    score = rep.score;
    report = rep;
    fixed_point = fixed_point_residual;
    x.assign(xt.begin(), xt.end());
    y.assign(yt.begin(), yt.end());
    reduced.assign(r.begin(), r.end());
  }
};

inline Residuals residuals_of(const OptimalityReport& rep, double fixed_point) {
  Residuals out;
  out.gap = rep.gap;
  out.primal = rep.primal_residual;
  out.dual = rep.dual_residual;
  out.fixed_point = fixed_point;
  return out;
}

}  // namespace detail

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
