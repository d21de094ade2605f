// batchlp/detail/device_solve.hpp — one batched solve through the C-ABI.
//
// Shared by solve() and solve_batch(): uploads (or reuses) the problem in
// HBM, marshals the override table, presets, initial weights and warm start
// into bl_solve_batch (include/batchlp_cuda.h), and turns the per-LP
// bl_column_result records back into SolveResult values in original column
// order, copying x / y / r and certificates back only as requested.
// Included by solver.hpp after the value types are declared.
#ifndef BATCHLP_B200_DETAIL_DEVICE_SOLVE_HPP
#define BATCHLP_B200_DETAIL_DEVICE_SOLVE_HPP

#include <cstdint>
#include <span>
#include <vector>

#include "batchlp/device.hpp"
#include "batchlp/problem.hpp"

namespace batchlp::detail {

struct DeviceRun {
  bl_summary summary{};
  std::vector<SolveResult> results;       // width entries; presets left default
  std::vector<RestartEvent> restart_log;
  std::vector<bl_kernel_stat> profile;    // in-situ kernel timing of the solve
};

inline bl_config to_abi(const SolverConfig& cfg, int vectors) {
  bl_config c;
  bl_config_default(&c);
  c.eps_opt = cfg.eps_opt;
  c.eps_infeas = cfg.eps_infeas;
  c.eps_dual = cfg.eps_dual;
  c.theta = cfg.theta;
  c.beta_sufficient = cfg.beta_sufficient;
  c.beta_necessary = cfg.beta_necessary;
  c.beta_artificial = cfg.beta_artificial;
  c.max_iterations = cfg.max_iterations;
  c.termination_check_period = cfg.termination_check_period;
  c.w_init = cfg.w_init;
  c.robust_bound_contribution = cfg.robust_bound_contribution ? 1 : 0;
  c.average_over_all_columns = cfg.average_over_all_columns ? 1 : 0;
  c.trace_iterates = cfg.trace_iterates ? 1 : 0;
  c.vectors = vectors;
  return c;
}

inline DeviceRun run_on_device(cuda::Context& ctx, const BatchProblem& batch,
                               const SolverConfig& cfg, std::span<const int> preset_columns,
                               std::span<const double> initial_weights, const WarmStart* warm,
                               int vectors) {
  const LpProblem& base = batch.base();
  const int width = batch.batch_width();
  const int n = base.num_cols(), m = base.num_rows();
  bl_problem* p = ctx.resident(base.A, base.objective, base.var_bounds.lower,
                               base.var_bounds.upper, base.row_bounds.lower,
                               base.row_bounds.upper);
  std::vector<bl_override> table;
  table.reserve(batch.all_overrides().size());
  for (const ColumnOverride& o : batch.all_overrides())
    table.push_back(bl_override{o.column, static_cast<std::int32_t>(o.kind), o.variable, 0,
                                o.value});
  std::vector<std::int32_t> presets(preset_columns.begin(), preset_columns.end());
  std::vector<double> wx, wy;
  if (warm != nullptr) {  // one column (solve): the ABI takes width x n / width x m
    wx = warm->x;
    wy = warm->y;
  }
  const bl_config c = to_abi(cfg, vectors);
  DeviceRun run;
  std::vector<bl_column_result> raw(static_cast<std::size_t>(width > 0 ? width : 1));
  cuda::check(ctx.handle(),
              bl_solve_batch(ctx.handle(), p, width, static_cast<std::int32_t>(batch.objective_mode()),
                             table.data(), static_cast<std::int32_t>(table.size()), &c,
                             presets.empty() ? nullptr : presets.data(),
                             static_cast<std::int32_t>(presets.size()),
                             initial_weights.empty() ? nullptr : initial_weights.data(),
                             warm ? wx.data() : nullptr, warm ? wy.data() : nullptr,
                             &run.summary, raw.data()));
  if (width == 0) return run;

  std::vector<char> is_preset(static_cast<std::size_t>(width), 0);
  for (int col : preset_columns) is_preset[col] = 1;
  run.results.resize(static_cast<std::size_t>(width));
  for (int j = 0; j < width; ++j) {
    if (is_preset[j]) continue;
    const bl_column_result& s = raw[j];
    SolveResult& r = run.results[j];
    r.status = static_cast<SolveStatus>(s.status);
    r.objective = s.objective;
    r.residuals = Residuals{s.gap, s.primal, s.dual, s.fixed_point};
    r.iterations = s.iterations;
    r.restarts = s.restarts;
    r.device.valid = true;
    r.device.vectors_exist = s.vectors_exist != 0;
    r.device.bound_support = s.bound_support;
    r.device.row_support = s.row_support;
    r.device.base_bound_support = s.base_bound_support;
    if (s.has_solution) {
      r.x.resize(n);
      r.y.resize(m);
      r.reduced_costs.resize(n);
      cuda::check(ctx.handle(), bl_fetch_solution(ctx.handle(), j, r.x.data(), r.y.data(),
                                                  r.reduced_costs.data()));
    }
    if (s.has_certificate) {
      InfeasibilityProbe& cert = r.certificate;
      cert.delta_x.resize(n);
      if (s.certificate_kind == 1) {
        cert.delta_y.resize(m);
        cert.delta_r.resize(n);
      }
      cuda::check(ctx.handle(),
                  bl_fetch_certificate(ctx.handle(), j, cert.delta_x.data(),
                                       cert.delta_y.empty() ? nullptr : cert.delta_y.data(),
                                       cert.delta_r.empty() ? nullptr : cert.delta_r.data()));
    }
  }
  if (run.summary.restart_log_size > 0) {
    std::vector<bl_restart_event> ev(static_cast<std::size_t>(run.summary.restart_log_size));
    std::int32_t got = 0;
    cuda::check(ctx.handle(), bl_fetch_restart_log(ctx.handle(), ev.data(),
                                                   static_cast<std::int32_t>(ev.size()), &got));
    run.restart_log.reserve(static_cast<std::size_t>(got));
    for (std::int32_t k = 0; k < got; ++k)
      run.restart_log.push_back(RestartEvent{ev[k].at_iteration,
                                             static_cast<RestartReason>(ev[k].reason),
                                             ev[k].residual, ev[k].anchor_residual});
  }
  run.profile.resize(16);
  std::int32_t kinds = 0;
  cuda::check(ctx.handle(), bl_fetch_profile(ctx.handle(), run.profile.data(), 16, &kinds));
  run.profile.resize(static_cast<std::size_t>(kinds));
  return run;
}

}  // namespace batchlp::detail

#endif  // BATCHLP_B200_DETAIL_DEVICE_SOLVE_HPP
