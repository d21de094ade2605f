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

#include <algorithm>
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

// One LP's record -> SolveResult; vectors fetched from `ctx` at the
// context-local column `local` when the solve kept them.
inline SolveResult from_record(cuda::Context& ctx, const bl_column_result& s, int local, int n,
                               int m) {
  SolveResult r;
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
    cuda::check(ctx.handle(), bl_fetch_solution(ctx.handle(), local, r.x.data(), r.y.data(),
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
                bl_fetch_certificate(ctx.handle(), local, cert.delta_x.data(),
                                     cert.delta_y.empty() ? nullptr : cert.delta_y.data(),
                                     cert.delta_r.empty() ? nullptr : cert.delta_r.data()));
  }
  return r;
}

inline std::vector<RestartEvent> fetch_log(cuda::Context& ctx, const bl_summary& sum) {
  std::vector<RestartEvent> out;
  if (sum.restart_log_size <= 0) return out;
  std::vector<bl_restart_event> ev(static_cast<std::size_t>(sum.restart_log_size));
  std::int32_t got = 0;
  cuda::check(ctx.handle(), bl_fetch_restart_log(ctx.handle(), ev.data(),
                                                 static_cast<std::int32_t>(ev.size()), &got));
  out.reserve(static_cast<std::size_t>(got));
  for (std::int32_t k = 0; k < got; ++k)
    out.push_back(RestartEvent{ev[k].at_iteration, static_cast<RestartReason>(ev[k].reason),
                               ev[k].residual, ev[k].anchor_residual});
  return out;
}

inline std::vector<bl_override> override_table(const BatchProblem& batch) {
  std::vector<bl_override> table;
  table.reserve(batch.all_overrides().size());
  for (const ColumnOverride& o : batch.all_overrides())
    table.push_back(bl_override{o.column, static_cast<std::int32_t>(o.kind), o.variable, 0,
                                o.value});
  return table;
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
  const std::vector<bl_override> table = override_table(batch);
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
  for (int j = 0; j < width; ++j)
    if (!is_preset[j]) run.results[j] = from_record(ctx, raw[j], j, n, m);
  run.restart_log = fetch_log(ctx, run.summary);
  run.profile.resize(16);
  std::int32_t kinds = 0;
  cuda::check(ctx.handle(), bl_fetch_profile(ctx.handle(), run.profile.data(), 16, &kinds));
  run.profile.resize(static_cast<std::size_t>(kinds));
  return run;
}

// The batch sharded over several contexts (bl_solve_batch_sharded, SURVEY
// §8(e)): each context holds its own replica of the problem and solves one
// contiguous column slice; per-LP records land in original column order.
// The merged summary: iterations = the longest shard, restarts and sparse
// products summed, the restart logs concatenated in shard order, the
// trajectory hash folded over the shards' hashes.
inline DeviceRun run_sharded(std::span<cuda::Context* const> ctxs, const BatchProblem& batch,
                             const SolverConfig& cfg, std::span<const int> preset_columns,
                             std::span<const double> initial_weights, int vectors) {
  const LpProblem& base = batch.base();
  const int width = batch.batch_width();
  const int n = base.num_cols(), m = base.num_rows();
  const int G = static_cast<int>(ctxs.size());
  std::vector<bl_ctx*> handles;
  std::vector<bl_problem*> probs;
  for (cuda::Context* c : ctxs) {
    handles.push_back(c->handle());
    probs.push_back(c->resident(base.A, base.objective, base.var_bounds.lower,
                                base.var_bounds.upper, base.row_bounds.lower,
                                base.row_bounds.upper));
  }
  const std::vector<bl_override> table = override_table(batch);
  std::vector<std::int32_t> presets(preset_columns.begin(), preset_columns.end());
  const bl_config c = to_abi(cfg, vectors);
  std::vector<bl_summary> sums(static_cast<std::size_t>(G));
  std::vector<bl_column_result> raw(static_cast<std::size_t>(width > 0 ? width : 1));
  cuda::check(handles[0],
              bl_solve_batch_sharded(handles.data(), probs.data(), G, width,
                                     static_cast<std::int32_t>(batch.objective_mode()),
                                     table.data(), static_cast<std::int32_t>(table.size()), &c,
                                     presets.empty() ? nullptr : presets.data(),
                                     static_cast<std::int32_t>(presets.size()),
                                     initial_weights.empty() ? nullptr : initial_weights.data(),
                                     sums.data(), raw.data()));
  DeviceRun run;
  run.summary.trajectory_hash = 1469598103934665603ull;
  if (width == 0) return run;
  std::vector<char> is_preset(static_cast<std::size_t>(width), 0);
  for (int col : preset_columns) is_preset[col] = 1;
  run.results.resize(static_cast<std::size_t>(width));
  for (int s = 0, b = 0; s < G; ++s) {
    const int w = width / G + (s < width % G ? 1 : 0);
    for (int j = b; j < b + w; ++j)
      if (!is_preset[j]) run.results[j] = from_record(*ctxs[s], raw[j], j - b, n, m);
    const bl_summary& q = sums[s];
    run.summary.iterations = std::max(run.summary.iterations, q.iterations);
    run.summary.restarts += q.restarts;
    run.summary.sparse_products += q.sparse_products;
    run.summary.device_ms = std::max(run.summary.device_ms, q.device_ms);
    run.summary.kernel_launches += q.kernel_launches;
    run.summary.loop_passes = std::max(run.summary.loop_passes, q.loop_passes);
    run.summary.eta = q.eta;
    run.summary.trajectory_hash =
        G == 1 ? q.trajectory_hash : (run.summary.trajectory_hash ^ q.trajectory_hash) * 1099511628211ull;
    std::vector<RestartEvent> log = fetch_log(*ctxs[s], q);
    run.restart_log.insert(run.restart_log.end(), log.begin(), log.end());
    b += w;
  }
  run.summary.restart_log_size = static_cast<std::int32_t>(run.restart_log.size());
  return run;
}

}  // namespace batchlp::detail

#endif  // BATCHLP_B200_DETAIL_DEVICE_SOLVE_HPP
