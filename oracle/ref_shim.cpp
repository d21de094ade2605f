// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (never shipped, never timed
// as the product).
//
// A C-ABI shim over the UNMODIFIED reference headers, compiled from where they
// lie under /root/reference/proj/include by oracle/Makefile into
// oracle/_ref/libbatchlp_ref.so. It lets the parity tests (tests/), smoke()
// and bench.py's cpu_baseline / --impl reference legs run the reference's own
// solve_batch / solve / run_fsb / run_obbt on exactly the arrays the CUDA path
// receives. Nothing here re-implements the algorithm; every entry forwards to
// the reference function named in its comment.
//
// Structs are the ones of include/batchlp_cuda.h so results compare field by
// field.

#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "batchlp/batch_solver.hpp"
#include "batchlp/generators.hpp"
#include "batchlp/obbt.hpp"
#include "batchlp/oracle.hpp"
#include "batchlp/problem.hpp"
#include "batchlp/solver.hpp"
#include "batchlp/sparse.hpp"
#include "batchlp/strong_branching.hpp"
#include "support/instances.hpp"

#include "batchlp_cuda.h"

using namespace batchlp;

namespace {

thread_local std::string g_error;

int fail(int code, const char* what) {
  g_error = what;
  return code;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return BL_OK;
  } catch (const std::out_of_range& e) {
    return fail(BL_ERR_OUT_OF_RANGE, e.what());
  } catch (const std::domain_error& e) {
    return fail(BL_ERR_DOMAIN, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(BL_ERR_INVALID_ARGUMENT, e.what());
  } catch (const std::logic_error& e) {
    return fail(BL_ERR_LOGIC, e.what());
  } catch (const std::exception& e) {
    return fail(BL_ERR_CUDA, e.what());
  }
}

SolverConfig to_cfg(const bl_config* c) {
  SolverConfig s;
  if (c == nullptr) return s;
  s.eps_opt = c->eps_opt;
  s.eps_infeas = c->eps_infeas;
  s.eps_dual = c->eps_dual;
  s.theta = c->theta;
  s.beta_sufficient = c->beta_sufficient;
  s.beta_necessary = c->beta_necessary;
  s.beta_artificial = c->beta_artificial;
  s.max_iterations = c->max_iterations;
  s.termination_check_period = c->termination_check_period;
  s.w_init = c->w_init;
  s.robust_bound_contribution = c->robust_bound_contribution != 0;
  s.average_over_all_columns = c->average_over_all_columns != 0;
  s.trace_iterates = c->trace_iterates != 0;
  return s;
}

double support_sum(std::span<const double> v, const std::vector<double>& lo,
                   const std::vector<double>& hi) {
  double t = 0.0;
  for (std::size_t i = 0; i < v.size(); ++i) t += support_term(v[i], lo[i], hi[i]);
  return t;
}

// Copies one SolveResult into the C structs / column-major blocks.
void export_result(const LpProblem& base, const ColumnView& view,
                   const SolveResult& r, int j, bl_column_result* out,
                   double* x, double* y, double* red) {
  const int n = base.num_cols();
  const int m = base.num_rows();
  bl_column_result& o = out[j];
  std::memset(&o, 0, sizeof(o));
  o.status = static_cast<int32_t>(r.status);
  o.restarts = r.restarts;
  o.iterations = r.iterations;
  o.objective = r.objective;
  o.gap = r.residuals.gap;
  o.primal = r.residuals.primal;
  o.dual = r.residuals.dual;
  o.fixed_point = r.residuals.fixed_point;
  o.has_solution = r.x.empty() ? 0 : 1;
  o.vectors_exist = o.has_solution;
  o.certificate_kind = r.certificate.delta_x.empty()
                           ? 0
                           : (r.certificate.delta_y.empty() ? 2 : 1);
  o.has_certificate = o.certificate_kind != 0;
  if (!r.reduced_costs.empty()) {
    double sr = 0.0;
    for (int i = 0; i < n; ++i)
      sr += support_term(r.reduced_costs[i], view.lower(i), view.upper(i));
    o.bound_support = sr;
    o.base_bound_support = support_sum(r.reduced_costs, base.var_bounds.lower,
                                       base.var_bounds.upper);
  }
  if (!r.y.empty())
    o.row_support = support_sum(r.y, base.row_bounds.lower, base.row_bounds.upper);
  if (x && !r.x.empty()) std::memcpy(x + static_cast<std::size_t>(j) * n, r.x.data(), n * 8);
  if (y && !r.y.empty()) std::memcpy(y + static_cast<std::size_t>(j) * m, r.y.data(), m * 8);
  if (red && !r.reduced_costs.empty())
    std::memcpy(red + static_cast<std::size_t>(j) * n, r.reduced_costs.data(), n * 8);
}

void export_log(const std::vector<RestartEvent>& log, bl_restart_event* out,
                int32_t cap) {
  if (out == nullptr) return;
  for (std::size_t i = 0; i < log.size() && static_cast<int32_t>(i) < cap; ++i) {
    out[i].at_iteration = log[i].at_iteration;
    out[i].reason = static_cast<int32_t>(log[i].reason);
    out[i].reserved = 0;
    out[i].residual = log[i].residual;
    out[i].anchor_residual = log[i].anchor_residual;
  }
}

LpProblem from_arrays(int32_t m, int32_t n, int64_t nnz, const int32_t* rowptr,
                      const int32_t* col, const double* val, const double* c,
                      const double* xl, const double* xu, const double* rl,
                      const double* ru) {
  std::vector<Triplet> t;
  t.reserve(static_cast<std::size_t>(nnz));
  for (int r = 0; r < m; ++r)
    for (int q = rowptr[r]; q < rowptr[r + 1]; ++q) t.push_back({r, col[q], val[q]});
  LpProblem p;
  p.A = SparseMatrix::from_triplets(std::move(t), m, n);
  p.objective.assign(c, c + n);
  p.var_bounds.lower.assign(xl, xl + n);
  p.var_bounds.upper.assign(xu, xu + n);
  p.row_bounds.lower.assign(rl, rl + m);
  p.row_bounds.upper.assign(ru, ru + m);
  return p;
}

std::vector<ColumnOverride> to_overrides(const bl_override* ov, int32_t n_ov) {
  std::vector<ColumnOverride> out;
  for (int i = 0; i < n_ov; ++i)
    out.push_back({ov[i].column, static_cast<OverrideKind>(ov[i].kind),
                   ov[i].variable, ov[i].value});
  return out;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_error.c_str(); }

// ---- problem handles ------------------------------------------------------
void* ref_lp_create(int32_t m, int32_t n, int64_t nnz, const int32_t* rowptr,
                    const int32_t* col, const double* val, const double* c,
                    const double* xl, const double* xu, const double* rl,
                    const double* ru) {
  LpProblem* p = nullptr;
  if (guarded([&] {
        p = new LpProblem(from_arrays(m, n, nnz, rowptr, col, val, c, xl, xu, rl, ru));
      }) != BL_OK)
    return nullptr;
  return p;
}

void ref_lp_free(void* h) { delete static_cast<LpProblem*>(h); }

void ref_lp_dims(void* h, int32_t* m, int32_t* n, int64_t* nnz) {
  const LpProblem& p = *static_cast<LpProblem*>(h);
  *m = p.num_rows();
  *n = p.num_cols();
  *nnz = p.A.nnz();
}

// Copies A, A' and the vectors out (buffers sized from ref_lp_dims).
void ref_lp_export(void* h, int32_t* rowptr, int32_t* col, double* val,
                   int32_t* t_rowptr, int32_t* t_col, double* t_val, double* c,
                   double* xl, double* xu, double* rl, double* ru) {
  const LpProblem& p = *static_cast<LpProblem*>(h);
  const CsrView a = p.A.view(), at = p.A.transpose_view();
  std::copy(a.offsets.begin(), a.offsets.end(), rowptr);
  std::copy(a.cols.begin(), a.cols.end(), col);
  std::copy(a.values.begin(), a.values.end(), val);
  std::copy(at.offsets.begin(), at.offsets.end(), t_rowptr);
  std::copy(at.cols.begin(), at.cols.end(), t_col);
  std::copy(at.values.begin(), at.values.end(), t_val);
  std::copy(p.objective.begin(), p.objective.end(), c);
  std::copy(p.var_bounds.lower.begin(), p.var_bounds.lower.end(), xl);
  std::copy(p.var_bounds.upper.begin(), p.var_bounds.upper.end(), xu);
  std::copy(p.row_bounds.lower.begin(), p.row_bounds.lower.end(), rl);
  std::copy(p.row_bounds.upper.begin(), p.row_bounds.upper.end(), ru);
}

// generate_set_cover, generators.hpp:76-109.
void* ref_gen_set_cover(int32_t rows, int32_t cols, double density, uint64_t seed) {
  LpProblem* p = nullptr;
  if (guarded([&] {
        p = new LpProblem(generate_set_cover(rows, cols, density, seed).problem);
      }) != BL_OK)
    return nullptr;
  return p;
}

// generate_comb_auction / generate_max_ind_set / generate_facility_location
// (generators.hpp), for the acceptance-3 style FSB cases.
void* ref_gen_family(int32_t family, int32_t a, int32_t b, int32_t c, uint64_t seed,
                     int32_t* integer_cols, int32_t* n_integer) {
  LpProblem* p = nullptr;
  if (guarded([&] {
        GeneratedInstance g;
        switch (family) {
          case 0: g = generate_set_cover(a, b, c / 100.0, seed); break;
          case 1: g = generate_comb_auction(a, b, seed); break;
          case 2: g = generate_max_ind_set(a, b, seed); break;
          default: g = generate_facility_location(a, b, c, seed); break;
        }
        if (integer_cols)
          std::copy(g.integer_columns.begin(), g.integer_columns.end(), integer_cols);
        if (n_integer) *n_integer = static_cast<int32_t>(g.integer_columns.size());
        p = new LpProblem(std::move(g.problem));
      }) != BL_OK)
    return nullptr;
  return p;
}

// testsupport fixtures (tests/support/instances.hpp): shape 0 feasible,
// 1 primal infeasible, 2 dual infeasible; 10 two_var_lp, 11 knapsack_lp.
void* ref_test_lp(int32_t shape, uint64_t seed) {
  LpProblem* p = nullptr;
  if (guarded([&] {
        switch (shape) {
          case 10: p = new LpProblem(testsupport::two_var_lp()); break;
          case 11: p = new LpProblem(testsupport::knapsack_lp()); break;
          default:
            p = new LpProblem(testsupport::random_lp(
                static_cast<testsupport::Shape>(shape), seed));
        }
      }) != BL_OK)
    return nullptr;
  return p;
}

// append_cutoff_row, problem.hpp:104-122.
void* ref_append_cutoff(void* h, double alpha) {
  LpProblem* p = nullptr;
  if (guarded([&] {
        p = new LpProblem(append_cutoff_row(*static_cast<LpProblem*>(h), alpha));
      }) != BL_OK)
    return nullptr;
  return p;
}

// ---- sparse ---------------------------------------------------------------
// spectral_norm, sparse.hpp:297-319.
int ref_spectral_norm(void* h, double* out) {
  return guarded([&] { *out = spectral_norm(static_cast<LpProblem*>(h)->A); });
}

// spmm, sparse.hpp:213-238 (column-major blocks, `width` columns).
int ref_spmm(void* h, int transpose, int32_t width, int32_t active,
             const double* x, double* out) {
  return guarded([&] {
    const SparseMatrix& a = static_cast<LpProblem*>(h)->A;
    const int rin = transpose ? a.n_rows() : a.n_cols();
    const int rout = transpose ? a.n_cols() : a.n_rows();
    DenseColumnBlock X(rin, width), O(rout, width);
    std::memcpy(X.data().data(), x, sizeof(double) * rin * width);
    std::memcpy(O.data().data(), out, sizeof(double) * rout * width);
    spmm(a, X, O, transpose != 0, active);
    std::memcpy(out, O.data().data(), sizeof(double) * rout * width);
  });
}

// ---- solvers --------------------------------------------------------------
// solve_batch, batch_solver.hpp:78-355. cutoff_set != 0 builds the batch with
// BatchProblem's cutoff row (problem.hpp:152). Preset results are default
// SolveResults with the given status/objective.
int ref_solve_batch(void* h, int32_t width, int32_t mode, const bl_override* ov,
                    int32_t n_ov, int32_t cutoff_set, double cutoff,
                    const bl_config* cfg, const int32_t* preset_cols,
                    const int32_t* preset_status, const double* preset_obj,
                    int32_t n_presets, const double* initial_weights,
                    bl_summary* summary, bl_column_result* results, double* x,
                    double* y, double* red, bl_restart_event* log,
                    int32_t log_cap) {
  return guarded([&] {
    const LpProblem& p = *static_cast<LpProblem*>(h);
    std::optional<double> co;
    if (cutoff_set) co = cutoff;
    BatchProblem batch(p, width, static_cast<ObjectiveMode>(mode),
                       to_overrides(ov, n_ov), co);
    std::vector<PresetColumn> presets;
    for (int i = 0; i < n_presets; ++i) {
      SolveResult r;
      r.status = static_cast<SolveStatus>(preset_status ? preset_status[i] : 1);
      if (preset_obj) r.objective = preset_obj[i];
      presets.push_back({preset_cols[i], r});
    }
    std::span<const double> w0;
    if (initial_weights) w0 = {initial_weights, static_cast<std::size_t>(width)};
    const BatchSolveSummary s = solve_batch(batch, to_cfg(cfg), presets, nullptr, w0);
    if (summary) {
      summary->iterations = s.iterations;
      summary->restarts = s.restarts;
      summary->restart_log_size = static_cast<int32_t>(s.restart_log.size());
      summary->sparse_products = s.sparse_products;
      summary->trajectory_hash = s.trajectory_hash;
      summary->eta = step_size_for(batch.base().A);
      summary->device_ms = 0.0;
    }
    for (int j = 0; j < width; ++j)
      export_result(batch.base(), resolve_column(batch, j), s.per_problem[j], j,
                    results, x, y, red);
    export_log(s.restart_log, log, log_cap);
  });
}

// solve, solver.hpp:569-703 (warm_x / warm_y may be NULL).
int ref_solve(void* h, const bl_config* cfg, const double* warm_x,
              const double* warm_y, bl_summary* summary, bl_column_result* result,
              double* x, double* y, double* red, bl_restart_event* log,
              int32_t log_cap) {
  return guarded([&] {
    const LpProblem& p = *static_cast<LpProblem*>(h);
    WarmStart ws;
    const WarmStart* wp = nullptr;
    if (warm_x && warm_y) {
      ws.x.assign(warm_x, warm_x + p.num_cols());
      ws.y.assign(warm_y, warm_y + p.num_rows());
      wp = &ws;
    }
    const SolveResult r = solve(p, to_cfg(cfg), wp);
    if (summary) {
      summary->iterations = r.iterations;
      summary->restarts = r.restarts;
      summary->restart_log_size = static_cast<int32_t>(r.restart_log.size());
      summary->sparse_products = r.sparse_products;
      summary->trajectory_hash = r.trajectory_hash;
      summary->eta = step_size_for(p.A);
      summary->device_ms = 0.0;
    }
    export_result(p, ColumnView(p), r, 0, result, x, y, red);
    export_log(r.restart_log, log, log_cap);
  });
}

// Certificate vectors of a single solve (InfeasibilityProbe, solver.hpp:123).
int ref_solve_certificate(void* h, const bl_config* cfg, double* dx, double* dy,
                          double* dr, int32_t* kind) {
  return guarded([&] {
    const LpProblem& p = *static_cast<LpProblem*>(h);
    const SolveResult r = solve(p, to_cfg(cfg));
    const InfeasibilityProbe& c = r.certificate;
    *kind = c.delta_x.empty() ? 0 : (c.delta_y.empty() ? 2 : 1);
    if (!c.delta_x.empty()) std::copy(c.delta_x.begin(), c.delta_x.end(), dx);
    if (!c.delta_y.empty()) std::copy(c.delta_y.begin(), c.delta_y.end(), dy);
    if (!c.delta_r.empty()) std::copy(c.delta_r.begin(), c.delta_r.end(), dr);
  });
}

// run_fsb, strong_branching.hpp:181-185. Per branch j: variable, up/down
// status, objective, iterations, delta, flagged, score.
int ref_run_fsb(void* h, const double* x_rel, const int32_t* frac, int32_t p_count,
                double integrality_tol, const bl_config* cfg, double infeasible_delta,
                int32_t* up_status, int32_t* down_status, double* up_obj,
                double* down_obj, int64_t* up_it, int64_t* down_it,
                double* delta_up, double* delta_down, int32_t* up_flag,
                int32_t* down_flag, double* score, double* root_obj,
                int64_t* iterations, int64_t* sparse_products) {
  return guarded([&] {
    const LpProblem& p = *static_cast<LpProblem*>(h);
    FsbRequest req;
    req.problem = p;
    req.x_rel.assign(x_rel, x_rel + p.num_cols());
    req.fractional_indices.assign(frac, frac + p_count);
    req.integrality_tol = integrality_tol;
    const FsbOutcome o = run_fsb(req, to_cfg(cfg), infeasible_delta);
    *root_obj = o.root_objective;
    *iterations = o.iterations;
    *sparse_products = o.sparse_products;
    for (std::size_t j = 0; j < o.branches.size(); ++j) {
      const FsbBranch& b = o.branches[j];
      up_status[j] = static_cast<int32_t>(b.up_status);
      down_status[j] = static_cast<int32_t>(b.down_status);
      up_obj[j] = b.up_objective;
      down_obj[j] = b.down_objective;
      up_it[j] = b.up_iterations;
      down_it[j] = b.down_iterations;
      delta_up[j] = b.delta_up;
      delta_down[j] = b.delta_down;
      up_flag[j] = b.up_flagged;
      down_flag[j] = b.down_flagged;
      score[j] = b.score;
    }
  });
}

// run_obbt, obbt.hpp:156-223. Per variable: new bounds, changed flags,
// margins, statuses. Scalars: counts, mean reduction, iterations.
int ref_run_obbt(void* h, double eps_opt, double eps_dual, double min_improvement,
                 int64_t max_iterations, int32_t cutoff_set, double cutoff,
                 int32_t lenient, const bl_config* solver, double* new_lower,
                 double* new_upper, int32_t* lower_changed, int32_t* upper_changed,
                 double* lower_margin, double* upper_margin, int32_t* lower_status,
                 int32_t* upper_status, int32_t* counts /* changed, solved, limit */,
                 double* mean_reduction, int64_t* iterations) {
  return guarded([&] {
    const LpProblem& p = *static_cast<LpProblem*>(h);
    ObbtConfig c;
    c.eps_opt = eps_opt;
    c.eps_dual = eps_dual;
    c.min_improvement = min_improvement;
    c.max_iterations = max_iterations;
    if (cutoff_set) c.cutoff = cutoff;
    c.lenient_iteration_limit = lenient != 0;
    c.solver = to_cfg(solver);
    const ObbtOutcome o = run_obbt(p, c);
    for (std::size_t i = 0; i < o.variables.size(); ++i) {
      const ObbtVariable& v = o.variables[i];
      new_lower[i] = v.new_lower;
      new_upper[i] = v.new_upper;
      lower_changed[i] = v.lower_changed;
      upper_changed[i] = v.upper_changed;
      lower_margin[i] = v.lower_margin;
      upper_margin[i] = v.upper_margin;
      lower_status[i] = static_cast<int32_t>(v.lower_status);
      upper_status[i] = static_cast<int32_t>(v.upper_status);
    }
    counts[0] = o.changed_count;
    counts[1] = o.solved_count;
    counts[2] = o.limit_count;
    *mean_reduction = o.mean_reduction_pct;
    *iterations = o.iterations;
  });
}

// oracle_solve (oracle.hpp:164-306): vertex enumeration ground truth for
// n + m <= 16. status: 0 optimal, 1 infeasible, 2 unbounded.
int ref_oracle_solve(void* h, int32_t* status, double* objective, double* vertex) {
  return guarded([&] {
    const LpProblem& p = *static_cast<LpProblem*>(h);
    const OracleResult r = oracle_solve(p);
    *status = static_cast<int32_t>(r.status);
    *objective = r.objective;
    if (vertex && !r.vertex.empty()) std::copy(r.vertex.begin(), r.vertex.end(), vertex);
  });
}

}  // extern "C"
