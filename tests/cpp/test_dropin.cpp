// tests/cpp/test_dropin.cpp — our own tests of the C++ drop-in API
// (include/batchlp/*.hpp over libbatchlp_cuda.so). Run by tests/test_cpp.py.
//
//   dropin_tests                      API cases (doctest shim)
//   dropin_tests --fsb-c1 FILE        C1 strong branching through run_fsb; FILE
//                                     holds "p" then p fractional indices then
//                                     n hex doubles of x_rel (from the golden
//                                     fixture); prints one line per branch
//   dropin_tests --obbt-c2            C2 OBBT batch through solve_batch and
//                                     run_obbt; prints one line per column
//   dropin_tests --write-mps R C D S FILE
//                                     generate_set_cover(R, C, D, S) written
//                                     as MPS (all columns integral)
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "batchlp/batchlp.hpp"
#include "doctest.h"

using namespace batchlp;

namespace {

LpProblem from_instance(bl_instance& in) {
  LpProblem p;
  const int m = in.m, n = in.n;
  p.A = SparseMatrix::from_csr(m, n, std::vector<int>(in.rowptr, in.rowptr + m + 1),
                               std::vector<int>(in.col, in.col + in.nnz),
                               std::vector<double>(in.val, in.val + in.nnz));
  p.objective.assign(in.objective, in.objective + n);
  p.var_bounds.lower.assign(in.var_lower, in.var_lower + n);
  p.var_bounds.upper.assign(in.var_upper, in.var_upper + n);
  p.row_bounds.lower.assign(in.row_lower, in.row_lower + m);
  p.row_bounds.upper.assign(in.row_upper, in.row_upper + m);
  bl_instance_free(&in);
  return p;
}

LpProblem set_cover_c1() {
  bl_instance in{};
  if (bl_gen_set_cover(1000, 2000, 0.01, 1, &in) != 0) std::abort();
  return from_instance(in);
}

LpProblem boxed_c2() {
  bl_instance in{};
  if (bl_gen_boxed_feasible(2000, 2000, 10, 11, &in) != 0) std::abort();
  return from_instance(in);
}

LpProblem tiny_lp() {  // min -x0 - x1, x0 + x1 <= 1, x in [0,1]^2; optimum -1
  LpProblem p;
  p.A = SparseMatrix::from_triplets({{0, 0, 1.0}, {0, 1, 1.0}}, 1, 2);
  p.objective = {-1.0, -1.0};
  p.row_bounds = Bounds(1, Interval{-kInf, 1.0});
  p.var_bounds = Bounds(2, Interval{0.0, 1.0});
  return p;
}

int fsb_c1(const char* path) {
  std::ifstream f(path);
  int p = 0;
  f >> p;
  FsbRequest req;
  req.problem = set_cover_c1();
  req.fractional_indices.resize(p);
  for (int& v : req.fractional_indices) f >> v;
  std::string tok;
  while (f >> tok) req.x_rel.push_back(std::strtod(tok.c_str(), nullptr));
  const FsbOutcome out = run_fsb(req);
  std::printf("iterations %lld\n", static_cast<long long>(out.iterations));
  for (const FsbBranch& b : out.branches)
    std::printf("%d %d %lld %a %d %lld %a\n", b.variable, static_cast<int>(b.up_status),
                static_cast<long long>(b.up_iterations), b.up_objective,
                static_cast<int>(b.down_status), static_cast<long long>(b.down_iterations),
                b.down_objective);
  return 0;
}

int obbt_c2() {
  const LpProblem p = boxed_c2();
  ObbtConfig cfg;
  const ObbtBatch built = build_obbt_batch(p, cfg);
  BatchOptions scalars;
  scalars.vectors = VectorMode::kNone;
  const BatchSolveSummary s =
      solve_batch(built.batch, cfg.solver_config(), built.presets, nullptr, {}, scalars);
  std::printf("iterations %lld restarts %d\n", static_cast<long long>(s.iterations), s.restarts);
  for (const SolveResult& r : s.per_problem)
    std::printf("%d %lld %a\n", static_cast<int>(r.status), static_cast<long long>(r.iterations),
                r.objective);
  const ObbtOutcome o = run_obbt(p, cfg);
  std::printf("obbt changed %d solved %d limit %d\n", o.changed_count, o.solved_count,
              o.limit_count);
  // every variable's tightened box (compared with the reference's run_obbt)
  for (const ObbtVariable& v : o.variables)
    std::printf("%d %d %a %d %a %d %d\n", v.variable, v.lower_changed ? 1 : 0, v.new_lower,
                v.upper_changed ? 1 : 0, v.new_upper, static_cast<int>(v.lower_status),
                static_cast<int>(v.upper_status));
  return 0;
}

}  // namespace

TEST_CASE("solve reaches the known optimum and returns vectors") {
  const SolveResult r = solve(tiny_lp());
  CHECK(r.status == SolveStatus::kOptimal);
  CHECK(r.objective == doctest::Approx(-1.0).epsilon(1e-4));
  CHECK(r.x.size() == 2);
  CHECK(r.y.size() == 1);
  CHECK(r.reduced_costs.size() == 2);
  CHECK(r.device.valid);
  CHECK(r.sparse_products > 0);
}

TEST_CASE("scalar-only batches skip vectors but keep every scalar") {
  const LpProblem p = tiny_lp();
  BatchProblem b(p, 3, ObjectiveMode::kSharedObjective, {});
  BatchOptions none;
  none.vectors = VectorMode::kNone;
  const BatchSolveSummary lean = solve_batch(b, {}, {}, nullptr, {}, none);
  const BatchSolveSummary full = solve_batch(b, {});
  REQUIRE(lean.per_problem.size() == 3);
  for (int j = 0; j < 3; ++j) {
    CHECK(lean.per_problem[j].x.empty());
    CHECK(full.per_problem[j].x.size() == 2);
    CHECK(lean.per_problem[j].status == full.per_problem[j].status);
    CHECK(lean.per_problem[j].iterations == full.per_problem[j].iterations);
    CHECK(lean.per_problem[j].objective == full.per_problem[j].objective);
  }
  CHECK(lean.iterations == full.iterations);
}

TEST_CASE("exceptions keep the reference's types") {
  const LpProblem p = tiny_lp();
  SolverConfig bad;
  bad.theta = 0.0;
  CHECK_THROWS_AS(solve(p, bad), std::invalid_argument);
  BatchProblem b(p, 2, ObjectiveMode::kSharedObjective, {});
  std::vector<PresetColumn> out_of_range(1);
  out_of_range[0].column = 5;
  CHECK_THROWS_AS(solve_batch(b, {}, out_of_range), std::out_of_range);
  std::vector<PresetColumn> dup(2);
  CHECK_THROWS_AS(solve_batch(b, {}, dup), std::invalid_argument);
  std::vector<double> w(3, 1.0);
  CHECK_THROWS_AS(solve_batch(b, {}, {}, nullptr, w), std::invalid_argument);
  CHECK_THROWS_AS(BatchProblem(p, 3, ObjectiveMode::kSignedUnitColumns, {}),
                  std::invalid_argument);
}

TEST_CASE("a workspace is reused across solves of different widths") {
  BatchWorkspace ws;
  const LpProblem p = tiny_lp();
  for (int width : {4, 1, 7}) {
    BatchProblem b(p, width, ObjectiveMode::kSharedObjective, {});
    const BatchSolveSummary s = solve_batch(b, {}, {}, &ws);
    REQUIRE(static_cast<int>(s.per_problem.size()) == width);
    for (const SolveResult& r : s.per_problem) CHECK(r.status == SolveStatus::kOptimal);
  }
}

TEST_CASE("sparse products match a hand product") {
  const SparseMatrix a = SparseMatrix::from_triplets({{0, 0, 2.0}, {1, 0, -1.0}, {1, 1, 3.0}}, 2, 2);
  DenseColumnBlock x(2, 2);
  x.at(0, 0) = 1.0;
  x.at(1, 0) = 2.0;
  x.at(0, 1) = -1.0;
  x.at(1, 1) = 0.5;
  const DenseColumnBlock y = spmm(a, x);
  CHECK(y.at(0, 0) == 2.0);
  CHECK(y.at(1, 0) == 5.0);
  CHECK(y.at(0, 1) == -2.0);
  CHECK(y.at(1, 1) == 2.5);
  const DenseColumnBlock yt = spmm(a, x, true);
  CHECK(yt.at(0, 0) == 0.0);
  CHECK(yt.at(1, 0) == 6.0);
}

TEST_CASE("a batch sharded over two contexts equals its slices solved one by one") {
  // OBBT on a small boxed LP: a signed-unit batch of 2n columns, split in two
  // contiguous slices (BatchOptions::devices = {0, 0}: two contexts, one GPU)
  bl_instance in{};
  REQUIRE(bl_gen_boxed_feasible(120, 150, 6, 3, &in) == 0);
  const LpProblem p = from_instance(in);
  ObbtConfig ocfg;
  const ObbtBatch built = build_obbt_batch(p, ocfg);
  BatchOptions two;
  two.vectors = VectorMode::kSolution;
  two.devices = {0, 0};
  const BatchSolveSummary whole =
      solve_batch(built.batch, ocfg.solver_config(), built.presets, nullptr, {}, two);
  const int width = built.batch.batch_width(), n = p.num_cols();
  REQUIRE(static_cast<int>(whole.per_problem.size()) == width);
  for (int half = 0; half < 2; ++half) {
    const int b = half * (width / 2), e = b + width / 2;
    // the slice as its own batch: signed units rewritten as objective entries
    LpProblem zero = p;
    zero.objective.assign(n, 0.0);
    std::vector<ColumnOverride> ov;
    for (int c = b; c < e; ++c)
      ov.push_back(ColumnOverride{c - b, OverrideKind::kObjectiveEntry, c < n ? c : c - n,
                                  c < n ? 1.0 : -1.0});
    const BatchProblem slice(zero, e - b, ObjectiveMode::kSharedObjective, ov);
    std::vector<PresetColumn> pre;
    for (const PresetColumn& q : built.presets)
      if (q.column >= b && q.column < e) pre.push_back(PresetColumn{q.column - b, q.result});
    BatchOptions one;
    one.vectors = VectorMode::kSolution;
    const BatchSolveSummary s =
        solve_batch(slice, ocfg.solver_config(), pre, nullptr, {}, one);
    for (int j = 0; j < e - b; ++j) {
      const SolveResult& g = whole.per_problem[b + j];
      const SolveResult& w = s.per_problem[j];
      CHECK(g.status == w.status);
      CHECK(g.iterations == w.iterations);
      CHECK(std::memcmp(&g.objective, &w.objective, sizeof(double)) == 0);
      CHECK(g.x == w.x);
    }
  }
}

int write_set_cover_mps(char** argv) {
  bl_instance in{};
  if (bl_gen_set_cover(std::atoi(argv[0]), std::atoi(argv[1]), std::atof(argv[2]),
                       std::strtoull(argv[3], nullptr, 10), &in) != 0)
    return 1;
  const LpProblem p = from_instance(in);
  std::vector<int> ints(static_cast<std::size_t>(p.num_cols()));
  for (int c = 0; c < p.num_cols(); ++c) ints[c] = c;
  std::ofstream out(argv[4]);
  write_mps(out, p, ints, "setcover");
  return out ? 0 : 1;
}

TEST_CASE("MPS round trip keeps every entry, bound and integrality mark") {
  bl_instance in{};
  REQUIRE(bl_gen_boxed_feasible(40, 50, 5, 9, &in) == 0);
  const LpProblem p = from_instance(in);
  std::ostringstream text;
  write_mps(text, p, {1, 2, 7}, "boxed");
  const MpsModel back = parse_mps_string(text.str());
  CHECK(back.name == "boxed");
  CHECK(back.integer_columns == std::vector<int>{1, 2, 7});
  REQUIRE(back.problem.A.nnz() == p.A.nnz());
  const CsrView a = p.A.view(), b = back.problem.A.view();
  for (std::size_t q = 0; q < a.values.size(); ++q) {
    CHECK(a.cols[q] == b.cols[q]);
    CHECK(a.values[q] == b.values[q]);  // %.17g: exact
  }
  CHECK(back.problem.objective == p.objective);
  CHECK(back.problem.var_bounds.lower == p.var_bounds.lower);
  CHECK(back.problem.var_bounds.upper == p.var_bounds.upper);
  CHECK(back.problem.row_bounds.lower == p.row_bounds.lower);
  CHECK(back.problem.row_bounds.upper == p.row_bounds.upper);
  CHECK_THROWS_AS(parse_mps_string("ROWS\n L r\nENDATA\n"), MpsParseError);
}

int main(int argc, char** argv) {
  if (argc > 6 && std::strcmp(argv[1], "--write-mps") == 0) return write_set_cover_mps(argv + 2);
  if (argc > 2 && std::strcmp(argv[1], "--fsb-c1") == 0) return fsb_c1(argv[2]);
  if (argc > 1 && std::strcmp(argv[1], "--obbt-c2") == 0) return obbt_c2();
  return doctest::shim::run_all(argc, argv);
}
