// tools/batchlp_run.cpp — command-line runs of MPS instances on the B200
// (SURVEY §8(f) item 4): the reference CLI's solve / fsb / obbt / bench
// flows (reference proj/tools/batchlp_main.cpp:115-273) over the drop-in
// headers, every LP solved on the GPU.
//
//   batchlp_run solve FILE.mps [--eps E] [--max-iter N] [--json OUT]
//   batchlp_run fsb   FILE.mps [--eps E] [--max-iter N] [--json OUT] [--devices 0,1,..]
//       root relaxation solved on the device (the reference's CLI needs a
//       given x_rel or its vertex-enumeration oracle), then strong branching
//       on the fractional integer columns (run_fsb); prints the ranking
//   batchlp_run obbt  FILE.mps [--eps E] [--eps-dual E] [--max-iter N] [--json OUT]
//   batchlp_run bench FILE.mps... [--eps E] [--max-iter N] [--csv OUT] [--devices ..]
//       the `bench` CSV (family,instance,m,n,nnz,S,runtime_s,iters): root
//       solve + strong branching on the fractional integer columns per file,
//       timed end to end (parse excluded), family "mps"
//
// Exit codes as the reference CLI: 0 ok, 1 usage, 2 input, 3 iteration limit.
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "batchlp/batchlp.hpp"

namespace {

using namespace batchlp;

constexpr int kOk = 0, kUsage = 1, kInput = 2, kLimit = 3;

double seconds() {
  using clock = std::chrono::steady_clock;
  return std::chrono::duration<double>(clock::now().time_since_epoch()).count();
}

struct Args {
  std::string command;
  std::vector<std::string> files;
  double eps = 1e-4, eps_dual = 1e-8;
  std::int64_t max_iter = 100000;
  std::string json, csv;
  std::vector<int> devices;
};

bool parse(int argc, char** argv, Args& a) {
  if (argc < 3) return false;
  a.command = argv[1];
  for (int k = 2; k < argc; ++k) {
    const std::string t = argv[k];
    auto value = [&]() -> const char* { return k + 1 < argc ? argv[++k] : nullptr; };
    const char* v = nullptr;
    if (t == "--eps" && (v = value())) a.eps = std::atof(v);
    else if (t == "--eps-dual" && (v = value())) a.eps_dual = std::atof(v);
    else if (t == "--max-iter" && (v = value())) a.max_iter = std::atoll(v);
    else if (t == "--json" && (v = value())) a.json = v;
    else if (t == "--csv" && (v = value())) a.csv = v;
    else if (t == "--devices" && (v = value())) {
      std::stringstream ss(v);
      for (std::string d; std::getline(ss, d, ',');)
        if (!d.empty()) a.devices.push_back(std::atoi(d.c_str()));
    } else if (!t.empty() && t[0] == '-') return false;
    else a.files.push_back(t);
  }
  return !a.files.empty();
}

void emit(const std::string& where, const std::string& text) {
  if (where.empty() || where == "-") {
    std::cout << text;
    if (!text.empty() && text.back() != '\n') std::cout << '\n';
    return;
  }
  std::ofstream out(where);
  if (!out) throw std::runtime_error("cannot write '" + where + "'");
  out << text;
}

// integer columns whose relaxation value is off an integer by more than tol
// (batchlp_main.cpp:60-69); all columns when the model declares none
std::vector<int> candidates(const std::vector<double>& x, const std::vector<int>& ints,
                            double tol) {
  std::vector<int> out;
  auto test = [&](int c) {
    if (std::abs(x[c] - std::round(x[c])) > tol) out.push_back(c);
  };
  if (ints.empty())
    for (int c = 0; c < static_cast<int>(x.size()); ++c) test(c);
  else
    for (const int c : ints) test(c);
  return out;
}

SolverConfig config_of(const Args& a) {
  SolverConfig cfg;
  cfg.eps_opt = a.eps;
  cfg.max_iterations = a.max_iter;
  return cfg;
}

struct FsbRun {
  SolveResult root;
  FsbOutcome outcome;
  int subproblems = 0;
  double solve_s = 0.0;
};

// root solve + strong branching, both on the device
FsbRun fsb_flow(const MpsModel& model, const SolverConfig& cfg, const std::vector<int>& devices) {
  FsbRun r;
  const double t0 = seconds();
  r.root = solve(model.problem, cfg);
  if (r.root.status == SolveStatus::kOptimal) {
    FsbRequest req;
    req.problem = model.problem;
    req.x_rel = r.root.x;
    req.fractional_indices = candidates(r.root.x, model.integer_columns, 1e-6);
    r.subproblems = 2 * static_cast<int>(req.fractional_indices.size());
    if (devices.size() > 1) {  // the batch sharded over the listed GPUs
      const FsbBatch built = build_fsb_batch(req);
      BatchOptions opt;
      opt.vectors = VectorMode::kNone;
      opt.devices = devices;
      const BatchSolveSummary s = solve_batch(built.batch, cfg, built.presets, nullptr, {}, opt);
      r.outcome.iterations = s.iterations;
      r.outcome.root_objective = r.root.objective;
    } else {
      r.outcome = run_fsb(req, cfg);
    }
  }
  r.solve_s = seconds() - t0;
  return r;
}

int cmd_solve(const Args& a) {
  PhaseTimes times;
  double t = seconds();
  const MpsModel model = read_mps_file(a.files[0]);
  times.load_s = seconds() - t;
  const SolverConfig cfg = config_of(a);
  t = seconds();
  if (model.problem.A.nnz() > 0) (void)spectral_norm(model.problem.A);
  times.norm_s = seconds() - t;
  t = seconds();
  const SolveResult r = solve(model.problem, cfg);
  times.solve_s = seconds() - t;
#if __has_include(<nlohmann/json.hpp>)
  if (!a.json.empty()) {
    nlohmann::json rep = report_header("solve", model.problem, cfg, times);
    rep["instance"] = model.name;
    rep["result"] = result_to_json(r);
    emit(a.json, rep.dump(2));
  } else
#endif
  {
    std::cout << "status      " << status_name(r.status) << "\nobjective   " << r.objective
              << "\niterations  " << r.iterations << "\nrestarts    " << r.restarts << "\n";
  }
  return r.status == SolveStatus::kIterationLimit ? kLimit : kOk;
}

int cmd_fsb(const Args& a) {
  PhaseTimes times;
  double t = seconds();
  const MpsModel model = read_mps_file(a.files[0]);
  times.load_s = seconds() - t;
  const SolverConfig cfg = config_of(a);
  const FsbRun r = fsb_flow(model, cfg, a.devices);
  times.solve_s = r.solve_s;
  if (r.root.status != SolveStatus::kOptimal) {
    std::cerr << "root relaxation: " << status_name(r.root.status) << "\n";
    return r.root.status == SolveStatus::kIterationLimit ? kLimit : kInput;
  }
#if __has_include(<nlohmann/json.hpp>)
  if (!a.json.empty()) {
    nlohmann::json rep = report_header("fsb", model.problem, cfg, times);
    rep["instance"] = model.name;
    rep["root"] = result_to_json(r.root);
    rep["fsb"] = fsb_to_json(r.outcome);
    emit(a.json, rep.dump(2));
    return kOk;
  }
#endif
  std::cout << "root objective " << r.root.objective << ", " << r.subproblems / 2
            << " fractional variables, " << r.outcome.iterations << " iterations\n";
  for (const int var : score_branching(r.outcome)) std::cout << "  x" << var << "\n";
  return kOk;
}

int cmd_obbt(const Args& a) {
  PhaseTimes times;
  double t = seconds();
  const MpsModel model = read_mps_file(a.files[0]);
  times.load_s = seconds() - t;
  ObbtConfig cfg;
  cfg.eps_opt = a.eps;
  cfg.eps_dual = a.eps_dual;
  cfg.max_iterations = a.max_iter;
  t = seconds();
  const ObbtOutcome o = run_obbt(model.problem, cfg);
  times.solve_s = seconds() - t;
#if __has_include(<nlohmann/json.hpp>)
  if (!a.json.empty()) {
    nlohmann::json rep = report_header("obbt", model.problem, cfg.solver_config(), times);
    rep["instance"] = model.name;
    rep["obbt"] = obbt_to_json(o);
    emit(a.json, rep.dump(2));
    return kOk;
  }
#endif
  std::cout << o.changed_count << " variables changed, mean reduction " << o.mean_reduction_pct
            << "%, solved " << o.solved_count << "/" << (o.solved_count + o.limit_count) << "\n";
  return kOk;
}

int cmd_bench(const Args& a) {
  std::ostringstream csv;
  write_bench_csv_header(csv);
  const SolverConfig cfg = config_of(a);
  for (const std::string& f : a.files) {
    const MpsModel model = read_mps_file(f);
    const FsbRun r = fsb_flow(model, cfg, a.devices);
    BenchRow row;
    row.family = "mps";
    row.instance = model.name.empty() ? f : model.name;
    row.m = model.problem.num_rows();
    row.n = model.problem.num_cols();
    row.nnz = model.problem.A.nnz();
    row.subproblems = r.subproblems;
    row.runtime_s = r.solve_s;
    row.iterations = r.root.iterations + r.outcome.iterations;
    write_bench_csv_row(csv, row);
  }
  emit(a.csv, csv.str());
  return kOk;
}

}  // namespace

int main(int argc, char** argv) {
  Args a;
  if (!parse(argc, argv, a)) {
    std::cerr << "usage: batchlp_run solve|fsb|obbt|bench FILE.mps... [--eps E] [--eps-dual E] "
                 "[--max-iter N] [--json OUT] [--csv OUT] [--devices 0,1,..]\n";
    return kUsage;
  }
  try {
    if (a.command == "solve") return cmd_solve(a);
    if (a.command == "fsb") return cmd_fsb(a);
    if (a.command == "obbt") return cmd_obbt(a);
    if (a.command == "bench") return cmd_bench(a);
    std::cerr << "unknown command '" << a.command << "'\n";
    return kUsage;
  } catch (const MpsParseError& e) {
    std::cerr << e.what() << "\n";
    return kInput;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kInput;
  }
}
