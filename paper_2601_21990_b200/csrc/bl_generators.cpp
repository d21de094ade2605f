// bl_generators.cpp — deterministic synthetic instances for the benchmarks
// (tools, not on the hot path). CSR assembly follows
// SparseMatrix::from_triplets semantics (reference sparse.hpp:99-163): entries
// sorted by (row, col), duplicates summed, exact zeros dropped, and the
// explicit transpose built by a counting pass in row order.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "batchlp_cuda.h"

namespace {

struct Trip {
  int r, c;
  double v;
};

// mt19937_64 draws with the reference generator's conversions
// (generators.hpp:45-61): uniform_int by modulo, uniform by 53 high bits.
class Rng {
 public:
  explicit Rng(uint64_t seed) : g_(seed) {}
  int uniform_int(int lo, int hi) {
    return lo + static_cast<int>(g_() % static_cast<uint64_t>(hi - lo + 1));
  }
  double uniform() { return (g_() >> 11) * 0x1.0p-53; }
  bool bernoulli(double p) { return uniform() < p; }

 private:
  std::mt19937_64 g_;
};

template <class T>
T* dup(const std::vector<T>& v) {
  T* p = static_cast<T*>(std::malloc(sizeof(T) * (v.size() ? v.size() : 1)));
  if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
  return p;
}

void assemble(std::vector<Trip> t, int m, int n, bl_instance* out) {
  std::stable_sort(t.begin(), t.end(), [](const Trip& a, const Trip& b) {
    return a.r != b.r ? a.r < b.r : a.c < b.c;
  });
  std::vector<int> rp(m + 1, 0), ci;
  std::vector<double> cv;
  ci.reserve(t.size());
  cv.reserve(t.size());
  size_t i = 0;
  while (i < t.size()) {
    const int r = t[i].r, c = t[i].c;
    double s = 0.0;
    while (i < t.size() && t[i].r == r && t[i].c == c) s += t[i++].v;
    if (s != 0.0) {
      ci.push_back(c);
      cv.push_back(s);
      ++rp[r + 1];
    }
  }
  for (int r = 0; r < m; ++r) rp[r + 1] += rp[r];
  std::vector<int> trp(n + 1, 0), tci(ci.size());
  std::vector<double> tcv(ci.size());
  for (int c : ci) ++trp[c + 1];
  for (int c = 0; c < n; ++c) trp[c + 1] += trp[c];
  std::vector<int> cur(trp.begin(), trp.end() - 1);
  for (int r = 0; r < m; ++r)
    for (int p = rp[r]; p < rp[r + 1]; ++p) {
      const int q = cur[ci[p]]++;
      tci[q] = r;
      tcv[q] = cv[p];
    }
  out->m = m;
  out->n = n;
  out->nnz = static_cast<int64_t>(ci.size());
  out->rowptr = dup(rp);
  out->col = dup(ci);
  out->val = dup(cv);
  out->t_rowptr = dup(trp);
  out->t_col = dup(tci);
  out->t_val = dup(tcv);
}

void set_vectors(bl_instance* out, const std::vector<double>& c, const std::vector<double>& xl,
                 const std::vector<double>& xu, const std::vector<double>& rl,
                 const std::vector<double>& ru) {
  out->objective = dup(c);
  out->var_lower = dup(xl);
  out->var_upper = dup(xu);
  out->row_lower = dup(rl);
  out->row_upper = dup(ru);
}

// k distinct values in [0, n) in ascending order (generators.hpp:61-65 style)
std::vector<int> sample_distinct(Rng& rng, int k, int n) {
  std::vector<int> picked;
  picked.reserve(k);
  while (static_cast<int>(picked.size()) < k) {
    const int v = rng.uniform_int(0, n - 1);
    if (std::find(picked.begin(), picked.end(), v) == picked.end()) picked.push_back(v);
  }
  std::sort(picked.begin(), picked.end());
  return picked;
}

}  // namespace

extern "C" {

// min c'x, A x >= 1, x in [0,1]^n: the draw sequence of generate_set_cover
// (reference generators.hpp:76-109), so seed s gives the reference instance.
int bl_gen_set_cover(int32_t rows, int32_t cols, double density, uint64_t seed,
                     bl_instance* out) {
  if (rows < 1 || cols < 1 || density <= 0.0 || density > 1.0) return BL_ERR_INVALID_ARGUMENT;
  Rng rng(seed);
  std::vector<Trip> t;
  std::vector<char> row_hit(rows, 0), col_hit(cols, 0);
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j)
      if (rng.bernoulli(density)) {
        t.push_back({i, j, 1.0});
        row_hit[i] = col_hit[j] = 1;
      }
  for (int i = 0; i < rows; ++i)
    if (!row_hit[i]) {
      const int j = rng.uniform_int(0, cols - 1);
      t.push_back({i, j, 1.0});
      col_hit[j] = 1;
    }
  for (int j = 0; j < cols; ++j)
    if (!col_hit[j]) t.push_back({rng.uniform_int(0, rows - 1), j, 1.0});
  assemble(std::move(t), rows, cols, out);
  std::vector<double> c(cols);
  for (int j = 0; j < cols; ++j) c[j] = rng.uniform_int(1, 100);
  set_vectors(out, c, std::vector<double>(cols, 0.0), std::vector<double>(cols, 1.0),
              std::vector<double>(rows, 1.0), std::vector<double>(rows, HUGE_VAL));
  return BL_OK;
}

// O(nnz) set-cover-like family: column j
// covers per_col distinct uniform rows; an uncovered row gets one random
// column; c in {1..100}; rows [1, inf); x in [0, 1].
int bl_gen_sparse_cover(int32_t rows, int32_t cols, int32_t per_col, uint64_t seed,
                        bl_instance* out) {
  if (rows < 1 || cols < 1 || per_col < 1 || per_col > rows) return BL_ERR_INVALID_ARGUMENT;
  Rng rng(seed);
  std::vector<Trip> t;
  t.reserve(static_cast<size_t>(cols) * per_col + rows / 8);
  std::vector<char> row_hit(rows, 0);
  for (int j = 0; j < cols; ++j)
    for (int r : sample_distinct(rng, per_col, rows)) {
      t.push_back({r, j, 1.0});
      row_hit[r] = 1;
    }
  for (int i = 0; i < rows; ++i)
    if (!row_hit[i]) t.push_back({i, rng.uniform_int(0, cols - 1), 1.0});
  assemble(std::move(t), rows, cols, out);
  std::vector<double> c(cols);
  for (int j = 0; j < cols; ++j) c[j] = rng.uniform_int(1, 100);
  set_vectors(out, c, std::vector<double>(cols, 0.0), std::vector<double>(cols, 1.0),
              std::vector<double>(rows, 1.0), std::vector<double>(rows, HUGE_VAL));
  return BL_OK;
}

// Scaled random_feasible_lp family (the shape of
// the reference fixture tests/support/instances.hpp:89-145): x in [0, U_j],
// U_j in {1..5}; a known point x0_j = U_j/2 * {0..2}/... on the half grid;
// each column has per_col distinct rows with coefficients in {-4..4}\{0};
// rows are two-sided / >= / <= around A x0 with slacks in 0.5 {1..6};
// c in {-5..5}. Feasible and bounded by construction.
int bl_gen_boxed_feasible(int32_t rows, int32_t cols, int32_t per_col, uint64_t seed,
                          bl_instance* out) {
  if (rows < 1 || cols < 1 || per_col < 1 || per_col > rows) return BL_ERR_INVALID_ARGUMENT;
  Rng rng(seed);
  std::vector<double> xu(cols), x0(cols);
  std::vector<Trip> t;
  t.reserve(static_cast<size_t>(cols) * per_col);
  for (int j = 0; j < cols; ++j) {
    const double hi = rng.uniform_int(1, 5);
    xu[j] = hi;
    x0[j] = 0.5 * rng.uniform_int(0, static_cast<int>(2 * hi));
    for (int r : sample_distinct(rng, per_col, rows)) {
      const int u = rng.uniform_int(1, 8);  // 1..8 -> -4..-1, 1..4
      t.push_back({r, j, static_cast<double>(u <= 4 ? u - 5 : u - 4)});
    }
  }
  assemble(std::move(t), rows, cols, out);
  std::vector<double> ax0(rows, 0.0);
  for (int r = 0; r < rows; ++r) {
    double acc = 0.0;
    for (int p = out->rowptr[r]; p < out->rowptr[r + 1]; ++p) acc += out->val[p] * x0[out->col[p]];
    ax0[r] = acc;
  }
  std::vector<double> rl(rows), ru(rows);
  for (int r = 0; r < rows; ++r) {
    const double slo = 0.5 * rng.uniform_int(1, 6);
    const double shi = 0.5 * rng.uniform_int(1, 6);
    switch (rng.uniform_int(0, 2)) {
      case 0: rl[r] = ax0[r] - slo; ru[r] = ax0[r] + shi; break;
      case 1: rl[r] = ax0[r] - slo; ru[r] = HUGE_VAL; break;
      default: rl[r] = -HUGE_VAL; ru[r] = ax0[r] + shi; break;
    }
  }
  std::vector<double> c(cols);
  for (int j = 0; j < cols; ++j) c[j] = rng.uniform_int(-5, 5);
  set_vectors(out, c, std::vector<double>(cols, 0.0), xu, rl, ru);
  return BL_OK;
}

void bl_instance_free(bl_instance* inst) {
  if (!inst) return;
  for (void* p : {static_cast<void*>(inst->rowptr), static_cast<void*>(inst->col),
                  static_cast<void*>(inst->val), static_cast<void*>(inst->t_rowptr),
                  static_cast<void*>(inst->t_col), static_cast<void*>(inst->t_val),
                  static_cast<void*>(inst->objective), static_cast<void*>(inst->var_lower),
                  static_cast<void*>(inst->var_upper), static_cast<void*>(inst->row_lower),
                  static_cast<void*>(inst->row_upper)})
    std::free(p);
  std::memset(inst, 0, sizeof(*inst));
}

}  // extern "C"
