// batchlp/device.hpp — the C++ side of the C-ABI boundary.
//
// Everything the drop-in headers need to reach the sm_100a kernels through
// include/batchlp_cuda.h (libbatchlp_cuda.so): status-code -> exception
// mapping (the reference's exception contract), an owning
// device context (one CUDA stream + grow-only workspace per host thread and
// device, like the reference's BatchWorkspace, batch_solver.hpp:59-67), and
// a residency cache that keeps a matrix's CSR / CSR' arrays in HBM across
// solves (the reference shares an immutable SparseMatrix across solves,
// sparse.hpp:90-92; here the device copy is what is shared).
//
// There is no CPU implementation behind these calls: if the CUDA library or
// a device is missing, every entry throws std::runtime_error.
#ifndef BATCHLP_B200_DEVICE_HPP
#define BATCHLP_B200_DEVICE_HPP

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "batchlp/detail/csr.hpp"
#include "batchlp_cuda.h"

namespace batchlp::cuda {

// bl_code -> the exception type the reference throws at the same point.
[[noreturn]] inline void raise_code(int code, const std::string& what) {
  switch (code) {
    case BL_ERR_INVALID_ARGUMENT: throw std::invalid_argument(what);
    case BL_ERR_OUT_OF_RANGE: throw std::out_of_range(what);
    case BL_ERR_DOMAIN: throw std::domain_error(what);
    case BL_ERR_LOGIC: throw std::logic_error(what);
    default: throw std::runtime_error("batchlp (CUDA): " + what);
  }
}

inline void check(const bl_ctx* ctx, int code) {
  if (code != BL_OK) raise_code(code, bl_last_error(ctx));
}

class Context {
 public:
  explicit Context(int device = default_device()) : device_(device) {
    bl_ctx* h = nullptr;
    check(nullptr, bl_ctx_create(device, &h));
    h_ = h;
  }
  ~Context() {
    for (Entry& e : cache_) bl_problem_free(e.handle);
    bl_ctx_destroy(h_);
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;

  bl_ctx* handle() const { return h_; }
  int device() const { return device_; }

  // A device-resident copy of (A, c, var bounds, row bounds). Matrices are
  // recognised by the identity of their shared storage, vectors by value;
  // at most kCacheSlots problems stay resident per context.
  bl_problem* resident(const SparseMatrix& a, std::span<const double> c,
                       std::span<const double> xl, std::span<const double> xu,
                       std::span<const double> rl, std::span<const double> ru) {
    const void* key = a.storage().get();
    ++clock_;
    for (Entry& e : cache_) {
      if (e.key == key && !e.owner.expired() && same(e.c, c) && same(e.xl, xl) &&
          same(e.xu, xu) && same(e.rl, rl) && same(e.ru, ru)) {
        e.last_use = clock_;
        return e.handle;
      }
    }
    const CsrView v = a.view(), t = a.transpose_view();
    bl_problem* p = nullptr;
    check(h_, bl_problem_upload(h_, v.n_rows, v.n_cols, a.nnz(), v.offsets.data(),
                                v.cols.data(), v.values.data(), t.offsets.data(),
                                t.cols.data(), t.values.data(), c.data(), xl.data(),
                                xu.data(), rl.data(), ru.data(), &p));
    Entry fresh{key, a.storage(), {c.begin(), c.end()}, {xl.begin(), xl.end()},
                {xu.begin(), xu.end()}, {rl.begin(), rl.end()}, {ru.begin(), ru.end()},
                p, clock_};
    if (cache_.size() < kCacheSlots) {
      cache_.push_back(std::move(fresh));
    } else {
      std::size_t victim = 0;
      for (std::size_t k = 1; k < cache_.size(); ++k)
        if (cache_[k].owner.expired() || cache_[k].last_use < cache_[victim].last_use)
          victim = k;
      bl_problem_free(cache_[victim].handle);
      cache_[victim] = std::move(fresh);
    }
    return p;
  }

  // A alone (zero objective, free boxes): sparse products and norms.
  bl_problem* resident_matrix(const SparseMatrix& a) {
    const std::size_t n = static_cast<std::size_t>(a.n_cols());
    const std::size_t m = static_cast<std::size_t>(a.n_rows());
    if (zeros_.size() < n) zeros_.assign(n, 0.0);
    if (neg_.size() < std::max(n, m)) {
      neg_.assign(std::max(n, m), -std::numeric_limits<double>::infinity());
      pos_.assign(std::max(n, m), std::numeric_limits<double>::infinity());
    }
    return resident(a, {zeros_.data(), n}, {neg_.data(), n}, {pos_.data(), n},
                    {neg_.data(), m}, {pos_.data(), m});
  }

  static int default_device() {
    const char* e = std::getenv("BATCHLP_DEVICE");
    return e ? std::atoi(e) : 0;
  }

 private:
  static constexpr std::size_t kCacheSlots = 4;
  struct Entry {
    const void* key;
    std::weak_ptr<const SparseMatrix::Storage> owner;
    std::vector<double> c, xl, xu, rl, ru;
    bl_problem* handle;
    std::uint64_t last_use;
  };
  static bool same(const std::vector<double>& a, std::span<const double> b) {
    if (a.size() != b.size()) return false;
    for (std::size_t k = 0; k < a.size(); ++k)  // bitwise: -0.0 / NaN payloads matter
      if (std::memcmp(&a[k], &b[k], sizeof(double)) != 0) return false;
    return true;
  }

  bl_ctx* h_ = nullptr;
  int device_ = 0;
  std::uint64_t clock_ = 0;
  std::vector<Entry> cache_;
  std::vector<double> zeros_, neg_, pos_;
};

// The context solves use when the caller passes no workspace: one per host
// thread (the reference allows concurrent solves over shared problems,
// SPEC.md:321,402; a bl_ctx must not be shared between threads).
inline Context& thread_context() {
  thread_local std::unique_ptr<Context> ctx;
  if (!ctx) ctx = std::make_unique<Context>();
  return *ctx;
}

// Contexts of a sharded solve (BatchOptions::devices): one per (device,
// occurrence) on this host thread, so a device listed twice gets two
// independent contexts (two streams on one GPU).
inline Context& shard_context(int device, int occurrence) {
  thread_local std::vector<std::unique_ptr<Context>> pool;
  thread_local std::vector<std::pair<int, int>> keys;
  for (std::size_t k = 0; k < keys.size(); ++k)
    if (keys[k] == std::pair<int, int>{device, occurrence}) return *pool[k];
  pool.push_back(std::make_unique<Context>(device));
  keys.emplace_back(device, occurrence);
  return *pool.back();
}

}  // namespace batchlp::cuda

#endif  // BATCHLP_B200_DEVICE_HPP
