// batchlp/detail/csr.hpp — host containers of the B200 drop-in.
//
// SparseMatrix keeps the reference's contract (reference
// proj/include/batchlp/sparse.hpp:30-171): CSR with columns sorted inside a
// row, duplicates summed in input order, exact cancellations dropped, and an
// eagerly built explicit transpose. The arrays live in one immutable,
// reference-counted block, so copies of a matrix (LpProblem, BatchProblem and
// the drivers copy freely) share it, and the device runtime can recognise a
// matrix it has already uploaded to HBM by the identity of that block
// (batchlp/device.hpp).
//
// DenseColumnBlock is the reference's column-major host block
// (sparse.hpp:46-88); the device never stores this layout.
#ifndef BATCHLP_B200_DETAIL_CSR_HPP
#define BATCHLP_B200_DETAIL_CSR_HPP

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <numeric>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace batchlp {

struct Triplet {
  int row = 0;
  int col = 0;
  double value = 0.0;
};

// Borrowed CSR arrays of one orientation (reference sparse.hpp:37-43).
struct CsrView {
  int n_rows = 0;
  int n_cols = 0;
  std::span<const int> offsets;
  std::span<const int> cols;
  std::span<const double> values;
};

class DenseColumnBlock {
 public:
  DenseColumnBlock() = default;
  DenseColumnBlock(int rows, int cols)
      : rows_(rows), cols_(cols), v_(static_cast<std::size_t>(rows) * cols, 0.0) {}

  int n_rows() const { return rows_; }
  int n_cols() const { return cols_; }
  double* col(int j) { return v_.data() + offset(j); }
  const double* col(int j) const { return v_.data() + offset(j); }
  std::span<double> col_span(int j) { return {col(j), static_cast<std::size_t>(rows_)}; }
  std::span<const double> col_span(int j) const {
    return {col(j), static_cast<std::size_t>(rows_)};
  }
  double& at(int i, int j) { return v_[offset(j) + i]; }
  double at(int i, int j) const { return v_[offset(j) + i]; }
  std::vector<double>& data() { return v_; }
  const std::vector<double>& data() const { return v_; }

  void swap_columns(int a, int b) {
    if (a != b) std::swap_ranges(col(a), col(a) + rows_, col(b));
  }
  void resize(int rows, int cols) {
    rows_ = rows;
    cols_ = cols;
    v_.resize(static_cast<std::size_t>(rows) * cols);
  }

 private:
  std::size_t offset(int j) const { return static_cast<std::size_t>(j) * rows_; }
  int rows_ = 0;
  int cols_ = 0;
  std::vector<double> v_;
};

class SparseMatrix {
 public:
  // Both orientations of one matrix; never mutated after construction.
  struct Storage {
    int rows = 0, cols = 0;
    std::vector<int> ptr, idx;        // A, CSR
    std::vector<double> val;
    std::vector<int> t_ptr, t_idx;    // A', CSR
    std::vector<double> t_val;
  };

  SparseMatrix() : s_(empty_storage()) {}

  // Coordinate input -> CSR (reference sparse.hpp:99-134). Entries are
  // bucketed by row keeping input order, then ordered by column inside the
  // row (stable), so duplicates are summed left to right exactly as the
  // reference's stable sort + sequential sum does.
  static SparseMatrix from_triplets(std::vector<Triplet> entries, int n_rows, int n_cols) {
    if (n_rows < 0 || n_cols < 0) throw std::invalid_argument("sparse: negative dimension");
    for (const Triplet& e : entries) {
      const bool row_ok = e.row >= 0 && e.row < n_rows;
      const bool col_ok = e.col >= 0 && e.col < n_cols;
      if (!row_ok || !col_ok)
        throw std::out_of_range("sparse: triplet index (" + std::to_string(e.row) + ", " +
                                std::to_string(e.col) + ") out of range");
    }
    auto st = std::make_shared<Storage>();
    st->rows = n_rows;
    st->cols = n_cols;
    // counting sort by row (stable)
    std::vector<std::size_t> start(static_cast<std::size_t>(n_rows) + 1, 0);
    for (const Triplet& e : entries) ++start[static_cast<std::size_t>(e.row) + 1];
    std::partial_sum(start.begin(), start.end(), start.begin());
    std::vector<std::size_t> order(entries.size());
    {
      std::vector<std::size_t> fill(start.begin(), start.end() - 1);
      for (std::size_t k = 0; k < entries.size(); ++k) order[fill[entries[k].row]++] = k;
    }
    st->ptr.assign(static_cast<std::size_t>(n_rows) + 1, 0);
    for (int r = 0; r < n_rows; ++r) {
      auto first = order.begin() + static_cast<std::ptrdiff_t>(start[r]);
      auto last = order.begin() + static_cast<std::ptrdiff_t>(start[r + 1]);
      std::stable_sort(first, last, [&](std::size_t a, std::size_t b) {
        return entries[a].col < entries[b].col;
      });
      for (auto it = first; it != last;) {
        const int c = entries[*it].col;
        double acc = 0.0;
        for (; it != last && entries[*it].col == c; ++it) acc += entries[*it].value;
        if (acc != 0.0) {
          st->idx.push_back(c);
          st->val.push_back(acc);
        }
      }
      st->ptr[r + 1] = static_cast<int>(st->idx.size());
    }
    build_transpose(*st);
    SparseMatrix out;
    out.s_ = std::move(st);
    return out;
  }

  // Adopts CSR arrays that already satisfy the invariants (sorted columns,
  // no duplicates, no explicit zeros) — the generators and the MPS-free
  // benchmark path build matrices this way without a triplet round trip.
  static SparseMatrix from_csr(int n_rows, int n_cols, std::vector<int> ptr,
                               std::vector<int> idx, std::vector<double> val) {
    if (n_rows < 0 || n_cols < 0) throw std::invalid_argument("sparse: negative dimension");
    if (ptr.size() != static_cast<std::size_t>(n_rows) + 1 || idx.size() != val.size() ||
        ptr.front() != 0 || static_cast<std::size_t>(ptr.back()) != idx.size())
      throw std::invalid_argument("sparse: malformed CSR arrays");
    auto st = std::make_shared<Storage>();
    st->rows = n_rows;
    st->cols = n_cols;
    st->ptr = std::move(ptr);
    st->idx = std::move(idx);
    st->val = std::move(val);
    for (int c : st->idx)
      if (c < 0 || c >= n_cols) throw std::out_of_range("sparse: column index out of range");
    build_transpose(*st);
    SparseMatrix out;
    out.s_ = std::move(st);
    return out;
  }

  int n_rows() const { return s_->rows; }
  int n_cols() const { return s_->cols; }
  std::int64_t nnz() const { return static_cast<std::int64_t>(s_->val.size()); }
  CsrView view() const { return {s_->rows, s_->cols, s_->ptr, s_->idx, s_->val}; }
  CsrView transpose_view() const { return {s_->cols, s_->rows, s_->t_ptr, s_->t_idx, s_->t_val}; }

  // Identity of the shared arrays (device residency cache key).
  const std::shared_ptr<const Storage>& storage() const { return s_; }

 private:
  static std::shared_ptr<const Storage> empty_storage() {
    auto st = std::make_shared<Storage>();
    st->ptr.assign(1, 0);
    st->t_ptr.assign(1, 0);
    return st;
  }

  // Scatter A's rows into A' rows; rows of A visited in order, so each row
  // of A' lists its entries by increasing column (reference sparse.hpp:148-163).
  static void build_transpose(Storage& st) {
    const std::size_t nz = st.val.size();
    st.t_ptr.assign(static_cast<std::size_t>(st.cols) + 1, 0);
    for (int c : st.idx) ++st.t_ptr[static_cast<std::size_t>(c) + 1];
    std::partial_sum(st.t_ptr.begin(), st.t_ptr.end(), st.t_ptr.begin());
    st.t_idx.resize(nz);
    st.t_val.resize(nz);
    std::vector<int> next(st.t_ptr.begin(), st.t_ptr.end() - 1);
    for (int r = 0; r < st.rows; ++r) {
      for (int q = st.ptr[r]; q < st.ptr[r + 1]; ++q) {
        const int slot = next[st.idx[q]]++;
        st.t_idx[slot] = r;
        st.t_val[slot] = st.val[q];
      }
    }
  }

  std::shared_ptr<const Storage> s_;
};

}  // namespace batchlp

#endif  // BATCHLP_B200_DETAIL_CSR_HPP
