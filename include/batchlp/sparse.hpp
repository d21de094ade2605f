// batchlp/sparse.hpp — sparse storage and products of the B200 drop-in.
//
// Source-compatible with the reference's sparse.hpp (reference
// proj/include/batchlp/sparse.hpp:28-319): the containers come from
// detail/csr.hpp, and the products run on the GPU through the C-ABI:
//   spmv / spmm      -> bl_spmm       (CSR SpMM kernel, row-major tiles;
//                                      entries bit-identical to csr_apply,
//                                      sparse.hpp:176-183)
//   csr_apply        -> bl_csr_apply  (the same kernel on a bare CsrView)
//   spectral_norm    -> bl_spectral_norm (device power iteration,
//                                      sparse.hpp:249-319)
// BATCHLP_THREADS (sparse.hpp:198-206) has no meaning here and is ignored.
#ifndef BATCHLP_B200_SPARSE_HPP
#define BATCHLP_B200_SPARSE_HPP

#include <cstdint>
#include <span>
#include <stdexcept>

#include "batchlp/detail/csr.hpp"
#include "batchlp/device.hpp"

namespace batchlp {

// out = M x on a bare view (reference sparse.hpp:173-183): the view need not
// belong to a resident SparseMatrix, so it is uploaded for this one product.
inline void csr_apply(const CsrView& mv, const double* x, double* out) {
  if (mv.n_rows == 0) return;
  cuda::Context& ctx = cuda::thread_context();
  cuda::check(ctx.handle(),
              bl_csr_apply(ctx.handle(), mv.n_rows, mv.n_cols,
                           static_cast<std::int64_t>(mv.values.size()), mv.offsets.data(),
                           mv.cols.data(), mv.values.data(), x, out));
}

// out.col(j) = op(A) x.col(j) for j < active_width; later columns of `out`
// keep their contents (reference sparse.hpp:213-238).
inline void spmm(const SparseMatrix& a, const DenseColumnBlock& x, DenseColumnBlock& out,
                 bool transpose_a = false, int active_width = -1) {
  const int in_rows = transpose_a ? a.n_rows() : a.n_cols();
  const int out_rows = transpose_a ? a.n_cols() : a.n_rows();
  if (x.n_rows() != in_rows || out.n_rows() != out_rows || out.n_cols() != x.n_cols())
    throw std::invalid_argument("spmm: dimension mismatch");
  const int width = x.n_cols();
  const int active = active_width < 0 ? width : active_width;
  if (active > width) throw std::invalid_argument("spmm: active width too large");
  if (active == 0 || out_rows == 0) return;
  cuda::Context& ctx = cuda::thread_context();
  bl_problem* p = ctx.resident_matrix(a);
  cuda::check(ctx.handle(), bl_spmm(ctx.handle(), p, transpose_a ? 1 : 0, width, active,
                                    x.data().data(), out.data().data()));
}

inline DenseColumnBlock spmm(const SparseMatrix& a, const DenseColumnBlock& x,
                             bool transpose_a = false) {
  DenseColumnBlock out(transpose_a ? a.n_cols() : a.n_rows(), x.n_cols());
  spmm(a, x, out, transpose_a);
  return out;
}

// One column of spmm (reference sparse.hpp:185-192).
inline void spmv(const SparseMatrix& a, std::span<const double> x, std::span<double> out,
                 bool transpose_a = false) {
  const CsrView v = transpose_a ? a.transpose_view() : a.view();
  if (static_cast<int>(x.size()) != v.n_cols || static_cast<int>(out.size()) != v.n_rows)
    throw std::invalid_argument("spmv: dimension mismatch");
  if (v.n_rows == 0) return;
  DenseColumnBlock xin(v.n_cols, 1), res(v.n_rows, 1);
  std::copy(x.begin(), x.end(), xin.col(0));
  spmm(a, xin, res, transpose_a, 1);
  std::copy(res.col(0), res.col(0) + v.n_rows, out.begin());
}

// ||A||_2 estimate x 1.01 (reference sparse.hpp:297-319), computed on the
// device; cached with the resident matrix.
inline double spectral_norm(const SparseMatrix& a) {
  if (a.nnz() == 0) throw std::invalid_argument("spectral_norm: zero matrix");
  cuda::Context& ctx = cuda::thread_context();
  bl_problem* p = ctx.resident_matrix(a);
  double out = 0.0;
  cuda::check(ctx.handle(), bl_spectral_norm(ctx.handle(), p, &out));
  return out;
}

}  // namespace batchlp

#endif  // BATCHLP_B200_SPARSE_HPP
