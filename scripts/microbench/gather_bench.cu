// gather_bench.cu — microbenchmark of the SpMM gather pattern of the solver
// (tuning tool, not product code). Y is m x K stored column-block tiled
// (blocks of W = 32 columns, row-major inside a block); out = A' Y over
// n rows, A' with `per_row` random nonzeros per row. Reports time and the
// algorithmic bandwidth 12 nnz + 8 K (m + n) per product, next to a plain
// streaming copy of the same dense bytes.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench gather_bench.cu
//   ./gather_bench m n per_row K
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      std::exit(1);                                                                \
    }                                                                              \
  } while (0)

constexpr int W = 32;

// L lanes per row, each lane V = W / L doubles (as V/2 double2 loads).
template <int L, int UNROLL>
__global__ void __launch_bounds__(256) k_gather(int n, int m, int nb, int R, const int* __restrict__ rp,
                                                const int* __restrict__ ci,
                                                const double* __restrict__ cv,
                                                const double* __restrict__ Y, double* __restrict__ out) {
  constexpr int V = W / L;   // doubles per lane
  constexpr int V2 = V / 2;  // double2 loads per lane
  constexpr int G = 256 / L;
  const int g = threadIdx.x / L, li = threadIdx.x % L;
  const int items = nb * R;
  const int per = (n + R - 1) / R;
  for (int w = blockIdx.x; w < items; w += gridDim.x) {
    const int b = w / R, r = w % R;
    const int r0 = min(n, r * per), r1 = min(n, r0 + per);
    const double* base = Y + (size_t)b * m * W + li * V;
    for (int i = r0 + g; i < r1; i += G) {
      double acc[V];
#pragma unroll
      for (int v = 0; v < V; ++v) acc[v] = 0.0;
      int p = __ldg(rp + i);
      const int e = __ldg(rp + i + 1);
      for (; p < e; p += UNROLL) {
        double2 x[UNROLL][V2];
        double a[UNROLL];
#pragma unroll
        for (int k = 0; k < UNROLL; ++k) {
          if (p + k < e) {
            const int c = __ldg(ci + p + k);
            a[k] = __ldg(cv + p + k);
#pragma unroll
            for (int q = 0; q < V2; ++q)
              x[k][q] = __ldg(reinterpret_cast<const double2*>(base + (size_t)c * W) + q);
          }
        }
#pragma unroll
        for (int k = 0; k < UNROLL; ++k) {
          if (p + k < e) {
#pragma unroll
            for (int q = 0; q < V2; ++q) {
              acc[2 * q] = __dadd_rn(acc[2 * q], __dmul_rn(a[k], x[k][q].x));
              acc[2 * q + 1] = __dadd_rn(acc[2 * q + 1], __dmul_rn(a[k], x[k][q].y));
            }
          }
        }
      }
      double* dst = out + ((size_t)b * n + i) * W + li * V;
#pragma unroll
      for (int q = 0; q < V2; ++q)
        __stcs(reinterpret_cast<double2*>(dst) + q, make_double2(acc[2 * q], acc[2 * q + 1]));
    }
  }
}

__global__ void k_copy(const double2* __restrict__ a, double2* __restrict__ b, size_t n2) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2;
       i += (size_t)gridDim.x * blockDim.x)
    __stcs(b + i, __ldcs(a + i));
}

template <int L, int U>
float run(int grid, int n, int m, int nb, int R, const int* rp, const int* ci, const double* cv,
          const double* Y, double* out, int reps) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  k_gather<L, U><<<grid, 256>>>(n, m, nb, R, rp, ci, cv, Y, out);
  CK(cudaEventRecord(e0));
  for (int k = 0; k < reps; ++k) k_gather<L, U><<<grid, 256>>>(n, m, nb, R, rp, ci, cv, Y, out);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  CK(cudaGetLastError());
  return ms / reps;
}

int main(int argc, char** argv) {
  const int m = argc > 1 ? std::atoi(argv[1]) : 20000;
  const int n = argc > 2 ? std::atoi(argv[2]) : 40000;
  const int per_row = argc > 3 ? std::atoi(argv[3]) : 10;
  const int K = argc > 4 ? std::atoi(argv[4]) : 1024;
  const int nb = K / W;
  std::mt19937_64 rng(7);
  std::vector<int> rp(n + 1), ci((size_t)n * per_row);
  std::vector<double> cv((size_t)n * per_row, 1.0);
  for (int i = 0; i < n; ++i) {
    rp[i] = i * per_row;
    std::vector<int> rows;
    while ((int)rows.size() < per_row) {
      int c = (int)(rng() % m);
      if (std::find(rows.begin(), rows.end(), c) == rows.end()) rows.push_back(c);
    }
    std::sort(rows.begin(), rows.end());
    for (int k = 0; k < per_row; ++k) ci[(size_t)i * per_row + k] = rows[k];
  }
  rp[n] = n * per_row;
  const size_t nnz = ci.size();
  int *drp, *dci;
  double *dcv, *dY, *dout;
  CK(cudaMalloc(&drp, sizeof(int) * (n + 1)));
  CK(cudaMalloc(&dci, sizeof(int) * nnz));
  CK(cudaMalloc(&dcv, sizeof(double) * nnz));
  CK(cudaMalloc(&dY, sizeof(double) * (size_t)m * K));
  CK(cudaMalloc(&dout, sizeof(double) * (size_t)n * K));
  CK(cudaMemcpy(drp, rp.data(), sizeof(int) * (n + 1), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dci, ci.data(), sizeof(int) * nnz, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dcv, cv.data(), sizeof(double) * nnz, cudaMemcpyHostToDevice));
  CK(cudaMemset(dY, 0, sizeof(double) * (size_t)m * K));
  int sms = 148;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const double alg = 12.0 * nnz + 8.0 * K * ((double)m + n);
  const double gathered = 8.0 * K * (double)nnz;
  std::printf("m=%d n=%d nnz=%zu K=%d  alg bytes %.1f MB, gathered bytes %.1f MB\n", m, n, nnz, K,
              alg / 1e6, gathered / 1e6);
  {  // streaming copy of the dense bytes (m + n) K
    const size_t n2 = (size_t)K * (m + n) / 4;  // double2 elements of half the bytes each way
    double2 *a, *b;
    CK(cudaMalloc(&a, n2 * 16));
    CK(cudaMalloc(&b, n2 * 16));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_copy<<<sms * 8, 256>>>(a, b, n2);
    cudaEventRecord(e0);
    for (int k = 0; k < 20; ++k) k_copy<<<sms * 8, 256>>>(a, b, n2);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 20;
    std::printf("copy %.1f MB: %.1f us  %.0f GB/s\n", 2.0 * n2 * 16 / 1e6, ms * 1e3,
                2.0 * n2 * 16 / (ms * 1e-3) / 1e9);
    cudaFree(a);
    cudaFree(b);
  }
  const int Rs[] = {1, 4, 16, 64, 256, 1024};
  for (int occ : {2, 4, 8}) {
    const int grid = sms * occ;
    for (int R : Rs) {
      if (R > n) continue;
      float t1 = run<16, 4>(grid, n, m, nb, R, drp, dci, dcv, dY, dout, 10);
      float t2 = run<16, 8>(grid, n, m, nb, R, drp, dci, dcv, dY, dout, 10);
      float t3 = run<16, 2>(grid, n, m, nb, R, drp, dci, dcv, dY, dout, 10);
      float t4 = run<8, 4>(grid, n, m, nb, R, drp, dci, dcv, dY, dout, 10);
      float t5 = run<4, 2>(grid, n, m, nb, R, drp, dci, dcv, dY, dout, 10);
      std::printf("grid=%5d R=%5d  L16U4 %8.1f us %6.0f GB/s | L16U8 %8.1f %6.0f | L16U2 %8.1f %6.0f | L8U4 %8.1f %6.0f | L4U2 %8.1f %6.0f\n",
                  grid, R, t1 * 1e3, alg / (t1 * 1e-3) / 1e9, t2 * 1e3, alg / (t2 * 1e-3) / 1e9,
                  t3 * 1e3, alg / (t3 * 1e-3) / 1e9, t4 * 1e3, alg / (t4 * 1e-3) / 1e9, t5 * 1e3,
                  alg / (t5 * 1e-3) / 1e9);
    }
  }
  return 0;
}
