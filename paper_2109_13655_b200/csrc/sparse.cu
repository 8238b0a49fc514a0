// Sparse operator ingest: compressed-sparse-column A (Eigen's SparseMatrix layout,
// proj/include/sssvd/problem.hpp:27-35) densified into the column-major HBM operator.
//
// The reference keeps A sparse and forms G = (A^T A) with a sparse product (problem.hpp:87-89),
// then applies A sparsely in the tail. On a B200 the dense Gram cap (n <= 8192, problem.hpp:84)
// bounds n, so A fits in HBM densified for every m up to ~2.7M rows at n = 8192 (180 GB); a
// dense DMMA Gram (gram.cu) and dense tail GEMMs then replace the sparse products. The zero
// products the dense form adds are exact zeros, so G and A*V agree with the sparse products to
// rounding (summation order only).
//
// Two kernels, both one warp per user column j:
//   csc_check   - colptr monotone with colptr[0] = 0 and colptr[cols] = nnz, every row index in
//                 [0, rows) and strictly increasing inside a column (compressed, no duplicates);
//                 any violation sets *bad. Index reads are clamped to [0, nnz) so a corrupt colptr
//                 cannot read out of bounds.
//   csc_scatter - Ad[j*ldp + r] = v (or Ad[r*ldp + j] when the operator is stored transposed,
//                 rows < cols). Ad must be zeroed first.
#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace sssvd_gpu {

__global__ void csc_check_kernel(const int64_t* __restrict__ colptr, const int64_t* __restrict__ rowind,
                                 int64_t rows, int64_t cols, int64_t nnz, int* __restrict__ bad) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t j = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); j < cols; j += warps) {
    const int64_t b = colptr[j], e = colptr[j + 1];
    int flag = 0;
    if (lane == 0) {
      if (b > e || b < 0 || e > nnz) flag = 1;
      if (j == 0 && b != 0) flag = 1;
      if (j == cols - 1 && e != nnz) flag = 1;
    }
    const int64_t lo = min(max(b, (int64_t)0), nnz), hi = min(max(e, lo), nnz);
    for (int64_t k = lo + lane; k < hi; k += 32) {
      const int64_t r = rowind[k];
      if (r < 0 || r >= rows) flag = 1;
      if (k > lo && rowind[k - 1] >= r) flag = 1;
    }
    if (__any_sync(0xffffffffu, flag) && lane == 0) atomicOr(bad, 1);
  }
}

__global__ void csc_scatter_kernel(const int64_t* __restrict__ colptr, const int64_t* __restrict__ rowind,
                                   const double* __restrict__ vals, int64_t cols, int transposed,
                                   double* __restrict__ Ad, int64_t ldp) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t j = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); j < cols; j += warps) {
    const int64_t b = colptr[j], e = colptr[j + 1];
    for (int64_t k = b + lane; k < e; k += 32) {
      const int64_t r = rowind[k];
      if (transposed)
        Ad[r * ldp + j] = vals[k];
      else
        Ad[j * ldp + r] = vals[k];
    }
  }
}

// *bad |= 1 if any entry is NaN or +-Inf (problem.hpp:56-58, :29-33). A flag rather than a sum of
// squares, which would overflow for finite entries above ~1e154.
__global__ void nonfinite_kernel(const double* __restrict__ a, long long count, int* __restrict__ bad) {
  int f = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x)
    f |= !isfinite(a[i]);
  if (__any_sync(0xffffffffu, f) && (threadIdx.x & 31) == 0) atomicOr(bad, 1);
}

namespace {
int warp_grid(int64_t cols) {
  // 8 warps per CTA; enough CTAs to cover the columns, capped at 148 SMs x 8 resident CTAs
  return (int)std::max<int64_t>(1, std::min<int64_t>((cols + 7) / 8, 148 * 8));
}
}  // namespace

cudaError_t csc_check(const int64_t* colptr, const int64_t* rowind, int64_t rows, int64_t cols, int64_t nnz,
                      int* bad, cudaStream_t s) {
  csc_check_kernel<<<warp_grid(cols), 256, 0, s>>>(colptr, rowind, rows, cols, nnz, bad);
  note_launch();
  return cudaGetLastError();
}

cudaError_t csc_scatter(const int64_t* colptr, const int64_t* rowind, const double* vals, int64_t cols,
                        bool transposed, double* Ad, int64_t ldp, cudaStream_t s) {
  csc_scatter_kernel<<<warp_grid(cols), 256, 0, s>>>(colptr, rowind, vals, cols, transposed ? 1 : 0, Ad, ldp);
  note_launch();
  return cudaGetLastError();
}

cudaError_t any_nonfinite(const double* a, long long count, int* bad, cudaStream_t s) {
  const int blocks = (int)std::max<long long>(1, std::min<long long>((count + 255) / 256, 148 * 8));
  nonfinite_kernel<<<blocks, 256, 0, s>>>(a, count, bad);
  note_launch();
  return cudaGetLastError();
}

}  // namespace sssvd_gpu
