// K7: fused moment accumulation, plus the small HBM-bound kernels of the tail.
//
// Reference: MomentAccumulator::accumulate (proj/include/sssvd/moments.hpp:132-147)
//   for k in 0..M: for j ascending: S_k += 2 Re(w_j t_j^k X_j); power_j *= t_j
// which re-reads every X_j M+1 times on one CPU thread. Here every X_j element is read once
// and all M+1 outputs are updated from registers. The coefficient table c[k][j] = w_j t_j^k is
// formed on the host with the reference's own std::complex power chain, and the real part is
// evaluated as 2*(cr*xr - ci*xi) with explicitly rounded (non-fused) operations, in ascending j
// for every k: given identical X_j the result is bitwise the reference's.
#include "common.cuh"
#include "kernels.h"

namespace sssvd_gpu {


// S is row-major [(M+1)][n][L]; X_j = rows 0..n-1, columns xcol..xcol+L-1 of mats[j].
// MMAX: compile-time bound on M (accumulators in registers), instantiated for 8, 16 and 32.
template <int MMAX>
__global__ void __launch_bounds__(256)
moments_kernel(const double2* __restrict__ mats, int ld, long long stride, int xcol, int n, int L,
               int nb, const double2* __restrict__ coef, int M, double* __restrict__ S) {
  extern __shared__ double2 cs[];   // [(M+1)][nb]
  for (int t = threadIdx.x; t < (M + 1) * nb; t += blockDim.x) cs[t] = coef[t];
  __syncthreads();
  const long long nl = (long long)n * L;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nl;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / L), c = (int)(e % L);
    double acc[MMAX + 1];
#pragma unroll
    for (int k = 0; k <= MMAX; ++k)
      if (k <= M) acc[k] = S[k * nl + e];
    // X_j loads in chunks of MCH shifts, all in flight before the (ascending-j) accumulation
    constexpr int MCH = 8;
    const double2* xp = mats + (size_t)i * ld + xcol + c;
    for (int j0 = 0; j0 < nb; j0 += MCH) {
      double2 xs[MCH];
#pragma unroll
      for (int u = 0; u < MCH; ++u) xs[u] = j0 + u < nb ? __ldcs(xp + (j0 + u) * stride) : make_double2(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < MCH; ++u) {
        if (j0 + u < nb) {
          const double2 x = xs[u];
          const int j = j0 + u;
#pragma unroll
          for (int k = 0; k <= MMAX; ++k) {
            if (k <= M) {
              const double2 w = cs[k * nb + j];
              const double re = __dsub_rn(__dmul_rn(w.x, x.x), __dmul_rn(w.y, x.y));
              acc[k] = __dadd_rn(acc[k], 2.0 * re);
            }
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k <= MMAX; ++k)
      if (k <= M) S[k * nl + e] = acc[k];
  }
}

cudaError_t moments(const double2* mats, int ld, long long stride, int xcol, int n, int L, int nb,
                    const double2* coef, int M, double* S, cudaStream_t s) {
  const long long nl = (long long)n * L;
  int blocks = (int)std::min<long long>((nl + 255) / 256, 148 * 8);
  // degrees in chunks of at most 33 (the register-resident accumulators): any M the reference
  // accepts (L M <= n) works; each chunk re-reads X_j once
  for (int k0 = 0; k0 <= M; k0 += 33) {
    const int mc = std::min(M - k0, 32);
    const double2* cc = coef + (size_t)k0 * nb;
    double* Sk = S + (size_t)k0 * nl;
    const size_t smem = (size_t)(mc + 1) * nb * sizeof(double2);
    if (mc <= 8)
      moments_kernel<8><<<blocks, 256, smem, s>>>(mats, ld, stride, xcol, n, L, nb, cc, mc, Sk);
    else if (mc <= 16)
      moments_kernel<16><<<blocks, 256, smem, s>>>(mats, ld, stride, xcol, n, L, nb, cc, mc, Sk);
    else
      moments_kernel<32><<<blocks, 256, smem, s>>>(mats, ld, stride, xcol, n, L, nb, cc, mc, Sk);
    note_launch();
  }
  return cudaGetLastError();
}

// [(M+1)][n][L] row-major  ->  column-major blocks [(M+1)][L][n] (stacked n x (M+1)L matrix)
__global__ void blocks_to_colmajor_kernel(const double* __restrict__ S, int n, int L, int nblk,
                                          double* __restrict__ out) {
  __shared__ double tile[32][33];
  const int k = blockIdx.z;
  const double* Sk = S + (size_t)k * n * L;
  double* Ok = out + (size_t)k * n * L;
  const int i0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    int i = i0 + r, c = c0 + threadIdx.x;
    if (i < n && c < L) tile[r][threadIdx.x] = Sk[(size_t)i * L + c];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    int c = c0 + r, i = i0 + threadIdx.x;
    if (i < n && c < L) Ok[(size_t)c * n + i] = tile[threadIdx.x][r];
  }
  (void)nblk;
}

cudaError_t blocks_to_colmajor(const double* S, int n, int L, int nblk, double* out, cudaStream_t s) {
  dim3 grid((n + 31) / 32, (L + 31) / 32, nblk);
  blocks_to_colmajor_kernel<<<grid, dim3(32, 8), 0, s>>>(S, n, L, nblk, out);
  note_launch();
  return cudaGetLastError();
}

// out[j] = || X[:, j] - s_j * Y[:, j] ||_2 for column-major X (ldx), Y (ldy), rows x cols.
// s == nullptr means s_j = 0. The residual kernel of the tail (postprocess.hpp:36-39 exact
// residual, pipeline.hpp:205-207 Galerkin, :91-95 estimate). HBM-bound: grid (column, row chunk
// of CN_ROWS), 8 independent loads in flight per thread, per-chunk partial sums, then one warp
// per column adds its chunks in a fixed order (deterministic) and takes the root.
constexpr int CN_THREADS = 256, CN_UNROLL = 8, CN_ROWS = CN_THREADS * CN_UNROLL;
__global__ void __launch_bounds__(CN_THREADS)
colnorm_partial_kernel(const double* __restrict__ X, int ldx, const double* __restrict__ Y, int ldy,
                       const double* __restrict__ s, int rows, double* __restrict__ part) {
  const int j = blockIdx.x, ch = blockIdx.y;
  const double sj = s ? s[j] : 0.0;
  const double* x = X + (size_t)j * ldx;
  const double* y = Y ? Y + (size_t)j * ldy : nullptr;
  const int r0 = ch * CN_ROWS + threadIdx.x;
  double xv[CN_UNROLL], yv[CN_UNROLL];
#pragma unroll
  for (int u = 0; u < CN_UNROLL; ++u) {
    const int r = r0 + u * CN_THREADS;
    xv[u] = r < rows ? __ldcs(x + r) : 0.0;
    yv[u] = (y && r < rows) ? __ldcs(y + r) : 0.0;
  }
  double acc = 0.0;
#pragma unroll
  for (int u = 0; u < CN_UNROLL; ++u) {
    const double v = xv[u] - sj * yv[u];
    acc += v * v;
  }
  __shared__ double red[CN_THREADS / 32];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < CN_THREADS / 32 ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (threadIdx.x == 0) part[(size_t)j * gridDim.y + ch] = acc;
  }
}

__global__ void colnorm_finish_kernel(const double* __restrict__ part, int chunks, int cols, double* __restrict__ out) {
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (j >= cols) return;
  double acc = 0.0;
  for (int c = lane; c < chunks; c += 32) acc += part[(size_t)j * chunks + c];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) out[j] = sqrt(acc);
}

size_t colnorm_scratch(int rows, int cols) { return (size_t)cols * ((rows + CN_ROWS - 1) / CN_ROWS); }

cudaError_t colnorm_diff(const double* X, int ldx, const double* Y, int ldy, const double* s, int rows,
                         int cols, double* out, double* part, cudaStream_t st) {
  if (cols <= 0) return cudaSuccess;
  const int chunks = (rows + CN_ROWS - 1) / CN_ROWS;
  colnorm_partial_kernel<<<dim3(cols, chunks), CN_THREADS, 0, st>>>(X, ldx, Y, ldy, s, rows, part);
  colnorm_finish_kernel<<<(cols + 7) / 8, 256, 0, st>>>(part, chunks, cols, out);
  note_launch(2);
  return cudaGetLastError();
}

// Spurious index and estimator coefficients of triplet i (one CTA per column of q, column-major
// rank x tcount), postprocess.hpp:56-60 and :86-93:
//   tau_i = ||q_i||^2 / sum_l q_li^2 / Sigma_l ,   qsc[:, i] = Sigma^+ q_i  (inv = Sigma^+ diagonal)
// (the sums are CTA reductions; the reference's order is Eigen's vectorised one, parity is by
// tolerance)
__global__ void tau_scale_kernel(const double* __restrict__ q, int rank, const double* __restrict__ sv,
                                 const double* __restrict__ inv, double* __restrict__ tau,
                                 double* __restrict__ qsc) {
  const int i = blockIdx.x;
  const double* qi = q + (size_t)i * rank;
  double num = 0.0, den = 0.0;
  for (int l = threadIdx.x; l < rank; l += blockDim.x) {
    const double v = qi[l], v2 = v * v;
    num += v2;
    den += v2 / sv[l];
    qsc[(size_t)i * rank + l] = inv[l] * v;
  }
  __shared__ double red[2][32];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    num += __shfl_xor_sync(0xffffffffu, num, off);
    den += __shfl_xor_sync(0xffffffffu, den, off);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = num;
    red[1][threadIdx.x >> 5] = den;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const bool in = threadIdx.x < (blockDim.x >> 5);
    num = in ? red[0][threadIdx.x] : 0.0;
    den = in ? red[1][threadIdx.x] : 0.0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      num += __shfl_xor_sync(0xffffffffu, num, off);
      den += __shfl_xor_sync(0xffffffffu, den, off);
    }
    if (threadIdx.x == 0) tau[i] = num / den;
  }
}

cudaError_t tau_scale(const double* q, int rank, int tcount, const double* sv, const double* inv, double* tau,
                      double* qsc, cudaStream_t st) {
  if (tcount <= 0) return cudaSuccess;
  tau_scale_kernel<<<tcount, 256, 0, st>>>(q, rank, sv, inv, tau, qsc);
  note_launch();
  return cudaGetLastError();
}

// dst[:, j] = src[:, perm[j]] * (scale ? scale[j] : 1)   (column gather, column-major)
__global__ void gather_cols_kernel(const double* __restrict__ src, int lds, const int* __restrict__ perm,
                                   const double* __restrict__ scale, int rows, double* __restrict__ dst,
                                   int ldd) {
  const int j = blockIdx.x;
  const double sc = scale ? scale[j] : 1.0;
  const double* s = src + (size_t)perm[j] * lds;
  double* d = dst + (size_t)j * ldd;
  for (int i = threadIdx.x; i < rows; i += blockDim.x) d[i] = s[i] * sc;
}

cudaError_t gather_cols(const double* src, int lds, const int* perm, const double* scale, int rows,
                        int cols, double* dst, int ldd, cudaStream_t st) {
  if (cols <= 0) return cudaSuccess;
  gather_cols_kernel<<<cols, 256, 0, st>>>(src, lds, perm, scale, rows, dst, ldd);
  note_launch();
  return cudaGetLastError();
}

// Frobenius norm squared (deterministic two-level reduction into out[0])
__global__ void sumsq_kernel(const double* __restrict__ a, long long count, double* __restrict__ partial) {
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x)
    acc += a[i] * a[i];
  __shared__ double red[32];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (threadIdx.x == 0) partial[blockIdx.x] = acc;
  }
}

__global__ void sum_partials_kernel(const double* __restrict__ partial, int cnt, double* out) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < cnt; i += 32) acc += partial[i];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (threadIdx.x == 0) out[0] = acc;
}

cudaError_t sumsq(const double* a, long long count, double* scratch /*>= 593 doubles*/, double* out,
                  cudaStream_t s) {
  const int blocks = 148 * 4;
  sumsq_kernel<<<blocks, 256, 0, s>>>(a, count, scratch);
  note_launch();
  sum_partials_kernel<<<1, 32, 0, s>>>(scratch, blocks, out);
  note_launch();
  return cudaGetLastError();
}

// column-major rows x cols (leading dim lds) -> column-major with leading dim ldd >= rows, zero rows beyond
__global__ void pad_copy_kernel(const double* __restrict__ src, int rows, int cols, int lds,
                                double* __restrict__ dst, int ldd) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)ldd * cols;
       e += (long long)gridDim.x * blockDim.x) {
    int c = (int)(e / ldd), r = (int)(e % ldd);
    dst[e] = r < rows ? src[(size_t)c * lds + r] : 0.0;
  }
}

cudaError_t pad_copy(const double* src, int rows, int cols, int lds, double* dst, int ldd, cudaStream_t s) {
  long long total = (long long)ldd * cols;
  int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 16);
  pad_copy_kernel<<<blocks, 256, 0, s>>>(src, rows, cols, lds, dst, ldd);
  note_launch();
  return cudaGetLastError();
}

}  // namespace sssvd_gpu
