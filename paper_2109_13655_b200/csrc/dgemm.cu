// Real FP64 GEMMs of the dense tail on the FP64 tensor cores (DMMA), column-major.
//
// Replaces the Eigen dense products of the extraction and postprocess steps of run_solve:
//   moments.hpp:207        U_S1 = Q U_R                   extract.hpp:46       A U_S1
//   extract.hpp:48,50      the Householder WY updates of HouseholderQR / householderQ()
//   extract.hpp:96-97      U~ p_i, U_S1 q_i               extract.hpp:112      U_S1^T G U_S1
//   postprocess.hpp:36-39  A^T u_i - sigma_i v_i          postprocess.hpp:91-93 S+ W Sigma^+ q_i
//   pipeline.hpp:203-208   A v_i - sigma_i u_i
// as   C (m x n) = alpha op(A) B + beta C,   op(A) = A (m x k, lda) or A^T (A stored k x m),
// and the residual form  out_j = || op(A) B[:, j] - d_j V[:, j] ||_2  with the subtraction and the
// column sums of squares fused into the epilogue (op(A) B is never written).
//
// CTA tile 64 x 64, 4 warps of 32 x 32 (4 x 4 DMMA m8n8k4 sub-tiles per warp, 32 accumulators per
// thread), K staged 16 deep through a 4-stage cp.async ring. Tile layouts in shared memory keep
// every fragment load conflict-free (a half-warp touches 16 distinct bank pairs):
//   op(A) = A   : [k][i], pitch 68  (global columns of A are contiguous along i)
//   op(A) = A^T : [i][k], pitch 20  (contiguous along k)         B : [j][k], pitch 20
// Operands whose base or leading dimension is not 16-byte aligned are staged 8 bytes per copy.
// Skinny outputs with deep K (fewer tiles than two waves of SMs: the Householder panel updates
// Y^T A, the block Gram Y^T Y) split K over blockIdx.z into a workspace that a second kernel sums
// in fixed z order, so every result is deterministic (no atomics anywhere).
#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace sssvd_gpu {
namespace {

constexpr int TBM = 64, TBN = 64, TBK = 16, TST = 4, TTHREADS = 128;
constexpr int PK = TBM + 4;   // [k][i] pitch
constexpr int PI = TBK + 4;   // [i][k] / [j][k] pitch
constexpr int A_ELEMS = (TBK * PK > TBM * PI) ? TBK * PK : TBM * PI;
constexpr int B_ELEMS = TBN * PI;
constexpr int STAGE = A_ELEMS + B_ELEMS;
constexpr size_t SMEM_BYTES = (size_t)TST * STAGE * sizeof(double);

enum { EPI_STORE = 0, EPI_SPLIT = 1, EPI_NORM = 2 };

// cp.async of VEC doubles (16 or 8 bytes) with src_bytes valid bytes; the rest is zero-filled
template <int VEC>
__device__ __forceinline__ void cp_vec(double* dst, const double* src, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  if (VEC == 2)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(src), "r"(src_bytes));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(src), "r"(src_bytes));
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// Operand contiguous along k (op(A) = A^T, and B): tile rows r (64) x k (16) -> smem [r][k].
template <int VEC>
struct RowLoader {
  static constexpr int C = TBK / VEC;              // chunks per tile row
  static constexpr int NP = TBM * C / TTHREADS;    // chunks per thread
  static constexpr int RSTEP = TTHREADS / C;       // tile-row step between a thread's chunks
  const double* g;
  long long rstep;
  int dst, kc, k, ke;
  unsigned rows_ok;
  __device__ __forceinline__ void init(const double* base, int ld, int r0, int R, int kb, int kend, int tid) {
    const int r = tid / C;
    kc = (tid % C) * VEC;
    g = base + (size_t)(r0 + r) * ld + kb + kc;
    rstep = (long long)RSTEP * ld;
    dst = r * PI + kc;
    k = kb;
    ke = kend;
    rows_ok = 0;
#pragma unroll
    for (int p = 0; p < NP; ++p) rows_ok |= (r0 + r + p * RSTEP < R ? 1u : 0u) << p;
  }
  __device__ __forceinline__ void load(double* tile, const double* fallback) {
    const int bytes = 8 * clampi(ke - (k + kc), 0, VEC);
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const bool ok = ((rows_ok >> p) & 1u) && bytes > 0;
      cp_vec<VEC>(tile + dst + p * RSTEP * PI, ok ? g + p * rstep : fallback, ok ? bytes : 0);
    }
    g += TBK;
    k += TBK;
  }
};

// op(A) = A (column-major, contiguous along i): tile k (16) x rows i (64) -> smem [k][i].
template <int VEC>
struct ColLoader {
  static constexpr int C = TBM / VEC;              // chunks per k-column
  static constexpr int NP = TBK * C / TTHREADS;
  static constexpr int KSTEP = TTHREADS / C;
  const double* g;
  long long kstep, kadv;
  int dst, kk, k, ke, bytes;
  __device__ __forceinline__ void init(const double* base, int ld, int m0, int M, int kb, int kend, int tid) {
    kk = tid / C;
    const int ic = (tid % C) * VEC;
    g = base + (size_t)(m0 + ic) + (size_t)(kb + kk) * ld;
    kstep = (long long)KSTEP * ld;
    kadv = (long long)TBK * ld;
    dst = kk * PK + ic;
    k = kb;
    ke = kend;
    bytes = 8 * clampi(M - (m0 + ic), 0, VEC);
  }
  __device__ __forceinline__ void load(double* tile, const double* fallback) {
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const bool ok = bytes > 0 && k + kk + p * KSTEP < ke;
      cp_vec<VEC>(tile + dst + p * KSTEP * PK, ok ? g + p * kstep : fallback, ok ? bytes : 0);
    }
    g += kadv;
    k += TBK;
  }
};

template <bool TA, int VA>
struct ALoader;
template <int VA>
struct ALoader<false, VA> : ColLoader<VA> {};
template <int VA>
struct ALoader<true, VA> : RowLoader<VA> {};

template <bool TA, int VA, int VB, int EPI>
__global__ void __launch_bounds__(TTHREADS, 2)
dgemm_kernel(int M, int N, int K, int kchunk, double alpha, const double* __restrict__ A, int lda,
             const double* __restrict__ B, int ldb, double beta, double* C, int ldc, const double* __restrict__ d,
             const double* __restrict__ V, int ldv, double* __restrict__ part) {
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  const int fr = lane >> 2, fc = lane & 3;
  const int m0 = blockIdx.y * TBM, n0 = blockIdx.x * TBN;
  const int kb = blockIdx.z * kchunk, ke = min(K, kb + kchunk);
  const int KT = ke > kb ? (ke - kb + TBK - 1) / TBK : 0;

  ALoader<TA, VA> la;
  la.init(A, lda, m0, M, kb, ke, tid);
  RowLoader<VB> lb;
  lb.init(B, ldb, n0, N, kb, ke, tid);

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < TST - 1; ++s) {
    if (s < KT) {
      la.load(sm + s * STAGE, A);
      lb.load(sm + s * STAGE + A_ELEMS, B);
    }
    cp_async_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<TST - 2>();
    __syncthreads();
    const int nk = kt + TST - 1;
    if (nk < KT) {
      la.load(sm + (nk % TST) * STAGE, A);
      lb.load(sm + (nk % TST) * STAGE + A_ELEMS, B);
    }
    cp_async_commit();
    const double* as = sm + (kt % TST) * STAGE;
    const double* bs = as + A_ELEMS + (wn * 32 + fr) * PI + fc;
#pragma unroll
    for (int kq = 0; kq < TBK / 4; ++kq) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        a[i] = TA ? as[(wm * 32 + i * 8 + fr) * PI + kq * 4 + fc] : as[(kq * 4 + fc) * PK + wm * 32 + i * 8 + fr];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = bs[j * 8 * PI + kq * 4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  cp_async_wait<0>();

  if (EPI == EPI_NORM) {
    // (acc - d_c V[r, c])^2 summed over the CTA's 64 rows, in fixed order: sub-tiles i, then the
    // fragment rows (lane bits 2..4), then the two row warps
    double cs[4][2];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = n0 + wn * 32 + j * 8 + 2 * fc + e;
        double sum = 0.0;
        if (c < N) {
          const double dc = d[c];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int r = m0 + wm * 32 + i * 8 + fr;
            if (r < M) {
              const double v = acc[i][j][e] - dc * V[(size_t)r + (size_t)c * ldv];
              sum = fma(v, v, sum);
            }
          }
        }
        cs[j][e] = sum;
      }
#pragma unroll
    for (int off = 4; off < 32; off <<= 1)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) cs[j][e] += __shfl_xor_sync(0xffffffffu, cs[j][e], off);
    __syncthreads();
    double* red = sm;   // [2][64]
    if (fr == 0) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) red[wm * 64 + wn * 32 + j * 8 + 2 * fc + e] = cs[j][e];
    }
    __syncthreads();
    if (tid < TBN && n0 + tid < N) part[(size_t)blockIdx.y * N + n0 + tid] = red[tid] + red[64 + tid];
    return;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = m0 + wm * 32 + i * 8 + fr;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = n0 + wn * 32 + j * 8 + 2 * fc + e;
        if (c >= N) continue;
        if (EPI == EPI_SPLIT) {
          part[(size_t)blockIdx.z * M * N + (size_t)r + (size_t)c * M] = acc[i][j][e];
        } else {
          double* cp = C + (size_t)r + (size_t)c * ldc;
          *cp = beta == 0.0 ? alpha * acc[i][j][e] : fma(alpha, acc[i][j][e], beta * *cp);
        }
      }
  }
}

// C = alpha sum_z part[z] + beta C, z ascending
__global__ void split_reduce_kernel(const double* __restrict__ part, int S, int M, int N, double alpha, double beta,
                                    double* C, int ldc) {
  const long long total = (long long)M * N;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    double s = part[e];
    for (int z = 1; z < S; ++z) s += part[(size_t)z * total + e];
    const int r = (int)(e % M), c = (int)(e / M);
    double* cp = C + (size_t)r + (size_t)c * ldc;
    *cp = beta == 0.0 ? alpha * s : fma(alpha, s, beta * *cp);
  }
}

// out[c] = sqrt(sum over row tiles t of part[t][c]), t ascending
__global__ void norm_finish_kernel(const double* __restrict__ part, int tiles, int N, double* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  double s = 0.0;
  for (int t = 0; t < tiles; ++t) s += part[(size_t)t * N + c];
  out[c] = sqrt(s);
}

bool aligned16(const double* p, int ld) { return ((uintptr_t)p & 15) == 0 && (ld & 1) == 0; }

template <bool TA, int VA, int VB, int EPI>
cudaError_t launch_k(dim3 grid, cudaStream_t s, int M, int N, int K, int kchunk, double alpha, const double* A, int lda,
                     const double* B, int ldb, double beta, double* C, int ldc, const double* d, const double* V, int ldv,
                     double* part) {
  auto kern = dgemm_kernel<TA, VA, VB, EPI>;
  SSSVD_CUDA_TRY(set_kernel_smem((const void*)kern, SMEM_BYTES, false));
  kern<<<grid, TTHREADS, SMEM_BYTES, s>>>(M, N, K, kchunk, alpha, A, lda, B, ldb, beta, C, ldc, d, V, ldv, part);
  note_launch();
  return cudaGetLastError();
}

template <int EPI>
cudaError_t dispatch(bool ta, bool va, bool vb, dim3 grid, cudaStream_t s, int M, int N, int K, int kchunk, double alpha,
                     const double* A, int lda, const double* B, int ldb, double beta, double* C, int ldc, const double* d,
                     const double* V, int ldv, double* part) {
#define SSSVD_DG(T, X, Y) \
  return launch_k<T, X, Y, EPI>(grid, s, M, N, K, kchunk, alpha, A, lda, B, ldb, beta, C, ldc, d, V, ldv, part)
  if (ta) {
    if (va) { if (vb) SSSVD_DG(true, 2, 2); else SSSVD_DG(true, 2, 1); }
    else { if (vb) SSSVD_DG(true, 1, 2); else SSSVD_DG(true, 1, 1); }
  } else {
    if (va) { if (vb) SSSVD_DG(false, 2, 2); else SSSVD_DG(false, 2, 1); }
    else { if (vb) SSSVD_DG(false, 1, 2); else SSSVD_DG(false, 1, 1); }
  }
#undef SSSVD_DG
}

}  // namespace

int dgemm_split_count(int m, int n, int k, size_t work_elems) {
  const long long tiles = (long long)((m + TBM - 1) / TBM) * ((n + TBN - 1) / TBN);
  if (tiles >= 2 * 148 || k < 512 || work_elems == 0) return 1;
  long long S = std::min<long long>((2 * 148 + tiles - 1) / tiles, k / 256);
  S = std::min<long long>(S, 64);
  while (S > 1 && (size_t)S * m * n > work_elems) --S;
  return (int)std::max<long long>(S, 1);
}

cudaError_t dgemm(bool ta, int m, int n, int k, double alpha, const double* A, int lda, const double* B, int ldb,
                  double beta, double* C, int ldc, double* work, size_t work_elems, cudaStream_t s) {
  if (m <= 0 || n <= 0) return cudaSuccess;
  k = std::max(k, 0);
  int S = dgemm_split_count(m, n, k, work_elems);
  int kchunk = k;
  if (S > 1) {
    kchunk = ((k + S - 1) / S + TBK - 1) / TBK * TBK;
    S = (k + kchunk - 1) / kchunk;
  }
  const dim3 grid((n + TBN - 1) / TBN, (m + TBM - 1) / TBM, S);
  const bool va = aligned16(A, lda), vb = aligned16(B, ldb);
  if (S == 1)
    return dispatch<EPI_STORE>(ta, va, vb, grid, s, m, n, k, std::max(kchunk, 1), alpha, A, lda, B, ldb, beta, C, ldc,
                               nullptr, nullptr, 0, nullptr);
  SSSVD_CUDA_TRY(dispatch<EPI_SPLIT>(ta, va, vb, grid, s, m, n, k, kchunk, 1.0, A, lda, B, ldb, 0.0, nullptr, 0,
                                     nullptr, nullptr, 0, work));
  const long long total = (long long)m * n;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 8);
  split_reduce_kernel<<<blocks, 256, 0, s>>>(work, S, m, n, alpha, beta, C, ldc);
  note_launch();
  return cudaGetLastError();
}

size_t dgemm_norm_scratch(int m, int n) { return (size_t)((m + TBM - 1) / TBM) * n; }

cudaError_t dgemm_colnorm_diff(bool ta, int m, int n, int k, const double* A, int lda, const double* B, int ldb,
                               const double* d, const double* V, int ldv, double* out, double* part, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int tiles = (m + TBM - 1) / TBM;
  if (m <= 0) return cudaMemsetAsync(out, 0, sizeof(double) * n, s);
  const dim3 grid((n + TBN - 1) / TBN, tiles, 1);
  SSSVD_CUDA_TRY(dispatch<EPI_NORM>(ta, aligned16(A, lda), aligned16(B, ldb), grid, s, m, n, std::max(k, 0),
                                    std::max(k, 1), 1.0, A, lda, B, ldb, 0.0, nullptr, 0, d, V, ldv, part));
  norm_finish_kernel<<<(n + 127) / 128, 128, 0, s>>>(part, tiles, n, out);
  note_launch();
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------- transpose
// out (cols x rows, ldo) = in^T (in: rows x cols, ldi), column-major; 32 x 32 tiles through
// shared memory (padded pitch: conflict-free both ways)
__global__ void transpose_kernel(const double* __restrict__ in, int rows, int cols, int ldi, double* __restrict__ out,
                                 int ldo) {
  __shared__ double t[32][33];
  const int r0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int r = r0 + threadIdx.x, c = c0 + y;
    if (r < rows && c < cols) t[y][threadIdx.x] = in[(size_t)r + (size_t)c * ldi];
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int c = c0 + threadIdx.x, r = r0 + y;
    if (r < rows && c < cols) out[(size_t)c + (size_t)r * ldo] = t[threadIdx.x][y];
  }
}

cudaError_t transpose(const double* in, int rows, int cols, int ldi, double* out, int ldo, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  transpose_kernel<<<dim3((rows + 31) / 32, (cols + 31) / 32), dim3(32, 8), 0, s>>>(in, rows, cols, ldi, out, ldo);
  note_launch();
  return cudaGetLastError();
}

// h <- (h + h^T) / 2 in place (extract.hpp:113), k x k column-major
__global__ void symmetrize_kernel(double* h, int k, int ldh) {
  const long long total = (long long)k * k;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % k), j = (int)(e / k);
    if (i <= j) continue;   // the lower-triangle thread owns the pair
    const double v = (h[(size_t)i + (size_t)j * ldh] + h[(size_t)j + (size_t)i * ldh]) / 2.0;
    h[(size_t)i + (size_t)j * ldh] = v;
    h[(size_t)j + (size_t)i * ldh] = v;
  }
}

cudaError_t symmetrize(double* h, int k, int ldh, cudaStream_t s) {
  if (k <= 0) return cudaSuccess;
  const long long total = (long long)k * k;
  symmetrize_kernel<<<(int)std::min<long long>((total + 255) / 256, 148 * 8), 256, 0, s>>>(h, k, ldh);
  note_launch();
  return cudaGetLastError();
}

// sgn[j] = sign(U[:, j] . V[:, j]) (+1 for a zero dot), one warp per column
__global__ void col_dot_sign_kernel(const double* __restrict__ U, const double* __restrict__ V, int rows, int cols,
                                    double* __restrict__ sgn) {
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (c >= cols) return;
  double s = 0.0;
  for (int r = lane; r < rows; r += 32) s = fma(U[(size_t)r + (size_t)c * rows], V[(size_t)r + (size_t)c * rows], s);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) sgn[c] = s < 0.0 ? -1.0 : 1.0;
}

cudaError_t col_dot_sign(const double* U, const double* V, int rows, int cols, double* sgn, cudaStream_t s) {
  if (cols <= 0) return cudaSuccess;
  col_dot_sign_kernel<<<(cols + 7) / 8, 256, 0, s>>>(U, V, rows, cols, sgn);
  note_launch();
  return cudaGetLastError();
}

}  // namespace sssvd_gpu
