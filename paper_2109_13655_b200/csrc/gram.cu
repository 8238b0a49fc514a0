// K0: Gram operator G = A^T A on the FP64 tensor cores, exactly symmetric.
//
// Replaces form_gram (proj/include/sssvd/problem.hpp:81-95): the reference forms the full
// product with Eigen and then symmetrises (G + G^T)/2. Here only the lower-triangle tiles are
// computed (half the flops) and mirrored, which makes G exactly symmetric by construction.
// A is column-major m x n with an even leading dimension lda (zero rows beyond m), so column i
// of A is row i of the k-contiguous operand: C[i][j] = sum_k P[i][k] P[j][k] (a "TN" GEMM).
// CTA tile 64x64, 4 warps (32x32 each), K staged 32 at a time through a 3-deep cp.async ring,
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4).
#include "common.cuh"
#include "kernels.h"
#include "partition.h"

namespace sssvd_gpu {

namespace {
constexpr int BM = kGramTile, BK = 32, STAGES = 3, THREADS = 128;
constexpr int LDS = BK + 4;  // 36 doubles (== 4 mod 16): conflict-free 8-byte fragment loads
constexpr int TILE = BM * LDS;

__device__ __forceinline__ void load_tile(double* Ps, double* Qs, const double* A, int lda, int n,
                                          int K, int i0, int j0, int k0, int tid) {
#pragma unroll
  for (int t = 0; t < (BM * BK / 2) / THREADS; ++t) {
    int idx = tid + t * THREADS;
    int r = idx / (BK / 2), kk = (idx % (BK / 2)) * 2;
    bool pi = (i0 + r < n) && (k0 + kk < K);
    bool pj = (j0 + r < n) && (k0 + kk < K);
    cp_async16(Ps + r * LDS + kk, pi ? A + (size_t)(i0 + r) * lda + k0 + kk : A, pi);
    cp_async16(Qs + r * LDS + kk, pj ? A + (size_t)(j0 + r) * lda + k0 + kk : A, pj);
  }
}
}  // namespace

// part/nparts: multi-GPU sharding - this launch computes the lower-triangle tiles
// t = part, part + nparts, ... (the other entries of G are left for the all-reduce)
__global__ void __launch_bounds__(THREADS, 2)
gram_kernel(const double* __restrict__ A, int lda, int K, int n, double* __restrict__ G, int ldg, int part,
            int nparts) {
  extern __shared__ __align__(16) double gsm[];
  double* Ps = gsm;
  double* Qs = gsm + STAGES * TILE;
  // decode lower-triangle tile (ti >= tj) from the linear block index
  const long long t = (long long)blockIdx.x * nparts + part;
  int ti, tj;
  gram_tile_decode(t, &ti, &tj);
  const int i0 = ti * BM, j0 = tj * BM;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  const int fr = lane >> 2, fc = lane & 3;

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int KT = (K + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_tile(Ps + s * TILE, Qs + s * TILE, A, lda, n, K, i0, j0, s * BK, tid);
    cp_async_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      int nk = kt + STAGES - 1;
      if (nk < KT) load_tile(Ps + (nk % STAGES) * TILE, Qs + (nk % STAGES) * TILE, A, lda, n, K, i0, j0, nk * BK, tid);
      cp_async_commit();
    }
    const double* ps = Ps + (kt % STAGES) * TILE + (wm * 32 + fr) * LDS + fc;
    const double* qs = Qs + (kt % STAGES) * TILE + (wn * 32 + fr) * LDS + fc;
#pragma unroll
    for (int kq = 0; kq < BK / 4; ++kq) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = ps[i * 8 * LDS + kq * 4];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = qs[j * 8 * LDS + kq * 4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = i0 + wm * 32 + i * 8 + fr;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = j0 + wn * 32 + j * 8 + 2 * fc + e;
        if (r < n && c < n && (ti != tj || r >= c)) {
          G[(size_t)r * ldg + c] = acc[i][j][e];
          G[(size_t)c * ldg + r] = acc[i][j][e];
        }
      }
    }
  }
}

cudaError_t gram(const double* A, int lda, int K, int n, double* G, int ldg, int part, int nparts, cudaStream_t s) {
  const size_t smem = (size_t)2 * STAGES * TILE * sizeof(double);
  SSSVD_CUDA_TRY(set_kernel_smem((const void*)gram_kernel, smem, false));
  const long long tiles = gram_tile_total(n);
  const long long mine = (tiles - part + nparts - 1) / nparts;
  if (mine <= 0) return cudaSuccess;
  gram_kernel<<<(unsigned)mine, THREADS, smem, s>>>(A, lda, K, n, G, ldg, part, nparts);
  note_launch();
  return cudaGetLastError();
}

}  // namespace sssvd_gpu
