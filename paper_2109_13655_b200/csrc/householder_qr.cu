// Householder QR of the tail (thin Q and R of an m x k column-major matrix, m >= k).
//
// Replaces the two HouseholderQR calls of the small dense tail: low_rank's QR of the stacked
// moments (proj/include/sssvd/moments.hpp:195-198) and project_qr's QR of A U_S1 (extract.hpp:
// 43-57), plus the preconditioning QR inside the Jacobi SVD. Same reflector convention as LAPACK
// dgeqrf / Eigen: beta = -sign(alpha) ||x||, tau = (beta - alpha) / beta, v = x / (alpha - beta)
// with v_0 = 1, so R and Q agree with the reference's to rounding.
//
// Blocked, compact-WY (LAPACK dgeqrf + dorgqr structure):
//   for each panel of w <= 32 columns at column j:
//     K1 qr_panel_kernel: one thread-block cluster factors A[j:m, j:j+w] with its rows split over
//        the CTAs and held in shared memory. Per column: a cluster-wide DSMEM reduction of the
//        tail norm (every CTA then derives the same beta / tau), then one of the w-1 dot products
//        v^T A[:, c'], then the rank-1 update of the CTA's own rows. A last reduction forms the
//        strictly upper part of Y^T Y, from which CTA 0 builds T (H_0..H_{w-1} = I - Y T Y^T).
//        Y (explicit unit diagonal and zeros) and T go to a workspace kept for the Q formation.
//     trailing columns: A[j:m, j+w:k] -= Y (T^T (Y^T A[j:m, j+w:k]))        (three DGEMMs)
//   Q = H_0 ... H_{p-1} [I_k; 0] by backward accumulation, Q[j:m, j:k] -= Y (T (Y^T Q[j:m, j:k])).
// The panel's 2w cluster reductions are the latency floor; the GEMMs carry the flops.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace sssvd_gpu {

namespace {
constexpr int QP_THREADS = 512;
constexpr int QP_WMAX = 32;
}  // namespace

// Cluster of `gridDim.x` CTAs; CTA c owns panel rows [c*rp, min((c+1)*rp, mp)) (relative to row j).
// Shared memory: P[w][rp] column-major, then the reduction slots.
// CLUSTER = false: a single CTA holds the whole panel; the cross-CTA exchanges become __syncthreads
// and local shared-memory reads (a one-CTA cluster barrier still pays the release/acquire fences).
template <bool CLUSTER>
__device__ __forceinline__ void qp_sync() {
  if constexpr (CLUSTER) cluster_sync_all();
  else __syncthreads();
}
template <bool CLUSTER>
__device__ __forceinline__ double qp_ld(const double* p, unsigned rank) {
  if constexpr (CLUSTER) return ld_dsmem_f64(dsmem_addr(p, rank));
  else return *p;
}

template <bool CLUSTER>
__global__ void __launch_bounds__(QP_THREADS, 1)
qr_panel_kernel(double* __restrict__ A, int lda, int m, int j, int w, int rp, double* __restrict__ Y, int ldy,
                double* __restrict__ Tout, double* __restrict__ tau_out) {
  extern __shared__ __align__(16) double qsm[];
  const int C = CLUSTER ? gridDim.x : 1;
  const unsigned crank = CLUSTER ? cluster_ctarank() : 0u;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int mp = m - j;
  const int lo = (int)crank * rp, hi = min(lo + rp, mp);
  const int nloc = max(hi - lo, 0);
  rp |= 1;                                          // odd pitch: conflict-free column-strided reads
  double* P = qsm;                                  // [w][rp]
  double* red1 = P + (size_t)w * rp;                // [2]: tail norm partial, alpha
  double* red2 = red1 + 2;                          // [QP_WMAX]: dot partials
  double* red3 = red2 + QP_WMAX;                    // [QP_WMAX * QP_WMAX]: Gram partial
  double* wsum = red3 + QP_WMAX * QP_WMAX;          // [QP_WMAX]: reduced dots
  double* wred = wsum + QP_WMAX;                    // [32][QP_WMAX]: per-warp partials, then G
  __shared__ double taus[QP_WMAX];
  __shared__ double gram[QP_WMAX * QP_WMAX];   // G[a][b] = y_a . y_b (a < b), filled column by column

  // panel rows -> shared memory (coalesced over rows)
  for (int c = 0; c < w; ++c)
    for (int i = tid; i < nloc; i += QP_THREADS) P[(size_t)c * rp + i] = A[(size_t)(j + c) * lda + j + lo + i];
  __syncthreads();

  for (int c = 0; c < w; ++c) {
    // ---- tail norm of column c below the diagonal (global relative row c)
    double ss = 0.0;
    for (int i = tid; i < nloc; i += QP_THREADS) {
      const int gi = lo + i;
      if (gi > c) {
        const double x = P[(size_t)c * rp + i];
        ss = fma(x, x, ss);
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    if (lane == 0) wred[warp] = ss;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int q = 0; q < QP_THREADS / 32; ++q) t += wred[q];
      red1[0] = t;
      red1[1] = (c >= lo && c < hi) ? P[(size_t)c * rp + (c - lo)] : 0.0;
    }
    qp_sync<CLUSTER>();
    // every CTA reduces the same partials in the same order: identical beta / tau everywhere
    double tail2 = 0.0, alpha = 0.0;
    for (int q = 0; q < C; ++q) {
      tail2 += qp_ld<CLUSTER>(red1, q);
      alpha += qp_ld<CLUSTER>(red1 + 1, q);
    }
    double tau = 0.0, beta = alpha, scale = 0.0;
    if (tail2 > 0.0) {
      beta = -copysign(sqrt(fma(alpha, alpha, tail2)), alpha);
      tau = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    if (tid == 0) taus[c] = tau;
    // v = x / (alpha - beta) below the diagonal (v_c = 1 implicit)
    for (int i = tid; i < nloc; i += QP_THREADS)
      if (lo + i > c) P[(size_t)c * rp + i] *= scale;
    __syncthreads();
    // ---- one reduction gives w_c' = v^T A[:, c'] for c' > c AND the Gram column
    //      G[q][c] = y_q^T y_c for q < c (y_c vanishes above row c, so only rows >= c contribute
    //      and there P[q] already holds y_q): T needs G, and no separate Y^T Y pass is required
    {
      double acc[QP_WMAX];
#pragma unroll
      for (int q = 0; q < QP_WMAX; ++q) acc[q] = 0.0;
      for (int i = tid; i < nloc; i += QP_THREADS) {
        const int gi = lo + i;
        if (gi < c) continue;
        const double v = gi == c ? 1.0 : P[(size_t)c * rp + i];
#pragma unroll
        for (int q = 0; q < QP_WMAX; ++q)
          if (q != c && q < w) acc[q] = fma(v, P[(size_t)q * rp + i], acc[q]);
      }
      // transpose-reduce the 32 partials across the warp (31 shuffle-adds): lane l ends up with
      // the warp sum of value l; then across warps through shared memory
#pragma unroll
      for (int h = 16; h >= 1; h >>= 1) {
        const bool upper = (lane & h) != 0;
#pragma unroll
        for (int q = 0; q < h; ++q) {
          const double send = upper ? acc[q] : acc[q + h];
          const double keep = upper ? acc[q + h] : acc[q];
          acc[q] = keep + __shfl_xor_sync(0xffffffffu, send, h);
        }
      }
      wred[warp * QP_WMAX + lane] = acc[0];
      __syncthreads();
      if (tid < w && tid != c) {
        double t = 0.0;
        for (int q = 0; q < QP_THREADS / 32; ++q) t += wred[q * QP_WMAX + tid];
        red2[tid] = t;
      }
      qp_sync<CLUSTER>();
      if (tid < w && tid != c) {
        double t = 0.0;
        for (int q = 0; q < C; ++q) t += qp_ld<CLUSTER>(red2 + tid, q);
        if (tid > c) wsum[tid] = tau * t;
        else gram[tid * QP_WMAX + c] = t;   // G[tid][c]
      }
      __syncthreads();
      // rank-1 update of this CTA's rows i >= c of the columns c' > c
      for (int i = tid; i < nloc; i += QP_THREADS) {
        const int gi = lo + i;
        if (gi < c) continue;
        const double v = gi == c ? 1.0 : P[(size_t)c * rp + i];
        for (int q = c + 1; q < w; ++q) P[(size_t)q * rp + i] = fma(-wsum[q], v, P[(size_t)q * rp + i]);
      }
    }
    // diagonal: R[c][c] = beta
    if (tid == 0 && c >= lo && c < hi) P[(size_t)c * rp + (c - lo)] = beta;
    __syncthreads();
  }

  // ---- write back: A holds R on/above the diagonal and v below; Y explicit (unit diagonal, zeros)
  for (int c = 0; c < w; ++c)
    for (int i = tid; i < nloc; i += QP_THREADS) {
      const int gi = lo + i;
      const double p = P[(size_t)c * rp + i];
      A[(size_t)(j + c) * lda + j + gi] = p;
      Y[(size_t)c * ldy + gi] = gi < c ? 0.0 : (gi == c ? 1.0 : p);
    }
  // red2 may still be read remotely by slower CTAs of the last column
  qp_sync<CLUSTER>();
  if (crank == 0 && warp == 0) {
    // dlarft (forward, columnwise): T[b][b] = tau_b, T[0:b, b] = -tau_b T[0:b, 0:b] G[0:b, b];
    // columns in order, lane a owns row a; T is staged in shared memory (red3 is free now)
    double* Ts = red3;   // [32][32] column-major
    for (int b = 0; b < QP_WMAX; ++b) {
      const double tb = b < w ? taus[b] : 0.0;
      double t = 0.0;
      if (lane < b && b < w)
        for (int q = lane; q < b; ++q) t = fma(Ts[q * QP_WMAX + lane], gram[q * QP_WMAX + b], t);
      Ts[b * QP_WMAX + lane] = lane < b ? -tb * t : (lane == b ? tb : 0.0);
      __syncwarp();
    }
    for (int e = lane; e < QP_WMAX * QP_WMAX; e += 32) Tout[e] = Ts[e];
    if (lane < w) tau_out[lane] = taus[lane];
  }
  // keep every CTA's shared memory alive until the remote reads above have finished
  qp_sync<CLUSTER>();
}

size_t qr_panel_smem(int rp, int w) {
  rp |= 1;
  return ((size_t)w * rp + 2 + QP_WMAX + QP_WMAX * QP_WMAX + QP_WMAX + QP_WMAX * QP_WMAX) * sizeof(double);
}

// rows per CTA and cluster size for a panel of mp rows and width w: the smallest cluster whose row
// slices fit (at most 512 rows per CTA unless 16 CTAs are needed); 0 if even 16 CTAs do not fit
int qr_panel_plan(int mp, int w, int* cluster) {
  for (int c = 1; c <= 16; c *= 2) {
    const int rp = (mp + c - 1) / c;
    if (qr_panel_smem(rp, w) <= 200 * 1024 && (rp <= (c == 1 ? 1024 : 512) || c == 16)) {
      *cluster = c;
      return rp;
    }
  }
  return 0;
}

cudaError_t qr_panel(double* A, int lda, int m, int j, int w, double* Y, int ldy, double* T, double* tau,
                     cudaStream_t s) {
  if (w < 1 || w > QP_WMAX) return cudaErrorInvalidValue;
  int C = 1;
  const int rp = qr_panel_plan(m - j, w, &C);
  if (rp == 0) return cudaErrorInvalidValue;
  const size_t smem = qr_panel_smem(rp, w);
  for (auto fn : {qr_panel_kernel<true>, qr_panel_kernel<false>}) SSSVD_CUDA_TRY(set_kernel_smem((const void*)fn, smem, true));
  cudaError_t e;
  if (C == 1) {
    qr_panel_kernel<false><<<1, QP_THREADS, smem, s>>>(A, lda, m, j, w, rp, Y, ldy, T, tau);
    e = cudaGetLastError();
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C, 1, 1);
    cfg.blockDim = dim3(QP_THREADS, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, qr_panel_kernel<true>, A, lda, m, j, w, rp, Y, ldy, T, tau);
  }
  note_launch();
  return e;
}

// ----------------------------------------------------------------------------- register panel
// Same panel factorisation with the panel held in REGISTERS: 256 threads per CTA, thread t owns
// rows lo + t + 256 r (r < RPT = 64 / W) of all W columns (64 doubles per thread). Per column: one
// CTA + cluster reduction for the tail norm, then one for the W dot products v^T A[:, q] (which
// also yield the Gram column y_q^T y_c for q < c), then the rank-1 update in registers. The
// shared-memory panel kernel above re-read the whole panel from shared memory for every column
// and was instruction-bound (ncu: IPC 1.64, ~1.4K instructions per warp per column).
constexpr int QR_THREADS = 256;

// lane l ends with the warp sum of acc[l % W] (transpose-reduce, W - 1 shuffles + log2(32 / W))
template <int W>
__device__ __forceinline__ double warp_transpose_reduce(double (&acc)[W], int lane) {
#pragma unroll
  for (int h = W / 2; h >= 1; h >>= 1) {
    const bool upper = (lane & h) != 0;
#pragma unroll
    for (int q = 0; q < h; ++q) {
      const double send = upper ? acc[q] : acc[q + h];
      const double keep = upper ? acc[q + h] : acc[q];
      acc[q] = keep + __shfl_xor_sync(0xffffffffu, send, h);
    }
  }
  double v = acc[0];
#pragma unroll
  for (int h = W; h < 32; h <<= 1) v += __shfl_xor_sync(0xffffffffu, v, h);
  return v;
}

template <int W, bool CLUSTER>
__global__ void __launch_bounds__(QR_THREADS, 1)
qr_panel_reg_kernel(double* __restrict__ A, int lda, int m, int j, int w, int rp, double* __restrict__ Y, int ldy,
                    double* __restrict__ Tout, double* __restrict__ tau_out) {
  constexpr int RPT = 64 / W;
  constexpr int NW = QR_THREADS / 32;
  __shared__ double red1[2];          // tail-norm partial, alpha (CTA 0 only)
  __shared__ double red2[W];          // dot partials of this CTA
  __shared__ double wred1[NW];
  __shared__ double wred2[NW][W];
  __shared__ double wsum[W];
  __shared__ double taus[32];
  __shared__ double gram[32 * 32];    // G[a][b] = y_a . y_b (a < b)
  __shared__ double Ts[32 * 32];
  const int C = CLUSTER ? gridDim.x : 1;
  const unsigned crank = CLUSTER ? cluster_ctarank() : 0u;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int mp = m - j;
  const int lo = (int)crank * rp, hi = min(lo + rp, mp);
  double x[RPT][W];
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int gi = lo + tid + QR_THREADS * r;
#pragma unroll
    for (int q = 0; q < W; ++q) x[r][q] = (gi < hi && q < w) ? A[(size_t)(j + q) * lda + j + gi] : 0.0;
  }
#pragma unroll
  for (int c = 0; c < W; ++c) {
    // ---- tail norm below the diagonal; alpha = A[c][c] (relative row c: CTA 0, thread c, r = 0)
    double ss = 0.0;
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int gi = lo + tid + QR_THREADS * r;
      if (gi > c && gi < hi) ss = fma(x[r][c], x[r][c], ss);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    if (lane == 0) wred1[warp] = ss;
    if (crank == 0 && tid == c) red1[1] = x[0][c];
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
#pragma unroll
      for (int q = 0; q < NW; ++q) t += wred1[q];
      red1[0] = t;
    }
    qp_sync<CLUSTER>();
    double tail2 = 0.0;
    for (int q = 0; q < C; ++q) tail2 += qp_ld<CLUSTER>(red1, q);
    const double alpha = qp_ld<CLUSTER>(red1 + 1, 0);
    double tau = 0.0, beta = alpha, scale = 0.0;
    if (tail2 > 0.0) {
      beta = -copysign(sqrt(fma(alpha, alpha, tail2)), alpha);
      tau = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    if (tid == 0) taus[c] = tau;
    // ---- v = x / (alpha - beta) below the diagonal, v_c = 1; one reduction gives v^T A[:, q]
    //      for q > c and the Gram column G[q][c] = y_q . y_c for q < c
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int gi = lo + tid + QR_THREADS * r;
      if (gi > c && gi < hi) x[r][c] *= scale;
    }
    // in groups of at most 16 columns (bounds the accumulator registers next to the panel)
    constexpr int WG = W < 16 ? W : 16;
#pragma unroll
    for (int g0 = 0; g0 < W; g0 += WG) {
      double acc[WG];
#pragma unroll
      for (int q = 0; q < WG; ++q) acc[q] = 0.0;
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        const int gi = lo + tid + QR_THREADS * r;
        if (gi >= c && gi < hi) {
          double v = x[r][c];   // (a select of the constant against the element would make the
          v = gi == c ? 1.0 : v; //  front end address the panel array: it would leave registers)
#pragma unroll
          for (int q = 0; q < WG; ++q)
            if (g0 + q != c) acc[q] = fma(v, x[r][g0 + q], acc[q]);
        }
      }
      const double part = warp_transpose_reduce<WG>(acc, lane);
      if (lane < WG) wred2[warp][g0 + lane] = part;
    }
    __syncthreads();
    if (tid < W) {
      double t = 0.0;
#pragma unroll
      for (int q = 0; q < NW; ++q) t += wred2[q][tid];
      red2[tid] = t;
    }
    qp_sync<CLUSTER>();
    if (tid < W && tid != c) {
      double t = 0.0;
      for (int q = 0; q < C; ++q) t += qp_ld<CLUSTER>(red2 + tid, q);
      if (tid > c) wsum[tid] = tau * t;
      else gram[tid * 32 + c] = t;
    }
    __syncthreads();
    // ---- rank-1 update of rows >= c of the columns q > c (registers); R[c][c] = beta
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int gi = lo + tid + QR_THREADS * r;
      if (gi >= c && gi < hi) {
        double v = x[r][c];   // (a select of the constant against the element would make the
          v = gi == c ? 1.0 : v; //  front end address the panel array: it would leave registers)
#pragma unroll
        for (int q = c + 1; q < W; ++q) x[r][q] = fma(-wsum[q], v, x[r][q]);
        if (gi == c) x[r][c] = beta;
      }
    }
  }
  // ---- write back: A holds R on/above the diagonal and v below; Y explicit (unit diagonal, zeros)
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int gi = lo + tid + QR_THREADS * r;
    if (gi < hi) {
#pragma unroll
      for (int q = 0; q < W; ++q)
        if (q < w) {
          A[(size_t)(j + q) * lda + j + gi] = x[r][q];
          Y[(size_t)q * ldy + gi] = gi < q ? 0.0 : (gi == q ? 1.0 : x[r][q]);
        }
    }
  }
  // red2 may still be read remotely by slower CTAs of the last column
  qp_sync<CLUSTER>();
  if (crank == 0 && warp == 0) {
    // dlarft (forward, columnwise) over the w columns, lane a owns row a
    for (int b = 0; b < 32; ++b) {
      const double tb = b < w ? taus[b] : 0.0;
      double t = 0.0;
      if (lane < b && b < w)
        for (int q = lane; q < b; ++q) t = fma(Ts[q * 32 + lane], gram[q * 32 + b], t);
      Ts[b * 32 + lane] = lane < b ? -tb * t : (lane == b ? tb : 0.0);
      __syncwarp();
    }
    for (int e = lane; e < 32 * 32; e += 32) Tout[e] = Ts[e];
    if (lane < w) tau_out[lane] = taus[lane];
  }
}

// rows capacity of one register panel CTA for width W: 256 threads x 64 / W rows
int qr_panel_reg_rows(int W) { return QR_THREADS * (64 / W); }

cudaError_t qr_panel_reg(double* A, int lda, int m, int j, int w, int W, double* Y, int ldy, double* T, double* tau,
                         cudaStream_t s) {
  if (w < 1 || w > W || (W != 8 && W != 16 && W != 32)) return cudaErrorInvalidValue;
  const int mp = m - j, cap = qr_panel_reg_rows(W);
  int C = 1;
  while (C < 16 && (mp + C - 1) / C > cap) C *= 2;
  const int rp = (mp + C - 1) / C;
  if (rp > cap) return cudaErrorInvalidValue;
  for (auto fn : {qr_panel_reg_kernel<8, true>, qr_panel_reg_kernel<16, true>, qr_panel_reg_kernel<32, true>})
    SSSVD_CUDA_TRY(set_kernel_smem((const void*)fn, 0, true));
  cudaError_t e;
  if (C == 1) {
    if (W == 8) qr_panel_reg_kernel<8, false><<<1, QR_THREADS, 0, s>>>(A, lda, m, j, w, rp, Y, ldy, T, tau);
    else if (W == 16) qr_panel_reg_kernel<16, false><<<1, QR_THREADS, 0, s>>>(A, lda, m, j, w, rp, Y, ldy, T, tau);
    else qr_panel_reg_kernel<32, false><<<1, QR_THREADS, 0, s>>>(A, lda, m, j, w, rp, Y, ldy, T, tau);
    e = cudaGetLastError();
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C, 1, 1);
    cfg.blockDim = dim3(QR_THREADS, 1, 1);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (W == 8) e = cudaLaunchKernelEx(&cfg, qr_panel_reg_kernel<8, true>, A, lda, m, j, w, rp, Y, ldy, T, tau);
    else if (W == 16) e = cudaLaunchKernelEx(&cfg, qr_panel_reg_kernel<16, true>, A, lda, m, j, w, rp, Y, ldy, T, tau);
    else e = cudaLaunchKernelEx(&cfg, qr_panel_reg_kernel<32, true>, A, lda, m, j, w, rp, Y, ldy, T, tau);
  }
  note_launch();
  return e;
}

// Block reflector factor of an outer block (LAPACK dlarft, forward / columnwise): H_0 ... H_{kb-1}
// = I - Y T Y^T with T upper triangular, T_ii = tau_i and T[0:i, i] = -tau_i T[0:i, 0:i] G[0:i, i],
// where G = Y^T Y (kb x kb, column-major, from one DGEMM). One CTA, T in shared memory.
__global__ void __launch_bounds__(128, 1)
larft_kernel(const double* __restrict__ G, int kb, const double* __restrict__ tau, double* __restrict__ T) {
  extern __shared__ double ts[];   // [kb][kb] column-major
  const int r = threadIdx.x;
  for (int e = r; e < kb * kb; e += blockDim.x) ts[e] = 0.0;
  __syncthreads();
  for (int i = 0; i < kb; ++i) {
    const double ti = tau[i];
    if (r < i) {
      double z = 0.0;
      for (int c = r; c < i; ++c) z = fma(ts[(size_t)c * kb + r], G[(size_t)i * kb + c], z);
      ts[(size_t)i * kb + r] = -ti * z;
    } else if (r == i) {
      ts[(size_t)i * kb + i] = ti;
    }
    __syncthreads();
  }
  for (int e = r; e < kb * kb; e += blockDim.x) T[e] = ts[e];
}

cudaError_t larft(const double* G, int kb, const double* tau, double* T, cudaStream_t s) {
  if (kb < 1 || kb > 128) return cudaErrorInvalidValue;
  const size_t smem = (size_t)kb * kb * sizeof(double);
  SSSVD_CUDA_TRY(set_kernel_smem((const void*)larft_kernel, 128 * 128 * 8, false));
  larft_kernel<<<1, 128, smem, s>>>(G, kb, tau, T);
  note_launch();
  return cudaGetLastError();
}

// [I_k; 0] into the m x k column-major Q
__global__ void eye_kernel(double* __restrict__ Q, int m, int k, int ldq) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)ldq * k;
       e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e / ldq), r = (int)(e % ldq);
    if (r < m) Q[e] = r == c ? 1.0 : 0.0;
  }
}

cudaError_t eye(double* Q, int m, int k, int ldq, cudaStream_t s) {
  const long long total = (long long)ldq * k;
  eye_kernel<<<(int)std::min<long long>((total + 255) / 256, 148 * 8), 256, 0, s>>>(Q, m, k, ldq);
  note_launch();
  return cudaGetLastError();
}

// R (k x k, upper, ldr = k) <- upper triangle of A's top k rows (zeros below the diagonal)
__global__ void copy_r_kernel(const double* __restrict__ A, int lda, int k, double* __restrict__ R) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)k * k;
       e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e / k), r = (int)(e % k);
    R[e] = r <= c ? A[(size_t)c * lda + r] : 0.0;
  }
}

cudaError_t copy_r(const double* A, int lda, int k, double* R, cudaStream_t s) {
  const long long total = (long long)k * k;
  copy_r_kernel<<<(int)std::min<long long>((total + 255) / 256, 148 * 8), 256, 0, s>>>(A, lda, k, R);
  note_launch();
  return cudaGetLastError();
}

}  // namespace sssvd_gpu
