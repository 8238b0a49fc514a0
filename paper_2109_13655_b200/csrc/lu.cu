// Blocked complex LU with partial (row) pivoting, batched over shifts, for sm_100a.
//
// Replaces Eigen::PartialPivLU<ComplexMatrix>::compute + solve on (z_j I - G)
// (proj/include/sssvd/shifted_solver.hpp:20-40), one factorisation per quadrature point
// (moments.hpp:113-114 / :158). Kernels in this file:
//   * assemble_kernel        : M_j = z_j I - G, augmented with the starting block V (K1)
//   * leaf_lu_kernel         : unblocked LU of an (m x W) leaf panel, one thread-block CLUSTER per
//                              shift, the leaf in distributed shared memory (K2)
//   * panel_prep2_kernel     : the panel's interchange map + L11^{-1} (K3 + K4)
//   * scatter_copy_kernel    : displaced rows + U12 written back
//   * trsm_upper_smem_kernel : X_b = U_bb^{-1} Y_b for the back substitution (K6)
//   * pivot_floor_kernel     : min |U_ii| against 1e-30 (max|G| + |z|) (shifted_solver.hpp:27-30)
// The trailing updates are zgemm_sub / zgemm_set_gather (zgemm.cu, DMMA).
#include <cooperative_groups.h>
#include <algorithm>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "kernels.h"

namespace sssvd_gpu {

// ----------------------------------------------------------------------------- K1 assembly
// Mj[i][c] = -G[i][c] + (i == c ? z_j : 0) for c < n ; V[i][c-n] for n <= c < n+L.
// G is symmetric, so reading it row-major is reading it column-major (shifted_solver.hpp:24-25).
// One CTA per row i; each thread reads two consecutive entries of the row ONCE and writes them to
// every shift of the batch (HBM: 8 n (n + L) bytes read, 16 B n (n + L) written per launch).
constexpr int ASM_THREADS = 256;
constexpr int ASM_MAXB = 64;
__global__ void __launch_bounds__(ASM_THREADS)
assemble_kernel(const double* __restrict__ G, int n, int ldg, const double* __restrict__ V, int L,
                const double2* __restrict__ shifts, double2* __restrict__ out, int ld, long long stride, int nb) {
  __shared__ double2 zs[ASM_MAXB];
  for (int b = threadIdx.x; b < nb; b += ASM_THREADS) zs[b] = shifts[b];
  __syncthreads();
  const int i = blockIdx.x;
  const int ncols = n + L;
  const double* grow = G + (size_t)i * ldg;
  for (int c = threadIdx.x; c < ncols; c += ASM_THREADS) {
    const double v = c < n ? -grow[c] : V[(size_t)(c - n) * n + i];
    double2* dst = out + (size_t)i * ld + c;
    if (c == i) {
      for (int b = 0; b < nb; ++b, dst += stride) __stcs(dst, make_double2(v + zs[b].x, zs[b].y));
    } else {
      for (int b = 0; b < nb; ++b, dst += stride) __stcs(dst, make_double2(v, 0.0));
    }
  }
}

// new right-hand side into the augmented columns n..n+L of resident factors (factor cache)
__global__ void load_rhs_kernel(const double* __restrict__ V, int n, int L, double2* __restrict__ out, int ld,
                                long long stride) {
  const int b = blockIdx.y;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)n * L;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / L), c = (int)(e % L);
    out[b * stride + (size_t)i * ld + n + c] = make_double2(V[(size_t)c * n + i], 0.0);
  }
}

cudaError_t load_rhs(const double* V, int n, int L, double2* out, int ld, long long stride, int batch, cudaStream_t s) {
  long long total = (long long)n * L;
  int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 4);
  load_rhs_kernel<<<dim3(blocks, batch), 256, 0, s>>>(V, n, L, out, ld, stride);
  note_launch();
  return cudaGetLastError();
}

cudaError_t assemble(const double* G, int n, int ldg, const double* V, int L, const double2* shifts,
                     double2* out, int ld, long long stride, int batch, cudaStream_t s) {
  for (int b0 = 0; b0 < batch; b0 += ASM_MAXB) {
    const int nbb = std::min(ASM_MAXB, batch - b0);
    assemble_kernel<<<n, ASM_THREADS, 0, s>>>(G, n, ldg, V, L, shifts + b0, out + (size_t)b0 * stride, ld, stride,
                                              nbb);
    note_launch();
  }
  return cudaGetLastError();
}

size_t leaf_smem_bytes(int n, int W, int cluster) {
  const int R = (n + cluster - 1) / cluster;
  return (size_t)R * (W + 1) * sizeof(double2) + (6 * W) * sizeof(double2) + 256;
}

// ----------------------------------------------------------------------------- pivot floor
// status[b] = 1 if min_i |U_ii| <= 1e-30 * (max|G| + |z_b|)  (shifted_solver.hpp:27-30)
__global__ void pivot_floor_kernel(const double2* mats, int ld, long long stride, int n,
                                   const double2* shifts, const double* gmax, int* status,
                                   double* minpiv) {
  const int b = blockIdx.x;
  const double2* Mb = mats + b * stride;
  double mn = 1e300;
  for (int i = threadIdx.x; i < n; i += blockDim.x) mn = fmin(mn, hypot(Mb[(size_t)i * ld + i].x, Mb[(size_t)i * ld + i].y));
  __shared__ double red[32];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, off));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mn;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mn = fmin(mn, red[w]);
    mn = fmin(mn, red[0]);
    const double floor = 1e-30 * (gmax[0] + hypot(shifts[b].x, shifts[b].y));
    status[b] = (mn <= floor || !(mn == mn)) ? 1 : 0;
    minpiv[b] = mn;
  }
}

cudaError_t pivot_floor(const double2* mats, int ld, long long stride, int n, const double2* shifts,
                        const double* gmax, int* status, double* minpiv, int batch, cudaStream_t s) {
  pivot_floor_kernel<<<batch, 256, 0, s>>>(mats, ld, stride, n, shifts, gmax, status, minpiv);
  note_launch();
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------- max |G|
__global__ void absmax_kernel(const double* __restrict__ a, long long count, double* out) {
  double m = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x)
    m = fmax(m, fabs(a[i]));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
    // values are >= 0: the IEEE bit pattern orders like the unsigned integer
    if (threadIdx.x == 0) atomicMax(reinterpret_cast<unsigned long long*>(out), (unsigned long long)__double_as_longlong(m));
  }
}

cudaError_t absmax(const double* a, long long count, double* out, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), s);
  if (e != cudaSuccess) return e;
  absmax_kernel<<<148 * 4, 256, 0, s>>>(a, count, out);
  note_launch();
  return cudaGetLastError();
}

// panel_prep, second form (default): 8 warps per CTA. The L11^{-1} columns of a CTA share the
// rows of L11, staged in shared memory R rows at a time by cp.async two chunks ahead (the
// single-warp prefetch of the first form waited on an L2 round trip per row); the interchange
// fold looks positions up in a row-indexed table instead of a warp-ballot search. Bitwise the
// first form: every dot product, reduction and fold step is unchanged.
template <int QMAX>
__global__ void __launch_bounds__(256)
panel_prep2_kernel(const double2* __restrict__ mats, int ld, long long stride, int r0, int np,
                   double2* __restrict__ linv, long long lstride, const int* __restrict__ ipiv, int n,
                   int* __restrict__ src, int* __restrict__ disp, int dstride) {
  constexpr int WPB = 8, R = 32 / QMAX, NP = 32 * QMAX;
  __shared__ __align__(16) double2 buf[2][R][NP];
  extern __shared__ int tbl[];   // build-moves CTA: [n - r0] slot of each row, then pos / cont
  const int b = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int nx = (np + WPB - 1) / WPB;
  if ((int)blockIdx.x == nx) {
    // ---- interchange map (semantics of build_moves_body)
    int* pos = tbl + (n - r0);
    int* cont = pos + 2 * np;
    __shared__ int kmv;
    const int* piv = ipiv + (size_t)b * n;
    for (int j = tid; j < np; j += blockDim.x) {
      tbl[j] = -1;
      tbl[piv[r0 + j] - r0] = -1;
    }
    __syncthreads();
    if (tid == 0) {
      int k = 0;
      for (int j = 0; j < np; ++j) {
        const int a = r0 + j, q = piv[r0 + j];
        int ia = tbl[a - r0];
        if (ia < 0) {
          pos[k] = a;
          cont[k] = a;
          tbl[a - r0] = k;
          ia = k++;
        }
        int iq = q == a ? ia : tbl[q - r0];
        if (iq < 0) {
          pos[k] = q;
          cont[k] = q;
          tbl[q - r0] = k;
          iq = k++;
        }
        if (ia != iq) {
          const int t = cont[ia];
          cont[ia] = cont[iq];
          cont[iq] = t;
        }
      }
      kmv = k;
    }
    __syncthreads();
    if (warp == 0) {
      const int k = kmv;
      int* so = src + (size_t)b * dstride;
      int* d = disp + (size_t)b * (2 * dstride + 1);
      int nd = 0;
      for (int base = 0; base < k; base += 32) {
        const int t = base + lane;
        const bool below = t < k && pos[t] >= r0 + np && cont[t] != pos[t];
        if (t < k && pos[t] < r0 + np) so[pos[t] - r0] = cont[t];
        const unsigned bal = __ballot_sync(0xffffffffu, below);
        if (below) {
          const int sl = nd + __popc(bal & ((1u << lane) - 1));
          d[1 + 2 * sl] = pos[t];
          d[2 + 2 * sl] = cont[t];
        }
        nd += __popc(bal);
      }
      if (lane == 0) d[0] = nd;
    }
    return;
  }
  // ---- L11^{-1} columns j0 .. j0 + WPB - 1 (semantics of trinv_lower_body)
  const int j0 = blockIdx.x * WPB, j = j0 + warp;
  const bool active = j < np;
  const double2* Mb = mats + b * stride + (size_t)r0 * ld + r0;
  double2* out = linv + (size_t)b * lstride;
  const int t0 = (j0 + 1) / R, T = (np + R - 1) / R;   // chunks of rows [t R, t R + R)
  auto load_chunk = [&](int t) {
    if (t < T) {
      for (int idx = tid; idx < R * np; idx += 32 * WPB) {
        const int sl = idx / np, l = idx - sl * np;
        const int i = t * R + sl;
        if (i < np) cp_async16(&buf[t & 1][sl][l], Mb + (size_t)i * ld + l);
      }
    }
    cp_async_commit();
  };
  load_chunk(t0);
  load_chunk(t0 + 1);
  double2 x[QMAX];
#pragma unroll
  for (int q = 0; q < QMAX; ++q) x[q] = make_double2((lane + 32 * q) == j ? 1.0 : 0.0, 0.0);
  for (int t = t0; t < T; ++t) {
    cp_async_wait<1>();
    __syncthreads();
    if (active) {
      for (int sl = 0; sl < R; ++sl) {
        const int i = t * R + sl;
        if (i <= j || i >= np) continue;
        const int qi = i >> 5, ii = i & 31;
        double sr = 0.0, si = 0.0;
#pragma unroll
        for (int q = 0; q < QMAX; ++q) {
          const int l = lane + 32 * q;
          if (q <= qi && l >= j && l < i) {
            const double2 lr = buf[t & 1][sl][l];
            sr += lr.x * x[q].x - lr.y * x[q].y;
            si += lr.x * x[q].y + lr.y * x[q].x;
          }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          sr += __shfl_xor_sync(0xffffffffu, sr, off);
          si += __shfl_xor_sync(0xffffffffu, si, off);
        }
#pragma unroll
        for (int q = 0; q < QMAX; ++q)
          if (q == qi && lane == ii) x[q] = make_double2(-sr, -si);
      }
    }
    __syncthreads();
    load_chunk(t + 2);
  }
  if (active) {
#pragma unroll
    for (int q = 0; q < QMAX; ++q) {
      const int i = lane + 32 * q;
      if (i < np) out[(size_t)i * np + j] = i >= j ? x[q] : make_double2(0.0, 0.0);
    }
  }
}

cudaError_t panel_prep(const double2* mats, int ld, long long stride, int r0, int np, double2* linv, long long lstride,
                       const int* ipiv, int n, int* src, int* disp, int dstride, int batch, cudaStream_t s) {
  if (np > 256) return cudaErrorInvalidValue;
  const size_t sm2 = (size_t)(n - r0 + 4 * np) * sizeof(int);
  SSSVD_CUDA_TRY(set_kernel_smem((const void*)panel_prep2_kernel<4>, sm2, false));
  SSSVD_CUDA_TRY(set_kernel_smem((const void*)panel_prep2_kernel<8>, sm2, false));
  dim3 grid2((np + 7) / 8 + 1, batch);
  if (np <= 128)
    panel_prep2_kernel<4><<<grid2, 256, sm2, s>>>(mats, ld, stride, r0, np, linv, lstride, ipiv, n, src, disp, dstride);
  else
    panel_prep2_kernel<8><<<grid2, 256, sm2, s>>>(mats, ld, stride, r0, np, linv, lstride, ipiv, n, src, disp, dstride);
  note_launch();
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------- scatter + copy
// Columns [c0, c1): displaced rows get their (original panel-row) content, then the panel rows
// r0..r0+np receive U12 = T (np x (c1-c0), pitch ldt). Each thread owns one column, so the
// panel rows are read (as displaced sources) before they are overwritten.
__global__ void scatter_copy_kernel(double2* mats, int ld, long long stride, int r0, int np, int c0, int c1,
                                    const int* __restrict__ disp, int dstride, const double2* __restrict__ T,
                                    int ldt, long long tstride) {
  const int b = blockIdx.y;
  const int c = c0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= c1) return;
  double2* Mb = mats + b * stride;
  const int* d = disp + (size_t)b * (2 * dstride + 1);
  const int nd = d[0];
  // sources of the displaced moves are panel rows and their destinations lie below the panel, so
  // the moves never alias: 8 loads are issued before their 8 stores (the compiler cannot prove
  // this and would otherwise serialise one load-store round trip per move)
  constexpr int U = 8;
  int t = 0;
  for (; t + U <= nd; t += U) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = Mb[(size_t)d[2 + 2 * (t + u)] * ld + c];
#pragma unroll
    for (int u = 0; u < U; ++u) Mb[(size_t)d[1 + 2 * (t + u)] * ld + c] = v[u];
  }
  for (; t < nd; ++t) Mb[(size_t)d[1 + 2 * t] * ld + c] = Mb[(size_t)d[2 + 2 * t] * ld + c];
  const double2* Tb = T + b * tstride;
  int q = 0;
  for (; q + U <= np; q += U) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = Tb[(size_t)(q + u) * ldt + (c - c0)];
#pragma unroll
    for (int u = 0; u < U; ++u) Mb[(size_t)(r0 + q + u) * ld + c] = v[u];
  }
  for (; q < np; ++q) Mb[(size_t)(r0 + q) * ld + c] = Tb[(size_t)q * ldt + (c - c0)];
}

cudaError_t scatter_copy(double2* mats, int ld, long long stride, int r0, int np, int c0, int c1, const int* disp,
                         int dstride, const double2* T, int ldt, long long tstride, int batch, cudaStream_t s) {
  if (c1 <= c0) return cudaSuccess;
  dim3 grid((c1 - c0 + 127) / 128, batch);
  scatter_copy_kernel<<<grid, 128, 0, s>>>(mats, ld, stride, r0, np, c0, c1, disp, dstride, T, ldt, tstride);
  note_launch();
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------- back substitution
// Rows r0..r0+np of the columns [c0,c1): x = U11^{-1} y by substitution (backward stable), one
// warp per (column, shift); lanes split each dot product; x stays distributed over the lanes.
// Same substitution (bitwise: identical per-row dot products and warp reductions), but the CTA's
// warps -- WPB right-hand-side columns of one shift -- share the rows of U11: chunks of R rows are
// staged in shared memory by cp.async two chunks ahead, instead of every warp fetching each row
// from L2 one row ahead. The per-row critical path drops from an L2 round trip to the shuffle
// reduction.
template <int QMAX, int WPB>
__global__ void __launch_bounds__(32 * WPB, 2)
trsm_upper_smem_kernel(double2* mats, int ld, long long stride, int r0, int np, int c0, int c1) {
  constexpr int R = 32 / QMAX;   // rows per chunk (one chunk never straddles a 32-row slot)
  constexpr int NP = 32 * QMAX;
  constexpr int T = NP / R;
  __shared__ __align__(16) double2 buf[2][R][NP];
  const int b = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = c0 + blockIdx.x * WPB + warp;
  const bool active = c < c1;
  double2* Mb = mats + b * stride;
  const double2* U = Mb + (size_t)r0 * ld + r0;
  // chunk t holds rows [NP - (t+1) R, NP - t R), highest first; rows >= np are not loaded
  auto load_chunk = [&](int t) {
    const int top = NP - t * R;
    for (int idx = threadIdx.x; idx < R * np; idx += 32 * WPB) {
      const int sl = idx / np, l = idx - sl * np;
      const int i = top - 1 - sl;
      if (i < np) cp_async16(&buf[t & 1][sl][l], U + (size_t)i * ld + l);
    }
    cp_async_commit();
  };
  load_chunk(0);
  load_chunk(1);
  double2 x[QMAX], invd[QMAX];
#pragma unroll
  for (int q = 0; q < QMAX; ++q) {
    const int i = lane + 32 * q;
    x[q] = (active && i < np) ? Mb[(size_t)(r0 + i) * ld + c] : make_double2(0.0, 0.0);
    const double2 u = i < np ? U[(size_t)i * ld + i] : make_double2(1.0, 0.0);
    invd[q] = cabs2(u) != 0.0 ? crecip(u) : make_double2(1.0, 0.0);
  }
  int t = 0;
#pragma unroll
  for (int qi = QMAX - 1; qi >= 0; --qi) {
    for (int tc = 0; tc < 32 / R; ++tc, ++t) {
      cp_async_wait<1>();
      __syncthreads();
      const int slot = t & 1;
      if (active) {
        for (int sl = 0; sl < R; ++sl) {
          const int ii = 31 - tc * R - sl;
          const int i = 32 * qi + ii;
          if (i >= np) continue;
          double sr = 0.0, si = 0.0;
#pragma unroll
          for (int q = qi; q < QMAX; ++q) {
            const int l = lane + 32 * q;
            if (l > i && l < np) {
              const double2 u = buf[slot][sl][l];
              sr += u.x * x[q].x - u.y * x[q].y;
              si += u.x * x[q].y + u.y * x[q].x;
            }
          }
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) {
            sr += __shfl_xor_sync(0xffffffffu, sr, off);
            si += __shfl_xor_sync(0xffffffffu, si, off);
          }
          if (lane == ii) x[qi] = cmul(make_double2(x[qi].x - sr, x[qi].y - si), invd[qi]);
        }
      }
      __syncthreads();
      if (t + 2 < T)
        load_chunk(t + 2);
      else
        cp_async_commit();   // keep one group per chunk so the wait count stays exact
    }
  }
  if (active) {
#pragma unroll
    for (int q = 0; q < QMAX; ++q) {
      const int i = lane + 32 * q;
      if (i < np) Mb[(size_t)(r0 + i) * ld + c] = x[q];
    }
  }
}

cudaError_t trsm_upper_blocks(double2* mats, int ld, long long stride, int r0, int np, int c0, int c1, int batch,
                            cudaStream_t s) {
  if (c1 <= c0 || np <= 0) return cudaSuccess;
  if (np > 256) return cudaErrorInvalidValue;
  constexpr int WPB = 8;
  dim3 grid((c1 - c0 + WPB - 1) / WPB, batch);
  if (np <= 128)
    trsm_upper_smem_kernel<4, WPB><<<grid, 32 * WPB, 0, s>>>(mats, ld, stride, r0, np, c0, c1);
  else
    trsm_upper_smem_kernel<8, WPB><<<grid, 32 * WPB, 0, s>>>(mats, ld, stride, r0, np, c0, c1);
  note_launch();
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------- K2 leaf panel
// One thread-block cluster per shift (blockIdx.y) holds the leaf columns [r0, r0 + w) in a
// shared-memory slab (R x (W+1) complex per CTA: CTA c owns rows [r0 + c R, r0 + (c+1) R)), and
// thread t owns slab rows t, t+NT, ...; for column j it scales its rows, applies
// the rank-1 update to their columns j+1..W-1 and scores column j+1 in the same pass, so the
// only barriers per column are: CTA argmax (1), cluster exchange (1), winner broadcast (1).
// Warp 0 publishes the CTA candidate and the diagonal row straight from the slab, reduces the C
// candidates over DSMEM, fetches the pivot row (and, in the winning CTA, the old diagonal row),
// and performs the interchange in the slab.
template <int W, int NT>
__global__ void __launch_bounds__(NT, 1)
leaf_lu_kernel(double2* mats, int ld, long long stride, int n, int r0, int w, int R, int* ipiv, int cb) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  constexpr int P = W + 1;
  double2* slab = reinterpret_cast<double2*>(sm_raw);   // R x P
  __shared__ double2 cand_vals[2][W];
  __shared__ double2 diag_vals[2][W];
  __shared__ double2 urow[W];
  __shared__ double cand_score[2];
  __shared__ int cand_row[2];
  __shared__ double red_s[NT / 32];
  __shared__ int red_r[NT / 32];
  __shared__ int win_row;

  const int C = gridDim.x;
  const unsigned rank = cluster_ctarank();
  const int b = blockIdx.y;
  double2* Mb = mats + b * stride;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int my0 = r0 + (int)rank * R;
  const int myn = max(0, min(R, n - my0));

  for (int e = tid; e < myn * W; e += NT) {
    const int i = e / W, c = e % W;
    slab[i * P + c] = (c < w) ? Mb[(size_t)(my0 + i) * ld + r0 + c] : make_double2(0.0, 0.0);
  }
  __syncthreads();

  // score of column 0 over the rows this thread owns
  double best = -1.0;
  int brow = 0x7fffffff;
  for (int i = tid; i < myn; i += NT) {
    const double s = cabs2(slab[i * P]);
    if (s > best) { best = s; brow = my0 + i; }
  }

  for (int j = 0; j < w; ++j) {
    const int d = r0 + j;
    const int par = j & 1;
    // ---- CTA argmax of column j (ties: smallest row)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double os = __shfl_xor_sync(0xffffffffu, best, off);
      const int orow = __shfl_xor_sync(0xffffffffu, brow, off);
      if (os > best || (os == best && orow < brow)) { best = os; brow = orow; }
    }
    if (lane == 0) { red_s[warp] = best; red_r[warp] = brow; }
    __syncthreads();
    if (warp == 0) {
      best = lane < NT / 32 ? red_s[lane] : -1.0;
      brow = lane < NT / 32 ? red_r[lane] : 0x7fffffff;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const double os = __shfl_xor_sync(0xffffffffu, best, off);
        const int orow = __shfl_xor_sync(0xffffffffu, brow, off);
        if (os > best || (os == best && orow < brow)) { best = os; brow = orow; }
      }
      if (lane == 0) { cand_score[par] = best; cand_row[par] = brow; }
      for (int c = lane; c < W; c += 32) {
        if (brow != 0x7fffffff) cand_vals[par][c] = slab[(brow - my0) * P + c];
        if (d >= my0 && d < my0 + myn) diag_vals[par][c] = slab[(d - my0) * P + c];
      }
    }
    cluster_sync_all();
    // ---- warp 0: winner over the C candidates, pivot row (+ old diagonal row), interchange
    if (warp == 0) {
      double s = -1.0;
      int r = 0x7fffffff, rk = lane;
      if (lane < C) {
        s = ld_dsmem_f64(dsmem_addr(&cand_score[par], lane));
        r = ld_dsmem_s32(dsmem_addr(&cand_row[par], lane));
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const double os = __shfl_xor_sync(0xffffffffu, s, off);
        const int orow = __shfl_xor_sync(0xffffffffu, r, off);
        const int ork = __shfl_xor_sync(0xffffffffu, rk, off);
        if (os > s || (os == s && orow < r)) { s = os; r = orow; rk = ork; }
      }
      const int downer = (d - r0) / R;
      for (int c = lane; c < W; c += 32) {
        const double2 u = ld_dsmem_f64x2(dsmem_addr(&cand_vals[par][c], rk));
        double2 dv = make_double2(0.0, 0.0);
        if (r != d && rk == (int)rank) dv = ld_dsmem_f64x2(dsmem_addr(&diag_vals[par][c], downer));
        urow[c] = u;
        if (d >= my0 && d < my0 + myn) slab[(d - my0) * P + c] = u;
        if (r != d && rk == (int)rank) slab[(r - my0) * P + c] = dv;
      }
      if (lane == 0) win_row = r;
      if (lane == 0 && rank == 0) ipiv[(size_t)b * n + d] = r;
    }
    __syncthreads();
    // ---- own rows: scale column j, rank-1 update of columns j+1.., score column j+1
    const double2 u = urow[j];
    const bool nz = cabs2(u) != 0.0;
    const double2 inv = nz ? crecip(u) : make_double2(0.0, 0.0);
    best = -1.0;
    brow = 0x7fffffff;
    const int first = max(0, d + 1 - my0);
    for (int i = first + ((tid - first) % NT + NT) % NT; i < myn; i += NT) {
      double2* row = slab + i * P;
      if (nz) {
        const double2 l = cmul(row[j], inv);
        row[j] = l;
#pragma unroll 4
        for (int c = j + 1; c < W; ++c) row[c] = cfms(row[c], l, urow[c]);
      }
      if (j + 1 < w) {
        const double sc = cabs2(row[j + 1]);
        if (sc > best) { best = sc; brow = my0 + i; }
      }
    }
    (void)win_row;
  }
  __syncthreads();
  for (int e = tid; e < myn * w; e += NT) {
    const int i = e / w, c = e % w;
    Mb[(size_t)(my0 + i) * ld + r0 + c] = slab[i * P + c];
  }
  cluster_sync_all();
  // ---- epilogue (rank 0): this leaf's w interchanges applied to the block columns on its left,
  // [cb, r0) (the separate swap_trsm launch of the recursive panel otherwise). Warp 0 folds the
  // sequential swaps into <= 2w (destination <- source) moves; each thread then gathers every
  // source of its column before scattering, so no load waits on a store. Only global rows of
  // columns the leaf never touches are involved, and the slab is free again after the barrier.
  if (cb < r0 && rank == 0) {
    int* pos = reinterpret_cast<int*>(sm_raw);        // [2W] touched rows
    int* cont = pos + 2 * W;                          // [2W] their final source rows
    double2* buf = reinterpret_cast<double2*>(sm_raw + 1024);
    __shared__ int kmv;
    const int* piv = ipiv + (size_t)b * n;
    if (warp == 0) {
      int k = 0;
      for (int j = 0; j < w; ++j) {
        const int a = r0 + j, q = piv[r0 + j];
        int ia = -1, iq = -1;
        for (int base = 0; base < k; base += 32) {
          const int t = base + lane;
          const int pv = t < k ? pos[t] : -1;
          const unsigned ba = __ballot_sync(0xffffffffu, pv == a);
          const unsigned bq = __ballot_sync(0xffffffffu, pv == q);
          if (ba && ia < 0) ia = base + __ffs(ba) - 1;
          if (bq && iq < 0) iq = base + __ffs(bq) - 1;
        }
        if (ia < 0) {
          if (lane == 0) { pos[k] = a; cont[k] = a; }
          ia = k++;
        }
        if (q == a) iq = ia;
        if (iq < 0) {
          if (lane == 0) { pos[k] = q; cont[k] = q; }
          iq = k++;
        }
        __syncwarp();
        if (lane == 0 && ia != iq) { const int t = cont[ia]; cont[ia] = cont[iq]; cont[iq] = t; }
        __syncwarp();
      }
      if (lane == 0) kmv = k;
    }
    __syncthreads();
    const int k = kmv, ncl = r0 - cb;
    for (int c = tid; c < ncl; c += NT) {
      for (int e = 0; e < k; ++e) buf[(size_t)e * ncl + c] = Mb[(size_t)cont[e] * ld + cb + c];
      for (int e = 0; e < k; ++e)
        if (pos[e] != cont[e]) Mb[(size_t)pos[e] * ld + cb + c] = buf[(size_t)e * ncl + c];
    }
  }
}

template <int W, int NT>
static cudaError_t launch_leaf(double2* mats, int ld, long long stride, int n, int r0, int w, int cluster,
                                  int* ipiv, int batch, cudaStream_t s, int cb) {
  const int m = n - r0;
  const int R = (m + cluster - 1) / cluster;
  // the slab, or the fused left-swap epilogue's move list + gather buffer if that is larger
  const size_t smem = std::max((size_t)R * (W + 1) * sizeof(double2),
                               cb < r0 ? 1024 + (size_t)2 * W * (r0 - cb) * sizeof(double2) : (size_t)0);
  SSSVD_CUDA_TRY(set_kernel_smem((const void*)leaf_lu_kernel<W, NT>, smem, true));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cluster, batch, 1);
  cfg.blockDim = dim3(NT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  note_launch();
  return cudaLaunchKernelEx(&cfg, leaf_lu_kernel<W, NT>, mats, ld, stride, n, r0, w, R, ipiv, cb);
}

cudaError_t leaf_lu(double2* mats, int ld, long long stride, int n, int r0, int w, int W, int cluster, int* ipiv,
                       int batch, cudaStream_t s, int cb) {
  if (cb > r0) return cudaErrorInvalidValue;
  switch (W) {
    case 8: return launch_leaf<8, 512>(mats, ld, stride, n, r0, w, cluster, ipiv, batch, s, cb);
    case 16: return launch_leaf<16, 512>(mats, ld, stride, n, r0, w, cluster, ipiv, batch, s, cb);
    case 32: return launch_leaf<32, 256>(mats, ld, stride, n, r0, w, cluster, ipiv, batch, s, cb);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace sssvd_gpu
