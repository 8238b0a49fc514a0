// Blocked complex LU with partial (row) pivoting, batched over shifts, for sm_100a.
//
// Replaces Eigen::PartialPivLU<ComplexMatrix>::compute + solve on (z_j I - G)
// (proj/include/sssvd/shifted_solver.hpp:20-40), one factorisation per quadrature point
// (moments.hpp:113-114 / :158). Kernels in this file:
//   * assemble_kernel    : M_j = z_j I - G, augmented with the starting block V (K1)
//   * leaf_lu_kernel     : unblocked LU of an (m x W) leaf panel. One thread-block CLUSTER
//                          per shift holds the whole leaf in distributed shared memory; the
//                          pivot search is a warp-shuffle argmax inside each CTA followed by
//                          a DSMEM exchange of the C per-CTA candidates, one cluster barrier
//                          per column (K2)
//   * swap_trsm_kernel   : applies a block of row interchanges to a column range (gather all
//                          sources, then scatter: no serial swap chain) and, optionally, the
//                          unit-lower triangular solve U12 = L11^{-1} A12 (K3 + K4)
//   * trsm_upper_kernel  : X_b = U_bb^{-1} Y_b for the back substitution (K6)
//   * pivot_floor_kernel : min |U_ii| against 1e-30 (max|G| + |z|) (shifted_solver.hpp:27-30)
// The trailing updates are zgemm_sub (zgemm.cu, DMMA).
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

// the per-shift variant (grid.y = shift): G is re-read once per shift (SSSVD_ASM=pershift)
__global__ void __launch_bounds__(ASM_THREADS)
assemble_pershift_kernel(const double* __restrict__ G, int n, int ldg, const double* __restrict__ V, int L,
                         const double2* __restrict__ shifts, double2* __restrict__ out, int ld, long long stride) {
  const int b = blockIdx.y;
  const double2 z = shifts[b];
  const int ncols = n + L;
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const double* grow = G + (size_t)i * ldg;
    double2* dst = out + b * stride + (size_t)i * ld;
    for (int c = threadIdx.x; c < ncols; c += ASM_THREADS) {
      const double v = c < n ? -grow[c] : V[(size_t)(c - n) * n + i];
      dst[c] = c == i ? make_double2(v + z.x, z.y) : make_double2(v, 0.0);
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
  static const char* env = std::getenv("SSSVD_ASM");
  if (env && std::string(env) == "pershift") {
    assemble_pershift_kernel<<<dim3(std::min(n, 148 * 4), batch), ASM_THREADS, 0, s>>>(G, n, ldg, V, L, shifts, out,
                                                                                      ld, stride);
    note_launch();
    return cudaGetLastError();
  }
  for (int b0 = 0; b0 < batch; b0 += ASM_MAXB) {
    const int nbb = std::min(ASM_MAXB, batch - b0);
    assemble_kernel<<<n, ASM_THREADS, 0, s>>>(G, n, ldg, V, L, shifts + b0, out + (size_t)b0 * stride, ld, stride,
                                              nbb);
    note_launch();
  }
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------- K2 leaf panel
// One cluster (gridDim.x == cluster size C) per shift (blockIdx.y). CTA c owns rows
// [r0 + c*R, r0 + (c+1)*R) of the leaf columns [r0, r0 + w). Panel pitch W+1 double2 keeps
// the column walk of the pivot search bank-conflict free.
template <int W>
__global__ void __launch_bounds__(256, 1)
leaf_lu_kernel(double2* mats, int ld, long long stride, int n, int r0, int w, int R, int* ipiv) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  constexpr int P = W + 1;
  double2* slab = reinterpret_cast<double2*>(sm_raw);                  // R x P
  double2* cand_vals = slab + (size_t)R * P;                           // [2][W]
  double2* diag_vals = cand_vals + 2 * W;                              // [2][W]
  double2* urow = diag_vals + 2 * W;                                   // [W]
  double2* drow = urow + W;                                            // [W]
  double* cand_score = reinterpret_cast<double*>(drow + W);            // [2]
  int* cand_row = reinterpret_cast<int*>(cand_score + 2);              // [2]
  double* red_s = reinterpret_cast<double*>(cand_row + 2);             // [8]
  int* red_r = reinterpret_cast<int*>(red_s + 8);                      // [8]
  int* win = red_r + 8;                                                // [2]: rank, row

  const int C = gridDim.x;
  const unsigned rank = cluster_ctarank();
  const int b = blockIdx.y;
  double2* Mb = mats + b * stride;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m = n - r0;
  const int my0 = r0 + (int)rank * R;                 // first global row of my slab
  const int myn = max(0, min(R, n - my0));            // rows I own

  // load my slab
  for (int e = tid; e < myn * W; e += blockDim.x) {
    int i = e / W, c = e % W;
    slab[i * P + c] = (c < w) ? Mb[(size_t)(my0 + i) * ld + r0 + c] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  (void)m;

  for (int j = 0; j < w; ++j) {
    const int d = r0 + j;           // diagonal row
    const int par = j & 1;
    // 1) local argmax of |a_ij|^2 over my rows i >= d (ties: smallest row)
    double best = -1.0;
    int brow = 0x7fffffff;
    for (int i = tid; i < myn; i += blockDim.x) {
      int gi = my0 + i;
      if (gi < d) continue;
      double s = cabs2(slab[i * P + j]);
      if (s > best || (s == best && gi < brow)) {
        best = s;
        brow = gi;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      double os = __shfl_xor_sync(0xffffffffu, best, off);
      int orow = __shfl_xor_sync(0xffffffffu, brow, off);
      if (os > best || (os == best && orow < brow)) {
        best = os;
        brow = orow;
      }
    }
    if (lane == 0) {
      red_s[warp] = best;
      red_r[warp] = brow;
    }
    __syncthreads();
    if (warp == 0) {
      best = lane < (int)(blockDim.x >> 5) ? red_s[lane] : -1.0;
      brow = lane < (int)(blockDim.x >> 5) ? red_r[lane] : 0x7fffffff;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        double os = __shfl_xor_sync(0xffffffffu, best, off);
        int orow = __shfl_xor_sync(0xffffffffu, brow, off);
        if (os > best || (os == best && orow < brow)) {
          best = os;
          brow = orow;
        }
      }
      if (lane == 0) {
        cand_score[par] = best;
        cand_row[par] = brow;
        red_r[0] = brow;
      }
    }
    __syncthreads();
    // 2) publish candidate row and (if owned) the diagonal row
    {
      const int crow = red_r[0];
      if (tid < W) {
        if (crow != 0x7fffffff) cand_vals[par * W + tid] = slab[(crow - my0) * P + tid];
        if (d >= my0 && d < my0 + myn) diag_vals[par * W + tid] = slab[(d - my0) * P + tid];
      }
    }
    // 3) cluster barrier: candidates of every CTA are visible
    cluster_sync_all();
    // 4) winner over the C candidates (DSMEM), same tie rule
    if (warp == 0) {
      double s = -1.0;
      int r = 0x7fffffff, rk = lane;
      if (lane < C) {
        s = ld_dsmem_f64(dsmem_addr(&cand_score[par], lane));
        r = ld_dsmem_s32(dsmem_addr(&cand_row[par], lane));
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        double os = __shfl_xor_sync(0xffffffffu, s, off);
        int orow = __shfl_xor_sync(0xffffffffu, r, off);
        int ork = __shfl_xor_sync(0xffffffffu, rk, off);
        if (os > s || (os == s && orow < r)) {
          s = os;
          r = orow;
          rk = ork;
        }
      }
      if (lane == 0) {
        win[0] = rk;
        win[1] = r;
      }
    }
    __syncthreads();
    const int wrank = win[0], p = win[1];
    const int downer = (d - r0) / R;
    if (tid < W) {
      urow[tid] = ld_dsmem_f64x2(dsmem_addr(&cand_vals[par * W + tid], wrank));
      if ((int)rank == wrank && p != d) drow[tid] = ld_dsmem_f64x2(dsmem_addr(&diag_vals[par * W + tid], downer));
    }
    __syncthreads();
    if (tid < W) {
      if (d >= my0 && d < my0 + myn) slab[(d - my0) * P + tid] = urow[tid];
      if ((int)rank == wrank && p != d) slab[(p - my0) * P + tid] = drow[tid];
    }
    if (rank == 0 && tid == 0) ipiv[(size_t)b * n + d] = p;
    __syncthreads();
    // 5) scale column j below the diagonal and rank-1 update the columns right of j
    const double2 u = urow[j];
    const bool nz = cabs2(u) != 0.0;
    const double2 inv = nz ? crecip(u) : make_double2(0.0, 0.0);
    const int first = max(0, d + 1 - my0);            // first local row strictly below d
    const int ncol = w - j - 1;
    if (nz && ncol > 0) {
      for (int e = tid; e < (myn - first) * ncol; e += blockDim.x) {
        int i = first + e / ncol, c = j + 1 + e % ncol;
        double2 l = cmul(slab[i * P + j], inv);
        slab[i * P + c] = cfms(slab[i * P + c], l, urow[c]);
      }
    }
    __syncthreads();
    if (nz)
      for (int i = first + tid; i < myn; i += blockDim.x) slab[i * P + j] = cmul(slab[i * P + j], inv);
    __syncthreads();
  }
  // write back (no other CTA reads my smem after the last barrier of the loop, but keep the
  // cluster alive until everybody finished its DSMEM reads of the last column)
  for (int e = tid; e < myn * w; e += blockDim.x) {
    int i = e / w, c = e % w;
    Mb[(size_t)(my0 + i) * ld + r0 + c] = slab[i * P + c];
  }
  cluster_sync_all();
}

template <int W>
static cudaError_t launch_leaf(double2* mats, int ld, long long stride, int n, int r0, int w,
                               int cluster, int* ipiv, int batch, cudaStream_t s) {
  const int m = n - r0;
  const int R = (m + cluster - 1) / cluster;
  const size_t smem = (size_t)R * (W + 1) * sizeof(double2) + (6 * W) * sizeof(double2) + 256;
  static size_t configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(leaf_lu_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(leaf_lu_kernel<W>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cluster, batch, 1);
  cfg.blockDim = dim3(256, 1, 1);
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
  return cudaLaunchKernelEx(&cfg, leaf_lu_kernel<W>, mats, ld, stride, n, r0, w, R, ipiv);
}

size_t leaf_smem_bytes(int n, int W, int cluster) {
  const int R = (n + cluster - 1) / cluster;
  return (size_t)R * (W + 1) * sizeof(double2) + (6 * W) * sizeof(double2) + 256;
}

cudaError_t leaf_lu(double2* mats, int ld, long long stride, int n, int r0, int w, int W,
                    int cluster, int* ipiv, int batch, cudaStream_t s) {
  switch (W) {
    case 8: return launch_leaf<8>(mats, ld, stride, n, r0, w, cluster, ipiv, batch, s);
    case 16: return launch_leaf<16>(mats, ld, stride, n, r0, w, cluster, ipiv, batch, s);
    case 32: return launch_leaf<32>(mats, ld, stride, n, r0, w, cluster, ipiv, batch, s);
    default: return cudaErrorInvalidValue;
  }
}

// ----------------------------------------------------------------------------- K3+K4 swap/TRSM
// For the pivots ipiv[r0 .. r0+np) (global row indices, LAPACK sequential-swap semantics) and
// the columns [c0, c1): (1) warp 0 folds the np swaps into a list of (dst <- src) moves over the
// <= 2 np touched rows; (2) each thread owns one column, gathers every source value, then
// scatters (no serial dependency chain); (3) optionally solves the unit-lower L11 (rows/cols
// r0..r0+np of the same matrix) against rows r0..r0+np of its column.
constexpr int ST_COLS = 32;

__global__ void __launch_bounds__(ST_COLS)
swap_trsm_kernel(double2* mats, int ld, long long stride, int n, int r0, int np, int c0, int c1,
                 const int* __restrict__ ipiv, int do_trsm) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  int* pos = reinterpret_cast<int*>(sm_raw);            // [2 np] touched positions
  int* cont = pos + 2 * np;                             // [2 np] current content (source row)
  int* slot = cont + 2 * np;                            // [np] list index of position r0+i
  double2* buf = reinterpret_cast<double2*>(
      (reinterpret_cast<uintptr_t>(slot + np) + 15) & ~uintptr_t(15));   // [2 np][ST_COLS]
  double2* xs = buf + (size_t)2 * np * ST_COLS;         // [np][ST_COLS] TRSM work
  const int b = blockIdx.y;
  double2* Mb = mats + b * stride;
  const int* piv = ipiv + (size_t)b * n;
  const int lane = threadIdx.x;   // one warp per CTA

  // fold the sequential interchanges into moves (warp-parallel ballot search)
  int k = 0;
  for (int j = 0; j < np; ++j) {
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
    if (lane == 0 && ia != iq) { int t = cont[ia]; cont[ia] = cont[iq]; cont[iq] = t; }
    __syncwarp();
  }
  for (int t = lane; t < k; t += 32)
    if (pos[t] >= r0 && pos[t] < r0 + np) slot[pos[t] - r0] = t;
  __syncwarp();
  const int c = c0 + blockIdx.x * ST_COLS + lane;
  if (c >= c1) return;
  // gather every source, then scatter the rows that leave the block
  for (int t = 0; t < k; ++t) buf[t * ST_COLS + lane] = Mb[(size_t)cont[t] * ld + c];
  for (int t = 0; t < k; ++t)
    if (pos[t] >= r0 + np) Mb[(size_t)pos[t] * ld + c] = buf[t * ST_COLS + lane];
  for (int i = 0; i < np; ++i) xs[i * ST_COLS + lane] = buf[slot[i] * ST_COLS + lane];
  if (do_trsm) {
    for (int i = 1; i < np; ++i) {
      double2 x = xs[i * ST_COLS + lane];
      const double2* Lrow = Mb + (size_t)(r0 + i) * ld + r0;
      for (int l = 0; l < i; ++l) x = cfms(x, Lrow[l], xs[l * ST_COLS + lane]);
      xs[i * ST_COLS + lane] = x;
    }
  }
  for (int i = 0; i < np; ++i) Mb[(size_t)(r0 + i) * ld + c] = xs[i * ST_COLS + lane];
}

size_t swap_trsm_smem(int np) {
  return (size_t)(5 * np + 8) * sizeof(int) + (size_t)3 * np * ST_COLS * sizeof(double2) + 64;
}

cudaError_t swap_trsm(double2* mats, int ld, long long stride, int n, int r0, int np, int c0,
                      int c1, const int* ipiv, bool do_trsm, int batch, cudaStream_t s) {
  if (c1 <= c0 || np <= 0) return cudaSuccess;
  const size_t smem = swap_trsm_smem(np);
  static size_t configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(swap_trsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  dim3 grid((c1 - c0 + ST_COLS - 1) / ST_COLS, batch);
  swap_trsm_kernel<<<grid, ST_COLS, smem, s>>>(mats, ld, stride, n, r0, np, c0, c1, ipiv, do_trsm ? 1 : 0);
  note_launch();
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------- K6 upper TRSM
// Rows r0..r0+np of the columns [c0, c1): x = U11^{-1} y, U11 non-unit upper (rows/cols r0..).
__global__ void trsm_upper_kernel(double2* mats, int ld, long long stride, int r0, int np, int c0, int c1) {
  extern __shared__ __align__(16) double2 xs[];   // [np][blockDim.x]
  const int b = blockIdx.y;
  double2* Mb = mats + b * stride;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int c = c0 + blockIdx.x * nt + tid;
  if (c >= c1) return;
  for (int i = 0; i < np; ++i) xs[i * nt + tid] = Mb[(size_t)(r0 + i) * ld + c];
  for (int i = np - 1; i >= 0; --i) {
    const double2* Urow = Mb + (size_t)(r0 + i) * ld + r0;
    double2 x = xs[i * nt + tid];
    for (int l = i + 1; l < np; ++l) x = cfms(x, Urow[l], xs[l * nt + tid]);
    const double2 u = Urow[i];
    x = cabs2(u) != 0.0 ? cmul(x, crecip(u)) : x;
    xs[i * nt + tid] = x;
  }
  for (int i = 0; i < np; ++i) Mb[(size_t)(r0 + i) * ld + c] = xs[i * nt + tid];
}

cudaError_t trsm_upper(double2* mats, int ld, long long stride, int r0, int np, int c0, int c1,
                       int batch, cudaStream_t s) {
  if (c1 <= c0 || np <= 0) return cudaSuccess;
  const int nt = 32;
  const size_t smem = (size_t)np * nt * sizeof(double2);
  static size_t configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(trsm_upper_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  dim3 grid((c1 - c0 + nt - 1) / nt, batch);
  trsm_upper_kernel<<<grid, nt, smem, s>>>(mats, ld, stride, r0, np, c0, c1);
  note_launch();
  return cudaGetLastError();
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

}  // namespace sssvd_gpu

namespace sssvd_gpu {

// ----------------------------------------------------------------------------- interchange map
// One warp per shift folds the np sequential interchanges (r0+j <-> ipiv[r0+j]) into
//   src[q]  (q < np): the ORIGINAL row whose content ends at position r0+q, and
//   disp    : the moves (dst >= r0+np <- src) of rows displaced below the panel.
// Every displaced row receives original content of a panel row (ipiv[r0+j] >= r0+j), so the
// displaced moves can be applied in place before the panel rows are overwritten.
__device__ __forceinline__ void build_moves_body(const int* __restrict__ ipiv, int n, int r0, int np,
                                                 int* __restrict__ src, int* __restrict__ disp, int stride, int b,
                                                 int* mv) {
  int* pos = mv;              // [2 np]
  int* cont = mv + 2 * np;    // [2 np]
  const int* piv = ipiv + (size_t)b * n;
  const int lane = threadIdx.x & 31;
  int k = 0;
  for (int j = 0; j < np; ++j) {
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
    if (lane == 0 && ia != iq) { int t = cont[ia]; cont[ia] = cont[iq]; cont[iq] = t; }
    __syncwarp();
  }
  int* s = src + (size_t)b * stride;
  int* d = disp + (size_t)b * (2 * stride + 1);
  // displaced moves, compacted with a warp ballot
  int nd = 0;
  for (int base = 0; base < k; base += 32) {
    const int t = base + lane;
    const bool below = t < k && pos[t] >= r0 + np && cont[t] != pos[t];
    if (t < k && pos[t] < r0 + np) s[pos[t] - r0] = cont[t];
    const unsigned bal = __ballot_sync(0xffffffffu, below);
    if (below) {
      const int slot = nd + __popc(bal & ((1u << lane) - 1));
      d[1 + 2 * slot] = pos[t];
      d[2 + 2 * slot] = cont[t];
    }
    nd += __popc(bal);
  }
  if (lane == 0) d[0] = nd;
}

__global__ void build_moves_kernel(const int* __restrict__ ipiv, int n, int r0, int np, int* __restrict__ src,
                                   int* __restrict__ disp, int stride) {
  extern __shared__ int mv[];
  build_moves_body(ipiv, n, r0, np, src, disp, stride, blockIdx.x, mv);
}

cudaError_t build_moves(const int* ipiv, int n, int r0, int np, int* src, int* disp, int stride, int batch,
                        cudaStream_t s) {
  build_moves_kernel<<<batch, 32, 4 * np * sizeof(int), s>>>(ipiv, n, r0, np, src, disp, stride);
  note_launch();
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------- L11^{-1}
// Linv = L11^{-1} for the unit-lower np x np block at (r0, r0): one warp per column j; lanes
// split each dot product, a warp reduction closes it. Row-major output with pitch np.
template <int QMAX>   // np <= 32 QMAX
__device__ __forceinline__ void trinv_lower_body(const double2* __restrict__ mats, int ld, long long stride, int r0,
                                                 int np, double2* __restrict__ linv, long long lstride, int b,
                                                 int j) {
  const int lane = threadIdx.x & 31;
  if (j >= np) return;
  const double2* Mb = mats + b * stride + (size_t)r0 * ld + r0;
  double2* out = linv + (size_t)b * lstride;
  double2 x[QMAX];
#pragma unroll
  for (int q = 0; q < QMAX; ++q) x[q] = make_double2((lane + 32 * q) == j ? 1.0 : 0.0, 0.0);
  // rows in ascending order; the owning slot qi of row i = 32 qi + ii is a compile-time index,
  // and row i's multipliers L[i][l] (l = lane + 32 q) are prefetched one row ahead
  double2 ln[QMAX];
#pragma unroll
  for (int q = 0; q < QMAX; ++q) {
    const int l = lane + 32 * q;
    ln[q] = (j + 1 < np && l < np) ? Mb[(size_t)(j + 1) * ld + l] : make_double2(0.0, 0.0);
  }
#pragma unroll
  for (int qi = 0; qi < QMAX; ++qi) {
    for (int ii = 0; ii < 32; ++ii) {
      const int i = 32 * qi + ii;
      if (i <= j || i >= np) continue;
      double2 lr[QMAX];
#pragma unroll
      for (int q = 0; q < QMAX; ++q) lr[q] = ln[q];
      if (i + 1 < np) {
#pragma unroll
        for (int q = 0; q < QMAX; ++q) {
          const int l = lane + 32 * q;
          ln[q] = l < np ? Mb[(size_t)(i + 1) * ld + l] : make_double2(0.0, 0.0);
        }
      }
      double sr = 0.0, si = 0.0;
#pragma unroll
      for (int q = 0; q <= qi; ++q) {
        const int l = lane + 32 * q;
        if (l >= j && l < i) {
          sr += lr[q].x * x[q].x - lr[q].y * x[q].y;
          si += lr[q].x * x[q].y + lr[q].y * x[q].x;
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        sr += __shfl_xor_sync(0xffffffffu, sr, off);
        si += __shfl_xor_sync(0xffffffffu, si, off);
      }
      if (lane == ii) x[qi] = make_double2(-sr, -si);
    }
  }
#pragma unroll
  for (int q = 0; q < QMAX; ++q) {
    const int i = lane + 32 * q;
    if (i < np) out[(size_t)i * np + j] = i >= j ? x[q] : make_double2(0.0, 0.0);
  }
}

template <int QMAX>
__global__ void trinv_lower_kernel(const double2* __restrict__ mats, int ld, long long stride, int r0, int np,
                                   double2* __restrict__ linv, long long lstride) {
  trinv_lower_body<QMAX>(mats, ld, stride, r0, np, linv, lstride, blockIdx.y,
                         blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5));
}

// build_moves and trinv_lower of one panel node in ONE launch: they are independent (the
// interchange map reads only ipiv, L11^{-1} only the factored panel), so the gather GEMM that
// needs both waits on one kernel instead of two in sequence. Blocks x < ceil(np/4) invert
// columns; block x = ceil(np/4) folds the interchanges (its first warp).
template <int QMAX>
__global__ void panel_prep_kernel(const double2* __restrict__ mats, int ld, long long stride, int r0, int np,
                                  double2* __restrict__ linv, long long lstride, const int* __restrict__ ipiv, int n,
                                  int* __restrict__ src, int* __restrict__ disp, int dstride) {
  extern __shared__ int mv[];
  const int nx = (np + 3) / 4;
  if ((int)blockIdx.x < nx)
    trinv_lower_body<QMAX>(mats, ld, stride, r0, np, linv, lstride, blockIdx.y, blockIdx.x * 4 + (threadIdx.x >> 5));
  else if (threadIdx.x < 32)
    build_moves_body(ipiv, n, r0, np, src, disp, dstride, blockIdx.y, mv);
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

// SSSVD_PANEL_PREP=v1: the 4-warp form with the ballot fold (read per call; graph key)
int panel_prep_variant() {
  const char* e = std::getenv("SSSVD_PANEL_PREP");
  return (e && std::string(e) == "v1") ? 1 : 0;
}

cudaError_t panel_prep(const double2* mats, int ld, long long stride, int r0, int np, double2* linv, long long lstride,
                       const int* ipiv, int n, int* src, int* disp, int dstride, int batch, cudaStream_t s) {
  if (np > 256) return cudaErrorInvalidValue;
  if (panel_prep_variant() == 0) {
    const size_t sm2 = (size_t)(n - r0 + 4 * np) * sizeof(int);
    static size_t configured = 0;
    if (sm2 > configured) {
      cudaError_t e = cudaFuncSetAttribute(panel_prep2_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(panel_prep2_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
      if (e != cudaSuccess) return e;
      configured = sm2;
    }
    dim3 grid2((np + 7) / 8 + 1, batch);
    if (np <= 128)
      panel_prep2_kernel<4><<<grid2, 256, sm2, s>>>(mats, ld, stride, r0, np, linv, lstride, ipiv, n, src, disp, dstride);
    else
      panel_prep2_kernel<8><<<grid2, 256, sm2, s>>>(mats, ld, stride, r0, np, linv, lstride, ipiv, n, src, disp, dstride);
    note_launch();
    return cudaGetLastError();
  }
  dim3 grid((np + 3) / 4 + 1, batch);
  const size_t sm = 4 * np * sizeof(int);
  if (np <= 128)
    panel_prep_kernel<4><<<grid, 128, sm, s>>>(mats, ld, stride, r0, np, linv, lstride, ipiv, n, src, disp, dstride);
  else
    panel_prep_kernel<8><<<grid, 128, sm, s>>>(mats, ld, stride, r0, np, linv, lstride, ipiv, n, src, disp, dstride);
  note_launch();
  return cudaGetLastError();
}

cudaError_t trinv_lower(const double2* mats, int ld, long long stride, int r0, int np, double2* linv,
                        long long lstride, int batch, cudaStream_t s) {
  if (np > 256) return cudaErrorInvalidValue;
  const int wpb = 4;
  dim3 grid((np + wpb - 1) / wpb, batch);
  if (np <= 128)
    trinv_lower_kernel<4><<<grid, 32 * wpb, 0, s>>>(mats, ld, stride, r0, np, linv, lstride);
  else
    trinv_lower_kernel<8><<<grid, 32 * wpb, 0, s>>>(mats, ld, stride, r0, np, linv, lstride);
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
template <int QMAX>   // np <= 32 QMAX
__global__ void trsm_upper_warp_kernel(double2* mats, int ld, long long stride, int r0, int np, int c0, int c1) {
  const int b = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = c0 + blockIdx.x * (blockDim.x >> 5) + warp;
  if (c >= c1) return;
  double2* Mb = mats + b * stride;
  const double2* U = Mb + (size_t)r0 * ld + r0;
  double2 x[QMAX], invd[QMAX];
#pragma unroll
  for (int q = 0; q < QMAX; ++q) {
    const int i = lane + 32 * q;
    x[q] = i < np ? Mb[(size_t)(r0 + i) * ld + c] : make_double2(0.0, 0.0);
    // reciprocal of the pivot of the row this lane owns, off the serial critical path
    const double2 u = i < np ? U[(size_t)i * ld + i] : make_double2(1.0, 0.0);
    invd[q] = cabs2(u) != 0.0 ? crecip(u) : make_double2(1.0, 0.0);
  }
  // row i's multipliers U[i][l] (l = lane + 32 q) are prefetched one row ahead
  double2 un[QMAX];
#pragma unroll
  for (int q = 0; q < QMAX; ++q) {
    const int l = lane + 32 * q;
    un[q] = l < np ? U[(size_t)(np - 1) * ld + l] : make_double2(0.0, 0.0);
  }
#pragma unroll
  for (int qi = QMAX - 1; qi >= 0; --qi) {
    for (int ii = 31; ii >= 0; --ii) {
      const int i = 32 * qi + ii;
      if (i >= np) continue;
      double2 ur[QMAX];
#pragma unroll
      for (int q = 0; q < QMAX; ++q) ur[q] = un[q];
      if (i > 0) {
#pragma unroll
        for (int q = 0; q < QMAX; ++q) {
          const int l = lane + 32 * q;
          un[q] = l < np ? U[(size_t)(i - 1) * ld + l] : make_double2(0.0, 0.0);
        }
      }
      double sr = 0.0, si = 0.0;
#pragma unroll
      for (int q = qi; q < QMAX; ++q) {
        const int l = lane + 32 * q;
        if (l > i && l < np) {
          sr += ur[q].x * x[q].x - ur[q].y * x[q].y;
          si += ur[q].x * x[q].y + ur[q].y * x[q].x;
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
#pragma unroll
  for (int q = 0; q < QMAX; ++q) {
    const int i = lane + 32 * q;
    if (i < np) Mb[(size_t)(r0 + i) * ld + c] = x[q];
  }
}

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

// SSSVD_TRSM=warp (1): every warp streams U11 itself (the previous kernel); read per call so tests
// can compare both (the shifted-solve graph key includes it)
int trsm_variant() {
  const char* tv = std::getenv("SSSVD_TRSM");
  return (tv && std::string(tv) == "warp") ? 1 : 0;
}

cudaError_t trsm_upper_warp(double2* mats, int ld, long long stride, int r0, int np, int c0, int c1, int batch,
                            cudaStream_t s) {
  if (c1 <= c0 || np <= 0) return cudaSuccess;
  if (np > 256) return cudaErrorInvalidValue;
  if (trsm_variant() == 0) {
    constexpr int WPB = 8;
    dim3 grid((c1 - c0 + WPB - 1) / WPB, batch);
    if (np <= 128)
      trsm_upper_smem_kernel<4, WPB><<<grid, 32 * WPB, 0, s>>>(mats, ld, stride, r0, np, c0, c1);
    else
      trsm_upper_smem_kernel<8, WPB><<<grid, 32 * WPB, 0, s>>>(mats, ld, stride, r0, np, c0, c1);
    note_launch();
    return cudaGetLastError();
  }
  const int wpb = 4;
  dim3 grid((c1 - c0 + wpb - 1) / wpb, batch);
  if (np <= 128)
    trsm_upper_warp_kernel<4><<<grid, 32 * wpb, 0, s>>>(mats, ld, stride, r0, np, c0, c1);
  else
    trsm_upper_warp_kernel<8><<<grid, 32 * wpb, 0, s>>>(mats, ld, stride, r0, np, c0, c1);
  note_launch();
  return cudaGetLastError();
}

}  // namespace sssvd_gpu

namespace sssvd_gpu {

// ----------------------------------------------------------------------------- K2 leaf, v2
// Register-resident leaf panel LU. One cluster of C CTAs per shift (blockIdx.y); CTA c owns
// rows [r0 + c R, r0 + (c+1) R) of the leaf columns [r0, r0 + w), thread t of that CTA owns
// rows t + q*NT (q < RPT) with all W columns in registers. The column loop is fully unrolled so
// every register index is static. Per column j:
//   scale + rank-1 update of the thread's own rows (no block barrier: rows are thread-private)
//   -> score of column j+1 fused into the same pass -> warp argmax -> CTA argmax (1 barrier)
//   -> candidate row / diagonal row published in shared memory -> cluster barrier
//   -> warp 0 reduces the C candidates over DSMEM (1 barrier) -> winner row fetched over DSMEM
//   (1 barrier) -> the owners of rows d and p swap contents.
__device__ unsigned long long g_leaf_prof[8];   // per-phase cycle sums (PROF instances only)

template <int W, int RPT, int NT, bool PROF = false>
__global__ void __launch_bounds__(NT, 1)
leaf_lu_v2_kernel(double2* mats, int ld, long long stride, int n, int r0, int w, int R, int* ipiv) {
  __shared__ double2 cand_vals[2][W];
  __shared__ double2 diag_vals[2][W];
  __shared__ double2 urow[W];
  __shared__ double2 drow[W];
  __shared__ double cand_score[2];
  __shared__ int cand_row[2];
  __shared__ double red_s[NT / 32];
  __shared__ int red_r[NT / 32];
  __shared__ int win[2];

  const int C = gridDim.x;
  const unsigned rank = cluster_ctarank();
  const int b = blockIdx.y;
  double2* Mb = mats + b * stride;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int my0 = r0 + (int)rank * R;
  const int myn = max(0, min(R, n - my0));

  const unsigned long long t_entry = PROF ? clock64() : 0ull;
  double2 a[RPT][W];
  int gi[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int li = tid + q * NT;
    gi[q] = li < myn ? my0 + li : 0x7fffffff;
#pragma unroll
    for (int c = 0; c < W; ++c)
      a[q][c] = (li < myn && c < w) ? Mb[(size_t)gi[q] * ld + r0 + c] : make_double2(0.0, 0.0);
  }

#pragma unroll
  for (int j = 0; j < W; ++j) {
    if (j < w) {
      const int d = r0 + j;
      const int par = j & 1;
      const bool rec = PROF && tid == 0 && rank == 0 && b == 0;
      unsigned long long t0 = 0, t1 = 0, t2 = 0, t3 = 0;
      if (rec) t0 = clock64();
      // ---- pivot search on column j (values already updated by the previous iteration)
      double best = -1.0;
      int brow = 0x7fffffff;
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        if (gi[q] >= d && gi[q] != 0x7fffffff) {
          const double s = cabs2(a[q][j]);
          if (s > best || (s == best && gi[q] < brow)) {
            best = s;
            brow = gi[q];
          }
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const double os = __shfl_xor_sync(0xffffffffu, best, off);
        const int orow = __shfl_xor_sync(0xffffffffu, brow, off);
        if (os > best || (os == best && orow < brow)) {
          best = os;
          brow = orow;
        }
      }
      if (lane == 0) {
        red_s[warp] = best;
        red_r[warp] = brow;
      }
      __syncthreads();
      if (rec) t1 = clock64();
      // every thread folds the NT/32 warp partials (so the owner of the CTA candidate knows)
      best = -1.0;
      brow = 0x7fffffff;
#pragma unroll
      for (int w2 = 0; w2 < NT / 32; ++w2) {
        const double os = red_s[w2];
        const int orow = red_r[w2];
        if (os > best || (os == best && orow < brow)) {
          best = os;
          brow = orow;
        }
      }
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        if (gi[q] == brow) {
#pragma unroll
          for (int c = 0; c < W; ++c) cand_vals[par][c] = a[q][c];
        }
        if (gi[q] == d) {
#pragma unroll
          for (int c = 0; c < W; ++c) diag_vals[par][c] = a[q][c];
        }
      }
      if (tid == 0) {
        cand_score[par] = best;
        cand_row[par] = brow;
      }
      cluster_sync_all();
      if (rec) t2 = clock64();
      // ---- winner over the C candidates (DSMEM)
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
          if (os > s || (os == s && orow < r)) {
            s = os;
            r = orow;
            rk = ork;
          }
        }
        if (lane == 0) {
          win[0] = rk;
          win[1] = r;
        }
        // winner's row and the old diagonal row, one element per lane, fetched in parallel
        // (every lane holds the reduced rank / row after the xor butterfly)
        const int downer_w = (d - r0) / R;
        for (int c = lane; c < W; c += 32) {
          urow[c] = ld_dsmem_f64x2(dsmem_addr(&cand_vals[par][c], rk));
          if (r != d && rk == (int)rank) drow[c] = ld_dsmem_f64x2(dsmem_addr(&diag_vals[par][c], downer_w));
        }
      }
      __syncthreads();
      if (rec) t3 = clock64();
      const int wrank = win[0], p = win[1];
      // ---- interchange rows d and p (owners only, from shared memory)
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        if (gi[q] == p && p != d) {
#pragma unroll
          for (int c = 0; c < W; ++c) a[q][c] = drow[c];
        } else if (gi[q] == d) {
#pragma unroll
          for (int c = 0; c < W; ++c) a[q][c] = urow[c];
        }
      }
      (void)wrank;
      if (rank == 0 && tid == 0) ipiv[(size_t)b * n + d] = p;
      // ---- scale column j below the diagonal, rank-1 update of the columns right of j
      const double2 u = urow[j];
      if (cabs2(u) != 0.0) {
        const double2 inv = crecip(u);
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
          if (gi[q] > d && gi[q] != 0x7fffffff) {
            const double2 l = cmul(a[q][j], inv);
            a[q][j] = l;
#pragma unroll
            for (int c = j + 1; c < W; ++c) a[q][c] = cfms(a[q][c], l, urow[c]);
          }
        }
      }
      if (rec) {
        const unsigned long long t4 = clock64();
        atomicAdd(&g_leaf_prof[0], t1 - t0);   // local search + warp/CTA argmax
        atomicAdd(&g_leaf_prof[1], t2 - t1);   // fold + publish + cluster barrier
        atomicAdd(&g_leaf_prof[2], t3 - t2);   // DSMEM winner + row fetch + barrier
        atomicAdd(&g_leaf_prof[3], t4 - t3);   // swap + scale + rank-1 update
        atomicAdd(&g_leaf_prof[4], 1ull);      // columns
      }
    }
  }
  // write back
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    if (gi[q] != 0x7fffffff) {
#pragma unroll
      for (int c = 0; c < W; ++c)
        if (c < w) Mb[(size_t)gi[q] * ld + r0 + c] = a[q][c];
    }
  }
  cluster_sync_all();   // keep every CTA's shared memory alive until all DSMEM reads are done
  if (PROF && tid == 0 && rank == 0 && b == 0) {
    atomicAdd(&g_leaf_prof[5], clock64() - t_entry);   // whole CTA lifetime
    atomicAdd(&g_leaf_prof[6], 1ull);                   // leaves
  }
}

template <int W, int RPT, int NT, bool PROF>
static cudaError_t launch_leaf_v2(double2* mats, int ld, long long stride, int n, int r0, int w, int cluster,
                                  int* ipiv, int batch, cudaStream_t s) {
  const int m = n - r0;
  const int R = (m + cluster - 1) / cluster;
  if (R > RPT * NT) return cudaErrorInvalidValue;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(leaf_lu_v2_kernel<W, RPT, NT, PROF>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cluster, batch, 1);
  cfg.blockDim = dim3(NT, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  note_launch();
  return cudaLaunchKernelEx(&cfg, leaf_lu_v2_kernel<W, RPT, NT, PROF>, mats, ld, stride, n, r0, w, R, ipiv);
}

// variant ids: 0: W32/RPT1/256  1: W16/RPT1/512  2: W8/RPT2/512
int leaf_v2_rows_per_cta(int variant) { return variant == 0 ? 256 : (variant == 1 ? 512 : 1024); }
int leaf_v2_width(int variant) { return variant == 0 ? 32 : (variant == 1 ? 16 : 8); }

static bool leaf_prof_on() {
  static const char* e = std::getenv("SSSVD_LEAF_PROF");
  return e && e[0] == '1';
}

cudaError_t leaf_lu_v2(double2* mats, int ld, long long stride, int n, int r0, int w, int variant, int cluster,
                       int* ipiv, int batch, cudaStream_t s) {
  const bool prof = leaf_prof_on();
  switch (variant) {
    case 0: return prof ? launch_leaf_v2<32, 1, 256, true>(mats, ld, stride, n, r0, w, cluster, ipiv, batch, s)
                        : launch_leaf_v2<32, 1, 256, false>(mats, ld, stride, n, r0, w, cluster, ipiv, batch, s);
    case 1: return prof ? launch_leaf_v2<16, 1, 512, true>(mats, ld, stride, n, r0, w, cluster, ipiv, batch, s)
                        : launch_leaf_v2<16, 1, 512, false>(mats, ld, stride, n, r0, w, cluster, ipiv, batch, s);
    case 2: return prof ? launch_leaf_v2<8, 2, 512, true>(mats, ld, stride, n, r0, w, cluster, ipiv, batch, s)
                        : launch_leaf_v2<8, 2, 512, false>(mats, ld, stride, n, r0, w, cluster, ipiv, batch, s);
    default: return cudaErrorInvalidValue;
  }
}

void leaf_profile_read(unsigned long long* out5, bool reset) {
  cudaMemcpyFromSymbol(out5, g_leaf_prof, 7 * sizeof(unsigned long long));
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_leaf_prof, z, sizeof(z));
  }
}

}  // namespace sssvd_gpu

namespace sssvd_gpu {

// ----------------------------------------------------------------------------- K2 leaf, v3
// Shared-memory slab (as v1: R x (W+1) complex per CTA, one cluster per shift) with thread-owned
// rows (as v2): thread t owns slab rows t, t+NT, ...; for column j it scales its rows, applies
// the rank-1 update to their columns j+1..W-1 and scores column j+1 in the same pass, so the
// only barriers per column are: CTA argmax (1), cluster exchange (1), winner broadcast (1).
// Warp 0 publishes the CTA candidate and the diagonal row straight from the slab, reduces the C
// candidates over DSMEM, fetches the pivot row (and, in the winning CTA, the old diagonal row),
// and performs the interchange in the slab.
template <int W, int NT>
__global__ void __launch_bounds__(NT, 1)
leaf_lu_v3_kernel(double2* mats, int ld, long long stride, int n, int r0, int w, int R, int* ipiv, int cb) {
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

// SSSVD_LEAF_SWAP=kernel: interchanges on the left block columns as a separate swap_trsm launch
// (the previous schedule; read per call for A/B tests, part of the shifted-solve graph key)
bool leaf_swap_fused() {
  const char* e = std::getenv("SSSVD_LEAF_SWAP");
  return !(e && std::string(e) == "kernel");
}

template <int W, int NT>
static cudaError_t launch_leaf_v3(double2* mats, int ld, long long stride, int n, int r0, int w, int cluster,
                                  int* ipiv, int batch, cudaStream_t s, int cb) {
  const int m = n - r0;
  const int R = (m + cluster - 1) / cluster;
  // the slab, or the fused left-swap epilogue's move list + gather buffer if that is larger
  const size_t smem = std::max((size_t)R * (W + 1) * sizeof(double2),
                               cb < r0 ? 1024 + (size_t)2 * W * (r0 - cb) * sizeof(double2) : (size_t)0);
  static size_t configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(leaf_lu_v3_kernel<W, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(leaf_lu_v3_kernel<W, NT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
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
  return cudaLaunchKernelEx(&cfg, leaf_lu_v3_kernel<W, NT>, mats, ld, stride, n, r0, w, R, ipiv, cb);
}

cudaError_t leaf_lu_v3(double2* mats, int ld, long long stride, int n, int r0, int w, int W, int cluster, int* ipiv,
                       int batch, cudaStream_t s, int cb) {
  if (cb > r0) return cudaErrorInvalidValue;
  switch (W) {
    case 8: return launch_leaf_v3<8, 512>(mats, ld, stride, n, r0, w, cluster, ipiv, batch, s, cb);
    case 16: return launch_leaf_v3<16, 512>(mats, ld, stride, n, r0, w, cluster, ipiv, batch, s, cb);
    case 32: return launch_leaf_v3<32, 256>(mats, ld, stride, n, r0, w, cluster, ipiv, batch, s, cb);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace sssvd_gpu
