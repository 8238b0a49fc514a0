// One-sided (Hestenes) Jacobi SVD of a square k x k matrix on the GPU.
//
// Replaces the Eigen::JacobiSVD calls of the small dense tail: low_rank
// (proj/include/sssvd/moments.hpp:199, SVD of the R factor of the stacked moments) and
// svd_small (proj/include/sssvd/extract.hpp:66-70, SVD of the projected triangular factor B).
// Jacobi keeps the small singular values of a graded triangular factor to high relative
// accuracy, and the spurious-triplet index tau (postprocess.hpp:56-60) is driven by exactly
// those values, so a Jacobi method is what keeps tau faithful to the reference.
//
// W = B (column-major), V = I. A sweep is k-1 rounds of a round-robin tournament; in a round the
// k/2 disjoint column pairs (p, q) are orthogonalised concurrently, one warp per pair:
//   alpha = |w_p|^2, beta = |w_q|^2, gamma = w_p . w_q  (warp reductions)
//   rotate iff |gamma| > tol sqrt(alpha beta):  zeta = (beta - alpha) / (2 gamma),
//   t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)), c = 1/sqrt(1 + t^2), s = c t
//   [w_p w_q] <- [w_p w_q] [c s; -s c],  same for V.
// The kernel is persistent (cooperative launch: all CTAs resident) and separates rounds with a
// sense-reversing software grid barrier; a sweep without any rotation ends the iteration.
// Afterwards sigma_j = |w_j|, u_j = w_j / sigma_j, sorted nonincreasing on the host.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace sssvd_gpu {

namespace {

struct GridBarrier {
  unsigned int* count;   // monotonic arrival counter (zeroed before the launch)
  unsigned int* unused;
};

// Software grid barrier over co-resident CTAs: every CTA adds one arrival (fire-and-forget
// release reduction) and polls the counter with acquire loads until all arrivals of this
// barrier instance are in. The counter only grows, so there is no reset and no second round
// trip; `target` is this CTA's running count of expected arrivals.
__device__ __forceinline__ void grid_barrier(GridBarrier b, unsigned int nblocks, unsigned int& target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    target += nblocks;
    __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(b.count) : "memory");
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(b.count) : "memory");
    } while ((int)(v - target) < 0);
    __threadfence();
  }
  __syncthreads();
}

// tournament position -> column index (player 0 fixed, the others rotate)
__device__ __forceinline__ int player(int pos, int round, int k) {
  return pos == 0 ? 0 : ((pos - 1 + round) % (k - 1)) + 1;
}

}  // namespace

__global__ void __launch_bounds__(256)
jacobi_svd_kernel(double* __restrict__ Wm, double* __restrict__ Vm, int k, int ldw, double tol, int max_sweeps,
                  unsigned int* __restrict__ bar, unsigned int* __restrict__ rot_count, int* __restrict__ sweeps_out) {
  GridBarrier gb{bar, bar + 1};
  unsigned int local_gen = 0;
  const int lane = threadIdx.x & 31;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int kk = k + (k & 1);   // odd k: a dummy player k sits out one pair per round
  const int npairs = kk / 2;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    for (int round = 0; round < kk - 1; ++round) {
      for (int pi = gwarp; pi < npairs; pi += nwarps) {
        int p = player(pi, round, kk), q = player(kk - 1 - pi, round, kk);
        if (p > q) { int t = p; p = q; q = t; }
        if (q >= k) continue;
        double* wp = Wm + (size_t)p * ldw;
        double* wq = Wm + (size_t)q * ldw;
        // pass 1: the 2x2 Gram entries. The grid barrier's gpu-scope fence invalidated this SM's
        // L1, so cached loads see the other CTAs' writes of the previous round.
        double a = 0.0, bb = 0.0, g = 0.0;
#pragma unroll 8
        for (int i = lane; i < k; i += 32) {
          const double x = wp[i], y = wq[i];
          a += x * x;
          bb += y * y;
          g += x * y;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          a += __shfl_xor_sync(0xffffffffu, a, off);
          bb += __shfl_xor_sync(0xffffffffu, bb, off);
          g += __shfl_xor_sync(0xffffffffu, g, off);
        }
        if (fabs(g) > tol * sqrt(a) * sqrt(bb) && g != 0.0) {
          const double zeta = (bb - a) / (2.0 * g);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
          // pass 2: rotate W and V columns (the reloads hit L1: this warp just read them)
          double* vp = Vm + (size_t)p * ldw;
          double* vq = Vm + (size_t)q * ldw;
#pragma unroll 4
          for (int i = lane; i < k; i += 32) {
            const double x = wp[i], y = wq[i];
            const double v1 = vp[i], v2 = vq[i];
            wp[i] = c * x - s * y;
            wq[i] = s * x + c * y;
            vp[i] = c * v1 - s * v2;
            vq[i] = s * v1 + c * v2;
          }
          if (lane == 0) atomicAdd(rot_count + (sweep & 1), 1u);
        }
      }
      grid_barrier(gb, gridDim.x, local_gen);
    }
    // sweep done: every CTA reads the rotation count of this sweep; the other slot is reset
    const unsigned int rc = *((volatile unsigned int*)(rot_count + (sweep & 1)));
    if (blockIdx.x == 0 && threadIdx.x == 0) rot_count[(sweep + 1) & 1] = 0;
    grid_barrier(gb, gridDim.x, local_gen);
    if (rc == 0) {
      ++sweep;
      break;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *sweeps_out = sweep;
}


// Same sweep, run by ONE thread-block cluster (16 CTAs x 512 threads): rounds are separated by
// the hardware cluster barrier (release/acquire at cluster scope; it also invalidates L1, so the
// global-memory columns written in one round are seen by every CTA in the next).
__global__ void __launch_bounds__(512, 1)
jacobi_svd_cluster_kernel(double* __restrict__ Wm, double* __restrict__ Vm, int k, int ldw, double tol,
                          int max_sweeps, unsigned int* __restrict__ rot_count, int* __restrict__ sweeps_out) {
  const int lane = threadIdx.x & 31;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int kk = k + (k & 1);
  const int npairs = kk / 2;
  __shared__ unsigned int cta_rot;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    unsigned int my_rot = 0;   // rotations by this warp in this sweep (no per-round atomics)
    if (threadIdx.x == 0) cta_rot = 0;
    for (int round = 0; round < kk - 1; ++round) {
      for (int pi = gwarp; pi < npairs; pi += nwarps) {
        int p = player(pi, round, kk), q = player(kk - 1 - pi, round, kk);
        if (p > q) { int t = p; p = q; q = t; }
        if (q >= k) continue;
        double* wp = Wm + (size_t)p * ldw;
        double* wq = Wm + (size_t)q * ldw;
        double a = 0.0, bb = 0.0, g = 0.0;
#pragma unroll 8
        for (int i = lane; i < k; i += 32) {
          const double x = wp[i], y = wq[i];
          a += x * x;
          bb += y * y;
          g += x * y;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          a += __shfl_xor_sync(0xffffffffu, a, off);
          bb += __shfl_xor_sync(0xffffffffu, bb, off);
          g += __shfl_xor_sync(0xffffffffu, g, off);
        }
        if (fabs(g) > tol * sqrt(a) * sqrt(bb) && g != 0.0) {
          const double zeta = (bb - a) / (2.0 * g);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
          double* vp = Vm + (size_t)p * ldw;
          double* vq = Vm + (size_t)q * ldw;
#pragma unroll 4
          for (int i = lane; i < k; i += 32) {
            const double x = wp[i], y = wq[i];
            const double v1 = vp[i], v2 = vq[i];
            wp[i] = c * x - s * y;
            wq[i] = s * x + c * y;
            vp[i] = c * v1 - s * v2;
            vq[i] = s * v1 + c * v2;
          }
          ++my_rot;
        }
      }
      cluster_sync_all();
    }
    // one atomic per CTA per sweep
    if (lane == 0 && my_rot) atomicAdd(&cta_rot, my_rot);
    __syncthreads();
    if (threadIdx.x == 0 && cta_rot) atomicAdd(rot_count + (sweep & 1), cta_rot);
    cluster_sync_all();
    const unsigned int rc = *((volatile unsigned int*)(rot_count + (sweep & 1)));
    if (blockIdx.x == 0 && threadIdx.x == 0) rot_count[(sweep + 1) & 1] = 0;
    cluster_sync_all();
    if (rc == 0) {
      ++sweep;
      break;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *sweeps_out = sweep;
}

// sigma_j = |w_j| and u_j = w_j / sigma_j (u_j = 0 when sigma_j = 0), column-major k x k
__global__ void jacobi_finish_kernel(double* __restrict__ Wm, int k, int ldw, double* __restrict__ S) {
  const int j = blockIdx.x;
  double* w = Wm + (size_t)j * ldw;
  double acc = 0.0;
  for (int i = threadIdx.x; i < k; i += blockDim.x) acc += w[i] * w[i];
  __shared__ double red[32];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (threadIdx.x == 0) red[0] = sqrt(acc);
  }
  __syncthreads();
  const double s = red[0];
  if (threadIdx.x == 0) S[j] = s;
  const double inv = s > 0.0 ? 1.0 / s : 0.0;
  for (int i = threadIdx.x; i < k; i += blockDim.x) w[i] *= inv;
}

__global__ void set_identity_kernel(double* __restrict__ V, int k, int ldv) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)k * ldv;
       e += (long long)gridDim.x * blockDim.x)
    V[e] = (e % ldv) == (e / ldv) ? 1.0 : 0.0;
}

cudaError_t jacobi_svd(double* W, double* V, int k, int ldw, double* S, double tol, int max_sweeps,
                       unsigned int* scratch /* >= 8 uints, zeroed by this call */, int* sweeps_out,
                       cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(scratch, 0, 8 * sizeof(unsigned int), s);
  if (e != cudaSuccess) return e;
  set_identity_kernel<<<148 * 4, 256, 0, s>>>(V, k, ldw);
  note_launch();
  if (k > 1) {
    e = set_kernel_smem((const void*)jacobi_svd_cluster_kernel, 0, true);
    if (e != cudaSuccess) return e;
    unsigned int* rot = scratch + 2;      // [2], [3] rotation counts (ping-pong by sweep parity)
    const int npairs = (k + (k & 1)) / 2;
    if (npairs > 256) {
      // large k (configs 3, 5: k = 1024, 2048): the whole GPU, one column pair per warp per round,
      // rounds separated by a software grid barrier over co-resident CTAs (cooperative launch)
      int ctas = std::min(148, (npairs + 7) / 8);
      unsigned int* bar = scratch;         // [0] arrivals, [1] generation (zeroed above)
      void* args[] = {&W, &V, &k, &ldw, &tol, &max_sweeps, &bar, &rot, &sweeps_out};
      e = cudaLaunchCooperativeKernel((const void*)jacobi_svd_kernel, dim3(ctas), dim3(256), args, 0, s);
      if (e != cudaSuccess) return e;
      note_launch();
      jacobi_finish_kernel<<<k, 256, 0, s>>>(W, k, ldw, S);
      note_launch();
      return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16, 1, 1);
    cfg.blockDim = dim3(512, 1, 1);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 16;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, jacobi_svd_cluster_kernel, W, V, k, ldw, tol, max_sweeps, rot, sweeps_out);
    if (e != cudaSuccess) return e;
    note_launch();
  }
  jacobi_finish_kernel<<<k, 256, 0, s>>>(W, k, ldw, S);
  note_launch();
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------- grid block Jacobi
// Block one-sided Jacobi (every k from 64 to 2048: the tail's k x k factors of configs 1-5) on the
// whole GPU. Cyclic block ordering: an outer tournament over nb blocks of b columns; round 0 of a
// sweep runs the full inner sweep of each block pair, later rounds only the b x b cross pairs. The
// block pairs are spread over one persistent CTA per SM and outer rounds are separated by the software grid barrier. b is the widest block whose
// pair fits shared memory, up to one warp per resident column (k = 2048: b = 7, 147 pairs on
// 148 SMs, 229 KB; k = 1024: b = 8, 64 pairs): nb - 1 grid barriers per sweep instead of the
// scalar kernel's k - 1, and the column traffic of the inner rounds stays on chip.
//
// Inner rounds: one warp owns one pair; lane t holds rows t + 32 i (i < RPL, RPL = 16 / 32 / 64
// for k <= 512 / 1024 / 2048) of the resident column x in registers and streams the partner
// column y from shared memory twice (dot products, then the rotation), so only x occupies
// registers (256 threads per CTA: up to 255 registers per thread).
constexpr int GB_THREADS = 256;

template <int RPL>
__device__ __forceinline__ void gb_load_x(double (&x)[RPL], const double* col, int k, int lane) {
#pragma unroll
  for (int i = 0; i < RPL; ++i) {
    const int r = lane + 32 * i;
    x[i] = r < k ? col[r] : 0.0;
  }
}
template <int RPL>
__device__ __forceinline__ void gb_store_x(const double (&x)[RPL], double* col, int k, int lane) {
#pragma unroll
  for (int i = 0; i < RPL; ++i) {
    const int r = lane + 32 * i;
    if (r < k) col[r] = x[i];
  }
}

// orthogonalise register column x against shared column y (rotating both); true iff rotated.
// Same test and rotation as pair_rotation.
// both columns in shared memory (outer round 0 only, where the pairs change every inner round)
__device__ __forceinline__ bool gb_visit_smem(double* x, double* y, int k, double tol, int lane, double& cs,
                                              double& sn, double& c2max) {
  double a = 0.0, bb = 0.0, g = 0.0;
#pragma unroll 8
  for (int r = lane; r < k; r += 32) {
    const double xv = x[r], yv = y[r];
    a = fma(xv, xv, a);
    bb = fma(yv, yv, bb);
    g = fma(xv, yv, g);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, off);
    bb += __shfl_xor_sync(0xffffffffu, bb, off);
    g += __shfl_xor_sync(0xffffffffu, g, off);
  }
  if (!(g * g > tol * tol * a * bb) || g == 0.0) return false;
  c2max = fmax(c2max, g * g / (a * bb));   // squared cosine of the largest angle rotated so far
  const double d = bb - a, g2x = 2.0 * g;
  const double tt = copysign(1.0, d) * g2x / (fabs(d) + sqrt(fma(d, d, g2x * g2x)));
  cs = rsqrt(fma(tt, tt, 1.0));
  sn = cs * tt;
#pragma unroll 8
  for (int r = lane; r < k; r += 32) {
    const double u = x[r], v = y[r];
    x[r] = cs * u - sn * v;
    y[r] = sn * u + cs * v;
  }
  return true;
}

template <int RPL>
__device__ __forceinline__ bool gb_visit(double (&x)[RPL], double* y, int k, double tol, int lane, double& cs,
                                         double& sn, double& c2max) {
  // four partial sums per product: 4x shorter FMA dependency chains
  double a4[4] = {0.0, 0.0, 0.0, 0.0}, b4[4] = {0.0, 0.0, 0.0, 0.0}, g4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int i = 0; i < RPL; ++i) {
    const int r = lane + 32 * i;
    const double yv = r < k ? y[r] : 0.0;
    a4[i & 3] = fma(x[i], x[i], a4[i & 3]);
    b4[i & 3] = fma(yv, yv, b4[i & 3]);
    g4[i & 3] = fma(x[i], yv, g4[i & 3]);
  }
  double a = (a4[0] + a4[1]) + (a4[2] + a4[3]);
  double bb = (b4[0] + b4[1]) + (b4[2] + b4[3]);
  double g = (g4[0] + g4[1]) + (g4[2] + g4[3]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, off);
    bb += __shfl_xor_sync(0xffffffffu, bb, off);
    g += __shfl_xor_sync(0xffffffffu, g, off);
  }
  if (!(g * g > tol * tol * a * bb) || g == 0.0) return false;
  c2max = fmax(c2max, g * g / (a * bb));   // squared cosine of the largest angle rotated so far
  const double d = bb - a, g2x = 2.0 * g;
  const double tt = copysign(1.0, d) * g2x / (fabs(d) + sqrt(fma(d, d, g2x * g2x)));
  cs = rsqrt(fma(tt, tt, 1.0));
  sn = cs * tt;
#pragma unroll
  for (int i = 0; i < RPL; ++i) {
    const int r = lane + 32 * i;
    if (r < k) {
      const double u = x[i], v = y[r];
      x[i] = cs * u - sn * v;
      y[r] = sn * u + cs * v;
    }
  }
  return true;
}

// V[:, pair] <- V[:, pair] Q of one outer round, captured in registers (Q's DMMA B fragments and
// the pair's column ids) so that it can run one round later, overlapped with the next block-pair
// load. V columns of a pair are touched by no other CTA until the round after next (blocks move
// on and every CTA defers its own update by exactly one round), so the deferral is race-free.
struct VUpdate {
  double bq[4][2];
  int acol[4], ocol[4];
  bool on;
};

__device__ __forceinline__ void vupdate_capture(VUpdate& u, const double* Qs, const int* colid, int w2, int lane,
                                                bool on) {
  const int fr = lane >> 2, fc = lane & 3;
  u.on = on;
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const int lc = 4 * kk + fc;
    u.acol[kk] = lc < w2 ? colid[lc] : -1;
#pragma unroll
    for (int nj = 0; nj < 2; ++nj) u.bq[kk][nj] = Qs[(size_t)(8 * nj + fr) * 16 + 4 * kk + fc];
  }
#pragma unroll
  for (int nj = 0; nj < 2; ++nj)
#pragma unroll
    for (int e2 = 0; e2 < 2; ++e2) {
      const int lc = 8 * nj + 2 * fc + e2;
      u.ocol[2 * nj + e2] = lc < w2 ? colid[lc] : -1;
    }
}

// DMMA m8n8k4 with the 2b <= 16 local columns zero-padded to 16: warp w owns rows
// [w k/8, (w+1) k/8), 64 rows per step; A fragments straight from L2, and each warp reads a
// step's rows completely before writing them back (in place)
__device__ __forceinline__ void vupdate_apply(const VUpdate& u, double* __restrict__ Vm, int k, int ldw, int warp,
                                              int lane) {
  const int fr = lane >> 2;
  const int rows_per_warp = (k + 8 * 64 - 1) / (8 * 64) * 64;
  const int rw0 = warp * rows_per_warp, rw1 = min(k, rw0 + rows_per_warp);
  for (int r0 = rw0; r0 < rw1; r0 += 64) {
    double a[4][8];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
#pragma unroll
      for (int mi = 0; mi < 8; ++mi) {
        const int r = r0 + 8 * mi + fr;
        a[kk][mi] = (u.acol[kk] >= 0 && r < rw1) ? __ldcg(Vm + (size_t)u.acol[kk] * ldw + r) : 0.0;
      }
    double acc[8][2][2];
#pragma unroll
    for (int mi = 0; mi < 8; ++mi)
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) acc[mi][nj][0] = acc[mi][nj][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
#pragma unroll
      for (int mi = 0; mi < 8; ++mi)
#pragma unroll
        for (int nj = 0; nj < 2; ++nj) dmma884(acc[mi][nj][0], acc[mi][nj][1], a[kk][mi], u.bq[kk][nj]);
#pragma unroll
    for (int mi = 0; mi < 8; ++mi) {
      const int r = r0 + 8 * mi + fr;
      if (r < rw1) {
#pragma unroll
        for (int nj = 0; nj < 2; ++nj)
#pragma unroll
          for (int e2 = 0; e2 < 2; ++e2)
            if (u.ocol[2 * nj + e2] >= 0) Vm[(size_t)u.ocol[2 * nj + e2] * ldw + r] = acc[mi][nj][e2];
      }
    }
  }
}

// one block pair per CTA per outer round (the plan guarantees nbe / 2 <= CTAs)
constexpr double kJacobiFinalCos = 1e-8;

template <int RPL, bool PROF>
__global__ void __launch_bounds__(GB_THREADS, 1)
jacobi_grid_block_kernel(double* __restrict__ Wm, double* __restrict__ Vm, int k, int ldw, int b, int nbe,
                         double tol, int max_sweeps, unsigned int* __restrict__ bar,
                         unsigned int* __restrict__ rot_count, int* __restrict__ sweeps_out,
                         unsigned long long* __restrict__ prof) {
  // rot_count[0..1]: rotations of the sweep (ping-pong by sweep parity); the two 64-bit words after
  // them: the largest squared cosine rotated in the sweep (double bits: order-preserving for >= 0)
  unsigned long long* c2_glob = reinterpret_cast<unsigned long long*>(rot_count + 2);
  extern __shared__ __align__(16) double gsm[];
  const int w2 = 2 * b;
  double* Ws = gsm;                        // [w2][k]
  double* Qs = Ws + (size_t)w2 * k;        // [16][16] column-major (2b <= 16, zero padded)
  __shared__ int colid[32];
  __shared__ unsigned int cta_rot;
  __shared__ unsigned long long cta_c2;
  __shared__ int pair_rot;
  __shared__ __align__(8) unsigned long long mbar;
  GridBarrier gb{bar, bar + 1};
  unsigned int local_gen = 0;
  unsigned phase = 0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool bulk = (k % 2) == 0 && (ldw % 2) == 0;
  if (tid == 0) mbar_init(&mbar, 1);
  __syncthreads();
  const int pi = blockIdx.x;
  const bool rec = PROF && blockIdx.x == 0 && tid == 0;
  unsigned long long t0 = 0, t1 = 0, t2 = 0, t3 = 0;
  VUpdate vu;
  vu.on = false;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    unsigned int my_rot = 0;
    double my_c2 = 0.0;
    if (tid == 0) {
      cta_rot = 0;
      cta_c2 = 0ull;
    }
    for (int round = 0; round < nbe - 1; ++round) {
      if (rec) t0 = clock64();
      const int bx = player(pi, round, nbe), by = player(nbe - 1 - pi, round, nbe);
      if (tid < w2) {
        const int blk = tid < b ? bx : by;
        const int gc = blk * b + (tid < b ? tid : tid - b);
        colid[tid] = gc < k ? gc : -1;
      }
      if (tid == 0) pair_rot = 0;
      __syncthreads();
      // block pair -> Ws (TMA bulk copies on one mbarrier), overlapped with the previous round's
      // V update; padding columns are zero-filled
      if (bulk) {
        if (tid == 0) {
          fence_proxy_async();
          unsigned bytes = 0;
          for (int lc = 0; lc < w2; ++lc)
            if (colid[lc] >= 0) bytes += (unsigned)k * 8u;
          mbar_expect_tx(&mbar, bytes);
        }
        __syncthreads();
        if (tid < w2 && colid[tid] >= 0)
          bulk_g2s(Ws + (size_t)tid * k, Wm + (size_t)colid[tid] * ldw, (unsigned)k * 8u, &mbar);
      } else {
        for (int lc = 0; lc < w2; ++lc) {
          const int gc = colid[lc];
          if (gc >= 0)
            for (int r = tid; r < k; r += GB_THREADS) Ws[(size_t)lc * k + r] = __ldcg(Wm + (size_t)gc * ldw + r);
        }
      }
      for (int lc = 0; lc < w2; ++lc)
        if (colid[lc] < 0)
          for (int r = tid; r < k; r += GB_THREADS) Ws[(size_t)lc * k + r] = 0.0;
      for (int e = tid; e < 256; e += GB_THREADS) Qs[e] = (e >> 4) == (e & 15) ? 1.0 : 0.0;
      if (vu.on) vupdate_apply(vu, Vm, k, ldw, warp, lane);
      if (bulk) {
        mbar_wait(&mbar, phase);
        phase ^= 1u;
      }
      __syncthreads();
      if (rec) t1 = clock64();
      if (round == 0) {
        // full inner sweep over the 2b local columns (intra-block + cross pairs)
        for (int ir = 0; ir < w2 - 1; ++ir) {
          for (int p0 = warp; p0 < b; p0 += GB_THREADS / 32) {
            int p = player(p0, ir, w2), q = player(w2 - 1 - p0, ir, w2);
            if (p > q) { int t = p; p = q; q = t; }
            double cs, sn;
            if (gb_visit_smem(Ws + (size_t)p * k, Ws + (size_t)q * k, k, tol, lane, cs, sn, my_c2)) {
              if (lane < w2) {
                double* qp = Qs + (size_t)p * 16;
                double* qq = Qs + (size_t)q * 16;
                const double u = qp[lane], v = qq[lane];
                qp[lane] = cs * u - sn * v;
                qq[lane] = sn * u + cs * v;
              }
              if (lane == 0) {
                ++my_rot;
                pair_rot = 1;
              }
            }
          }
          __syncthreads();
        }
      } else {
        // cross pairs only: warp p keeps local column p resident, partners b + (p + ir) mod b
        // rotate past it one per inner round (the plan guarantees b <= warps)
        const int p = warp;
        const bool active = p < b;
        double x[RPL];
        if (active) gb_load_x<RPL>(x, Ws + (size_t)p * k, k, lane);
        bool moved = false;
        for (int ir = 0; ir < b; ++ir) {
          if (active) {
            const int q = b + (p + ir) % b;
            double cs, sn;
            if (gb_visit<RPL>(x, Ws + (size_t)q * k, k, tol, lane, cs, sn, my_c2)) {
              if (lane < w2) {
                double* qp = Qs + (size_t)p * 16;
                double* qq = Qs + (size_t)q * 16;
                const double u = qp[lane], v = qq[lane];
                qp[lane] = cs * u - sn * v;
                qq[lane] = sn * u + cs * v;
              }
              moved = true;
              if (lane == 0) ++my_rot;
            }
          }
          __syncthreads();   // partner columns move on to the next warp
        }
        if (active && moved) {
          gb_store_x<RPL>(x, Ws + (size_t)p * k, k, lane);
          if (lane == 0) pair_rot = 1;
        }
        __syncthreads();
      }
      if (rec) t2 = clock64();
      // a pair without rotations leaves W and V unchanged: no write-back, no V update
      const bool rotated = pair_rot != 0;
      vupdate_capture(vu, Qs, colid, w2, lane, rotated);
      if (rotated) {
        if (bulk) {
          fence_proxy_async();
          __syncthreads();
          if (tid < w2 && colid[tid] >= 0)
            bulk_s2g(Wm + (size_t)colid[tid] * ldw, Ws + (size_t)tid * k, (unsigned)k * 8u);
          if (tid < w2) {
            bulk_commit();
            bulk_wait_all();
            __threadfence();
          }
        } else {
          for (int lc = 0; lc < w2; ++lc) {
            const int gc = colid[lc];
            if (gc >= 0)
              for (int r = tid; r < k; r += GB_THREADS) Wm[(size_t)gc * ldw + r] = Ws[(size_t)lc * k + r];
          }
        }
      }
      if (rec) t3 = clock64();
      grid_barrier(gb, gridDim.x, local_gen);
      if (rec) {
        const unsigned long long t4 = clock64();
        prof[0] += t1 - t0;   // block pair load (+ the previous round's V update)
        prof[1] += t2 - t1;   // inner rounds
        prof[2] += t3 - t2;   // write back
        prof[3] += t4 - t3;   // grid barrier
        prof[4] += 1;
        if (round == 0) prof[5] += t2 - t1;   // inner rounds of outer round 0 (full inner sweep)
      }
    }
    if (lane == 0 && my_rot) {
      atomicAdd(&cta_rot, my_rot);
      atomicMax(&cta_c2, (unsigned long long)__double_as_longlong(my_c2));
    }
    __syncthreads();
    if (tid == 0 && cta_rot) {
      atomicAdd(rot_count + (sweep & 1), cta_rot);
      atomicMax(c2_glob + (sweep & 1), cta_c2);
    }
    grid_barrier(gb, gridDim.x, local_gen);
    const unsigned int rc = *((volatile unsigned int*)(rot_count + (sweep & 1)));
    const double c2 = __longlong_as_double((long long)*((volatile unsigned long long*)(c2_glob + (sweep & 1))));
    if (blockIdx.x == 0 && tid == 0) {
      rot_count[(sweep + 1) & 1] = 0;
      c2_glob[(sweep + 1) & 1] = 0ull;
    }
    grid_barrier(gb, gridDim.x, local_gen);
    // converged: no rotation, or only rotations by angles whose cosine is below kJacobiFinalCos.
    // Rotating two columns by such an angle changes any cosine by O(c^2) <= 1e-16 < tol, so the next
    // sweep would find nothing to rotate: the sweep that would only confirm it is skipped.
    if (rc == 0 || c2 < kJacobiFinalCos * kJacobiFinalCos) {
      ++sweep;
      break;
    }
  }
  if (vu.on) vupdate_apply(vu, Vm, k, ldw, warp, lane);   // the last round's deferred update
  if (blockIdx.x == 0 && tid == 0) *sweeps_out = sweep;
}

// plan for the grid block Jacobi: b columns per block, padded block count, rows per lane;
// false when the shape does not fit (callers fall back to the scalar grid kernel)
bool jacobi_grid_block_plan(int k, int sms, int* b_out, int* nbe_out, int* rpl_out, size_t* smem_out) {
  if (k < 64 || k > 32 * 64) return false;
  const int rpl = k <= 32 * 16 ? 16 : k <= 32 * 32 ? 32 : 64;
  // widest block (fewest outer rounds, i.e. grid barriers, per sweep) with one warp per resident
  // column and the pair in shared memory; at least enough blocks to cover the SMs once
  int b = GB_THREADS / 32;
  {
    // measurement override: a narrower block (more pairs per round, more rounds per sweep)
    static const char* be = std::getenv("SSSVD_JACOBI_B");
    if (be && std::atoi(be) >= 2 && std::atoi(be) < b) b = std::atoi(be);
  }
  const size_t limit = 232448 - 1024;   // 227 KB opt-in per CTA, less the static shared memory
  while (b > 2 && ((size_t)2 * b * k + 256) * sizeof(double) > limit) --b;
  if (b < (k + 2 * sms - 1) / (2 * sms)) return false;
  const size_t smem = ((size_t)2 * b * k + 256) * sizeof(double);
  if (smem > limit) return false;
  const int nb = (k + b - 1) / b;
  *b_out = b;
  *nbe_out = nb + (nb & 1);
  *rpl_out = rpl;
  *smem_out = smem;
  return true;
}

cudaError_t jacobi_svd_grid_block(double* W, double* V, int k, int ldw, double* S, double tol, int max_sweeps,
                                  unsigned int* scratch, int* sweeps_out, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int b, nbe, rpl;
  size_t smem;
  if (!jacobi_grid_block_plan(k, sms, &b, &nbe, &rpl, &smem)) return cudaErrorInvalidValue;
  cudaError_t e = cudaMemsetAsync(scratch, 0, 8 * sizeof(unsigned int), s);
  if (e != cudaSuccess) return e;
  set_identity_kernel<<<148 * 4, 256, 0, s>>>(V, k, ldw);
  note_launch();
  static const bool prof_on = std::getenv("SSSVD_JACOBI_PROF") != nullptr;
  static unsigned long long* dprof = nullptr;
  if (prof_on && !dprof) cudaMalloc(&dprof, 8 * sizeof(unsigned long long));
  if (prof_on) cudaMemsetAsync(dprof, 0, 8 * sizeof(unsigned long long), s);
  const void* fn = rpl == 16   ? (prof_on ? (const void*)jacobi_grid_block_kernel<16, true>
                                          : (const void*)jacobi_grid_block_kernel<16, false>)
                   : rpl == 32 ? (prof_on ? (const void*)jacobi_grid_block_kernel<32, true>
                                          : (const void*)jacobi_grid_block_kernel<32, false>)
                               : (prof_on ? (const void*)jacobi_grid_block_kernel<64, true>
                                          : (const void*)jacobi_grid_block_kernel<64, false>);
  e = set_kernel_smem(fn, smem, false);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, GB_THREADS, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  if (nbe / 2 > sms * per_sm) return cudaErrorInvalidConfiguration;
  int ctas = nbe / 2;
  unsigned int* bar = scratch;
  unsigned int* rot = scratch + 2;
  unsigned long long* pr = dprof;
  void* args[] = {&W, &V, &k, &ldw, &b, &nbe, &tol, &max_sweeps, &bar, &rot, &sweeps_out, &pr};
  e = cudaLaunchCooperativeKernel(fn, dim3(ctas), dim3(GB_THREADS), args, smem, s);
  if (e != cudaSuccess) return e;
  note_launch();
  if (prof_on) {
    unsigned long long v[8];
    cudaMemcpyAsync(v, dprof, sizeof(v), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    if (v[4])
      std::fprintf(stderr, "[sssvd] grid block jacobi k=%d b=%d ctas=%d: cycles/outer round: load+V %llu inner %llu "
                   "store %llu barrier %llu (round-0 inner total %llu, rounds %llu)\n", k, b, ctas, v[0] / v[4],
                   v[1] / v[4], v[2] / v[4], v[3] / v[4], v[5], v[4]);
  }
  jacobi_finish_kernel<<<k, 256, 0, s>>>(W, k, ldw, S);
  note_launch();
  return cudaGetLastError();
}

}  // namespace sssvd_gpu
