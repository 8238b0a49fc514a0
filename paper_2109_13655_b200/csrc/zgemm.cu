// Batched complex update  C[MxN] -= A[MxK] * B[KxN]  on the FP64 tensor cores (DMMA).
//
// This is the trailing update of the blocked LU (A = L21, B = U12, C = A22) and the block
// update of the back substitution. The reference does this inside Eigen::PartialPivLU
// (proj/include/sssvd/shifted_solver.hpp:26) on one CPU thread per shift.
//
// All operands are ROW-MAJOR interleaved complex128 (double2) with leading dimensions in
// elements; blockIdx.z walks the batch of shifts. Complex products use the 4-real-product
// form on mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4):
//   Cre += Are*Bre + (-Aim)*Bim ,  Cim += Are*Bim + Aim*Bre
// CTA tile 64x64 (4 warps, 32x32 each), K staged 16 at a time through a 3-deep cp.async ring.
// Shared-memory row pitches are padded (A: 20, B: 66 double2) so every fragment load is one
// conflict-free LDS.128 per quarter-warp.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace sssvd_gpu {

static std::atomic<unsigned long long> g_launches{0};
void note_launch(unsigned long long c) { g_launches += c; }
void unnote_launch(unsigned long long c) { g_launches -= c; }
unsigned long long launch_count() { return g_launches.load(); }

// Live timing of the DMMA GEMMs without extra stream or graph nodes: inside a shifted-solve pass
// every launch gets a stamp slot; thread 0 of each CTA folds %globaltimer into the slot's start
// (atomicMin at entry) and end (atomicMax at exit). The slots are reset by two memsets at the
// start of the pass (captured with it when the pass is a CUDA graph) and harvested after the
// pass has synchronised, so graph replays and eager runs are timed alike.
struct GemmProf {
  bool on = false;
  unsigned long long* d_stamp = nullptr;   // [cap] starts, then [cap] ends (ns)
  int cap = 0;
  bool in_pass = false;
  std::vector<double> flops;               // per slot of the pass being enqueued
  double acc_ms = 0, acc_flops = 0;
  unsigned long long acc_launches = 0;
};
static GemmProf g_prof;
constexpr int kStampSlots = 8192;

void zgemm_profile_enable(bool on) {
  g_prof.on = on;
  g_prof.acc_ms = g_prof.acc_flops = 0;
  g_prof.acc_launches = 0;
}

cudaError_t zgemm_stamp_pass_begin(cudaStream_t s) {
  if (!g_prof.d_stamp) {
    cudaError_t e = cudaMalloc(&g_prof.d_stamp, sizeof(unsigned long long) * 2 * kStampSlots);
    if (e != cudaSuccess) return e;
    g_prof.cap = kStampSlots;
  }
  g_prof.in_pass = true;
  g_prof.flops.clear();
  cudaError_t e = cudaMemsetAsync(g_prof.d_stamp, 0xff, sizeof(unsigned long long) * g_prof.cap, s);
  if (e != cudaSuccess) return e;
  return cudaMemsetAsync(g_prof.d_stamp + g_prof.cap, 0, sizeof(unsigned long long) * g_prof.cap, s);
}

std::vector<double> zgemm_stamp_pass_end() {
  g_prof.in_pass = false;
  return g_prof.flops;
}

// GEMM-BUSY time of one pass: the length of the union of its launch intervals (the shift groups
// run their trailing updates concurrently, so summing per-launch durations would count shared
// time once per overlapping launch); added to the running totals when profiling is on
void zgemm_stamp_harvest(const std::vector<double>& flops) {
  if (!g_prof.on || flops.empty() || !g_prof.d_stamp) return;
  const size_t cnt = flops.size();
  std::vector<unsigned long long> st(cnt), en(cnt);
  cudaMemcpy(st.data(), g_prof.d_stamp, sizeof(unsigned long long) * cnt, cudaMemcpyDeviceToHost);
  cudaMemcpy(en.data(), g_prof.d_stamp + g_prof.cap, sizeof(unsigned long long) * cnt, cudaMemcpyDeviceToHost);
  std::vector<std::pair<unsigned long long, unsigned long long>> iv;
  double f = 0;
  for (size_t i = 0; i < cnt; ++i) {
    if (en[i] == 0 || st[i] == ~0ull) continue;   // empty launch
    iv.emplace_back(st[i], en[i]);
    f += flops[i];
  }
  std::sort(iv.begin(), iv.end());
  double t = 0;
  unsigned long long cs = 0, ce = 0;
  bool open = false;
  for (const auto& [a, b] : iv) {
    if (!open || a > ce) {
      if (open) t += (double)(ce - cs);
      cs = a;
      ce = b;
      open = true;
    } else {
      ce = std::max(ce, b);
    }
  }
  if (open) t += (double)(ce - cs);
  g_prof.acc_ms += t * 1e-6;
  g_prof.acc_flops += f;
  g_prof.acc_launches += iv.size();
}

void zgemm_profile_collect(double* ms, double* flops, unsigned long long* launches) {
  *ms = g_prof.acc_ms;
  *flops = g_prof.acc_flops;
  *launches = g_prof.acc_launches;
  g_prof.acc_ms = g_prof.acc_flops = 0;
  g_prof.acc_launches = 0;
}

namespace {
// CTA tile BM x BN = 64 x 64 complex, K staged BK = 16 at a time through a STAGES-deep cp.async
// ring. The warp tile is (8 WI) x (8 WJ): WI x WJ DMMA sub-tiles; (64 / 8WI) x (64 / 8WJ) warps.
//   <4,4>:  4 warps of 32x32 (the original tile)      <4,2>: 8 warps of 32x16
//   <2,4>:  8 warps of 16x32                           <2,2>: 16 warps of 16x16
// More warps per SM shorten the gaps in the DMMA pipe left by one warp's fixed-latency waits.
constexpr int BM = 64, BN = 64, BK = 16, STAGES = 3;
constexpr int LDA_S = BK + 4;   // 20 double2: row pitch of the A tile (== 4 mod 8)
constexpr int LDB_S = BN + 2;   // 66 double2: row pitch of the B tile (== 2 mod 8)
constexpr int A_STAGE = BM * LDA_S;
constexpr int B_STAGE = BK * LDB_S;

template <int THREADS, bool GATHER>
__device__ __forceinline__ void load_stage(double2* As, double2* Bs, const double2* A, int lda,
                                           const double2* B, int ldb, const int* brow, int M, int N, int K,
                                           int m0, int n0, int k0, int tid) {
#pragma unroll
  for (int i = 0; i < (BM * BK) / THREADS; ++i) {
    int idx = tid + i * THREADS;
    int r = idx / BK, kk = idx % BK;
    bool p = (m0 + r < M) && (k0 + kk < K);
    const double2* src = p ? A + (size_t)(m0 + r) * lda + (k0 + kk) : A;
    cp_async16(As + r * LDA_S + kk, src, p);
  }
#pragma unroll
  for (int i = 0; i < (BK * BN) / THREADS; ++i) {
    int idx = tid + i * THREADS;
    int kk = idx / BN, c = idx % BN;
    bool p = (k0 + kk < K) && (n0 + c < N);
    const int row = p ? (GATHER ? brow[k0 + kk] : k0 + kk) : 0;
    const double2* src = p ? B + (size_t)row * ldb + (n0 + c) : B;
    cp_async16(Bs + kk * LDB_S + c, src, p);
  }
}
// Stage loader of the non-gathering GEMMs: every address is precomputed once per tile, so a
// k-stage costs one pointer bump per operand plus the cp.async issue (the generic load_stage spends
// ~10 integer instructions per 16-byte copy, and those fixed-latency chains left gaps in the DMMA
// pipe: ncu "wait" stalls, 1.39x the instructions of a CUTLASS 64x64x16x3 z884 kernel).
template <int THREADS>
struct StageLoader {
  static constexpr int AN = BM * BK / THREADS;   // A elements per thread per stage
  static constexpr int AR = THREADS / BK;        // row step between them
  static constexpr int BNE = BK * BN / THREADS;  // B elements per thread per stage
  static constexpr int BR = THREADS / BN;        // k-row step between them
  const double2* a;
  const double2* b;
  long long a_step, b_step, b_adv;
  int a_dst, b_dst, a_k, b_k;
  unsigned a_rows;
  bool b_col;
  __device__ __forceinline__ void init(const double2* A, int lda, const double2* B, int ldb, int M, int N, int m0,
                                       int n0, int tid) {
    const int ar = tid / BK;
    a_k = tid % BK;
    a = A + (size_t)(m0 + ar) * lda + a_k;
    a_step = (long long)AR * lda;
    a_dst = ar * LDA_S + a_k;
    a_rows = 0;
#pragma unroll
    for (int i = 0; i < AN; ++i) a_rows |= (m0 + ar + i * AR < M ? 1u : 0u) << i;
    b_k = tid / BN;
    const int bc = tid % BN;
    b = B + (size_t)b_k * ldb + n0 + bc;
    b_step = (long long)BR * ldb;
    b_adv = (long long)BK * ldb;
    b_dst = b_k * LDB_S + bc;
    b_col = n0 + bc < N;
  }
  // the next k-stage (kleft = K - k0 columns of A / rows of B remain); interior tiles with a full
  // k-stage skip every predicate
  __device__ __forceinline__ void load(double2* As, double2* Bs, int kleft, bool interior) {
    if (interior && kleft >= BK) {
#pragma unroll
      for (int i = 0; i < AN; ++i) cp_async16(As + a_dst + i * AR * LDA_S, a + i * a_step);
#pragma unroll
      for (int i = 0; i < BNE; ++i) cp_async16(Bs + b_dst + i * BR * LDB_S, b + i * b_step);
    } else {
      const bool ak = a_k < kleft;
#pragma unroll
      for (int i = 0; i < AN; ++i) cp_async16(As + a_dst + i * AR * LDA_S, a + i * a_step, ak && ((a_rows >> i) & 1u));
#pragma unroll
      for (int i = 0; i < BNE; ++i)
        cp_async16(Bs + b_dst + i * BR * LDB_S, b + i * b_step, b_col && (b_k + i * BR < kleft));
    }
    a += BK;
    b += b_adv;
  }
};

// C half-tile h (rows 32h..32h+32 of the 64x64 tile) -> a free pipeline stage, pitch CP
constexpr int CP = BN + 1;   // 65 double2: conflict-free fragment-pattern reads in the epilogue
static_assert(32 * CP <= A_STAGE + B_STAGE, "C half-tile must fit one pipeline stage");
template <int THREADS>
__device__ __forceinline__ void load_c_half(double2* dst, const double2* C, int ldc, int M, int N, int m0,
                                            int n0, int h, int tid) {
#pragma unroll
  for (int i = 0; i < (32 * BN) / THREADS; ++i) {
    const int idx = tid + i * THREADS;
    const int r = idx / BN, c = idx % BN;
    const bool p = (m0 + 32 * h + r < M) && (n0 + c < N);
    cp_async16(dst + r * CP + c, p ? C + (size_t)(m0 + 32 * h + r) * ldc + n0 + c : C, p);
  }
}
}  // namespace

// SET: C = A B (C is not read); otherwise C -= A B. GATHER: row k of B is row brow[k] of the
// B matrix (the pivoted rows of the panel block, read straight from their pre-interchange place).
template <int WI, int WJ, bool SET, bool GATHER, int ISSUE_AT = 0>
__global__ void __launch_bounds__((64 / (8 * WI)) * (64 / (8 * WJ)) * 32, WI * WJ >= 8 ? 2 : 1)
zgemm_kernel(int M, int N, int K, const double2* __restrict__ A, int lda, long long sA,
             const double2* __restrict__ B, int ldb, long long sB, const int* __restrict__ brow, int sR,
             double2* C, int ldc, long long sC, unsigned long long* __restrict__ stamp, int stamp_cap) {
  constexpr int WARPS_N = 64 / (8 * WJ);
  constexpr int THREADS = (64 / (8 * WI)) * WARPS_N * 32;
  extern __shared__ __align__(16) double2 smem[];
  if (stamp && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMin(stamp, t);
  }
  // stage s occupies [s*(A_STAGE+B_STAGE), (s+1)*(A_STAGE+B_STAGE)): A tile then B tile
  double2* As = smem;
  double2* Bs = smem + A_STAGE;
  constexpr int SSTRIDE = A_STAGE + B_STAGE;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WARPS_N, wn = warp % WARPS_N;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  A += blockIdx.z * sA;
  B += blockIdx.z * sB;
  C += blockIdx.z * sC;
  if (GATHER) brow += blockIdx.z * sR;

  double acc_re[WI][WJ][2], acc_im[WI][WJ][2];
#pragma unroll
  for (int i = 0; i < WI; ++i)
#pragma unroll
    for (int j = 0; j < WJ; ++j) {
      acc_re[i][j][0] = acc_re[i][j][1] = 0.0;
      acc_im[i][j][0] = acc_im[i][j][1] = 0.0;
    }

  const int KT = (K + BK - 1) / BK;
  // C is prefetched into the two stages the k-loop no longer needs: half h goes to stage
  // (KT + h) % 3, issued at iteration KT - 2 + h (or in the prologue when that is < 0)
  auto c_stage = [&](int h) { return smem + ((KT + h) % STAGES) * (A_STAGE + B_STAGE); };
  StageLoader<THREADS> ld;
  if (!GATHER) ld.init(A, lda, B, ldb, M, N, m0, n0, tid);
  const bool interior = m0 + BM <= M && n0 + BN <= N;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) {
      if (GATHER)
        load_stage<THREADS, GATHER>(As + s * SSTRIDE, Bs + s * SSTRIDE, A, lda, B, ldb, brow, M, N, K, m0, n0, s * BK, tid);
      else
        ld.load(As + s * SSTRIDE, Bs + s * SSTRIDE, K - s * BK, interior);
    }
    if (!SET) {
      for (int h = 0; h < 2; ++h)
        if (KT - 2 + h < 0 && s == 0) load_c_half<THREADS>(c_stage(h), C, ldc, M, N, m0, n0, h, tid);
    }
    cp_async_commit();
  }
  const int fr = lane >> 2, fc = lane & 3;
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    // the next stage's copies (or a C half-tile): issued at the top (ISSUE_AT = 0) or after
    // ISSUE_AT k-quads of this stage, spreading the integer work between DMMA blocks
    auto issue_next = [&]() {
      int nk = kt + STAGES - 1;
      if (nk < KT) {
        int st = nk % STAGES;
        if (GATHER)
          load_stage<THREADS, GATHER>(As + st * SSTRIDE, Bs + st * SSTRIDE, A, lda, B, ldb, brow, M, N, K, m0, n0,
                                      nk * BK, tid);
        else
          ld.load(As + st * SSTRIDE, Bs + st * SSTRIDE, K - nk * BK, interior);
      } else if (!SET) {
        const int h = kt - (KT - 2);
        if (h >= 0 && h < 2) load_c_half<THREADS>(c_stage(h), C, ldc, M, N, m0, n0, h, tid);
      }
      cp_async_commit();
    };
    if (ISSUE_AT == 0) issue_next();
    const double2* as = As + (kt % STAGES) * SSTRIDE + (wm * 8 * WI + fr) * LDA_S + fc;
    const double2* bs = Bs + (kt % STAGES) * SSTRIDE + fc * LDB_S + wn * 8 * WJ + fr;
#pragma unroll
    for (int kq = 0; kq < BK / 4; ++kq) {
      if (ISSUE_AT > 0 && kq == ISSUE_AT) issue_next();
      double2 a[WI], b[WJ];
#pragma unroll
      for (int i = 0; i < WI; ++i) a[i] = as[i * 8 * LDA_S + kq * 4];
#pragma unroll
      for (int j = 0; j < WJ; ++j) b[j] = bs[kq * 4 * LDB_S + j * 8];
      double nai[WI];
#pragma unroll
      for (int i = 0; i < WI; ++i) nai[i] = -a[i].y;
      // four passes over the WI x WJ independent accumulators: the two DMMAs feeding the same
      // accumulator are 2 WI WJ instructions apart
#pragma unroll
      for (int i = 0; i < WI; ++i)
#pragma unroll
        for (int j = 0; j < WJ; ++j) dmma884(acc_re[i][j][0], acc_re[i][j][1], a[i].x, b[j].x);
#pragma unroll
      for (int i = 0; i < WI; ++i)
#pragma unroll
        for (int j = 0; j < WJ; ++j) dmma884(acc_im[i][j][0], acc_im[i][j][1], a[i].x, b[j].y);
#pragma unroll
      for (int i = 0; i < WI; ++i)
#pragma unroll
        for (int j = 0; j < WJ; ++j) dmma884(acc_re[i][j][0], acc_re[i][j][1], nai[i], b[j].y);
#pragma unroll
      for (int i = 0; i < WI; ++i)
#pragma unroll
        for (int j = 0; j < WJ; ++j) dmma884(acc_im[i][j][0], acc_im[i][j][1], a[i].y, b[j].x);
    }
  }
  cp_async_wait<0>();
  __syncthreads();

  // epilogue: C -= acc (fragment rows fr, cols 2*fc, 2*fc+1 of each 8x8 sub-tile). The C values
  // of a row block are loaded together before any store, so their latencies overlap.
#pragma unroll
  for (int i = 0; i < WI; ++i) {
    const int rt = wm * 8 * WI + i * 8 + fr;   // row inside the 64-row tile
    const int r = m0 + rt;
    if (r >= M) continue;
    double2* crow = C + (size_t)r * ldc + n0 + wn * 8 * WJ + 2 * fc;
    const int cbase = n0 + wn * 8 * WJ + 2 * fc;
    if (SET) {
#pragma unroll
      for (int j = 0; j < WJ; ++j) {
        const int c = cbase + j * 8;
        if (c < N) crow[j * 8] = make_double2(acc_re[i][j][0], acc_im[i][j][0]);
        if (c + 1 < N) crow[j * 8 + 1] = make_double2(acc_re[i][j][1], acc_im[i][j][1]);
      }
    } else {
      // the row lives in the prefetched half-tile rt / 32 (row rt % 32, pitch CP)
      const double2* cs = c_stage(rt >> 5) + (rt & 31) * CP + wn * 8 * WJ + 2 * fc;
      double2 v[WJ][2];
#pragma unroll
      for (int j = 0; j < WJ; ++j) {
        v[j][0] = cs[j * 8];
        v[j][1] = cs[j * 8 + 1];
      }
#pragma unroll
      for (int j = 0; j < WJ; ++j) {
        const int c = cbase + j * 8;
        if (c < N) crow[j * 8] = make_double2(v[j][0].x - acc_re[i][j][0], v[j][0].y - acc_im[i][j][0]);
        if (c + 1 < N) crow[j * 8 + 1] = make_double2(v[j][1].x - acc_re[i][j][1], v[j][1].y - acc_im[i][j][1]);
      }
    }
  }
  if (stamp) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      atomicMax(stamp + stamp_cap, t);
    }
  }
}

// Persistent form of the 32x32-warp-tile kernel (variants 4, 5): the cp.async ring runs across
// tiles, so the next tile's first k-stages load while this tile's last ones compute, and C -= AB
// leaves through fire-and-forget red.global.add.f64 of -acc (fl(c + (-x)) == fl(c - x): bitwise
// the read-modify-write epilogue, with no C read into the SM and no C staging). Tiles are walked
// t = blockIdx.x + i * gridDim.x over (batch, m-tile, n-tile); grid = 2 CTAs per SM (variant 4)
// or one CTA per tile (variant 5, the red epilogue alone).
__device__ __forceinline__ void red_add_f64(double* p, double v) {
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

template <bool SET, bool GATHER>
__global__ void __launch_bounds__(128, 2)
zgemm_persist_kernel(int M, int N, int K, const double2* __restrict__ A, int lda, long long sA,
                     const double2* __restrict__ B, int ldb, long long sB, const int* __restrict__ brow, int sR,
                     double2* C, int ldc, long long sC, int batch, unsigned long long* __restrict__ stamp,
                     int stamp_cap) {
  constexpr int THREADS = 128, WI = 4, WJ = 4;
  extern __shared__ __align__(16) double2 smem[];
  if (stamp && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMin(stamp, t);
  }
  constexpr int SSTRIDE = A_STAGE + B_STAGE;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  const int tm = (M + BM - 1) / BM, tn = (N + BN - 1) / BN;
  const int per = tm * tn, total = per * batch;
  const int KT = (K + BK - 1) / BK;
  const int ntiles = blockIdx.x < total ? (total - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int steps = ntiles * KT;

  // producer state: the (tile, k-stage) of the next load
  int ld_tile = 0, ld_kt = 0;
  auto issue = [&](int slot) {
    const int t = blockIdx.x + ld_tile * gridDim.x;
    const int z = t / per, rem = t - z * per;
    const int m0 = (rem / tn) * BM, n0 = (rem % tn) * BN;
    load_stage<THREADS, GATHER>(smem + slot * SSTRIDE, smem + slot * SSTRIDE + A_STAGE, A + z * sA, lda, B + z * sB,
                                ldb, GATHER ? brow + z * sR : brow, M, N, K, m0, n0, ld_kt * BK, tid);
    if (++ld_kt == KT) {
      ld_kt = 0;
      ++ld_tile;
    }
  };
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < steps) issue(s);
    cp_async_commit();
  }

  double acc_re[WI][WJ][2], acc_im[WI][WJ][2];
#pragma unroll
  for (int i = 0; i < WI; ++i)
#pragma unroll
    for (int j = 0; j < WJ; ++j) {
      acc_re[i][j][0] = acc_re[i][j][1] = 0.0;
      acc_im[i][j][0] = acc_im[i][j][1] = 0.0;
    }
  const int fr = lane >> 2, fc = lane & 3;
  int cur_tile = 0, cur_kt = 0;
  for (int g = 0; g < steps; ++g) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    if (g + STAGES - 1 < steps) issue((g + STAGES - 1) % STAGES);
    cp_async_commit();
    const double2* as = smem + (g % STAGES) * SSTRIDE + (wm * 32 + fr) * LDA_S + fc;
    const double2* bs = smem + (g % STAGES) * SSTRIDE + A_STAGE + fc * LDB_S + wn * 32 + fr;
#pragma unroll
    for (int kq = 0; kq < BK / 4; ++kq) {
      double2 a[WI], b[WJ];
#pragma unroll
      for (int i = 0; i < WI; ++i) a[i] = as[i * 8 * LDA_S + kq * 4];
#pragma unroll
      for (int j = 0; j < WJ; ++j) b[j] = bs[kq * 4 * LDB_S + j * 8];
      double nai[WI];
#pragma unroll
      for (int i = 0; i < WI; ++i) nai[i] = -a[i].y;
#pragma unroll
      for (int i = 0; i < WI; ++i)
#pragma unroll
        for (int j = 0; j < WJ; ++j) dmma884(acc_re[i][j][0], acc_re[i][j][1], a[i].x, b[j].x);
#pragma unroll
      for (int i = 0; i < WI; ++i)
#pragma unroll
        for (int j = 0; j < WJ; ++j) dmma884(acc_im[i][j][0], acc_im[i][j][1], a[i].x, b[j].y);
#pragma unroll
      for (int i = 0; i < WI; ++i)
#pragma unroll
        for (int j = 0; j < WJ; ++j) dmma884(acc_re[i][j][0], acc_re[i][j][1], nai[i], b[j].y);
#pragma unroll
      for (int i = 0; i < WI; ++i)
#pragma unroll
        for (int j = 0; j < WJ; ++j) dmma884(acc_im[i][j][0], acc_im[i][j][1], a[i].y, b[j].x);
    }
    if (++cur_kt == KT) {
      // tile epilogue: the accumulators leave as stores (SET) or reductions (C -= AB); the next
      // tile's first stages are already in flight
      const int t = blockIdx.x + cur_tile * gridDim.x;
      const int z = t / per, rem = t - z * per;
      const int m0 = (rem / tn) * BM, n0 = (rem % tn) * BN;
      double2* Cz = C + z * sC;
#pragma unroll
      for (int i = 0; i < WI; ++i) {
        const int r = m0 + wm * 32 + i * 8 + fr;
        if (r < M) {
          double2* crow = Cz + (size_t)r * ldc + n0 + wn * 32 + 2 * fc;
          const int cbase = n0 + wn * 32 + 2 * fc;
#pragma unroll
          for (int j = 0; j < WJ; ++j) {
            const int c = cbase + j * 8;
            if (SET) {
              if (c < N) crow[j * 8] = make_double2(acc_re[i][j][0], acc_im[i][j][0]);
              if (c + 1 < N) crow[j * 8 + 1] = make_double2(acc_re[i][j][1], acc_im[i][j][1]);
            } else {
              if (c < N) {
                red_add_f64(&crow[j * 8].x, -acc_re[i][j][0]);
                red_add_f64(&crow[j * 8].y, -acc_im[i][j][0]);
              }
              if (c + 1 < N) {
                red_add_f64(&crow[j * 8 + 1].x, -acc_re[i][j][1]);
                red_add_f64(&crow[j * 8 + 1].y, -acc_im[i][j][1]);
              }
            }
          }
        }
#pragma unroll
        for (int j = 0; j < WJ; ++j) {
          acc_re[i][j][0] = acc_re[i][j][1] = 0.0;
          acc_im[i][j][0] = acc_im[i][j][1] = 0.0;
        }
      }
      cur_kt = 0;
      ++cur_tile;
    }
  }
  cp_async_wait<0>();
  if (stamp) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      atomicMax(stamp + stamp_cap, t);
    }
  }
}

// Persistent, C-buffered form (variants 6, 7): one CTA of 8 warps (32x16 warp tiles) per SM walks
// its tiles t = blockIdx.x + i * gridDim.x. The cp.async ring of PS stages runs across tiles (the
// next tile's first k-stages load under this tile's last ones), and the tile's C block is
// prefetched into its own shared buffer with the tile's first k-stage, so the read-modify-write
// epilogue never waits on HBM. Each CTA start, prologue and C fetch is paid once per SM instead of
// once per tile.
template <int PS>
constexpr size_t persist2_smem() {
  return ((size_t)PS * (A_STAGE + B_STAGE) + (size_t)BM * CP) * sizeof(double2);
}

template <int PS, bool SET, bool GATHER>
__global__ void __launch_bounds__(256, 1)
zgemm_persist2_kernel(int M, int N, int K, const double2* __restrict__ A, int lda, long long sA,
                      const double2* __restrict__ B, int ldb, long long sB, const int* __restrict__ brow, int sR,
                      double2* C, int ldc, long long sC, int batch, unsigned long long* __restrict__ stamp,
                      int stamp_cap) {
  constexpr int THREADS = 256, WI = 4, WJ = 2, WARPS_N = 4;
  extern __shared__ __align__(16) double2 smem[];
  if (stamp && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMin(stamp, t);
  }
  constexpr int SSTRIDE = A_STAGE + B_STAGE;
  double2* Cs = smem + PS * SSTRIDE;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WARPS_N, wn = warp % WARPS_N;
  const int tm = (M + BM - 1) / BM, tn = (N + BN - 1) / BN;
  const int per = tm * tn, total = per * batch;
  const int KT = (K + BK - 1) / BK;
  const int ntiles = blockIdx.x < total ? (total - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int steps = ntiles * KT;

  // producer: (tile, k-stage) of the next load
  int p_tile = 0, p_kt = 0;
  StageLoader<THREADS> ld;
  auto issue = [&](int slot) {
    const int t = blockIdx.x + p_tile * gridDim.x;
    const int z = t / per, rem = t - z * per;
    const int m0 = (rem / tn) * BM, n0 = (rem % tn) * BN;
    double2* As = smem + slot * SSTRIDE;
    if (GATHER) {
      load_stage<THREADS, GATHER>(As, As + A_STAGE, A + z * sA, lda, B + z * sB, ldb, brow + z * sR, M, N, K, m0, n0,
                                  p_kt * BK, tid);
    } else {
      if (p_kt == 0) ld.init(A + z * sA, lda, B + z * sB, ldb, M, N, m0, n0, tid);
      ld.load(As, As + A_STAGE, K - p_kt * BK, false);
    }
    if (++p_kt == KT) {
      p_kt = 0;
      ++p_tile;
    }
  };
  auto fetch_c = [&](int tile) {   // C block of `tile` -> Cs (pitch CP)
    const int t = blockIdx.x + tile * gridDim.x;
    const int z = t / per, rem = t - z * per;
    const int m0 = (rem / tn) * BM, n0 = (rem % tn) * BN;
    const double2* Cz = C + z * sC;
#pragma unroll
    for (int i = 0; i < (BM * BN) / THREADS; ++i) {
      const int idx = tid + i * THREADS;
      const int r = idx / BN, c = idx % BN;
      const bool p = (m0 + r < M) && (n0 + c < N);
      cp_async16(Cs + r * CP + c, p ? Cz + (size_t)(m0 + r) * ldc + n0 + c : Cz, p);
    }
  };
#pragma unroll
  for (int s = 0; s < PS - 1; ++s) {
    if (s < steps) issue(s);
    if (!SET && s == 0 && steps > 0) fetch_c(0);
    cp_async_commit();
  }

  double acc_re[WI][WJ][2], acc_im[WI][WJ][2];
#pragma unroll
  for (int i = 0; i < WI; ++i)
#pragma unroll
    for (int j = 0; j < WJ; ++j) {
      acc_re[i][j][0] = acc_re[i][j][1] = 0.0;
      acc_im[i][j][0] = acc_im[i][j][1] = 0.0;
    }
  const int fr = lane >> 2, fc = lane & 3;
  int c_tile = 0, c_kt = 0;
  for (int g = 0; g < steps; ++g) {
    cp_async_wait<PS - 2>();
    __syncthreads();
    if (g + PS - 1 < steps) issue((g + PS - 1) % PS);
    // the C block of this tile rides with the tile's first k-step (the buffer was released by the
    // previous tile's epilogue before the barrier above)
    if (!SET && c_kt == 0 && g > 0) fetch_c(c_tile);
    cp_async_commit();
    const double2* as = smem + (g % PS) * SSTRIDE + (wm * 8 * WI + fr) * LDA_S + fc;
    const double2* bs = smem + (g % PS) * SSTRIDE + A_STAGE + fc * LDB_S + wn * 8 * WJ + fr;
#pragma unroll
    for (int kq = 0; kq < BK / 4; ++kq) {
      double2 a[WI], b[WJ];
#pragma unroll
      for (int i = 0; i < WI; ++i) a[i] = as[i * 8 * LDA_S + kq * 4];
#pragma unroll
      for (int j = 0; j < WJ; ++j) b[j] = bs[kq * 4 * LDB_S + j * 8];
      double nai[WI];
#pragma unroll
      for (int i = 0; i < WI; ++i) nai[i] = -a[i].y;
#pragma unroll
      for (int i = 0; i < WI; ++i)
#pragma unroll
        for (int j = 0; j < WJ; ++j) dmma884(acc_re[i][j][0], acc_re[i][j][1], a[i].x, b[j].x);
#pragma unroll
      for (int i = 0; i < WI; ++i)
#pragma unroll
        for (int j = 0; j < WJ; ++j) dmma884(acc_im[i][j][0], acc_im[i][j][1], a[i].x, b[j].y);
#pragma unroll
      for (int i = 0; i < WI; ++i)
#pragma unroll
        for (int j = 0; j < WJ; ++j) dmma884(acc_re[i][j][0], acc_re[i][j][1], nai[i], b[j].y);
#pragma unroll
      for (int i = 0; i < WI; ++i)
#pragma unroll
        for (int j = 0; j < WJ; ++j) dmma884(acc_im[i][j][0], acc_im[i][j][1], a[i].y, b[j].x);
    }
    if (++c_kt == KT) {
      // epilogue of tile c_tile. Its C group was committed with the tile's first step; the wait at
      // the top of step x leaves only the newest PS - 2 groups pending, so with KT >= PS the wait +
      // barrier of this step already covered it, else wait for it here
      if (!SET && KT < PS) {
        cp_async_wait<0>();
        __syncthreads();
      }
      const int t = blockIdx.x + c_tile * gridDim.x;
      const int z = t / per, rem = t - z * per;
      const int m0 = (rem / tn) * BM, n0 = (rem % tn) * BN;
      double2* Cz = C + z * sC;
#pragma unroll
      for (int i = 0; i < WI; ++i) {
        const int rt = wm * 8 * WI + i * 8 + fr;
        const int r = m0 + rt;
        if (r < M) {
          double2* crow = Cz + (size_t)r * ldc + n0 + wn * 8 * WJ + 2 * fc;
          const int cbase = n0 + wn * 8 * WJ + 2 * fc;
          const double2* cs = Cs + rt * CP + wn * 8 * WJ + 2 * fc;
#pragma unroll
          for (int j = 0; j < WJ; ++j) {
            const int c = cbase + j * 8;
            if (SET) {
              if (c < N) crow[j * 8] = make_double2(acc_re[i][j][0], acc_im[i][j][0]);
              if (c + 1 < N) crow[j * 8 + 1] = make_double2(acc_re[i][j][1], acc_im[i][j][1]);
            } else {
              const double2 v0 = cs[j * 8], v1 = cs[j * 8 + 1];
              if (c < N) crow[j * 8] = make_double2(v0.x - acc_re[i][j][0], v0.y - acc_im[i][j][0]);
              if (c + 1 < N) crow[j * 8 + 1] = make_double2(v1.x - acc_re[i][j][1], v1.y - acc_im[i][j][1]);
            }
          }
        }
#pragma unroll
        for (int j = 0; j < WJ; ++j) {
          acc_re[i][j][0] = acc_re[i][j][1] = 0.0;
          acc_im[i][j][0] = acc_im[i][j][1] = 0.0;
        }
      }
      c_kt = 0;
      ++c_tile;
    }
  }
  cp_async_wait<0>();
  if (stamp) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      atomicMax(stamp + stamp_cap, t);
    }
  }
}

size_t zgemm_sub_smem() { return (size_t)STAGES * (A_STAGE + B_STAGE) * sizeof(double2); }

// variant of the trailing-update GEMM: SSSVD_ZGEMM_V (warp tiles 0: 32x32, 1: 32x16, 2: 16x32,
// 3: 16x16; 4: persistent 32x32 with the red epilogue; 5: one CTA per tile with the red epilogue;
// 6 / 7: persistent 8-warp CTA per SM with a C buffer, 3 / 4 k-stages; 8 / 9: 32x32 with the next
// stage issued after the first / second k-quad instead of at the top)
// or zgemm_set_variant (measurement hook)
static int g_variant = -1;
void zgemm_set_variant(int v) { g_variant = v; }
static int zgemm_variant() {
  if (g_variant < 0) {
    // default 8: the next stage's copies go out after the first k-quad's DMMAs (+1 % over the
    // top-of-stage issue, tools/zgemm_variants.py; bitwise identical)
    const char* e = std::getenv("SSSVD_ZGEMM_V");
    g_variant = e ? std::atoi(e) : 8;
    if (g_variant < 0 || g_variant > 9) g_variant = 8;
  }
  return g_variant;
}

template <int WI, int WJ, bool SET, bool GATHER, int ISSUE_AT = 0>
static cudaError_t launch_v(int M, int N, int K, const double2* A, int lda, long long sA, const double2* B, int ldb,
                            long long sB, const int* brow, int sR, double2* C, int ldc, long long sC, int batch,
                            cudaStream_t stream, unsigned long long* stamp) {
  constexpr int THREADS = (64 / (8 * WI)) * (64 / (8 * WJ)) * 32;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(zgemm_kernel<WI, WJ, SET, GATHER, ISSUE_AT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)zgemm_sub_smem());
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM, batch);
  zgemm_kernel<WI, WJ, SET, GATHER, ISSUE_AT><<<grid, THREADS, zgemm_sub_smem(), stream>>>(
      M, N, K, A, lda, sA, B, ldb, sB, brow, sR, C, ldc, sC, stamp, g_prof.cap);
  return cudaGetLastError();
}

template <bool SET, bool GATHER>
static cudaError_t launch_persist(int M, int N, int K, const double2* A, int lda, long long sA, const double2* B,
                                  int ldb, long long sB, const int* brow, int sR, double2* C, int ldc, long long sC,
                                  int batch, cudaStream_t stream, unsigned long long* stamp, bool persistent) {
  static bool configured = false;
  static int sms = 148;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(zgemm_persist_kernel<SET, GATHER>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)zgemm_sub_smem());
    if (e != cudaSuccess) return e;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    configured = true;
  }
  const long long total = (long long)((M + BM - 1) / BM) * ((N + BN - 1) / BN) * batch;
  const int grid = (int)(persistent ? std::min<long long>(total, 2LL * sms) : total);
  zgemm_persist_kernel<SET, GATHER><<<grid, 128, zgemm_sub_smem(), stream>>>(M, N, K, A, lda, sA, B, ldb, sB, brow, sR,
                                                                             C, ldc, sC, batch, stamp, g_prof.cap);
  return cudaGetLastError();
}

template <int PS, bool SET, bool GATHER>
static cudaError_t launch_persist2(int M, int N, int K, const double2* A, int lda, long long sA, const double2* B,
                                   int ldb, long long sB, const int* brow, int sR, double2* C, int ldc, long long sC,
                                   int batch, cudaStream_t stream, unsigned long long* stamp) {
  static bool configured = false;
  static int sms = 148;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(zgemm_persist2_kernel<PS, SET, GATHER>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)persist2_smem<PS>());
    if (e != cudaSuccess) return e;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    configured = true;
  }
  const long long total = (long long)((M + BM - 1) / BM) * ((N + BN - 1) / BN) * batch;
  const int grid = (int)std::min<long long>(total, sms);
  zgemm_persist2_kernel<PS, SET, GATHER><<<grid, 256, persist2_smem<PS>(), stream>>>(
      M, N, K, A, lda, sA, B, ldb, sB, brow, sR, C, ldc, sC, batch, stamp, g_prof.cap);
  return cudaGetLastError();
}

template <bool SET, bool GATHER>
static cudaError_t launch(int M, int N, int K, const double2* A, int lda, long long sA, const double2* B, int ldb,
                          long long sB, const int* brow, int sR, double2* C, int ldc, long long sC, int batch,
                          cudaStream_t stream) {
  if (M <= 0 || N <= 0 || K <= 0 || batch <= 0) return cudaSuccess;
  unsigned long long* stamp = nullptr;
  if (g_prof.in_pass && (int)g_prof.flops.size() < g_prof.cap) {
    stamp = g_prof.d_stamp + g_prof.flops.size();
    g_prof.flops.push_back(8.0 * M * (double)N * K * batch);
  }
  note_launch();
  switch (zgemm_variant()) {
    case 1: return launch_v<4, 2, SET, GATHER>(M, N, K, A, lda, sA, B, ldb, sB, brow, sR, C, ldc, sC, batch, stream, stamp);
    case 2: return launch_v<2, 4, SET, GATHER>(M, N, K, A, lda, sA, B, ldb, sB, brow, sR, C, ldc, sC, batch, stream, stamp);
    case 3: return launch_v<2, 2, SET, GATHER>(M, N, K, A, lda, sA, B, ldb, sB, brow, sR, C, ldc, sC, batch, stream, stamp);
    case 4: return launch_persist<SET, GATHER>(M, N, K, A, lda, sA, B, ldb, sB, brow, sR, C, ldc, sC, batch, stream, stamp, true);
    case 5: return launch_persist<SET, GATHER>(M, N, K, A, lda, sA, B, ldb, sB, brow, sR, C, ldc, sC, batch, stream, stamp, false);
    case 6: return launch_persist2<3, SET, GATHER>(M, N, K, A, lda, sA, B, ldb, sB, brow, sR, C, ldc, sC, batch, stream, stamp);
    case 7: return launch_persist2<4, SET, GATHER>(M, N, K, A, lda, sA, B, ldb, sB, brow, sR, C, ldc, sC, batch, stream, stamp);
    case 9: return launch_v<4, 4, SET, GATHER, 2>(M, N, K, A, lda, sA, B, ldb, sB, brow, sR, C, ldc, sC, batch, stream, stamp);
    case 0: return launch_v<4, 4, SET, GATHER>(M, N, K, A, lda, sA, B, ldb, sB, brow, sR, C, ldc, sC, batch, stream, stamp);
    default: return launch_v<4, 4, SET, GATHER, 1>(M, N, K, A, lda, sA, B, ldb, sB, brow, sR, C, ldc, sC, batch, stream, stamp);
  }
}

cudaError_t zgemm_sub(int M, int N, int K, const double2* A, int lda, long long sA,
                      const double2* B, int ldb, long long sB, double2* C, int ldc, long long sC,
                      int batch, cudaStream_t stream) {
  return launch<false, false>(M, N, K, A, lda, sA, B, ldb, sB, nullptr, 0, C, ldc, sC, batch, stream);
}

cudaError_t zgemm_set_gather(int M, int N, int K, const double2* A, int lda, long long sA, const double2* B,
                             int ldb, long long sB, const int* brow, int sR, double2* C, int ldc, long long sC,
                             int batch, cudaStream_t stream) {
  return launch<true, true>(M, N, K, A, lda, sA, B, ldb, sB, brow, sR, C, ldc, sC, batch, stream);
}

}  // namespace sssvd_gpu
