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
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <atomic>
#include <map>
#include <mutex>
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
  std::vector<double> flops;               // per slot of the pass being enqueued: executed tensor flops,
                                           // negated for 3M launches (algorithmic = 4/3 executed)
  double acc_ms = 0, acc_flops = 0, acc_alg = 0;
  unsigned long long acc_launches = 0;
};
static GemmProf g_prof;
constexpr int kStampSlots = 32768;   // config 5 issues ~16.6k GEMM launches per 32-shift pass

void zgemm_profile_enable(bool on) {
  g_prof.on = on;
  g_prof.acc_ms = g_prof.acc_flops = g_prof.acc_alg = 0;
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
  double f = 0, falg = 0;
  for (size_t i = 0; i < cnt; ++i) {
    if (en[i] == 0 || st[i] == ~0ull) continue;   // empty launch
    iv.emplace_back(st[i], en[i]);
    f += std::fabs(flops[i]);
    falg += flops[i] < 0 ? -flops[i] * (4.0 / 3.0) : flops[i];
  }
  // SSSVD_GEMM_DUMP=<path>: append every launch of the pass as "start_ns end_ns flops" (tools/gemm_timeline.py)
  if (const char* dump = std::getenv("SSSVD_GEMM_DUMP")) {
    if (FILE* fp = std::fopen(dump, "a")) {
      std::fprintf(fp, "# pass %zu launches\n", cnt);
      for (size_t i = 0; i < cnt; ++i)
        if (en[i] != 0 && st[i] != ~0ull) std::fprintf(fp, "%llu %llu %.0f\n", st[i], en[i], std::fabs(flops[i]));
      std::fclose(fp);
    }
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
  g_prof.acc_alg += falg;
  g_prof.acc_launches += iv.size();
}

void zgemm_profile_collect(double* ms, double* flops, double* algorithmic, unsigned long long* launches) {
  *ms = g_prof.acc_ms;
  *flops = g_prof.acc_flops;
  *algorithmic = g_prof.acc_alg;
  *launches = g_prof.acc_launches;
  g_prof.acc_ms = g_prof.acc_flops = g_prof.acc_alg = 0;
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
             double2* C, int ldc, long long sC, unsigned long long* __restrict__ stamp, int stamp_cap,
             unsigned* desync, int desync_first, unsigned desync_ns, int group_m) {
  constexpr int WARPS_N = 64 / (8 * WJ);
  constexpr int THREADS = (64 / (8 * WI)) * WARPS_N * 32;
  extern __shared__ __align__(16) double2 smem[];
  if (stamp && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMin(stamp, t);
  }
  // The two CTAs resident on an SM start together and run identical work, so their prologues and
  // epilogues (no DMMA) coincide for the whole launch. Every second CTA to arrive on an SM in the
  // first wave waits about half a tile time once; the offset then persists through the launch,
  // so one CTA's epilogue runs under the other's main loop.
  if (desync) {
    const int lin = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    if (lin < desync_first) {
      if (threadIdx.x == 0) {
        unsigned sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        if (atomicAdd(desync + sm, 1u) & 1u) {
          unsigned long long t0, t1;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
          do {
            __nanosleep(1000);
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
          } while (t1 - t0 < desync_ns);
        }
      }
      __syncthreads();
    }
  }
  // stage s occupies [s*(A_STAGE+B_STAGE), (s+1)*(A_STAGE+B_STAGE)): A tile then B tile
  double2* As = smem;
  double2* Bs = smem + A_STAGE;
  constexpr int SSTRIDE = A_STAGE + B_STAGE;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WARPS_N, wn = warp % WARPS_N;
  // Tile order: CTAs are dispatched x-fastest; walking a whole row of n-tiles per m-tile streams all
  // of B (66 MB per shift at n = 16384) between two uses of a B tile, and the C traffic evicts it
  // from L2 meanwhile (ncu: 15.3 GB read for 8.7 GB algorithmic). Instead consecutive CTAs walk
  // down GROUP_M m-tiles of one n-tile before moving to the next n-tile, so a B tile is reused
  // GROUP_M times back to back and the group's A rows (GROUP_M x 256 KB at K = 256) stay in L2.
  // The host picks GROUP_M = 32 when one shift's B operand would not stay in L2 beside the C
  // stream, else 1 (the plain order: measured 2 % faster on the config-2 shapes, whose A and B
  // fit L2 together).
  const int GROUP_M = group_m;
  int tile_m, tile_n;
  {
    const int tiles_n = gridDim.x, tiles_m = gridDim.y;
    const int lin_t = blockIdx.y * tiles_n + blockIdx.x;
    const int per_group = GROUP_M * tiles_n;
    const int g = lin_t / per_group, within = lin_t - g * per_group;
    const int gm = min(GROUP_M, tiles_m - g * GROUP_M);
    tile_n = within / gm;
    tile_m = g * GROUP_M + (within - tile_n * gm);
  }
  const int m0 = tile_m * BM, n0 = tile_n * BN;
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

size_t zgemm_sub_smem() { return (size_t)STAGES * (A_STAGE + B_STAGE) * sizeof(double2); }

// ----------------------------------------------------------------------------- 3M form
// C -= A B with THREE real products per complex multiply-add instead of four:
//   P1 = Are Bre,  P2 = Aim Bim,  P3 = (Are + Aim)(Bre + Bim);   Re = P1 - P2,  Im = P3 - P1 - P2
// (the "3M" complex GEMM; Higham, "Stability of a method for multiplying complex matrices with
// three real matrix multiplications", SIMAX 1992: normwise the same error bound as the 4-product
// form). 25 % fewer DMMAs per complex flop; the price is a third accumulator set, so the CTA tile
// is 64 x (16 WJ) with 4 warps of 32 x (8 WJ): WJ = 3 (64 x 48) keeps 144 accumulator registers per
// thread; WJ = 4 needs 192 + operands > 255 and spills inside the k-loop (measured slower).
// The operand sums are formed from the fragments in registers (one DADD per fragment element).
// Same cp.async ring, C prefetch, tile order and first-wave offset as zgemm_kernel.
template <int WJ>
struct Tile3M {
  static constexpr int BN3 = 16 * WJ;
  static constexpr int LDB3 = BN3 + 2;            // == 2 mod 8 for WJ = 3, 4
  static constexpr int B_STAGE3 = BK * LDB3;
  static constexpr int SSTRIDE3 = A_STAGE + B_STAGE3;
  static constexpr int CP3 = BN3 + 1;
  static_assert(32 * CP3 <= SSTRIDE3, "C half-tile must fit one pipeline stage");
  static constexpr size_t SMEM = (size_t)STAGES * SSTRIDE3 * sizeof(double2);
};

template <int WJ, bool SET = false, bool GATHER = false>
__global__ void __launch_bounds__(128, 2)
zgemm3m_kernel(int M, int N, int K, const double2* __restrict__ A, int lda, long long sA,
               const double2* __restrict__ B, int ldb, long long sB, const int* __restrict__ brow, int sR,
               double2* C, int ldc, long long sC,
               unsigned long long* __restrict__ stamp, int stamp_cap, unsigned* desync, int desync_first,
               unsigned desync_ns, int group_m) {
  using T = Tile3M<WJ>;
  constexpr int BN3 = T::BN3, LDB3 = T::LDB3, SSTRIDE = T::SSTRIDE3, CP3 = T::CP3;
  constexpr int THREADS = 128, WI = 4;
  extern __shared__ __align__(16) double2 smem[];
  if (stamp && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMin(stamp, t);
  }
  if (desync) {
    const int lin = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    if (lin < desync_first) {
      if (threadIdx.x == 0) {
        unsigned sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        if (atomicAdd(desync + sm, 1u) & 1u) {
          unsigned long long t0, t1;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
          do {
            __nanosleep(1000);
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
          } while (t1 - t0 < desync_ns);
        }
      }
      __syncthreads();
    }
  }
  double2* As = smem;
  double2* Bs = smem + A_STAGE;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  int tile_m, tile_n;
  {
    const int tiles_n = gridDim.x, tiles_m = gridDim.y;
    const int lin_t = blockIdx.y * tiles_n + blockIdx.x;
    const int per_group = group_m * tiles_n;
    const int g = lin_t / per_group, within = lin_t - g * per_group;
    const int gm = min(group_m, tiles_m - g * group_m);
    tile_n = within / gm;
    tile_m = g * group_m + (within - tile_n * gm);
  }
  const int m0 = tile_m * BM, n0 = tile_n * BN3;
  A += blockIdx.z * sA;
  B += blockIdx.z * sB;
  C += blockIdx.z * sC;
  if (GATHER) brow += blockIdx.z * sR;

  double p1[WI][WJ][2], p2[WI][WJ][2], p3[WI][WJ][2];
#pragma unroll
  for (int i = 0; i < WI; ++i)
#pragma unroll
    for (int j = 0; j < WJ; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) p1[i][j][e] = p2[i][j][e] = p3[i][j][e] = 0.0;

  const int KT = (K + BK - 1) / BK;
  auto c_stage = [&](int h) { return smem + ((KT + h) % STAGES) * SSTRIDE; };
  // stage loader: A as in StageLoader (thread = one k column, 8 rows); B: thread = one k row of
  // the stage and every 8th column of it (8 consecutive lanes copy 128 contiguous bytes)
  constexpr int AN = BM * BK / THREADS, AR = THREADS / BK, BNE = BN3 / 8;
  const int a_k = tid % BK, ar = tid / BK;
  const double2* ap = A + (size_t)(m0 + ar) * lda + a_k;
  const long long a_step = (long long)AR * lda;
  const int a_dst = ar * LDA_S + a_k;
  unsigned a_rows = 0;
#pragma unroll
  for (int i = 0; i < AN; ++i) a_rows |= (m0 + ar + i * AR < M ? 1u : 0u) << i;
  const int b_k = tid >> 3, bc = tid & 7;
  const double2* bp = B + (size_t)b_k * ldb + n0 + bc;
  // GATHER: row k of the B operand is row brow[k] of B; the index of the NEXT stage's row is
  // fetched one stage ahead so its latency never sits in front of a cp.async
  int gk = b_k, grow = 0;
  if (GATHER) grow = gk < K ? brow[gk] : 0;
  const long long b_adv = (long long)BK * ldb;
  const int b_dst = b_k * LDB3 + bc;
  unsigned b_cols = 0;
#pragma unroll
  for (int i = 0; i < BNE; ++i) b_cols |= (n0 + bc + 8 * i < N ? 1u : 0u) << i;
  const bool interior = m0 + BM <= M && n0 + BN3 <= N;
  auto load = [&](double2* as_, double2* bs_, int kleft) {
    const double2* bsrc = GATHER ? B + (size_t)grow * ldb + n0 + bc : bp;
    if (interior && kleft >= BK) {
#pragma unroll
      for (int i = 0; i < AN; ++i) cp_async16(as_ + a_dst + i * AR * LDA_S, ap + i * a_step);
#pragma unroll
      for (int i = 0; i < BNE; ++i) cp_async16(bs_ + b_dst + 8 * i, bsrc + 8 * i);
    } else {
      const bool ak = a_k < kleft, bk = b_k < kleft;
#pragma unroll
      for (int i = 0; i < AN; ++i) cp_async16(as_ + a_dst + i * AR * LDA_S, ap + i * a_step, ak && ((a_rows >> i) & 1u));
#pragma unroll
      for (int i = 0; i < BNE; ++i) cp_async16(bs_ + b_dst + 8 * i, bsrc + 8 * i, bk && ((b_cols >> i) & 1u));
    }
    ap += BK;
    if (GATHER) {
      gk += BK;
      grow = gk < K ? brow[gk] : 0;
    } else {
      bp += b_adv;
    }
  };
  auto load_c = [&](double2* dst, int h) {
#pragma unroll
    for (int i = 0; i < (32 * BN3) / THREADS; ++i) {
      const int idx = tid + i * THREADS;
      const int r = idx / BN3, c = idx % BN3;
      const bool p = (m0 + 32 * h + r < M) && (n0 + c < N);
      cp_async16(dst + r * CP3 + c, p ? C + (size_t)(m0 + 32 * h + r) * ldc + n0 + c : C, p);
    }
  };
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load(As + s * SSTRIDE, Bs + s * SSTRIDE, K - s * BK);
    if (!SET) {
      for (int h = 0; h < 2; ++h)
        if (KT - 2 + h < 0 && s == 0) load_c(c_stage(h), h);
    }
    cp_async_commit();
  }
  const int fr = lane >> 2, fc = lane & 3;
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const double2* as = As + (kt % STAGES) * SSTRIDE + (wm * 32 + fr) * LDA_S + fc;
    const double2* bs = Bs + (kt % STAGES) * SSTRIDE + fc * LDB3 + wn * 8 * WJ + fr;
#pragma unroll
    for (int kq = 0; kq < BK / 4; ++kq) {
      if (kq == 1) {
        const int nk = kt + STAGES - 1;
        if (nk < KT) {
          const int st = nk % STAGES;
          load(As + st * SSTRIDE, Bs + st * SSTRIDE, K - nk * BK);
        } else if (!SET) {
          const int h = kt - (KT - 2);
          if (h >= 0 && h < 2) load_c(c_stage(h), h);
        }
        cp_async_commit();
      }
      double2 a[WI], b[WJ];
      double sa[WI], sb[WJ];
#pragma unroll
      for (int i = 0; i < WI; ++i) a[i] = as[i * 8 * LDA_S + kq * 4];
#pragma unroll
      for (int j = 0; j < WJ; ++j) b[j] = bs[kq * 4 * LDB3 + j * 8];
#pragma unroll
      for (int i = 0; i < WI; ++i)
#pragma unroll
        for (int j = 0; j < WJ; ++j) dmma884(p1[i][j][0], p1[i][j][1], a[i].x, b[j].x);
#pragma unroll
      for (int i = 0; i < WI; ++i)
#pragma unroll
        for (int j = 0; j < WJ; ++j) dmma884(p2[i][j][0], p2[i][j][1], a[i].y, b[j].y);
      // the operand sums, pinned (volatile) between the P2 and the P3 pass: left to ptxas they are
      // spread among the P1 DMMAs, measured 0.8 % slower (41.95 -> 42.30 TF/s, bitwise equal)
#pragma unroll
      for (int i = 0; i < WI; ++i) asm volatile("add.f64 %0, %1, %2;" : "=d"(sa[i]) : "d"(a[i].x), "d"(a[i].y));
#pragma unroll
      for (int j = 0; j < WJ; ++j) asm volatile("add.f64 %0, %1, %2;" : "=d"(sb[j]) : "d"(b[j].x), "d"(b[j].y));
#pragma unroll
      for (int i = 0; i < WI; ++i)
#pragma unroll
        for (int j = 0; j < WJ; ++j) dmma884(p3[i][j][0], p3[i][j][1], sa[i], sb[j]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();
#pragma unroll
  for (int i = 0; i < WI; ++i) {
    const int rt = wm * 32 + i * 8 + fr;
    const int r = m0 + rt;
    if (r >= M) continue;
    const int cbase = n0 + wn * 8 * WJ + 2 * fc;
    double2* crow = C + (size_t)r * ldc + cbase;
    if (SET) {
#pragma unroll
      for (int j = 0; j < WJ; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = cbase + j * 8 + e;
          if (c < N)
            crow[j * 8 + e] = make_double2(p1[i][j][e] - p2[i][j][e], (p3[i][j][e] - p1[i][j][e]) - p2[i][j][e]);
        }
      continue;
    }
    const double2* cs = c_stage(rt >> 5) + (rt & 31) * CP3 + wn * 8 * WJ + 2 * fc;
    double2 v[WJ][2];
#pragma unroll
    for (int j = 0; j < WJ; ++j) {
      v[j][0] = cs[j * 8];
      v[j][1] = cs[j * 8 + 1];
    }
#pragma unroll
    for (int j = 0; j < WJ; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = cbase + j * 8 + e;
        if (c < N)
          crow[j * 8 + e] = make_double2(v[j][e].x - (p1[i][j][e] - p2[i][j][e]),
                                         v[j][e].y - ((p3[i][j][e] - p1[i][j][e]) - p2[i][j][e]));
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

// ----------------------------------------------------------------------------- TMA form
// Persistent, warp-specialised form of C -= A B (the same DMMA chain per entry as zgemm_kernel,
// so bitwise the same result): 4 consumer warps (32 x 32 warp tiles of a 64 x 64 CTA tile) and
// one producer warp whose elected lane streams the K-stages with TMA (cp.async.bulk.tensor, SASS
// UTMALDG) into a ring of TMA_STAGES stages guarded by full / empty mbarriers, so the consumers
// never hit a CTA-wide barrier and the next tile's stages load under this tile's last k-steps
// and epilogue. Two CTAs per SM: one CTA's epilogue (C read-modify-write) overlaps the other's
// DMMA main loop. Tiles t = blockIdx.x + i gridDim.x over (shift, m-tile, n-tile).
// Shared-memory layouts (dense, TMA writes them as is):
//   A stage: 4 boxes (one per k-quad) of 64 rows x 4 complex (64 B rows, no swizzle): a DMMA A
//            fragment (rows fr, fr+1 of a phase x 4 k) covers 128 contiguous bytes;
//   B stage: 8 boxes of 16 k-rows x 8 complex (128 B rows, 128B swizzle: chunk ^= row % 8). Lane
//            fr of a DMMA B fragment reads column x(fr) = 4 (fr & 1) + fr / 2 of its 8-column box,
//            so the two columns of a phase sit in opposite halves of the swizzled row.
constexpr int TMA_STAGES = 3, TMA_THREADS = 160;
constexpr int TMA_A_BYTES = 64 * BK * 16, TMA_B_BYTES = BK * 64 * 16;
constexpr int TMA_STAGE_BYTES = TMA_A_BYTES + TMA_B_BYTES;
constexpr size_t TMA_SMEM = (size_t)TMA_STAGES * TMA_STAGE_BYTES + 1024 + 64;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void tma_load3(void* dst, const CUtensorMap* map, int c0, int c1, int c2, void* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(void* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__global__ void __maxnreg__(200)
zgemm_tma_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, int M, int N,
                 int K, double2* C, int ldc, long long sC, int batch, unsigned long long* __restrict__ stamp,
                 int stamp_cap) {
  extern __shared__ unsigned char tsm_raw[];
  // 1024-byte aligned ring (the 128B swizzle atom), derived from the shared array itself so the
  // fragment loads stay LDS
  unsigned char* base = tsm_raw + (((smem_u32(tsm_raw) + 1023u) & ~1023u) - smem_u32(tsm_raw));
  unsigned long long* full = reinterpret_cast<unsigned long long*>(base + TMA_STAGES * TMA_STAGE_BYTES);
  unsigned long long* empty = full + TMA_STAGES;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (stamp && tid == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMin(stamp, t);
  }
  if (tid == 0) {
    for (int s = 0; s < TMA_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
  }
  __syncthreads();
  const int tm = (M + BM - 1) / BM, tn = (N + BN - 1) / BN;
  const int per = tm * tn, total = per * batch;
  const int KT = (K + BK - 1) / BK;
  if (warp == 4) {
    // ---- producer: one elected lane issues every TMA of every stage of every tile of this CTA
    if (lane == 0) {
      int stage = 0;
      unsigned phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const int z = t / per, rem = t - z * per;
        const int m0 = (rem / tn) * BM, n0 = (rem % tn) * BN;
        for (int kt = 0; kt < KT; ++kt) {
          mbar_wait(&empty[stage], phase ^ 1u);
          mbar_expect_tx(&full[stage], TMA_STAGE_BYTES);
          unsigned char* sa = base + stage * TMA_STAGE_BYTES;
          unsigned char* sb = sa + TMA_A_BYTES;
#pragma unroll
          for (int q = 0; q < BK / 4; ++q) tma_load3(sa + q * (64 * 64), &mapA, 2 * (kt * BK + 4 * q), m0, z, &full[stage]);
#pragma unroll
          for (int bx = 0; bx < 8; ++bx) tma_load3(sb + bx * (BK * 128), &mapB, 2 * (n0 + 8 * bx), kt * BK, z, &full[stage]);
          if (++stage == TMA_STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
    __syncwarp();   // the producer warp reconverges before the closing barrier
  } else {
    // ---- consumers: warp (wm, wn) owns rows 32 wm.., columns 32 wn.. of each tile
    const int wm = warp >> 1, wn = warp & 1;
    const int fr = lane >> 2, fc = lane & 3;
    const int xcol = 4 * (fr & 1) + (fr >> 1);   // this lane's B column inside an 8-column box
    int stage = 0;
    unsigned phase = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      const int z = t / per, rem = t - z * per;
      const int m0 = (rem / tn) * BM, n0 = (rem % tn) * BN;
      double2* Cz = C + z * sC;
      // pull this warp's C rows toward L2 while the main loop runs
      for (int r = lane; r < 32; r += 32) {
        const int row = m0 + wm * 32 + r;
        if (row < M) {
          const char* p = reinterpret_cast<const char*>(Cz + (size_t)row * ldc + n0 + wn * 32);
#pragma unroll
          for (int c = 0; c < 4; ++c) asm volatile("prefetch.global.L2 [%0];" ::"l"(p + 128 * c));
        }
      }
      double acc_re[4][4][2], acc_im[4][4][2];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc_re[i][j][0] = acc_re[i][j][1] = 0.0;
          acc_im[i][j][0] = acc_im[i][j][1] = 0.0;
        }
      for (int kt = 0; kt < KT; ++kt) {
        mbar_wait(&full[stage], phase);
        const unsigned char* sa = base + stage * TMA_STAGE_BYTES;
        const unsigned char* sb = sa + TMA_A_BYTES;
#pragma unroll
        for (int kq = 0; kq < BK / 4; ++kq) {
          double2 a[4], b[4];
#pragma unroll
          for (int i = 0; i < 4; ++i)
            a[i] = *reinterpret_cast<const double2*>(sa + kq * (64 * 64) + (wm * 32 + i * 8 + fr) * 64 + fc * 16);
          const int krow = kq * 4 + fc;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            b[j] = *reinterpret_cast<const double2*>(sb + (wn * 4 + j) * (BK * 128) + krow * 128 +
                                                     ((xcol ^ (krow & 7)) << 4));
          double nai[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) nai[i] = -a[i].y;
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma884(acc_re[i][j][0], acc_re[i][j][1], a[i].x, b[j].x);
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma884(acc_im[i][j][0], acc_im[i][j][1], a[i].x, b[j].y);
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma884(acc_re[i][j][0], acc_re[i][j][1], nai[i], b[j].y);
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma884(acc_im[i][j][0], acc_im[i][j][1], a[i].y, b[j].x);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == TMA_STAGES) {
          stage = 0;
          phase ^= 1u;
        }
      }
      // epilogue: accumulator (fr, 2 fc + e) of sub-tile j is tile column 8 (4 wn + j) + 4 e + fc
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = m0 + wm * 32 + i * 8 + fr;
        if (r >= M) continue;
        double2* crow = Cz + (size_t)r * ldc + n0;
        double2 v[4][2];
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int c = 8 * (4 * wn + j) + 4 * e + fc;
            v[j][e] = n0 + c < N ? __ldcg(crow + c) : make_double2(0.0, 0.0);   // L2: never a stale L1 line
          }
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int c = 8 * (4 * wn + j) + 4 * e + fc;
            if (n0 + c < N) __stcg(crow + c, make_double2(v[j][e].x - acc_re[i][j][e], v[j][e].y - acc_im[i][j][e]));
          }
      }
    }
  }
  if (stamp) {
    __syncthreads();
    if (tid == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      atomicMax(stamp + stamp_cap, t);
    }
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 3-D map over [batch][rows][2 cols] doubles of a row-major complex matrix (pitch ld complex,
// batch stride sb complex): box = box_cols complex x box_rows rows x 1
static bool encode_map(CUtensorMap* map, const double2* p, int rows, int cols, int ld, long long sb, int batch,
                       int box_cols, int box_rows, bool swizzle128) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)2 * cols, (cuuint64_t)rows, (cuuint64_t)batch};
  const cuuint64_t strides[2] = {(cuuint64_t)ld * 16, (cuuint64_t)std::max<long long>(sb, 1) * 16};
  const cuuint32_t box[3] = {(cuuint32_t)(2 * box_cols), (cuuint32_t)box_rows, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double2*>(p), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Kernel of the C -= A B updates and of the gather-GEMM C = A B[brow]: 1 = 4-product cp.async kernel, 2 = its TMA form, 3 = the 3-product
// (3M) kernel, the default (measured: config-5 step 24.0 -> 20.2 s, isolated trailing update 34.8 ->
// 41.9 TF/s in 8 M N K units). Forms of the 3M kernel measured slower and not kept
// (profiles/r02_3m_zgemm.txt): 64 x 64 tiles (255 registers, spills: 39.3), 8 warps of 16 x 24
// (40.5), a multi-tile CTA with cross-tile stage prefetch and a global-memory C epilogue (40.7).
// SSSVD_ZGEMM = 4m | tma selects another kernel for A/B measurements (read per call); zgemm_force
// (debug comparisons) overrides.
static int g_force = 0;
void zgemm_force(int kernel) { g_force = kernel; }
static int sub_kernel() {
  if (g_force) return g_force;
  const char* e = std::getenv("SSSVD_ZGEMM");
  if (!e) return 3;
  const std::string v(e);
  return v == "4m" ? 1 : v == "tma" ? 2 : 3;
}

static cudaError_t launch_tma(int M, int N, int K, const double2* A, int lda, long long sA, const double2* B, int ldb,
                              long long sB, double2* C, int ldc, long long sC, int batch, cudaStream_t stream,
                              unsigned long long* stamp, bool* done) {
  *done = false;
  // the pitches and bases must satisfy TMA's 16-byte rules (always true for double2 buffers)
  if (((uintptr_t)A & 15) || ((uintptr_t)B & 15)) return cudaSuccess;
  if ((long long)batch > 1 && (sA <= 0 || sB <= 0)) return cudaSuccess;
  CUtensorMap ma, mb;
  if (!encode_map(&ma, A, M, K, lda, sA, batch, 4, 64, false)) return cudaSuccess;
  if (!encode_map(&mb, B, K, N, ldb, sB, batch, 8, BK, true)) return cudaSuccess;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  SSSVD_CUDA_TRY(set_kernel_smem((const void*)zgemm_tma_kernel, TMA_SMEM, false));
  const long long total = (long long)((M + BM - 1) / BM) * ((N + BN - 1) / BN) * batch;
  const int grid = (int)std::min<long long>(total, 2LL * sms);
  zgemm_tma_kernel<<<grid, TMA_THREADS, TMA_SMEM, stream>>>(ma, mb, M, N, K, C, ldc, sC, batch, stamp, g_prof.cap);
  *done = true;
  return cudaGetLastError();
}

// Per-device kernel attributes: cudaFuncSetAttribute applies to the current device only, so the
// largest dynamic shared-memory size set so far is remembered per (kernel, device).
cudaError_t set_kernel_smem(const void* fn, size_t bytes, bool nonportable_cluster) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;   // bytes + 1 once configured
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  size_t& cur = done[{fn, dev}];
  if (cur > bytes) return cudaSuccess;
  if (bytes > 48 * 1024 || cur == 0) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(bytes, 48 * 1024));
    if (e != cudaSuccess) return e;
  }
  if (nonportable_cluster) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cur = bytes + 1;
  return cudaSuccess;
}

// per-device arrival counters of the first-wave offset (monotonic, never reset: only the parity
// of consecutive arrivals on one SM matters)
static unsigned* desync_counters(int* sms_out) {
  static std::mutex mu;
  static std::map<int, std::pair<unsigned*, int>> per_dev;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  auto it = per_dev.find(dev);
  if (it == per_dev.end()) {
    int sms = 0;
    unsigned* p = nullptr;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaMalloc(&p, 1024 * sizeof(unsigned)) != cudaSuccess) return nullptr;
    cudaMemset(p, 0, 1024 * sizeof(unsigned));
    it = per_dev.emplace(dev, std::make_pair(p, sms)).first;
  }
  *sms_out = it->second.second;
  return it->second.first;
}
// the offset pays only on launches of many waves (a first-wave CTA idles for half a tile time);
// SSSVD_ZGEMM_DESYNC_WAVES overrides the threshold (measurement)
static long long desync_min_waves() {
  const char* e = std::getenv("SSSVD_ZGEMM_DESYNC_WAVES");
  return e ? std::max(1, std::atoi(e)) : 32;
}

void zgemm_init_device() {
  int sms = 0;
  (void)desync_counters(&sms);
}

// The first-wave offset in ns for a launch of KT k-stages: about half the time one 64 x 64 tile
// takes when it has the SM's DMMA pipe to itself (2.1 us per k-stage + ~6 us of prologue and
// epilogue). Measured on the isolated trailing updates (profiles/r02_zgemm_desync.txt): K = 128
// 31.5 -> 33.5 TF/s, K = 256 33.9 -> 35.1 TF/s; offsets near a whole tile time re-align the two
// CTAs and gain nothing. SSSVD_ZGEMM_DESYNC=0 turns it off, a positive value is ns per k-stage
// (measurement override); read per call.
static unsigned desync_ns(int KT) {
  const char* e = std::getenv("SSSVD_ZGEMM_DESYNC");
  if (!e) return 1050u * (unsigned)KT + 3000u;
  const int v = std::atoi(e);
  return v > 0 ? (unsigned)v * (unsigned)KT : 0u;
}

template <int WJ, bool SET, bool GATHER>
static cudaError_t launch_3m(int M, int N, int K, const double2* A, int lda, long long sA, const double2* B, int ldb,
                             long long sB, const int* brow, int sR, double2* C, int ldc, long long sC, int batch,
                             cudaStream_t stream, unsigned long long* stamp) {
  using T = Tile3M<WJ>;
  auto kern = zgemm3m_kernel<WJ, SET, GATHER>;
  SSSVD_CUDA_TRY(set_kernel_smem((const void*)kern, T::SMEM, false));
  dim3 grid((N + T::BN3 - 1) / T::BN3, (M + BM - 1) / BM, batch);
  // first-wave offset as in the 4-product launcher (measured neutral on this kernel: 41.88-41.90
  // TF/s at every offset from 0 to 1200 ns per k-stage, profiles/r02_3m_zgemm.txt)
  unsigned* desync = nullptr;
  int first = 0;
  unsigned ns = 0;
  const int KT = (K + BK - 1) / BK;
  const long long ctas = (long long)grid.x * grid.y * grid.z;
  if (!SET && KT >= 4 && desync_ns(KT) > 0) {
    int sms = 0;
    unsigned* ctr = desync_counters(&sms);
    if (ctr && ctas >= desync_min_waves() * 2LL * sms) {
      desync = ctr;
      first = 2 * sms;
      ns = desync_ns(KT) * (3 * WJ) / 16;   // a tile's DMMA time relative to the 64 x 64 4-product tile
    }
  }
  const int group_m = (double)K * N * sizeof(double2) > 24e6 ? 32 : 1;
  kern<<<grid, 128, T::SMEM, stream>>>(M, N, K, A, lda, sA, B, ldb, sB, brow, sR, C, ldc, sC, stamp, g_prof.cap, desync,
                                       first, ns, group_m);
  return cudaGetLastError();
}

// C -= A B (SET = false) or C = A B[brow] (SET = GATHER = true). The next k-stage's copies are
// issued after the first k-quad's DMMAs (measured +1 % over issuing them at the top of the stage;
// bitwise identical).
template <bool SET, bool GATHER>
static cudaError_t launch(int M, int N, int K, const double2* A, int lda, long long sA, const double2* B, int ldb,
                          long long sB, const int* brow, int sR, double2* C, int ldc, long long sC, int batch,
                          cudaStream_t stream) {
  if (M <= 0 || N <= 0 || K <= 0 || batch <= 0) return cudaSuccess;
  // the gather-GEMM (SET && GATHER) follows the 3M / 4-product choice; the TMA form covers only C -= A B
  const int which = (SET == GATHER) ? (SET && sub_kernel() == 2 ? 1 : sub_kernel()) : 1;
  unsigned long long* stamp = nullptr;
  if (g_prof.in_pass && (int)g_prof.flops.size() < g_prof.cap) {
    stamp = g_prof.d_stamp + g_prof.flops.size();
    // EXECUTED tensor flops: 4 real products per complex multiply-add, 3 in the 3M kernels
    g_prof.flops.push_back((which >= 3 ? -6.0 : 8.0) * M * (double)N * K * batch);
  }
  note_launch();
  if (which == 2) {
    bool done = false;
    SSSVD_CUDA_TRY(launch_tma(M, N, K, A, lda, sA, B, ldb, sB, C, ldc, sC, batch, stream, stamp, &done));
    if (done) return cudaSuccess;
  }
  if (which == 3)
    return launch_3m<3, SET, GATHER>(M, N, K, A, lda, sA, B, ldb, sB, brow, sR, C, ldc, sC, batch, stream, stamp);
  auto kern = zgemm_kernel<4, 4, SET, GATHER, 1>;
  SSSVD_CUDA_TRY(set_kernel_smem((const void*)kern, zgemm_sub_smem(), false));
  dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM, batch);
  // first-wave offset of the two co-resident CTAs (large launches only)
  unsigned* desync = nullptr;
  int first = 0;
  unsigned ns = 0;
  const int KT = (K + BK - 1) / BK;
  const long long ctas = (long long)grid.x * grid.y * grid.z;
  if (!SET && KT >= 4 && desync_ns(KT) > 0) {
    int sms = 0;
    unsigned* ctr = desync_counters(&sms);
    if (ctr && ctas >= desync_min_waves() * 2LL * sms) {
      desync = ctr;
      first = 2 * sms;
      ns = desync_ns(KT);
    }
  }
  const int group_m = (double)K * N * sizeof(double2) > 24e6 ? 32 : 1;
  kern<<<grid, 128, zgemm_sub_smem(), stream>>>(M, N, K, A, lda, sA, B, ldb, sB, brow, sR, C, ldc, sC, stamp,
                                                  g_prof.cap, desync, first, ns, group_m);
  return cudaGetLastError();
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
