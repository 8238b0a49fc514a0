// C-ABI implementation and host orchestration of the B200 shifted-solve path.
//
// Follows run_solve (proj/include/sssvd/pipeline.hpp:112-231) step for step:
//   steps 1-2 : form_gram (K0) -> per shift batch: assemble (K1), blocked LU with the starting
//               block riding as extra columns (K2-K5), back substitution (K6, K5), fused moment
//               accumulation (K7) -> one ncclAllReduce over ranks
//   step 3    : low_rank (QR + SVD of R)            \
//   step 4    : project_qr (A U_S1, QR)              |  round-1 interim: cuSOLVER / cuBLAS
//   step 5    : svd_small + assemble_triplets        |  (plain library QR/SVD/GEMM), the
//   postproc. : tau, residual estimate, exact, Galerkin residual norms on the residual kernel
// There is no CPU fallback: every numerical step runs on the GPU.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <future>
#include <mutex>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/sssvd_gpu.h"
#include "host_mirror.h"
#include "kernels.h"

namespace sssvd_gpu {

cudaError_t cuda_fail(cudaError_t e, const char*, const char*, int) { return e; }

struct Status : std::runtime_error {
  sssvd_status code;
  Status(sssvd_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CK(expr)                                                                                 \
  do {                                                                                           \
    cudaError_t _e = (expr);                                                                     \
    if (_e != cudaSuccess)                                                                       \
      throw Status(_e == cudaErrorMemoryAllocation ? SSSVD_E_OOM : SSSVD_E_CUDA,                 \
                   std::string(#expr) + ": " + cudaGetErrorString(_e));                          \
  } while (0)
#define CKN(expr)                                                                                \
  do {                                                                                           \
    ncclResult_t _r = (expr);                                                                    \
    if (_r != ncclSuccess) throw Status(SSSVD_E_NCCL, std::string(#expr) + ": " + nccl().GetErrorString(_r)); \
  } while (0)

// device buffer with grow-only capacity
struct DBuf {
  void* p = nullptr;
  size_t cap = 0;
  void* get(size_t bytes) {
    if (bytes > cap) {
      if (p) cudaFree(p);
      p = nullptr;
      cap = 0;
      CK(cudaMalloc(&p, std::max<size_t>(bytes, 256)));
      cap = std::max<size_t>(bytes, 256);
    }
    return p;
  }
  template <typename T>
  T* as(size_t count) { return static_cast<T*>(get(count * sizeof(T))); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// NCCL is resolved at run time (dlopen of the libnccl.so.2 already loaded by the host process,
// e.g. torch's, else the system one) and only when a communicator is requested, so loading this
// library never pins an NCCL version for the rest of the process.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

static NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
      api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
      api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
      api.Broadcast = (decltype(api.Broadcast))dlsym(h, "ncclBroadcast");
      api.CommCount = (decltype(api.CommCount))dlsym(h, "ncclCommCount");
      api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
      api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
      api.ok = api.GetUniqueId && api.CommInitRank && api.AllReduce && api.Broadcast && api.CommDestroy &&
               api.GetErrorString;
    }
  }
  if (!api.ok) throw Status(SSSVD_E_NCCL, "libnccl.so.2 not found");
  return api;
}

static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// SSSVD_TAIL_PROF=1: synchronised checkpoints through the tail (stderr), for measurement only
struct TailProf {
  cudaStream_t s;
  bool on;
  double t;
  explicit TailProf(cudaStream_t st) : s(st), on(std::getenv("SSSVD_TAIL_PROF") != nullptr), t(now_s()) {}
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const double t1 = now_s();
    std::fprintf(stderr, "[sssvd] tail %-28s %8.2f ms\n", what, (t1 - t) * 1e3);
    t = t1;
  }
};

}  // namespace sssvd_gpu

using namespace sssvd_gpu;

enum TailBuf { T_SC, T_Q, T_R, T_UR, T_VR, T_SV, T_US1, T_QM, T_LEFT, T_RIGHT, T_PERM, T_UT, T_BM, T_PM, T_PHI,
               T_QS, T_SIG, T_PS, T_QSC, T_COEFF, T_X, T_IMG, T_NRM, T_INV, T_TAU, T_Y, T_CNP, T_EU, T_EV, T_ES,
               T_COUNT };

struct sssvd_gpu_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  int max_batch = 0;
  std::string err;
  // operator (internal orientation: rows >= cols), column-major, lda even with zero padding
  int64_t m = 0, n = 0, lda = 0;
  bool transposed = false;
  bool has_gram = false;
  DBuf A, G, gmax, mats, ipiv, shifts, coef, S, V, status, minpiv, scratch;
  DBuf t0, t1, t2, t7, gwork;
  DBuf lw_linv, lw_T, lw_src, lw_disp, lw2_linv, lw2_T, lw2_src, lw2_disp, jscr, jperm, jq, jr, jj, qy, qt, qw, ts_tmp, ts_rs, ts_r;
  // factor cache (moments.hpp:106-116): the last pass left shifts [fact_jb, fact_je) factored in
  // one resident batch of `mats`, so a later pass with the same operator/shifts/L only replays the
  // forward elimination of its new right-hand side and the back substitution
  bool fact_valid = false;
  int64_t fact_jb = 0, fact_je = 0;
  int fact_n = 0, fact_L = 0;
  std::vector<std::complex<double>> fact_shifts;
  static constexpr int kMaxGroups = 8;
  cudaStream_t gstream[kMaxGroups] = {};      // high priority: panels, small kernels
  cudaStream_t gstream_lo[kMaxGroups] = {};   // low priority: the big trailing-update GEMMs
  cudaEvent_t ev_fork = nullptr, ev_join[kMaxGroups] = {};
  cudaEvent_t ev_pre[kMaxGroups] = {}, ev_gemm[kMaxGroups] = {};
  DBuf tail[T_COUNT];
  // CUDA graphs of the shifted-solve pass (assemble -> grouped LU -> pivot floor -> moments), keyed
  // by the plan and every device pointer they bake in; captured on the second sighting of a key
  struct LuGraph {
    std::vector<uintptr_t> key;
    cudaGraphExec_t exec = nullptr;
    std::vector<double> gemm_flops;   // per stamp slot
    unsigned long long launches = 0;
  };
  std::vector<LuGraph> lu_graphs;
  std::vector<uintptr_t> lu_warm_key;
  cudaStream_t cstream = nullptr;   // result device->host copies, overlapped with the tail
  cudaEvent_t ev_copy = nullptr;
  double t_gram = 0, t_solves = 0, t_allreduce = 0, solve_flops = 0;
  // the last starting block (random_start is a pure function of n, L, seed: ~1 ms of mt19937_64
  // draws at n = 4096, L = 32, repeated by every run_solve of the same shape)
  int64_t v0_n = -1, v0_L = -1;
  uint64_t v0_seed = 0;
  std::vector<double> v0;
};

// Page-locked host arrays for the large result fields (moment blocks, triplet vectors): their
// device->host copies run asynchronously on the context's copy stream, overlapped with the tail.
// Blocks come from a process-wide cache, so steady-state runs allocate no pinned memory.
class PinnedPool {
 public:
  static double* get(size_t count) {
    std::lock_guard<std::mutex> lk(mu());
    auto& f = free_list();
    // best fit: a small request must not take a large block, or the next large request has to
    // page-lock a new one (~0.3 s per GB) inside a run
    size_t best = f.size();
    for (size_t i = 0; i < f.size(); ++i)
      if (f[i].second >= count && (best == f.size() || f[i].second < f[best].second)) best = i;
    if (best < f.size()) {
      double* p = f[best].first;
      f.erase(f.begin() + (long)best);
      return p;
    }
    void* p = nullptr;
    if (cudaMallocHost(&p, std::max<size_t>(count, 1) * sizeof(double)) != cudaSuccess)
      throw std::bad_alloc();
    sizes()[p] = std::max<size_t>(count, 1);
    return static_cast<double*>(p);
  }
  static void put(double* p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(mu());
    free_list().emplace_back(p, sizes()[p]);
  }

 private:
  static std::mutex& mu() { static std::mutex m; return m; }
  static std::vector<std::pair<double*, size_t>>& free_list() { static std::vector<std::pair<double*, size_t>> f; return f; }
  static std::map<void*, size_t>& sizes() { static std::map<void*, size_t> m; return m; }
};

struct PinnedArray {
  double* p = nullptr;
  size_t n = 0;
  PinnedArray() = default;
  PinnedArray(const PinnedArray&) = delete;
  PinnedArray& operator=(const PinnedArray&) = delete;
  PinnedArray(PinnedArray&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  PinnedArray& operator=(PinnedArray&& o) noexcept {
    std::swap(p, o.p);
    std::swap(n, o.n);
    return *this;
  }
  ~PinnedArray() { PinnedPool::put(p); }
  void resize(size_t count) {
    PinnedPool::put(p);
    p = count ? PinnedPool::get(count) : nullptr;
    n = count;
  }
  bool empty() const { return n == 0; }
  size_t size() const { return n; }
  const double* data() const { return p; }
  double* data() { return p; }
  const double& operator[](size_t i) const { return p[i]; }
};

struct sssvd_gpu_result {
  sssvd_result_info info{};
  std::vector<double> sigma, tau, estimated, exact, galerkin, basis_sv;
  PinnedArray left, right, blocks, q;
  std::vector<int32_t> in_interval, spurious, invalid;
  std::string note;
};

namespace sssvd_gpu {

// ----------------------------------------------------------------------------- LU driver
struct LuPlan {
  int n, L, ld, NB, W, cluster;
  long long stride;
};

static constexpr size_t kLeafSlabBudget = 200 * 1024;

// Cluster size of a leaf with m rows left: the smallest power of two (up to the plan's) whose slab
// fits. Late panels have few rows, so their leaves hold fewer SMs and cross a smaller cluster
// barrier (config-5 phase 23.38 -> 23.32 s, config 4 1.546 -> 1.542 s; the factors are bitwise
// the same: a row's arithmetic and the pivot choice do not depend on which CTA holds the row).
static int leaf_cluster_for(const LuPlan& P, int m) {
  for (int c = 1; c < P.cluster; c *= 2)
    if (leaf_smem_bytes(m, P.W, c) <= kLeafSlabBudget) return c;
  return P.cluster;
}

static LuPlan make_plan(int n, int L) {
  LuPlan p;
  p.n = n;
  p.L = L;
  p.ld = ((n + L) + 7) / 8 * 8;
  p.stride = (long long)n * p.ld;
  // outer block: the trailing update runs K = NB deep (the 256-wide block recurses once more inside
  // the panel). Measured (tools/shard_sweep.py): n >= 8192 prefers 256 (config 4 1.72 -> 1.60 s,
  // config-5 shard 3.23 -> 3.08 s: the K = 256 trailing GEMM halves the C traffic per flop), n = 4096
  // prefers 128 (0.125 vs 0.138 s: the wider panel's latency is no longer hidden). SSSVD_NB overrides.
  static const char* nb_env = std::getenv("SSSVD_NB");
  p.NB = n >= 8192 ? 256 : 128;
  if (nb_env && (std::atoi(nb_env) == 128 || std::atoi(nb_env) == 256)) p.NB = std::atoi(nb_env);
  // leaf width W and cluster size C: the leaf slab (ceil(n/C) x (W+1) complex) must fit ~200 KB
  const size_t budget = kLeafSlabBudget;
  p.W = 8;
  p.cluster = 16;
  const int Ws[3] = {32, 16, 8};
  bool found = false;
  for (int wi = 0; wi < 3 && !found; ++wi)
    for (int c = 1; c <= 8 && !found; c *= 2)
      if (leaf_smem_bytes(n, Ws[wi], c) <= budget) {
        p.W = Ws[wi];
        p.cluster = c;
        found = true;
      }
  if (!found) {
    for (int wi = 0; wi < 3 && !found; ++wi)
      if (leaf_smem_bytes(n, Ws[wi], 16) <= budget) {
        p.W = Ws[wi];
        p.cluster = 16;
        found = true;
      }
  }
  if (!found) throw Status(SSSVD_E_LENGTH, "operator too large for the on-chip leaf panel");
  {
    // measurement overrides: leaf width / cluster size (used only if the slab fits)
    const char* wenv = std::getenv("SSSVD_LEAF_W");
    const char* cenv = std::getenv("SSSVD_LEAF_C");
    const int w = wenv ? std::atoi(wenv) : p.W, c = cenv ? std::atoi(cenv) : p.cluster;
    if ((w == 8 || w == 16 || w == 32) && (c == 1 || c == 2 || c == 4 || c == 8 || c == 16) &&
        leaf_smem_bytes(n, w, c) <= budget) {
      p.W = w;
      p.cluster = c;
    }
  }
  return p;
}

// Workspace of the batched LU: L11^{-1} per shift, the U12 staging block T, the interchange map.
struct LuWork {
  double2* linv;   // [nb][NB][NB]
  double2* T;      // [nb][NB][n + L]
  int* src;        // [nb][NB]
  int* disp;       // [nb][2 NB + 1]
  long long tstride;
};

// Applies the interchanges + unit-lower factor of the panel block (rows/cols r0..r0+np) to the
// columns [c0, c1) and updates rows [r0+np, n) of those columns:
//   T = L11^{-1} P A12  (DMMA GEMM gathering the pivoted rows on load)  -> U12
//   displaced rows + U12 written back (scatter_copy), then A22 -= L21 T (DMMA GEMM)
static void apply_panel(const LuPlan& P, const LuWork& W, double2* mats, const int* ipiv, int nb, cudaStream_t s,
                        int r0, int np, int c0, int c1, cudaStream_t s_gemm = nullptr, cudaEvent_t ev_pre = nullptr,
                        cudaEvent_t ev_done = nullptr) {
  const int n = P.n, N = c1 - c0;
  if (N <= 0) return;
  CK(panel_prep(mats, P.ld, P.stride, r0, np, W.linv, (long long)P.NB * P.NB, ipiv, n, W.src, W.disp, P.NB, nb, s));
  CK(zgemm_set_gather(np, N, np, W.linv, np, (long long)P.NB * P.NB, mats + c0, P.ld, P.stride, W.src, P.NB, W.T, N,
                      W.tstride, nb, s));
  CK(scatter_copy(mats, P.ld, P.stride, r0, np, c0, c1, W.disp, P.NB, W.T, N, W.tstride, nb, s));
  const int M = n - (r0 + np);
  cudaStream_t sg = s;
  if (s_gemm) {
    // the trailing GEMM runs on a low-priority stream, so pending panel CTAs of other groups
    // are scheduled ahead of its queued tiles
    CK(cudaEventRecord(ev_pre, s));
    CK(cudaStreamWaitEvent(s_gemm, ev_pre, 0));
    sg = s_gemm;
  }
  if (M > 0)
    CK(zgemm_sub(M, N, np, mats + (size_t)(r0 + np) * P.ld + r0, P.ld, P.stride, W.T, N, W.tstride,
                 mats + (size_t)(r0 + np) * P.ld + c0, P.ld, P.stride, nb, sg));
  if (s_gemm) {
    CK(cudaEventRecord(ev_done, s_gemm));
    CK(cudaStreamWaitEvent(s, ev_done, 0));
  }
}

// Recursive (getrf2-style) factorisation of the panel columns [c0, c0+w) over rows [c0, n),
// confined to the current NB block starting at column cb: leaves of width <= W run the cluster
// kernel; an internal node factors its left half, applies it to its right half (apply_panel,
// K = left width), then factors the right half. Each leaf applies its interchanges to the
// block columns on its left; the columns on its right receive them from the lowest common
// ancestor, so every block column sees every interchange of the block once and in order.
static void factor_rec(const LuPlan& P, const LuWork& W, double2* mats, int* ipiv, int nb, cudaStream_t s, int c0,
                       int w, int cb) {
  const int n = P.n;
  if (w <= P.W) {
    // the leaf applies its interchanges to the block columns [cb, c0) in its own epilogue
    CK(leaf_lu(mats, P.ld, P.stride, n, c0, w, P.W, leaf_cluster_for(P, n - c0), ipiv, nb, s, cb));
    return;
  }
  int wl = ((w / 2) + P.W - 1) / P.W * P.W;
  if (wl >= w) wl = w - P.W;
  factor_rec(P, W, mats, ipiv, nb, s, c0, wl, cb);
  apply_panel(P, W, mats, ipiv, nb, s, c0, wl, c0 + wl, c0 + w);
  factor_rec(P, W, mats, ipiv, nb, s, c0 + wl, w - wl, cb);
}

// back substitution on the RHS columns [n, n+L): substitution per diagonal block (warp per
// column), DMMA GEMM for the off-diagonal blocks
static void back_substitute(const LuPlan& P, double2* mats, int nb, cudaStream_t s) {
  const int n = P.n, ncols = n + P.L;
  const int nblocks = (n + P.NB - 1) / P.NB;
  for (int bi = nblocks - 1; bi >= 0; --bi) {
    const int kb = bi * P.NB, nbk = std::min(P.NB, n - kb);
    CK(trsm_upper_blocks(mats, P.ld, P.stride, kb, nbk, n, ncols, nb, s));
    if (kb > 0)
      CK(zgemm_sub(kb, P.L, nbk, mats + kb, P.ld, P.stride, mats + (size_t)kb * P.ld + n, P.ld, P.stride,
                   mats + n, P.ld, P.stride, nb, s));
  }
}

// LU of nb augmented matrices [z I - G | V] in place (rows 0..n-1, cols 0..n+L-1), then the
// back substitution U^{-1} on the L right-hand-side columns. ipiv: nb x n.
static void lu_solve_batch(const LuPlan& P, const LuWork& W, double2* mats, int* ipiv, int nb, cudaStream_t s) {
  const int n = P.n, ncols = n + P.L;
  for (int kb = 0; kb < n; kb += P.NB) {
    const int nbk = std::min(P.NB, n - kb);
    factor_rec(P, W, mats, ipiv, nb, s, kb, nbk, kb);
    // trailing columns (incl. the right-hand side): all NB interchanges, U12, A22 -= L21 U12
    apply_panel(P, W, mats, ipiv, nb, s, kb, nbk, kb + nbk, ncols);
  }
  back_substitute(P, mats, nb, s);
}

// Independent shift groups of one batch, each on its own stream; the host interleaves their
// launches block by block so a group's latency-bound panel overlaps another group's DMMA
// trailing update (no data is shared between groups).
struct LuGroup {
  double2* mats;
  int* ipiv;
  LuWork W;
  int nb;
  cudaStream_t s;      // high priority
  cudaStream_t s_lo;   // low priority (trailing GEMMs)
  cudaEvent_t ev_pre, ev_gemm;
  LuWork Wb;           // look-ahead: workspace of the far trailing update on s_lo
};

static void lu_solve_groups(const LuPlan& P, std::vector<LuGroup>& G) {
  const int n = P.n, ncols = n + P.L;
  for (int kb = 0; kb < n; kb += P.NB) {
    const int nbk = std::min(P.NB, n - kb);
    for (auto& g : G) {
      factor_rec(P, g.W, g.mats, g.ipiv, g.nb, g.s, kb, nbk, kb);
      apply_panel(P, g.W, g.mats, g.ipiv, g.nb, g.s, kb, nbk, kb + nbk, ncols, g.s_lo, g.ev_pre, g.ev_gemm);
    }
  }
  const int nblocks = (n + P.NB - 1) / P.NB;
  for (int bi = nblocks - 1; bi >= 0; --bi) {
    const int kb = bi * P.NB, nbk = std::min(P.NB, n - kb);
    for (auto& g : G) {
      CK(trsm_upper_blocks(g.mats, P.ld, P.stride, kb, nbk, n, ncols, g.nb, g.s));
      if (kb > 0)
        CK(zgemm_sub(kb, P.L, nbk, g.mats + kb, P.ld, P.stride, g.mats + (size_t)kb * P.ld + n, P.ld, P.stride,
                     g.mats + n, P.ld, P.stride, g.nb, g.s));
    }
  }
}

// Look-ahead (depth 1) version of lu_solve_groups. Block k's trailing update is split into the
// next block's columns A(k) = [kb+NB, kb+2NB) and the far columns B(k) = [kb+2NB, n+L):
//   s    (high priority): panel(k) -> [wait B(k-1)] -> A(k) -> panel(k+1) -> [wait B(k)] -> A(k+1) ...
//   s_lo (low priority) :   [wait panel(k)] -> B(k) -> [wait panel(k+1)] -> B(k+1) ...
// so panel k+1 factors while B(k) -- the big GEMM -- runs, instead of after it. A(k) and B(k)
// read panel k and write disjoint columns; B(k-1) precedes A(k) because both update block k+1's
// columns (blocks k-1 then k, the reference's order). Every column still receives every update
// in the same order through the same kernels, so the factors are bitwise those of
// lu_solve_groups. B(k) keeps its own interchange map / L11^-1 / U12 staging (Wb) because the
// panel recursion on s reuses W meanwhile.
static void lu_solve_groups_lookahead(const LuPlan& P, std::vector<LuGroup>& G) {
  const int n = P.n, ncols = n + P.L;
  for (int kb = 0; kb < n; kb += P.NB) {
    const int nbk = std::min(P.NB, n - kb);
    const int a_lo = kb + nbk;
    const int a_hi = a_lo < n ? std::min(a_lo + P.NB, n) : a_lo;
    for (auto& g : G) {
      factor_rec(P, g.W, g.mats, g.ipiv, g.nb, g.s, kb, nbk, kb);
      CK(cudaEventRecord(g.ev_pre, g.s));                       // panel k done
      if (kb > 0) CK(cudaStreamWaitEvent(g.s, g.ev_gemm, 0));   // B(k-1) done
      if (a_hi > a_lo) apply_panel(P, g.W, g.mats, g.ipiv, g.nb, g.s, kb, nbk, a_lo, a_hi);
      CK(cudaStreamWaitEvent(g.s_lo, g.ev_pre, 0));
      apply_panel(P, g.Wb, g.mats, g.ipiv, g.nb, g.s_lo, kb, nbk, a_hi, ncols);
      CK(cudaEventRecord(g.ev_gemm, g.s_lo));
    }
  }
  for (auto& g : G) CK(cudaStreamWaitEvent(g.s, g.ev_gemm, 0));   // the last B (the right-hand side)
  const int nblocks = (n + P.NB - 1) / P.NB;
  for (int bi = nblocks - 1; bi >= 0; --bi) {
    const int kb = bi * P.NB, nbk = std::min(P.NB, n - kb);
    for (auto& g : G) {
      CK(trsm_upper_blocks(g.mats, P.ld, P.stride, kb, nbk, n, ncols, g.nb, g.s));
      if (kb > 0)
        CK(zgemm_sub(kb, P.L, nbk, g.mats + kb, P.ld, P.stride, g.mats + (size_t)kb * P.ld + n, P.ld, P.stride,
                     g.mats + n, P.ld, P.stride, g.nb, g.s));
    }
  }
}

// SSSVD_LOOKAHEAD=1 selects the look-ahead schedule (read per pass, so tests can compare both).
// Off by default: measured equal to the plain grouped schedule (cfg2 phase 128-129 ms either way,
// cfg4 1.62-1.66 s), because the other shift groups' GEMMs already fill the GPU during a panel.
static bool lookahead_on() {
  const char* e = std::getenv("SSSVD_LOOKAHEAD");
  return e && std::string(e) == "1";
}

static LuWork make_work(sssvd_gpu_ctx* ctx, const LuPlan& P, int B) {
  LuWork W;
  W.tstride = (long long)P.NB * (P.n + P.L);
  W.linv = ctx->lw_linv.as<double2>((size_t)B * P.NB * P.NB);
  W.T = ctx->lw_T.as<double2>((size_t)B * W.tstride);
  W.src = ctx->lw_src.as<int>((size_t)B * P.NB);
  W.disp = ctx->lw_disp.as<int>((size_t)B * (2 * P.NB + 1));
  return W;
}

// the second workspace of the look-ahead far update (same shapes)
static LuWork make_work2(sssvd_gpu_ctx* ctx, const LuPlan& P, int B) {
  LuWork W;
  W.tstride = (long long)P.NB * (P.n + P.L);
  W.linv = ctx->lw2_linv.as<double2>((size_t)B * P.NB * P.NB);
  W.T = ctx->lw2_T.as<double2>((size_t)B * W.tstride);
  W.src = ctx->lw2_src.as<int>((size_t)B * P.NB);
  W.disp = ctx->lw2_disp.as<int>((size_t)B * (2 * P.NB + 1));
  return W;
}

// the slice of a batch workspace that belongs to shifts [b0, ...)
static LuWork work_slice(const LuWork& W, const LuPlan& P, int b0) {
  LuWork g = W;
  g.linv += (size_t)b0 * P.NB * P.NB;
  g.T += (size_t)b0 * W.tstride;
  g.src += (size_t)b0 * P.NB;
  g.disp += (size_t)b0 * (2 * P.NB + 1);
  return g;
}

static size_t bytes_per_shift(const LuPlan& P) {
  // mats + ipiv + two LU workspaces (the look-ahead far update keeps its own)
  return (size_t)P.stride * sizeof(double2) + (size_t)P.n * sizeof(int) +
         2 * (size_t)P.NB * (P.n + P.L + P.NB) * sizeof(double2);
}

static int choose_batch(sssvd_gpu_ctx* ctx, const LuPlan& P, int64_t shifts) {
  size_t free_b = 0, total_b = 0;
  CK(cudaMemGetInfo(&free_b, &total_b));
  // keep what is already allocated for mats reusable; leave 4 GiB headroom for the tail
  size_t avail = free_b + ctx->mats.cap + ctx->ipiv.cap + ctx->lw_T.cap + ctx->lw_linv.cap + ctx->lw2_T.cap +
                 ctx->lw2_linv.cap;
  const size_t headroom = (size_t)4 << 30;
  avail = avail > headroom ? avail - headroom : avail / 2;
  int64_t b = std::max<int64_t>(1, (int64_t)(avail / bytes_per_shift(P)));
  b = std::min<int64_t>(b, shifts);
  b = std::min<int64_t>(b, 32);
  if (ctx->max_batch > 0) b = std::min<int64_t>(b, ctx->max_batch);
  return (int)std::max<int64_t>(1, b);
}

// One pass over this rank's shifts [jb, je): S_dev (row-major [(M+1)][n][L]) is zeroed and
// receives sum_j 2 Re(c[k][j] X_j) in ascending j. V_dev: n x L column-major (real).
static void moment_pass(sssvd_gpu_ctx* ctx, const std::vector<std::complex<double>>& shifts,
                        const std::vector<std::complex<double>>& coef, int64_t h, int64_t jb, int64_t je,
                        const double* V_dev, int L, int M, double* S_dev) {
  cudaStream_t s = ctx->stream;
  const double t_entry = now_s();
  const int n = (int)ctx->n;
  LuPlan P = make_plan(n, L);
  CK(cudaMemsetAsync(S_dev, 0, sizeof(double) * (size_t)(M + 1) * n * L, s));
  if (je <= jb) return;
  const bool reuse = ctx->fact_valid && ctx->fact_jb == jb && ctx->fact_je == je && ctx->fact_n == n &&
                     ctx->fact_L == L && ctx->fact_shifts == std::vector<std::complex<double>>(shifts.begin() + jb,
                                                                                               shifts.begin() + je);
  const int B = reuse ? (int)(je - jb) : choose_batch(ctx, P, je - jb);
  double2* mats = ctx->mats.as<double2>((size_t)B * P.stride);
  int* ipiv = ctx->ipiv.as<int>((size_t)B * n);
  double2* dshift = ctx->shifts.as<double2>(B);
  double2* dcoef = ctx->coef.as<double2>((size_t)(M + 1) * B);
  int* dstatus = ctx->status.as<int>(B);
  double* dmin = ctx->minpiv.as<double>(B);
  const LuWork work = make_work(ctx, P, B);
  const bool lookahead = lookahead_on() && !reuse;
  const LuWork work2 = lookahead ? make_work2(ctx, P, B) : LuWork{};
  std::vector<double2> hshift(B), hcoef((size_t)(M + 1) * B);
  std::vector<int> hstatus(B);
  for (int64_t j0 = jb; j0 < je; j0 += B) {
    const int nb = (int)std::min<int64_t>(B, je - j0);
    for (int b = 0; b < nb; ++b) hshift[b] = make_double2(shifts[j0 + b].real(), shifts[j0 + b].imag());
    for (int k = 0; k <= M; ++k)
      for (int b = 0; b < nb; ++b) {
        const auto c = coef[(size_t)k * h + j0 + b];
        hcoef[(size_t)k * nb + b] = make_double2(c.real(), c.imag());
      }
    CK(cudaMemcpyAsync(dshift, hshift.data(), sizeof(double2) * nb, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dcoef, hcoef.data(), sizeof(double2) * (M + 1) * nb, cudaMemcpyHostToDevice, s));
    if (reuse) {
      // cached factors: new RHS into the augmented columns, forward elimination, back substitution
      CK(load_rhs(V_dev, n, L, mats, P.ld, P.stride, nb, s));
      for (int kb = 0; kb < n; kb += P.NB)
        apply_panel(P, work, mats, ipiv, nb, s, kb, std::min(P.NB, n - kb), n, n + L);
      back_substitute(P, mats, nb, s);
      CK(moments(mats, P.ld, P.stride, n, n, L, nb, dcoef, M, S_dev, s));
      CK(cudaStreamSynchronize(s));
      ctx->solve_flops += nb * (8.0 * (double)n * n * L);
      continue;
    }
    // independent shift groups: 8 for the 128-wide outer block (n < 8192; config-2 phase 118.0 ->
    // 116.4 ms), 4 for the 256-wide one (configs 3 / 4 / 5 measured 1-2 % faster with 4 than 8)
    static const char* genv = std::getenv("SSSVD_GROUPS");
    const int gdef = P.NB == 128 ? 8 : 4;
    const int ng = std::max(1, std::min({nb / 2, sssvd_gpu_ctx::kMaxGroups, genv ? std::atoi(genv) : gdef}));
    // the whole pass on the device: the host issues ~5000 launches per pass, which at ~17 us each
    // would make the GPU wait on the host; replaying a captured graph removes that
    std::vector<double> pass_flops;
    auto enqueue = [&](bool capturing) {
      CK(zgemm_stamp_pass_begin(s));
      CK(assemble(ctx->G.as<double>(0), n, n, V_dev, L, dshift, mats, P.ld, P.stride, nb, s));
      if (ng <= 1) {
        lu_solve_batch(P, work, mats, ipiv, nb, s);
      } else {
        std::vector<LuGroup> groups;
        CK(cudaEventRecord(ctx->ev_fork, s));
        int b0 = 0;
        for (int g = 0; g < ng; ++g) {
          const int cnt = nb / ng + (g < nb % ng ? 1 : 0);
          CK(cudaStreamWaitEvent(ctx->gstream[g], ctx->ev_fork, 0));
          groups.push_back({mats + (size_t)b0 * P.stride, ipiv + (size_t)b0 * n, work_slice(work, P, b0), cnt,
                            ctx->gstream[g], ctx->gstream_lo[g], ctx->ev_pre[g], ctx->ev_gemm[g],
                            lookahead ? work_slice(work2, P, b0) : LuWork{}});
          b0 += cnt;
        }
        const double th0 = now_s();
        if (lookahead)
          lu_solve_groups_lookahead(P, groups);
        else
          lu_solve_groups(P, groups);
        const double th1 = now_s();
        for (int g = 0; g < ng; ++g) {
          CK(cudaEventRecord(ctx->ev_join[g], ctx->gstream[g]));
          CK(cudaStreamWaitEvent(s, ctx->ev_join[g], 0));
        }
        static const bool dbg_issue = std::getenv("SSSVD_DEBUG_ISSUE") != nullptr;
        if (dbg_issue && !capturing) {
          CK(cudaStreamSynchronize(s));
          std::fprintf(stderr, "[sssvd] LU host issue %.1f ms, host issue + device drain %.1f ms\n",
                       (th1 - th0) * 1e3, (now_s() - th0) * 1e3);
        }
      }
      CK(pivot_floor(mats, P.ld, P.stride, n, dshift, ctx->gmax.as<double>(1), dstatus, dmin, nb, s));
      CK(moments(mats, P.ld, P.stride, n, n, L, nb, dcoef, M, S_dev, s));
      pass_flops = zgemm_stamp_pass_end();
    };
    static const bool no_graph = std::getenv("SSSVD_NO_GRAPH") != nullptr;
    sssvd_gpu_ctx::LuGraph* replayed = nullptr;
    if (no_graph) {
      enqueue(false);
    } else {
      const std::vector<uintptr_t> key = {
          (uintptr_t)n, (uintptr_t)L, (uintptr_t)M, (uintptr_t)nb, (uintptr_t)ng, (uintptr_t)P.NB, (uintptr_t)P.W,
          (uintptr_t)P.cluster, (uintptr_t)P.ld, (uintptr_t)ctx->G.p,
          (uintptr_t)V_dev, (uintptr_t)mats, (uintptr_t)ipiv, (uintptr_t)work.linv, (uintptr_t)work.T,
          (uintptr_t)work.src, (uintptr_t)work.disp, (uintptr_t)dshift, (uintptr_t)dcoef, (uintptr_t)S_dev,
          (uintptr_t)ctx->gmax.p, (uintptr_t)dstatus, (uintptr_t)dmin, (uintptr_t)lookahead,
          (uintptr_t)work2.linv, (uintptr_t)work2.T, (uintptr_t)work2.src, (uintptr_t)work2.disp};
      for (auto& g : ctx->lu_graphs)
        if (g.key == key) replayed = &g;
      if (replayed) {
        // SSSVD_DEBUG_PHASE=1: split the pass into host preparation (since moment_pass entry) and
        // the graph's own device time (measurement only)
        static const bool dbg_phase = std::getenv("SSSVD_DEBUG_PHASE") != nullptr;
        cudaEvent_t g0 = nullptr, g1 = nullptr;
        if (dbg_phase) {
          cudaEventCreate(&g0);
          cudaEventCreate(&g1);
          cudaEventRecord(g0, s);
        }
        CK(cudaGraphLaunch(replayed->exec, s));
        if (dbg_phase) {
          cudaEventRecord(g1, s);
          cudaEventSynchronize(g1);
          float gm = 0;
          cudaEventElapsedTime(&gm, g0, g1);
          std::fprintf(stderr, "[sssvd] phase host prep %.3f ms, graph device %.3f ms\n", (now_s() - t_entry) * 1e3 - gm,
                       gm);
          cudaEventDestroy(g0);
          cudaEventDestroy(g1);
        }
        note_launch(replayed->launches);
      } else if (ctx->lu_warm_key == key) {
        // second sighting: capture (the eager first run has set every kernel attribute)
        sssvd_gpu_ctx::LuGraph g;
        g.key = key;
        const unsigned long long l0 = launch_count();
        cudaGraph_t graph = nullptr;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        try {
          enqueue(true);
        } catch (...) {
          cudaStreamEndCapture(s, &graph);
          if (graph) cudaGraphDestroy(graph);
          zgemm_stamp_pass_end();
          throw;
        }
        g.gemm_flops = pass_flops;
        CK(cudaStreamEndCapture(s, &graph));
        g.launches = launch_count() - l0;
        unnote_launch(g.launches);
        CK(cudaGraphInstantiateWithFlags(&g.exec, graph, cudaGraphInstantiateFlagUseNodePriority));
        CK(cudaGraphDestroy(graph));
        if (ctx->lu_graphs.size() >= 4) {
          if (ctx->lu_graphs.front().exec) cudaGraphExecDestroy(ctx->lu_graphs.front().exec);
          ctx->lu_graphs.erase(ctx->lu_graphs.begin());
        }
        ctx->lu_graphs.push_back(g);
        replayed = &ctx->lu_graphs.back();
        CK(cudaGraphLaunch(replayed->exec, s));
        note_launch(replayed->launches);
      } else {
        enqueue(false);
        ctx->lu_warm_key = key;
      }
    }
    CK(cudaMemcpyAsync(hstatus.data(), dstatus, sizeof(int) * nb, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    zgemm_stamp_harvest(replayed ? replayed->gemm_flops : pass_flops);
    for (int b = 0; b < nb; ++b)
      if (hstatus[b]) throw Status(SSSVD_E_NUMERICAL, "ShiftedFactorization: shift numerically on the spectrum");
    ctx->solve_flops += nb * (8.0 * n * (double)n * n / 3.0 + 8.0 * (double)n * n * L);
  }
  // the factors stay resident when the whole shard fit one batch
  ctx->fact_valid = (je - jb) <= B;
  if (ctx->fact_valid) {
    ctx->fact_jb = jb;
    ctx->fact_je = je;
    ctx->fact_n = n;
    ctx->fact_L = L;
    ctx->fact_shifts.assign(shifts.begin() + jb, shifts.begin() + je);
  }
}

// Every rank calls this after its shifted-solve pass and before the moment all-reduce. A failure on
// any rank (a shift on the spectrum, a device error) is agreed on first (one int all-reduce, max),
// so every rank throws together instead of the healthy ranks waiting forever in a collective the
// failed rank never reaches. The reference simply propagates the exception (parallel.hpp:44-50).
static void agree_status(sssvd_gpu_ctx* ctx, int code, const std::string& msg) {
  if (ctx->comm) {   // a 1-rank communicator runs the collective too (the tests' single-GPU check)
    int* d = ctx->scratch.as<int>(2048) + 2046;
    int h = code;
    CK(cudaMemcpyAsync(d, &h, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    CKN(nccl().AllReduce(d, d, 1, ncclInt32, ncclMax, ctx->comm, ctx->stream));
    CK(cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (h != SSSVD_OK && code == SSSVD_OK)
      throw Status((sssvd_status)h, "shifted solves failed on another rank (status " + std::to_string(h) + ")");
  }
  if (code != SSSVD_OK) throw Status((sssvd_status)code, msg);
}

// moment_pass on every rank, then the failure agreement above
static void moment_pass_agreed(sssvd_gpu_ctx* ctx, const std::vector<std::complex<double>>& shifts,
                               const std::vector<std::complex<double>>& coef, int64_t h, int64_t jb, int64_t je,
                               const double* V_dev, int L, int M, double* S_dev) {
  int code = SSSVD_OK;
  std::string msg;
  try {
    moment_pass(ctx, shifts, coef, h, jb, je, V_dev, L, M, S_dev);
  } catch (const Status& e) {
    code = e.code;
    msg = e.what();
  }
  agree_status(ctx, code, msg);
}

static void allreduce_S(sssvd_gpu_ctx* ctx, double* S, size_t count) {
  if (!ctx->comm) return;   // a 1-rank communicator still runs the collective (exercised by the tests)
  CKN(nccl().AllReduce(S, S, count, ncclDouble, ncclSum, ctx->comm, ctx->stream));
}

// common tail of set_operator / set_operator_csc: NaN / Inf check (problem.hpp:56-58, :29-33 for
// sparse) and the operator bookkeeping
static void finish_operator(sssvd_gpu_ctx* ctx, int64_t m, int64_t n, int64_t ldp, bool tr) {
  cudaStream_t s = ctx->stream;
  int* bad = ctx->scratch.as<int>(2048) + 2044;
  CK(cudaMemsetAsync(bad, 0, sizeof(int), s));
  CK(any_nonfinite(ctx->A.as<double>(0), (long long)ldp * n, bad, s));
  int hbad = 0;
  CK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (hbad) throw Status(SSSVD_E_INVALID_ARGUMENT, "ProblemMatrix: NaN/Inf entry");
  ctx->m = m;
  ctx->n = n;
  ctx->lda = ldp;
  ctx->transposed = tr;
  ctx->has_gram = false;
  ctx->fact_valid = false;
}

// ProblemMatrix::from_dense (problem.hpp:47-58) into HBM: A (rows x cols, column-major, lda) is
// staged on the device, transposed there when rows < cols (the reference's auto-transpose), and
// padded to the internal operator (m x n, m >= n, leading dimension ldp = roundup(m, 8), zero rows)
static void upload_operator(sssvd_gpu_ctx* ctx, const double* a, int64_t rows, int64_t cols, int64_t lda,
                            int on_device, int64_t* m_out, int64_t* n_out, int64_t* ldp_out, bool* tr_out) {
  if (rows <= 0 || cols <= 0 || lda < rows) throw Status(SSSVD_E_INVALID_ARGUMENT, "set_operator: bad shape");
  if (!a) throw Status(SSSVD_E_INVALID_ARGUMENT, "set_operator: null matrix");
  cudaStream_t s = ctx->stream;
  const bool tr = rows < cols;
  const int64_t m = tr ? cols : rows, n = tr ? rows : cols;
  const int64_t ldp = (m + 7) / 8 * 8;
  double* Ad = ctx->A.as<double>((size_t)ldp * n);
  double* stage;
  if (on_device) {
    stage = const_cast<double*>(a);
  } else {
    stage = ctx->t0.as<double>((size_t)lda * cols);
    CK(cudaMemcpyAsync(stage, a, sizeof(double) * lda * cols, cudaMemcpyHostToDevice, s));
  }
  if (!tr) {
    CK(pad_copy(stage, (int)rows, (int)cols, (int)lda, Ad, (int)ldp, s));
  } else {
    // A^T into a dense m x n buffer (transpose kernel), then pad
    double* tmp = ctx->t1.as<double>((size_t)m * n);
    CK(transpose(stage, (int)rows, (int)cols, (int)lda, tmp, (int)m, s));
    CK(pad_copy(tmp, (int)m, (int)n, (int)m, Ad, (int)ldp, s));
  }
  *m_out = m;
  *n_out = n;
  *ldp_out = ldp;
  *tr_out = tr;
}

// Gram of the current operator into ctx->G (row-major == column-major, symmetric) + max|G|
static void ensure_gram(sssvd_gpu_ctx* ctx, int64_t cap) {
  if (ctx->n <= 0) throw Status(SSSVD_E_INVALID_ARGUMENT, "no operator set");
  if (ctx->n > cap) throw Status(SSSVD_E_LENGTH, "form_gram: column count exceeds the dense Gram cap");
  if (ctx->has_gram) return;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, ctx->stream));
  double* G = ctx->G.as<double>((size_t)ctx->n * ctx->n);
  if (ctx->comm && ctx->nranks > 1) {
    // multi-GPU: each rank forms its share of the lower-triangle tiles, one all-reduce assembles
    // G (every entry is written by exactly one rank, so the sum is exact)
    CK(cudaMemsetAsync(G, 0, sizeof(double) * ctx->n * ctx->n, ctx->stream));
    CK(gram(ctx->A.as<double>(0), (int)ctx->lda, (int)ctx->lda, (int)ctx->n, G, (int)ctx->n, ctx->rank, ctx->nranks,
            ctx->stream));
    CKN(nccl().AllReduce(G, G, (size_t)ctx->n * ctx->n, ncclDouble, ncclSum, ctx->comm, ctx->stream));
  } else {
    CK(gram(ctx->A.as<double>(0), (int)ctx->lda, (int)ctx->lda, (int)ctx->n, G, (int)ctx->n, 0, 1, ctx->stream));
  }
  CK(absmax(G, (long long)ctx->n * ctx->n, ctx->gmax.as<double>(1), ctx->stream));
  CK(cudaEventRecord(e1, ctx->stream));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  ctx->t_gram = ms * 1e-3;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  ctx->has_gram = true;
}

// ----------------------------------------------------------------------------- dense tail helpers
// column-major C = alpha op(A) B + beta C on ctx->stream (dgemm.cu: DMMA, split-K through the
// context's GEMM workspace for deep skinny products)
static constexpr size_t kGemmWork = (size_t)4 << 20;   // doubles (32 MB)
static void dgemm(sssvd_gpu_ctx* ctx, bool ta, int m, int n, int k, double alpha, const double* A, int lda,
                  const double* B, int ldb, double beta, double* C, int ldc) {
  if (m <= 0 || n <= 0) return;
  double* work = ctx->gwork.as<double>(kGemmWork);
  CK(sssvd_gpu::dgemm(ta, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, work, kGemmWork, ctx->stream));
}

// thin QR: A (m x k, lda=m) is overwritten by Q; R (k x k upper, ldr = k) returned
// QR panel plan for m rows: panel width w, 32 halved until the tallest panel's rows fit one
// cluster (register panel: 16 CTAs x 256 threads x 64 / w rows); beyond that the shared-memory
// panel (its slab budget; also SSSVD_QR_PANEL=smem). False: no panel holds m rows on chip
// (about 368k rows at w = 1), checked by run_solve before the shifted-solve phase.
static bool qr_plan(int m, int* w_out, bool* reg_out) {
  static const char* pe = std::getenv("SSSVD_QR_PANEL");
  const bool reg_panel = !(pe && std::string(pe) == "smem");
  int w = 32, c = 0;
  if (reg_panel)
    while (w > 8 && m > 16 * qr_panel_reg_rows(w)) w /= 2;
  const bool use_reg = reg_panel && m <= 16 * qr_panel_reg_rows(w);
  if (!use_reg) {
    w = 32;
    while (w > 1 && qr_panel_plan(m, w, &c) == 0) w /= 2;
    if (qr_panel_plan(m, w, &c) == 0) return false;
  }
  *w_out = w;
  *reg_out = use_reg;
  return true;
}

static void thin_qr_oneshot(sssvd_gpu_ctx* ctx, double* A, int m, int k, double* R) {
  // hand-written blocked Householder QR (householder_qr.cu), two levels: cluster panels of w
  // columns, whose updates stay inside an outer block of NBO columns; the outer block's reflectors
  // are merged into one compact-WY factor (T from G = Y^T Y, larft) and applied to the trailing
  // matrix and in the Q formation as K = NBO DGEMMs (the rank-w updates re-read the whole trailing
  // matrix once per panel)
  cudaStream_t s = ctx->stream;
  int w = 32;
  bool use_reg = true;
  if (!qr_plan(m, &w, &use_reg)) throw Status(SSSVD_E_LENGTH, "thin_qr: operator too tall for the on-chip QR panel");
  static const char* nbo_env = std::getenv("SSSVD_QR_NB");
  // measured (tools/qr_time.py): the merged factor pays off from k ~ 1024 (16384 x 2048: 52 -> 35
  // ms); below, the larft + Y^T Y overhead outweighs the saved re-reads (4096 x 512: 4.4 vs 4.8 ms)
  const int nbo_default = k >= 1024 ? 128 : w;
  const int NBO = std::max(w, std::min(128, nbo_env ? std::atoi(nbo_env) / w * w : nbo_default));
  const int npanel = (k + w - 1) / w;
  const int nblock = (k + NBO - 1) / NBO;
  double* Y = ctx->qy.as<double>((size_t)m * k);
  double* T = ctx->qt.as<double>((size_t)npanel * 1024 + (size_t)nblock * NBO * NBO + (size_t)NBO * NBO);
  double* Tb = T + (size_t)npanel * 1024;                 // [nblock][NBO][NBO]
  double* Gb = Tb + (size_t)nblock * NBO * NBO;            // [NBO][NBO]
  double* Wt = ctx->qw.as<double>((size_t)2 * NBO * k + 64);
  double* W2 = Wt + (size_t)NBO * k;
  double* tau = ctx->t7.as<double>(k + 64);
  // the block reflector Y_b spans rows jb..m: the rows above each panel's diagonal must be zero
  CK(cudaMemsetAsync(Y, 0, sizeof(double) * m * k, s));
  for (int jb = 0; jb < k; jb += NBO) {
    const int kb = std::min(NBO, k - jb), mb = m - jb;
    for (int j = jb; j < jb + kb; j += w) {
      const int p = j / w, wp = std::min(w, jb + kb - j), mp = m - j, ntb = jb + kb - j - wp;
      if (use_reg)
        CK(qr_panel_reg(A, m, m, j, wp, w, Y + (size_t)j * m + j, m, T + (size_t)p * 1024, tau + j, s));
      else
        CK(qr_panel(A, m, m, j, wp, Y + (size_t)j * m + j, m, T + (size_t)p * 1024, tau + j, s));
      if (ntb > 0) {
        // inside the outer block: A[j:m, j+wp:jb+kb] -= Y (T^T (Y^T A[j:m, j+wp:jb+kb]))
        dgemm(ctx, true, wp, ntb, mp, 1.0, Y + (size_t)j * m + j, m, A + (size_t)(j + wp) * m + j, m, 0.0, Wt, wp);
        dgemm(ctx, true, wp, ntb, wp, 1.0, T + (size_t)p * 1024, 32, Wt, wp, 0.0, W2, wp);
        dgemm(ctx, false, mp, ntb, wp, -1.0, Y + (size_t)j * m + j, m, W2, wp, 1.0,
              A + (size_t)(j + wp) * m + j, m);
      }
    }
    double* Yb = Y + (size_t)jb * m + jb;
    double* Tbb = Tb + (size_t)(jb / NBO) * NBO * NBO;
    if (kb > w) {
      dgemm(ctx, true, kb, kb, mb, 1.0, Yb, m, Yb, m, 0.0, Gb, kb);
      CK(larft(Gb, kb, tau + jb, Tbb, s));
    }
    const int nt = k - jb - kb;
    if (nt > 0) {
      // trailing columns: A[jb:m, jb+kb:k] -= Y_b (T_b^T (Y_b^T A[jb:m, jb+kb:k]))
      const double* Tuse = kb > w ? Tbb : T + (size_t)(jb / w) * 1024;
      const int ldt = kb > w ? kb : 32;
      dgemm(ctx, true, kb, nt, mb, 1.0, Yb, m, A + (size_t)(jb + kb) * m + jb, m, 0.0, Wt, kb);
      dgemm(ctx, true, kb, nt, kb, 1.0, Tuse, ldt, Wt, kb, 0.0, W2, kb);
      dgemm(ctx, false, mb, nt, kb, -1.0, Yb, m, W2, kb, 1.0, A + (size_t)(jb + kb) * m + jb, m);
    }
  }
  CK(copy_r(A, m, k, R, s));
  // Q = H_0 ... H_{p-1} [I; 0], backward over the outer blocks: Q[jb:m, jb:k] -= Y_b (T_b (Y_b^T Q[jb:m, jb:k]))
  CK(eye(A, m, k, m, s));
  for (int jb = (nblock - 1) * NBO; jb >= 0; jb -= NBO) {
    const int kb = std::min(NBO, k - jb), mb = m - jb, nq = k - jb;
    double* Yb = Y + (size_t)jb * m + jb;
    const double* Tuse = kb > w ? Tb + (size_t)(jb / NBO) * NBO * NBO : T + (size_t)(jb / w) * 1024;
    const int ldt = kb > w ? kb : 32;
    dgemm(ctx, true, kb, nq, mb, 1.0, Yb, m, A + (size_t)jb * m + jb, m, 0.0, Wt, kb);
    dgemm(ctx, false, kb, nq, kb, 1.0, Tuse, ldt, Wt, kb, 0.0, W2, kb);
    dgemm(ctx, false, mb, nq, kb, -1.0, Yb, m, W2, kb, 1.0, A + (size_t)jb * m + jb, m);
  }
}

// Rows per chunk of the tall-skinny QR below: the tallest panel the register kernel holds (w = 8).
static constexpr int kQrChunkRows = 32768;

// thin QR of any height. Up to kQrChunkRows rows the blocked Householder QR above factors the
// matrix in one shot (R agrees with LAPACK / Eigen to rounding, signs included). Taller matrices
// (the reference's HouseholderQR has no row limit: moments.hpp:195-198, extract.hpp:46-52) go
// through one level of TSQR: each row chunk A_i = Q_i R_i, the stacked R_i (p k x k) = Q_s R, and
// Q's rows of chunk i = Q_i Q_s[i k : (i+1) k, :]. Q R = A and Q^T Q = I hold to the same 1e-15
// level; R can differ from the one-shot factor in the signs of its rows (Q's columns flip with
// them), which no consumer of the tail depends on (|R_ii| for the rank flag, the SVD of R, and the
// products Q U_R / Q p are invariant).
static void thin_qr(sssvd_gpu_ctx* ctx, double* A, int m, int k, double* R) {
  if (m <= kQrChunkRows) {
    thin_qr_oneshot(ctx, A, m, k, R);
    return;
  }
  cudaStream_t s = ctx->stream;
  const int p = (m + kQrChunkRows - 1) / kQrChunkRows;
  const int mc = (m + p - 1) / p;   // rows per chunk (the last one may be shorter)
  if (m - (p - 1) * mc < k)
    throw Status(SSSVD_E_LENGTH, "thin_qr: more columns than rows in a row chunk of the tall-skinny QR");
  double* tmp = ctx->ts_tmp.as<double>((size_t)mc * k);
  double* Rs = ctx->ts_rs.as<double>((size_t)p * k * k);
  double* Ri = ctx->ts_r.as<double>((size_t)k * k);
  const int ldrs = p * k;
  for (int i = 0; i < p; ++i) {
    const int o = i * mc, mi = std::min(mc, m - o);
    CK(cudaMemcpy2DAsync(tmp, sizeof(double) * mi, A + o, sizeof(double) * m, sizeof(double) * mi, k,
                         cudaMemcpyDeviceToDevice, s));
    thin_qr_oneshot(ctx, tmp, mi, k, Ri);
    CK(cudaMemcpy2DAsync(Rs + (size_t)i * k, sizeof(double) * ldrs, Ri, sizeof(double) * k, sizeof(double) * k, k,
                         cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpy2DAsync(A + o, sizeof(double) * m, tmp, sizeof(double) * mi, sizeof(double) * mi, k,
                         cudaMemcpyDeviceToDevice, s));
  }
  // Rs <- Q_s: one shot (above kQrChunkRows stacked rows the shared-memory panel takes over, up to
  // ~368k rows, i.e. m ~ 1.4 M rows at k = 8192)
  thin_qr_oneshot(ctx, Rs, ldrs, k, R);
  for (int i = 0; i < p; ++i) {
    const int o = i * mc, mi = std::min(mc, m - o);
    CK(cudaMemcpy2DAsync(tmp, sizeof(double) * mi, A + o, sizeof(double) * m, sizeof(double) * mi, k,
                         cudaMemcpyDeviceToDevice, s));
    dgemm(ctx, false, mi, k, k, 1.0, tmp, mi, Rs + (size_t)i * k, ldrs, 0.0, A + o, m);
  }
}

// full SVD of a square k x k matrix B (destroyed): U (k x k), S (k, descending), V (k x k), by the
// hand-written one-sided Jacobi SVD (jacobi_svd.cu) with dgejsv-style QR preconditioning (below).
// Jacobi, like the reference's JacobiSVD, keeps the roundoff-level singular values that drive the
// spurious index tau; a polar-decomposition SVD (measured: cuSOLVER gesvdp) moves tau on the
// degenerate configs (cfg2 NT-off: 20 non-spurious vs 0 for the reference restatement).
static std::vector<double> d2h(const double* d, size_t count, cudaStream_t s) {
  std::vector<double> h(count);
  if (count) {
    CK(cudaMemcpyAsync(h.data(), d, sizeof(double) * count, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  return h;
}

// start an asynchronous device->host copy of `count` doubles into a pinned result array, ordered
// after the work queued so far on ctx->stream; completion is awaited by CopyFence at run end
static void d2h_async(sssvd_gpu_ctx* ctx, const double* d, size_t count, PinnedArray& out) {
  out.resize(count);
  if (!count) return;
  CK(cudaEventRecord(ctx->ev_copy, ctx->stream));
  CK(cudaStreamWaitEvent(ctx->cstream, ctx->ev_copy, 0));
  CK(cudaMemcpyAsync(out.data(), d, sizeof(double) * count, cudaMemcpyDeviceToHost, ctx->cstream));
}
struct CopyFence {
  cudaStream_t s;
  ~CopyFence() { cudaStreamSynchronize(s); }
};

static void svd_square(sssvd_gpu_ctx* ctx, double* B, int k, double* U, double* S, double* V) {
  // hand-written one-sided Jacobi (jacobi_svd.cu) with dgejsv-style preconditioning: B^T = Q2 R2
  // (QR), one-sided Jacobi on X = R2^T (lower triangular, nearly orthogonal columns: far fewer
  // sweeps than on B itself): X J = W = U S  =>  B = R2^T Q2^T = U S (Q2 J)^T, so U_B = W S^{-1}
  // and V_B = Q2 J. Columns sorted by nonincreasing sigma (stable).
  cudaStream_t st = ctx->stream;
  unsigned int* scr = static_cast<unsigned int*>(ctx->jscr.get(64));
  int* sweeps = reinterpret_cast<int*>(scr + 8);
  const double tol = (double)k * 2.220446049250313e-16;   // cosine noise is ~sqrt(k) eps
  double* Q2 = ctx->jq.as<double>((size_t)k * k);
  double* R2 = ctx->jr.as<double>((size_t)k * k);
  CK(transpose(B, k, k, k, Q2, k, st));
  thin_qr(ctx, Q2, k, k, R2);                     // Q2 <- Q, R2 <- R of B^T
  CK(transpose(R2, k, k, k, U, k, st));           // X = R2^T
  double* J = ctx->jj.as<double>((size_t)k * k);
  // the grid-wide block Jacobi (one block pair per SM per outer round) where a block plan fits
  // (64 <= k <= 2048), else the scalar round-robin kernel
  int gb_b, gb_nbe, gb_rpl;
  size_t gb_smem;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  if (jacobi_grid_block_plan(k, sms, &gb_b, &gb_nbe, &gb_rpl, &gb_smem))
    CK(jacobi_svd_grid_block(U, J, k, k, S, tol, 60, scr, sweeps, st));
  else
    CK(jacobi_svd(U, J, k, k, S, tol, 60, scr, sweeps, st));   // U <- W S^-1, S
  dgemm(ctx, false, k, k, k, 1.0, Q2, k, J, k, 0.0, V, k);
  std::vector<double> sv = d2h(S, k, st);
  std::vector<int> order(k);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return sv[a] > sv[b]; });
  std::vector<double> sorted(k);
  for (int i = 0; i < k; ++i) sorted[i] = sv[order[i]];
  int* perm = static_cast<int*>(ctx->jperm.get(sizeof(int) * k));
  double* tmp = ctx->t7.as<double>((size_t)k * k + 64);
  CK(cudaMemcpyAsync(perm, order.data(), sizeof(int) * k, cudaMemcpyHostToDevice, st));
  CK(gather_cols(U, k, perm, nullptr, k, k, tmp, k, st));
  CK(cudaMemcpyAsync(U, tmp, sizeof(double) * k * k, cudaMemcpyDeviceToDevice, st));
  CK(gather_cols(V, k, perm, nullptr, k, k, tmp, k, st));
  CK(cudaMemcpyAsync(V, tmp, sizeof(double) * k * k, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(S, sorted.data(), sizeof(double) * k, cudaMemcpyHostToDevice, st));
  CK(cudaStreamSynchronize(st));
}

// Symmetric eigendecomposition H = Q diag(theta) Q^T (theta ascending), standing in for
// Eigen::SelfAdjointEigenSolver in naive_eigen_route (extract.hpp:114). H (k x k, destroyed) is
// symmetric, so its SVD is U = Q sign(Lambda), V = Q, S = |Lambda|: theta_i = s_i sign(u_i . v_i)
// and the eigenvectors are the right singular vectors, reordered by ascending theta (stable).
static std::vector<double> sym_eig(sssvd_gpu_ctx* ctx, double* H, int k, double* Qout) {
  cudaStream_t st = ctx->stream;
  double* U = ctx->tail[T_EU].as<double>((size_t)k * k);
  double* V = ctx->tail[T_EV].as<double>((size_t)k * k);
  double* S = ctx->tail[T_ES].as<double>(k);
  svd_square(ctx, H, k, U, S, V);
  double* sgn = ctx->t2.as<double>(k);
  CK(col_dot_sign(U, V, k, k, sgn, st));
  std::vector<double> sv = d2h(S, k, st), sg = d2h(sgn, k, st);
  std::vector<double> theta(k);
  for (int i = 0; i < k; ++i) theta[i] = sg[i] * sv[i];
  std::vector<int> order(k);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return theta[a] < theta[b]; });
  std::vector<double> out(k);
  for (int i = 0; i < k; ++i) out[i] = theta[order[i]];
  int* perm = static_cast<int*>(ctx->jperm.get(sizeof(int) * k));
  CK(cudaMemcpyAsync(perm, order.data(), sizeof(int) * k, cudaMemcpyHostToDevice, st));
  CK(gather_cols(V, k, perm, nullptr, k, k, Qout, k, st));
  CK(cudaStreamSynchronize(st));
  return out;
}

static bool near_endpoint(double sigma, double endpoint) {
  return std::abs(sigma - endpoint) <= 1e-9 * std::max(std::abs(endpoint), sigma);
}

static const char* kEmptyNote = "filter annihilated the starting block: no singular values inside the interval";

// ----------------------------------------------------------------------------- run_solve
static void run_solve_impl(sssvd_gpu_ctx* ctx, const sssvd_config& cfg, sssvd_gpu_result* res) {
  cudaStream_t s = ctx->stream;
  const int64_t n = ctx->n, m = ctx->m;
  if (n <= 0) throw Status(SSSVD_E_INVALID_ARGUMENT, "no operator set");
  validate_params(cfg.params, n);
  CopyFence copy_fence{ctx->cstream};   // every return path waits for the result copies
  const bool use_exp = cfg.mode == SSSVD_MODE_SS_SVD_NT || cfg.mode == SSSVD_MODE_NAIVE_NT;
  const bool naive = cfg.mode == SSSVD_MODE_NAIVE || cfg.mode == SSSVD_MODE_NAIVE_NT;
  Contour rule = make_contour(cfg.interval_a, cfg.interval_b, cfg.params.quadrature_count, cfg.aspect, use_exp);
  const int L = (int)cfg.params.block_size, M = (int)cfg.params.moment_degree;
  const int64_t h = cfg.params.quadrature_count / 2;
  auto& info = res->info;
  info.input_transposed = ctx->transposed;
  info.n_internal = n;
  info.block_size = L;
  info.moment_degree = M;
  info.calibration_index = -1;
  info.rows = ctx->transposed ? n : m;
  info.cols = ctx->transposed ? m : n;
  ctx->t_solves = ctx->t_allreduce = ctx->solve_flops = 0;

  // ---- steps 1-2 (form_gram is part of steps 1-2 in every run, pipeline.hpp:124-125); the factor
  // cache lives only inside one solve, like the reference's per-accumulator cache
  double t0 = now_s();
  TailProf tp12(s);
  ctx->has_gram = false;
  ctx->fact_valid = false;
  ensure_gram(ctx, cfg.gram_cap > 0 ? cfg.gram_cap : 8192);
  tp12.mark("form_gram");
  if (ctx->v0_n != n || ctx->v0_L != L || ctx->v0_seed != cfg.params.seed) {
    ctx->v0 = random_start(n, L, cfg.params.seed);
    ctx->v0_n = n;
    ctx->v0_L = L;
    ctx->v0_seed = cfg.params.seed;
  }
  const std::vector<double>& v0 = ctx->v0;
  double start_norm2 = 0;
  for (double x : v0) start_norm2 += x * x;
  const double starting_norm = std::sqrt(start_norm2);
  std::vector<std::complex<double>> shifts(h);
  for (int64_t j = 0; j < h; ++j) shifts[j] = rule.shift(j);
  std::vector<std::complex<double>> w(rule.weights.begin(), rule.weights.begin() + h);
  std::vector<std::complex<double>> t(rule.nodes.begin(), rule.nodes.begin() + h);
  int64_t jb = 0, je = h;
  shard_range(h, ctx->nranks, ctx->rank, &jb, &je);
  {
    // measurement only (tools/scale_estimate.py): SSSVD_SIM_RANKS="G:r" factors just rank r's
    // shard of a G-rank run on this single GPU (no collective; the moments are partial sums)
    static const char* sim = std::getenv("SSSVD_SIM_RANKS");
    int sg = 0, sr = 0;
    if (sim && std::sscanf(sim, "%d:%d", &sg, &sr) == 2 && sg > 0 && sr >= 0 && sr < sg)
      shard_range(h, sg, sr, &jb, &je);
  }
  double* Vd = ctx->V.as<double>((size_t)n * L);
  CK(cudaMemcpyAsync(Vd, v0.data(), sizeof(double) * n * L, cudaMemcpyHostToDevice, s));
  double* S = ctx->S.as<double>((size_t)(M + 1) * n * L);
  cudaEvent_t e0, e1, e2;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventCreate(&e2));
  for (int64_t nu = 1; nu < cfg.params.refinement_steps; ++nu) {
    // refine (moments.hpp:121-128): S0 <- 2 sum_j Re(w_j X_j) == moment pass with M = 0
    CK(cudaEventRecord(e0, s));
    moment_pass_agreed(ctx, shifts, w, h, jb, je, Vd, L, 0, S);
    CK(cudaEventRecord(e1, s));
    allreduce_S(ctx, S, (size_t)n * L);
    CK(cudaEventRecord(e2, s));
    CK(cudaEventSynchronize(e2));
    float a = 0, b = 0;
    CK(cudaEventElapsedTime(&a, e0, e1));
    CK(cudaEventElapsedTime(&b, e1, e2));
    ctx->t_solves += a * 1e-3;
    ctx->t_allreduce += b * 1e-3;
    // S0 row-major [n][L] -> column-major V
    CK(blocks_to_colmajor(S, (int)n, L, 1, Vd, s));
  }
  auto coef = moment_coefficients(w, t, h, M);
  tp12.mark("start block + contour (host)");
  // while the shifted-solve pass runs, a helper thread takes the pinned result buffers from the
  // pool at their largest sizes (page-locking hundreds of MB costs ~0.3 s per GB when the pool
  // has to grow)
  auto reserve = std::async(std::launch::async, [res, m, n, L, M, dev = ctx->device] {
    cudaSetDevice(dev);   // page-locked allocations from this thread must not create a context on GPU 0
    const size_t rmax = (size_t)L * M;
    res->left.resize((size_t)m * rmax);
    res->right.resize((size_t)n * rmax);
    res->blocks.resize((size_t)(M + 1) * n * L);
    res->q.resize(rmax * rmax);
  });
  CK(cudaEventRecord(e0, s));
  moment_pass_agreed(ctx, shifts, coef, h, jb, je, Vd, L, M, S);
  CK(cudaEventRecord(e1, s));
  allreduce_S(ctx, S, (size_t)(M + 1) * n * L);
  CK(cudaEventRecord(e2, s));
  CK(cudaEventSynchronize(e2));
  tp12.mark("shifted solves + moments");
  reserve.get();
  tp12.mark("result buffer reservation");
  {
    float a = 0, b = 0;
    CK(cudaEventElapsedTime(&a, e0, e1));
    CK(cudaEventElapsedTime(&b, e1, e2));
    ctx->t_solves += a * 1e-3;
    ctx->t_allreduce += b * 1e-3;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(e2);
  // column-major blocks: Sc = [S_0 .. S_M] (n x (M+1)L); stacked = Sc[:, :LM], S+ = Sc[:, L:]
  const int r = L * M;
  auto& B = ctx->tail;
  double* Sc = B[T_SC].as<double>((size_t)(M + 1) * n * L);
  CK(blocks_to_colmajor(S, (int)n, L, M + 1, Sc, s));
  CK(cudaStreamSynchronize(s));
  tp12.mark("moment blocks layout");
  info.steps_1_2 = now_s() - t0;
  info.t_gram = ctx->t_gram;
  info.t_shifted_solves = ctx->t_solves;
  info.t_allreduce = ctx->t_allreduce;
  info.shifted_solve_flops = ctx->solve_flops;
  d2h_async(ctx, Sc, (size_t)(M + 1) * n * L, res->blocks);   // Sc is read-only from here on

  // ---- step 3: low_rank (moments.hpp:190-211)
  t0 = now_s();
  double* scratch = ctx->scratch.as<double>(1024);
  CK(sumsq(Sc, (long long)n * r, scratch, scratch + 1000, s));
  const double snorm = std::sqrt(d2h(scratch + 1000, 1, s)[0]);
  if (!(snorm > 1e-12 * starting_norm)) {   // pipeline.hpp:141-148
    info.empty = 1;
    res->note = kEmptyNote;
    res->left.resize(0);
    res->right.resize(0);
    res->q.resize(0);
    info.step_3 = now_s() - t0;
    return;
  }
  TailProf tp(s);
  double* Q = B[T_Q].as<double>((size_t)n * r);
  CK(cudaMemcpyAsync(Q, Sc, sizeof(double) * n * r, cudaMemcpyDeviceToDevice, s));
  double* R = B[T_R].as<double>((size_t)r * r);
  thin_qr(ctx, Q, (int)n, r, R);
  tp.mark("low_rank thin_qr");
  double* UR = B[T_UR].as<double>((size_t)r * r);
  double* VR = B[T_VR].as<double>((size_t)r * r);   // W_S1 = VR[:, :rank]
  double* SV = B[T_SV].as<double>(r);
  svd_square(ctx, R, r, UR, SV, VR);
  tp.mark("low_rank svd_square");
  std::vector<double> sv = d2h(SV, r, s);
  if (sv.empty() || !(sv[0] > 0)) {   // EmptySubspaceError caught at pipeline.hpp:151-156
    info.empty = 1;
    res->note = kEmptyNote;
    res->left.resize(0);
    res->right.resize(0);
    res->q.resize(0);
    info.step_3 = now_s() - t0;
    return;
  }
  int rank = 0;
  while (rank < r && sv[rank] >= cfg.params.lowrank_threshold * sv[0]) ++rank;
  info.retained_rank = rank;
  res->basis_sv.assign(sv.begin(), sv.begin() + rank);
  double* US1 = B[T_US1].as<double>((size_t)n * rank);
  dgemm(ctx, false, (int)n, rank, r, 1.0, Q, (int)n, UR, r, 0.0, US1, (int)n);
  CK(cudaStreamSynchronize(s));
  tp.mark("U_S1 gemm");
  info.step_3 = now_s() - t0;

  const double* Ad = ctx->A.as<double>(0);
  const int lda = (int)ctx->lda;
  const int tcount = rank;
  std::vector<double> sigma(tcount);
  std::vector<int> order(tcount);
  std::vector<int32_t> invalid(tcount, 0);
  std::iota(order.begin(), order.end(), 0);
  double* Qm = B[T_QM].as<double>((size_t)rank * rank);
  double* leftv = B[T_LEFT].as<double>((size_t)m * rank);
  double* right = B[T_RIGHT].as<double>((size_t)n * rank);
  int* perm_d = B[T_PERM].as<int>(rank);
  double* Ut = nullptr;
  double* Pm = nullptr;
  double* Yk = nullptr;
  if (!naive) {
    // ---- step 4: project_qr (extract.hpp:43-57)
    t0 = now_s();
    Ut = B[T_UT].as<double>((size_t)m * rank);
    dgemm(ctx, false, (int)m, rank, (int)n, 1.0, Ad, lda, US1, (int)n, 0.0, Ut, (int)m);
    Yk = B[T_Y].as<double>((size_t)m * rank);   // Y = A U_S1, kept for the Galerkin residuals
    CK(cudaMemcpyAsync(Yk, Ut, sizeof(double) * m * rank, cudaMemcpyDeviceToDevice, s));
    double* Bm = B[T_BM].as<double>((size_t)rank * rank);
    tp.mark("project gemm");
    thin_qr(ctx, Ut, (int)m, rank, Bm);
    tp.mark("project thin_qr");
    std::vector<double> bd(rank);   // the diagonal of B only (a strided copy)
    CK(cudaMemcpy2DAsync(bd.data(), sizeof(double), Bm, sizeof(double) * (rank + 1), sizeof(double), rank,
                         cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const double lead = std::abs(bd[0]);
    for (int i = 0; i < rank; ++i)
      if (std::abs(bd[i]) <= 1e-14 * lead) info.rank_deficient_qr = 1;
    tp.mark("project rank flag d2h");
    info.step_4 = now_s() - t0;
    // ---- step 5: svd_small + assemble_triplets (extract.hpp:66-102)
    t0 = now_s();
    Pm = B[T_PM].as<double>((size_t)rank * rank);
    double* phi_d = B[T_PHI].as<double>(rank);
    svd_square(ctx, Bm, rank, Pm, phi_d, Qm);
    tp.mark("svd_small svd_square");
    std::vector<double> phi = d2h(phi_d, rank, s);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return phi[a] < phi[b]; });
    for (int i = 0; i < rank; ++i) sigma[i] = phi[order[i]];
  } else {
    // ---- naive_eigen_route (extract.hpp:108-139): Rayleigh-Ritz on G in span(U_S1)
    t0 = now_s();
    double* GU = B[T_UT].as<double>((size_t)n * rank);
    dgemm(ctx, false, (int)n, rank, (int)n, 1.0, ctx->G.as<double>(0), (int)n, US1, (int)n, 0.0, GU, (int)n);
    double* H = B[T_BM].as<double>((size_t)rank * rank);
    dgemm(ctx, true, rank, rank, (int)n, 1.0, US1, (int)n, GU, (int)n, 0.0, H, rank);
    CK(symmetrize(H, rank, rank, s));                  // (h + h^T) / 2 (extract.hpp:113)
    std::vector<double> theta = sym_eig(ctx, H, rank, Qm);   // ascending, eigenvectors -> Qm
    for (int i = 0; i < rank; ++i) {
      sigma[i] = std::sqrt(std::max(theta[i], 0.0));
      invalid[i] = theta[i] > 0 ? 0 : 1;
    }
  }
  CK(cudaMemcpyAsync(perm_d, order.data(), sizeof(int) * rank, cudaMemcpyHostToDevice, s));
  double* qs = B[T_QS].as<double>((size_t)rank * rank);           // q = Q[:, order]
  CK(gather_cols(Qm, rank, perm_d, nullptr, rank, rank, qs, rank, s));
  // q (part of the result) goes out first, ahead of the triplet vectors on the copy engine
  res->q.resize((size_t)rank * rank);
  CK(cudaMemcpyAsync(res->q.data(), qs, sizeof(double) * rank * rank, cudaMemcpyDeviceToHost, s));
  dgemm(ctx, false, (int)n, rank, rank, 1.0, US1, (int)n, qs, rank, 0.0, right, (int)n);
  double* sig_d = B[T_SIG].as<double>(rank);
  if (!naive) {
    double* ps = B[T_PS].as<double>((size_t)rank * rank);         // P[:, order]
    CK(gather_cols(Pm, rank, perm_d, nullptr, rank, rank, ps, rank, s));
    dgemm(ctx, false, (int)m, rank, rank, 1.0, Ut, (int)m, ps, rank, 0.0, leftv, (int)m);
  } else {
    double* av = B[T_UT].as<double>((size_t)m * rank);
    dgemm(ctx, false, (int)m, rank, (int)n, 1.0, Ad, lda, right, (int)n, 0.0, av, (int)m);
    std::vector<double> inv(rank);
    for (int i = 0; i < rank; ++i) inv[i] = invalid[i] ? 0.0 : 1.0 / sigma[i];
    CK(cudaMemcpyAsync(sig_d, inv.data(), sizeof(double) * rank, cudaMemcpyHostToDevice, s));
    std::vector<int> idn(rank);
    std::iota(idn.begin(), idn.end(), 0);
    CK(cudaMemcpyAsync(perm_d, idn.data(), sizeof(int) * rank, cudaMemcpyHostToDevice, s));
    CK(gather_cols(av, (int)m, perm_d, sig_d, (int)m, rank, leftv, (int)m, s));
  }
  // the triplet vectors are final: copy them out while the postprocess runs
  d2h_async(ctx, leftv, (size_t)m * tcount, res->left);
  d2h_async(ctx, right, (size_t)n * tcount, res->right);
  tp.mark("assemble gemms");
  info.step_5 = now_s() - t0;

  // ---- postprocess (pipeline.hpp:179-208)
  t0 = now_s();
  info.count = tcount;
  res->sigma = sigma;
  res->in_interval.resize(tcount);
  for (int i = 0; i < tcount; ++i) res->in_interval[i] = (sigma[i] >= cfg.interval_a && sigma[i] <= cfg.interval_b);
  // detect_spurious (postprocess.hpp:47-62)
  const double sv_max = *std::max_element(res->basis_sv.begin(), res->basis_sv.end());
  for (double x : res->basis_sv)
    if (!(x > 0)) throw Status(SSSVD_E_INVALID_ARGUMENT, "detect_spurious: Sigma_S1 must be positive");
  info.spurious_threshold = cfg.params.spurious_threshold * sv_max;
  // tau (postprocess.hpp:56-60) and the estimator's Sigma^+ q (:86-93) in one pass over q on the
  // device; transformed residual norms (postprocess.hpp:76-97):
  //   ||S+ W Sigma^+ q_i - img_i U_S1 q_i|| / sigma_i
  const double rcond = use_exp ? cfg.estimator_rcond_exp : cfg.estimator_rcond_identity;
  std::vector<double> inv(rank);
  for (int l = 0; l < rank; ++l) inv[l] = res->basis_sv[l] >= rcond * sv_max ? 1.0 / res->basis_sv[l] : 0.0;
  double* inv_d = B[T_INV].as<double>(rank);
  double* tau_d = B[T_TAU].as<double>(tcount);
  double* qsc_d = B[T_QSC].as<double>((size_t)rank * tcount);
  CK(cudaMemcpyAsync(inv_d, inv.data(), sizeof(double) * rank, cudaMemcpyHostToDevice, s));
  CK(tau_scale(qs, rank, tcount, SV, inv_d, tau_d, qsc_d, s));
  tp.mark("tau + Sigma^+ q");
  {
    double* coeff = B[T_COEFF].as<double>((size_t)r * tcount);
    dgemm(ctx, false, r, tcount, rank, 1.0, VR, r, qsc_d, rank, 0.0, coeff, r);
    std::vector<double> images(tcount);
    for (int i = 0; i < tcount; ++i) {
      if (use_exp) images[i] = sigma[i] > 1e-30 ? std::log(sigma[i] * sigma[i]) : 0.0;   // g^{-1}(sigma^2)
      else images[i] = sigma[i] * sigma[i];
    }
    double* img_d = B[T_IMG].as<double>(tcount);
    CK(cudaMemcpyAsync(img_d, images.data(), sizeof(double) * tcount, cudaMemcpyHostToDevice, s));
    double* out_d = B[T_NRM].as<double>(3 * (size_t)tcount);
    double* part = B[T_CNP].as<double>(dgemm_norm_scratch((int)std::max(n, m), tcount));
    // the three residual norms as GEMMs with the fused "- d_i w_i, column norm" epilogue:
    //   transformed ||S+ (W Sigma^+ q_i) - img_i v_i|| (postprocess.hpp:91-95)
    CK(dgemm_colnorm_diff(false, (int)n, tcount, r, Sc + (size_t)n * L, (int)n, coeff, r, img_d, right, (int)n, out_d,
                          part, s));
    tp.mark("transformed residual");
    //   exact ||A^T u_i - sigma_i v_i|| (postprocess.hpp:34-41)
    CK(cudaMemcpyAsync(sig_d, sigma.data(), sizeof(double) * tcount, cudaMemcpyHostToDevice, s));
    CK(dgemm_colnorm_diff(true, (int)n, tcount, (int)m, Ad, lda, leftv, (int)m, sig_d, right, (int)n, out_d + tcount,
                          part, s));
    //   Galerkin ||A v_i - sigma_i u_i|| (pipeline.hpp:203-208); A v_i = A U_S1 q_i = Y q_i with Y = A U_S1
    //   kept from project_qr: an m x r x r product instead of m x n x r (equal up to rounding)
    if (Yk)
      CK(dgemm_colnorm_diff(false, (int)m, tcount, rank, Yk, (int)m, qs, rank, sig_d, leftv, (int)m,
                            out_d + 2 * tcount, part, s));
    else
      CK(dgemm_colnorm_diff(false, (int)m, tcount, (int)n, Ad, lda, right, (int)n, sig_d, leftv, (int)m,
                            out_d + 2 * tcount, part, s));
    // one small read-back at the end: the copy engine is busy with the triplet vectors meanwhile
    std::vector<double> norms = d2h(out_d, 3 * (size_t)tcount, s);
    res->tau = d2h(tau_d, tcount, s);
    res->spurious.resize(tcount);
    for (int i = 0; i < tcount; ++i) res->spurious[i] = (res->tau[i] < info.spurious_threshold) || invalid[i];
    res->invalid = invalid;
    tp.mark("exact + galerkin residuals");
    res->estimated.assign(norms.begin(), norms.begin() + tcount);
    for (int i = 0; i < tcount; ++i)
      res->estimated[i] = sigma[i] <= 1e-30 ? std::numeric_limits<double>::infinity() : res->estimated[i] / sigma[i];
    res->exact.assign(norms.begin() + tcount, norms.begin() + 2 * tcount);
    res->galerkin.assign(norms.begin() + 2 * tcount, norms.end());
  }
  if (use_exp) {
    // estimate_residual_nonlinear calibration (postprocess.hpp:121-156)
    int best = -1;
    for (int i = 0; i < tcount; ++i) {
      if (!res->in_interval[i] || res->spurious[i]) continue;
      if (best < 0 || res->tau[i] > res->tau[best]) best = i;
    }
    if (best < 0) {
      std::fill(res->estimated.begin(), res->estimated.end(), std::numeric_limits<double>::quiet_NaN());
      res->note = "nonlinear residual calibration impossible: all candidates spurious";
    } else {
      const double exact_best = res->exact[best];
      const double mu = exact_best / res->estimated[best];
      for (auto& x : res->estimated) x *= mu;
      res->estimated[best] = exact_best;
      info.calibration_index = best;
      info.mu = mu;
    }
  }
  CK(cudaStreamSynchronize(ctx->cstream));
  tp.mark("calibration + result copies");
  info.postprocess = now_s() - t0;
  if (ctx->transposed) {   // pipeline.hpp:214-217
    std::swap(res->left, res->right);
    std::swap(res->exact, res->galerkin);
  }
  for (int i = 0; i < tcount; ++i) {   // pipeline.hpp:219-229
    if (!res->in_interval[i]) continue;
    ++info.count_in_interval;
    if (!res->spurious[i]) ++info.count_nonspurious_in_interval;
    if (near_endpoint(sigma[i], cfg.interval_a) || near_endpoint(sigma[i], cfg.interval_b)) ++info.count_boundary;
    else ++info.count_interior;
  }
}

}  // namespace sssvd_gpu

// ----------------------------------------------------------------------------- C ABI
template <typename F>
static sssvd_status guarded(sssvd_gpu_ctx* ctx, F&& body) {
  try {
    body();
    return SSSVD_OK;
  } catch (const Status& st) {
    if (ctx) ctx->err = st.what();
    return st.code;
  } catch (const std::domain_error& ex) {
    if (ctx) ctx->err = ex.what();
    return SSSVD_E_DOMAIN;
  } catch (const std::length_error& ex) {
    if (ctx) ctx->err = ex.what();
    return SSSVD_E_LENGTH;
  } catch (const std::invalid_argument& ex) {
    if (ctx) ctx->err = ex.what();
    return SSSVD_E_INVALID_ARGUMENT;
  } catch (const std::bad_alloc& ex) {
    if (ctx) ctx->err = ex.what();
    return SSSVD_E_OOM;
  } catch (const std::exception& ex) {
    if (ctx) ctx->err = ex.what();
    return SSSVD_E_CUDA;
  }
}

extern "C" {

uint64_t sssvd_gpu_launch_count(void) { return launch_count(); }
void sssvd_gpu_profile_gemm(int enable) { zgemm_profile_enable(enable != 0); }
void sssvd_gpu_profile_gemm_collect2(double* ms, double* executed_flops, double* algorithmic_flops, uint64_t* launches) {
  unsigned long long n = 0;
  zgemm_profile_collect(ms, executed_flops, algorithmic_flops, &n);
  *launches = n;
}
void sssvd_gpu_profile_gemm_collect(double* ms, double* flops, uint64_t* launches) {
  double alg = 0;
  sssvd_gpu_profile_gemm_collect2(ms, flops, &alg, launches);
}

const char* sssvd_build_info(void) {
  return "sssvd_gpu: sm_100a (compute_100a) DMMA/FP64 kernels";
}

sssvd_status sssvd_gpu_create(int device, sssvd_gpu_ctx** out) {
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count <= device) return SSSVD_E_CUDA;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return SSSVD_E_CUDA;
  if (prop.major != 10) return SSSVD_E_CUDA;  // sm_100a binary only
  auto* ctx = new sssvd_gpu_ctx();
  ctx->device = device;
  if (cudaSetDevice(device) != cudaSuccess || cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return SSSVD_E_CUDA;
  }
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  for (int g = 0; g < sssvd_gpu_ctx::kMaxGroups; ++g) {
    cudaStreamCreateWithPriority(&ctx->gstream[g], cudaStreamNonBlocking, prio_hi);
    cudaStreamCreateWithPriority(&ctx->gstream_lo[g], cudaStreamNonBlocking, prio_lo);
    cudaEventCreateWithFlags(&ctx->ev_join[g], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->ev_pre[g], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->ev_gemm[g], cudaEventDisableTiming);
  }
  cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming);
  cudaStreamCreateWithFlags(&ctx->cstream, cudaStreamNonBlocking);
  cudaEventCreateWithFlags(&ctx->ev_copy, cudaEventDisableTiming);
  zgemm_init_device();   // per-device counters of the GEMM's first-wave offset (never inside a capture)
  *out = ctx;
  return SSSVD_OK;
}

void sssvd_gpu_destroy(sssvd_gpu_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  DBuf* bufs[] = {&ctx->A, &ctx->G, &ctx->gmax, &ctx->mats, &ctx->ipiv, &ctx->shifts, &ctx->coef, &ctx->S, &ctx->V,
                  &ctx->status, &ctx->minpiv, &ctx->scratch, &ctx->t0, &ctx->t1, &ctx->t2, &ctx->t7, &ctx->gwork,
                  &ctx->lw_linv, &ctx->lw_T, &ctx->lw_src, &ctx->lw_disp, &ctx->lw2_linv, &ctx->lw2_T, &ctx->lw2_src, &ctx->lw2_disp, &ctx->jscr, &ctx->jperm, &ctx->jq, &ctx->jr, &ctx->jj,
                  &ctx->qy, &ctx->qt, &ctx->qw, &ctx->ts_tmp, &ctx->ts_rs, &ctx->ts_r};
  for (DBuf* b : bufs) b->release();
  for (auto& b : ctx->tail) b.release();
  if (ctx->comm) nccl().CommDestroy(ctx->comm);
  for (int g = 0; g < sssvd_gpu_ctx::kMaxGroups; ++g) {
    if (ctx->gstream[g]) cudaStreamDestroy(ctx->gstream[g]);
    if (ctx->gstream_lo[g]) cudaStreamDestroy(ctx->gstream_lo[g]);
    if (ctx->ev_join[g]) cudaEventDestroy(ctx->ev_join[g]);
    if (ctx->ev_pre[g]) cudaEventDestroy(ctx->ev_pre[g]);
    if (ctx->ev_gemm[g]) cudaEventDestroy(ctx->ev_gemm[g]);
  }
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->cstream) {
    cudaStreamSynchronize(ctx->cstream);
    cudaStreamDestroy(ctx->cstream);
  }
  if (ctx->ev_copy) cudaEventDestroy(ctx->ev_copy);
  for (auto& g : ctx->lu_graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char* sssvd_gpu_last_error(const sssvd_gpu_ctx* ctx) { return ctx ? ctx->err.c_str() : "no context"; }

sssvd_status sssvd_gpu_set_batch(sssvd_gpu_ctx* ctx, int max_shifts) {
  ctx->max_batch = max_shifts;
  return SSSVD_OK;
}

sssvd_status sssvd_gpu_nccl_unique_id(void* out128) {
  ncclUniqueId id;
  try {
    if (nccl().GetUniqueId(&id) != ncclSuccess) return SSSVD_E_NCCL;
  } catch (const Status& st) {
    return st.code;
  }
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(out128, &id, sizeof(id));
  return SSSVD_OK;
}

sssvd_status sssvd_gpu_init_comm(sssvd_gpu_ctx* ctx, const void* uid, int nranks, int rank) {
  return guarded(ctx, [&]() {
    CK(cudaSetDevice(ctx->device));
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof(id));
    if (ctx->comm) nccl().CommDestroy(ctx->comm);
    ctx->comm = nullptr;
    CKN(nccl().CommInitRank(&ctx->comm, nranks, id, rank));
    ctx->nranks = nranks;
    ctx->rank = rank;
  });
}

sssvd_status sssvd_gpu_set_operator(sssvd_gpu_ctx* ctx, const double* a, int64_t rows, int64_t cols, int64_t lda,
                                    int on_device) {
  return guarded(ctx, [&]() {
    CK(cudaSetDevice(ctx->device));
    int64_t m, n, ldp;
    bool tr;
    upload_operator(ctx, a, rows, cols, lda, on_device, &m, &n, &ldp, &tr);
    finish_operator(ctx, m, n, ldp, tr);
  });
}

sssvd_status sssvd_gpu_set_operator_root(sssvd_gpu_ctx* ctx, const double* a, int64_t rows, int64_t cols,
                                         int64_t lda, int on_device, int root) {
  return guarded(ctx, [&]() {
    CK(cudaSetDevice(ctx->device));
    if (!ctx->comm) {   // no communicator: plain upload (a 1-rank communicator broadcasts to itself)
      int64_t m, n, ldp;
      bool tr;
      upload_operator(ctx, a, rows, cols, lda, on_device, &m, &n, &ldp, &tr);
      finish_operator(ctx, m, n, ldp, tr);
      return;
    }
    if (root < 0 || root >= ctx->nranks) throw Status(SSSVD_E_INVALID_ARGUMENT, "set_operator_root: bad root");
    if (rows <= 0 || cols <= 0) throw Status(SSSVD_E_INVALID_ARGUMENT, "set_operator: bad shape");
    const bool tr = rows < cols;
    const int64_t m = tr ? cols : rows, n = tr ? rows : cols;
    const int64_t ldp = (m + 7) / 8 * 8;
    int code = SSSVD_OK;
    std::string msg;
    if (ctx->rank == root) {
      try {
        int64_t m2, n2, ldp2;
        bool tr2;
        upload_operator(ctx, a, rows, cols, lda, on_device, &m2, &n2, &ldp2, &tr2);
      } catch (const Status& e) {
        code = e.code;
        msg = e.what();
      }
    }
    agree_status(ctx, code, msg);   // the root's upload failed: every rank returns its status
    // one broadcast of the padded internal operator (ldp x n, m >= n) from the root over NVLink
    double* Ad = ctx->A.as<double>((size_t)ldp * n);
    CKN(nccl().Broadcast(Ad, Ad, (size_t)ldp * n, ncclDouble, root, ctx->comm, ctx->stream));
    finish_operator(ctx, m, n, ldp, tr);
  });
}

sssvd_status sssvd_gpu_comm_size(sssvd_gpu_ctx* ctx, int* nranks) {
  return guarded(ctx, [&]() {
    if (!ctx->comm) {
      *nranks = 1;
      return;
    }
    int c = ctx->nranks;
    if (nccl().CommCount) CKN(nccl().CommCount(ctx->comm, &c));
    *nranks = c;
  });
}

sssvd_status sssvd_gpu_set_operator_csc(sssvd_gpu_ctx* ctx, int64_t rows, int64_t cols, int64_t nnz,
                                        const int64_t* colptr, const int64_t* rowind, const double* values,
                                        int on_device) {
  return guarded(ctx, [&]() {
    if (rows <= 0 || cols <= 0 || nnz < 0) throw Status(SSSVD_E_INVALID_ARGUMENT, "set_operator_csc: bad shape");
    if (!colptr || (nnz > 0 && (!rowind || !values)))
      throw Status(SSSVD_E_INVALID_ARGUMENT, "set_operator_csc: null array");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const bool tr = rows < cols;
    const int64_t m = tr ? cols : rows, n = tr ? rows : cols;
    const int64_t ldp = (m + 7) / 8 * 8;
    // stage colptr | rowind | values in one device buffer (8-byte elements throughout)
    const int64_t nz = std::max<int64_t>(nnz, 1);
    const int64_t *cp = colptr, *ri = rowind;
    const double* va = values;
    if (!on_device) {
      int64_t* st = ctx->t0.as<int64_t>((size_t)(cols + 1 + 2 * nz));
      CK(cudaMemcpyAsync(st, colptr, sizeof(int64_t) * (cols + 1), cudaMemcpyHostToDevice, s));
      if (nnz > 0) {
        CK(cudaMemcpyAsync(st + cols + 1, rowind, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(st + cols + 1 + nz, values, sizeof(double) * nnz, cudaMemcpyHostToDevice, s));
      }
      cp = st;
      ri = st + cols + 1;
      va = reinterpret_cast<const double*>(st + cols + 1 + nz);
    }
    int* bad = ctx->scratch.as<int>(2048) + 2040;   // past the doubles sumsq uses (<= index 1000)
    CK(cudaMemsetAsync(bad, 0, sizeof(int), s));
    CK(csc_check(cp, ri, rows, cols, nnz, bad, s));
    int hbad = 0;
    CK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (hbad)
      throw Status(SSSVD_E_INVALID_ARGUMENT,
                   "set_operator_csc: not a compressed CSC matrix (colptr/rowind out of range or unsorted)");
    double* Ad = ctx->A.as<double>((size_t)ldp * n);
    CK(cudaMemsetAsync(Ad, 0, sizeof(double) * ldp * n, s));
    CK(csc_scatter(cp, ri, va, cols, tr, Ad, ldp, s));
    finish_operator(ctx, m, n, ldp, tr);
  });
}

sssvd_status sssvd_gpu_form_gram(sssvd_gpu_ctx* ctx, int64_t cap, double* g_out) {
  return guarded(ctx, [&]() {
    CK(cudaSetDevice(ctx->device));
    ensure_gram(ctx, cap > 0 ? cap : 8192);
    if (g_out) {
      CK(cudaMemcpyAsync(g_out, ctx->G.as<double>(0), sizeof(double) * ctx->n * ctx->n, cudaMemcpyDeviceToHost,
                         ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
    }
  });
}

// debug: the lower-triangle tile share `part` of `nparts` of the Gram (the multi-GPU sharding of
// form_gram), zeros elsewhere; column-major n x n into g_out
sssvd_status sssvd_debug_gram_part(sssvd_gpu_ctx* ctx, int part, int nparts, double* g_out) {
  return guarded(ctx, [&]() {
    if (ctx->n <= 0 || nparts < 1 || part < 0 || part >= nparts) throw Status(SSSVD_E_INVALID_ARGUMENT, "bad part");
    CK(cudaSetDevice(ctx->device));
    double* G = ctx->t2.as<double>((size_t)ctx->n * ctx->n);
    CK(cudaMemsetAsync(G, 0, sizeof(double) * ctx->n * ctx->n, ctx->stream));
    CK(gram(ctx->A.as<double>(0), (int)ctx->lda, (int)ctx->lda, (int)ctx->n, G, (int)ctx->n, part, nparts, ctx->stream));
    CK(cudaMemcpyAsync(g_out, G, sizeof(double) * ctx->n * ctx->n, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

sssvd_status sssvd_debug_thin_qr(sssvd_gpu_ctx* ctx, const double* a, int64_t m, int64_t k, double* q_out,
                                 double* r_out) {
  return guarded(ctx, [&]() {
    if (m < 1 || k < 1 || m < k) throw Status(SSSVD_E_INVALID_ARGUMENT, "thin_qr: need m >= k >= 1");
    CK(cudaSetDevice(ctx->device));
    double* A = ctx->t1.as<double>((size_t)m * k);
    double* R = ctx->t2.as<double>((size_t)k * k);
    CK(cudaMemcpyAsync(A, a, sizeof(double) * m * k, cudaMemcpyHostToDevice, ctx->stream));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, ctx->stream));
    thin_qr(ctx, A, (int)m, (int)k, R);
    CK(cudaEventRecord(e1, ctx->stream));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (std::getenv("SSSVD_DEBUG")) std::fprintf(stderr, "[sssvd] thin_qr %lld x %lld: %.3f ms\n", (long long)m, (long long)k, ms);
    CK(cudaMemcpyAsync(q_out, A, sizeof(double) * m * k, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(r_out, R, sizeof(double) * k * k, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

sssvd_status sssvd_debug_svd_square(sssvd_gpu_ctx* ctx, const double* b, int64_t k, double* u_out, double* s_out,
                                    double* v_out) {
  return guarded(ctx, [&]() {
    if (k < 1) throw Status(SSSVD_E_INVALID_ARGUMENT, "svd_square: need k >= 1");
    CK(cudaSetDevice(ctx->device));
    double* B = ctx->t1.as<double>((size_t)3 * k * k + k);
    double *U = B + (size_t)k * k, *V = U + (size_t)k * k, *S = V + (size_t)k * k;
    CK(cudaMemcpyAsync(B, b, sizeof(double) * k * k, cudaMemcpyHostToDevice, ctx->stream));
    svd_square(ctx, B, (int)k, U, S, V);
    CK(cudaMemcpyAsync(u_out, U, sizeof(double) * k * k, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(v_out, V, sizeof(double) * k * k, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(s_out, S, sizeof(double) * k, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

namespace {
__global__ void debug_fill_kernel(double* p, long long cnt, unsigned long long seed) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cnt; i += (long long)gridDim.x * blockDim.x) {
    unsigned long long x = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
    x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 29;
    p[i] = (double)(x >> 11) * (1.0 / 9007199254740992.0) - 0.5;
  }
}
__global__ void debug_diff_kernel(const double* a, const double* b, long long cnt, double tol,
                                  unsigned long long* out) {
  unsigned long long c = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cnt; i += (long long)gridDim.x * blockDim.x)
    c += !(fabs(a[i] - b[i]) <= tol);
  if (c) atomicAdd(out, c);
}
}  // namespace

// debug: times the trailing-update GEMM C -= A B (complex, row-major, batched) on seeded data.
// variant 0: the 4-product cp.async kernel, 1: its TMA form, 2: the 3-product (3M) kernel (the product
// default). *mismatches_out counts the entries that differ from the 4-product cp.async kernel's
// result on the same inputs: bitwise for variants 0 and 1, by more than the 3M rounding bound
// (K * 1e-15 on operands in [-0.5, 0.5]) for variant 2.
sssvd_status sssvd_debug_zgemm(sssvd_gpu_ctx* ctx, int variant, int64_t m, int64_t n, int64_t k, int64_t batch,
                               int reps, double* ms_out, int64_t* mismatches_out) {
  return guarded(ctx, [&]() {
    if (m < 1 || n < 1 || k < 1 || batch < 1 || reps < 1 || variant < 0 || variant > 2)
      throw Status(SSSVD_E_INVALID_ARGUMENT, "debug_zgemm: bad arguments");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const size_t na = (size_t)batch * m * k, nb = (size_t)batch * k * n, nc = (size_t)batch * m * n;
    double2 *A = nullptr, *B = nullptr, *C0 = nullptr, *C1 = nullptr, *C2 = nullptr;
    unsigned long long* cnt = nullptr;
    auto release = [&]() {
      zgemm_force(0);
      cudaFree(A); cudaFree(B); cudaFree(C0); cudaFree(C1); cudaFree(C2); cudaFree(cnt);
    };
    try {
      CK(cudaMalloc(&A, na * sizeof(double2)));
      CK(cudaMalloc(&B, nb * sizeof(double2)));
      CK(cudaMalloc(&C0, nc * sizeof(double2)));
      CK(cudaMalloc(&C1, nc * sizeof(double2)));
      CK(cudaMalloc(&C2, nc * sizeof(double2)));
      CK(cudaMalloc(&cnt, sizeof(unsigned long long)));
      debug_fill_kernel<<<1184, 256, 0, s>>>((double*)A, 2 * (long long)na, 1);
      debug_fill_kernel<<<1184, 256, 0, s>>>((double*)B, 2 * (long long)nb, 2);
      debug_fill_kernel<<<1184, 256, 0, s>>>((double*)C0, 2 * (long long)nc, 3);
      CK(cudaMemcpyAsync(C1, C0, nc * sizeof(double2), cudaMemcpyDeviceToDevice, s));
      CK(cudaMemcpyAsync(C2, C0, nc * sizeof(double2), cudaMemcpyDeviceToDevice, s));
      zgemm_force(1);
      CK(zgemm_sub((int)m, (int)n, (int)k, A, (int)k, m * k, B, (int)n, k * n, C2, (int)n, m * n, (int)batch, s));
      zgemm_force(variant + 1);
      CK(zgemm_sub((int)m, (int)n, (int)k, A, (int)k, m * k, B, (int)n, k * n, C1, (int)n, m * n, (int)batch, s));
      CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), s));
      debug_diff_kernel<<<1184, 256, 0, s>>>((const double*)C1, (const double*)C2, 2 * (long long)nc,
                                             variant >= 2 ? 1e-15 * (double)k : 0.0, cnt);
      unsigned long long h = 0;
      CK(cudaMemcpyAsync(&h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s));
      cudaEvent_t e0, e1;
      CK(cudaEventCreate(&e0));
      CK(cudaEventCreate(&e1));
      CK(cudaEventRecord(e0, s));
      for (int r = 0; r < reps; ++r)
        CK(zgemm_sub((int)m, (int)n, (int)k, A, (int)k, m * k, B, (int)n, k * n, C1, (int)n, m * n, (int)batch, s));
      CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      *ms_out = ms / reps;
      *mismatches_out = (int64_t)h;
    } catch (...) {
      release();
      throw;
    }
    release();
  });
}

// debug: C = alpha op(A) B + beta C through the tail GEMM (dgemm.cu), host column-major buffers
// (C in/out); mode 1: out[j] = ||op(A) B[:, j] - d_j V[:, j]|| (the fused residual form) into c_out
sssvd_status sssvd_debug_dgemm(sssvd_gpu_ctx* ctx, int mode, int ta, int64_t m, int64_t n, int64_t k, double alpha,
                               const double* a, int64_t lda, const double* b, int64_t ldb, double beta,
                               const double* d, const double* v, double* c_io, int64_t ldc) {
  return guarded(ctx, [&]() {
    if (m < 1 || n < 1 || k < 0 || lda < (ta ? std::max<int64_t>(k, 1) : m) || ldb < std::max<int64_t>(k, 1) ||
        ldc < m || (mode != 0 && mode != 1))
      throw Status(SSSVD_E_INVALID_ARGUMENT, "debug_dgemm: bad arguments");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const size_t na = (size_t)lda * (ta ? m : std::max<int64_t>(k, 1)), nb = (size_t)ldb * n, nc = (size_t)ldc * n;
    double* A = ctx->t0.as<double>(na + nb + 2 * nc + n);
    double *B = A + na, *C = B + nb, *Vd = C + nc, *dd = Vd + nc;
    CK(cudaMemcpyAsync(A, a, sizeof(double) * na, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(B, b, sizeof(double) * nb, cudaMemcpyHostToDevice, s));
    if (mode == 0) {
      CK(cudaMemcpyAsync(C, c_io, sizeof(double) * nc, cudaMemcpyHostToDevice, s));
      dgemm(ctx, ta != 0, (int)m, (int)n, (int)k, alpha, A, (int)lda, B, (int)ldb, beta, C, (int)ldc);
      CK(cudaMemcpyAsync(c_io, C, sizeof(double) * nc, cudaMemcpyDeviceToHost, s));
    } else {
      CK(cudaMemcpyAsync(Vd, v, sizeof(double) * nc, cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(dd, d, sizeof(double) * n, cudaMemcpyHostToDevice, s));
      double* part = ctx->t2.as<double>(dgemm_norm_scratch((int)m, (int)n));
      CK(dgemm_colnorm_diff(ta != 0, (int)m, (int)n, (int)k, A, (int)lda, B, (int)ldb, dd, Vd, (int)ldc, C, part, s));
      CK(cudaMemcpyAsync(c_io, C, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
  });
}

sssvd_status sssvd_gpu_shifted_solve(sssvd_gpu_ctx* ctx, const double* g, int64_t n, double zr, double zi,
                                     const double* rhs, int64_t rhs_rows, int64_t L, double* x_out) {
  return guarded(ctx, [&]() {
    if (n <= 0 || L <= 0) throw Status(SSSVD_E_INVALID_ARGUMENT, "ShiftedFactorization: empty system");
    if (rhs_rows != n) throw std::invalid_argument("ShiftedFactorization: right-hand side dimension mismatch");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    LuPlan P = make_plan((int)n, (int)L);
    ctx->fact_valid = false;   // this entry point overwrites the factor workspace
    double2* mats = ctx->mats.as<double2>(P.stride);
    int* ipiv = ctx->ipiv.as<int>(n);
    double* Gd = ctx->t0.as<double>((size_t)n * n);
    CK(cudaMemcpyAsync(Gd, g, sizeof(double) * n * n, cudaMemcpyHostToDevice, s));
    double* gmax = ctx->t2.as<double>(1);
    CK(absmax(Gd, (long long)n * n, gmax, s));
    double2* dz = ctx->shifts.as<double2>(1);
    double2 hz = make_double2(zr, zi);
    CK(cudaMemcpyAsync(dz, &hz, sizeof(double2), cudaMemcpyHostToDevice, s));
    // assemble with a zero RHS block, then write the complex RHS into the augmented columns
    double* Vz = ctx->t1.as<double>((size_t)n * L);
    CK(cudaMemsetAsync(Vz, 0, sizeof(double) * n * L, s));
    CK(assemble(Gd, (int)n, (int)n, Vz, (int)L, dz, mats, P.ld, P.stride, 1, s));
    // rhs: column-major complex n x L -> row-major columns n..n+L of mats
    std::vector<double2> hrow((size_t)n * L);
    for (int64_t c = 0; c < L; ++c)
      for (int64_t i = 0; i < n; ++i) hrow[(size_t)i * L + c] = make_double2(rhs[2 * (c * n + i)], rhs[2 * (c * n + i) + 1]);
    CK(cudaMemcpy2DAsync(mats + n, sizeof(double2) * P.ld, hrow.data(), sizeof(double2) * L, sizeof(double2) * L, n,
                         cudaMemcpyHostToDevice, s));
    lu_solve_batch(P, make_work(ctx, P, 1), mats, ipiv, 1, s);
    int* dstatus = ctx->status.as<int>(1);
    double* dmin = ctx->minpiv.as<double>(1);
    CK(pivot_floor(mats, P.ld, P.stride, (int)n, dz, gmax, dstatus, dmin, 1, s));
    int hs = 0;
    CK(cudaMemcpyAsync(&hs, dstatus, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpy2DAsync(hrow.data(), sizeof(double2) * L, mats + n, sizeof(double2) * P.ld, sizeof(double2) * L, n,
                         cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (hs) throw Status(SSSVD_E_NUMERICAL, "ShiftedFactorization: shift numerically on the spectrum");
    for (int64_t c = 0; c < L; ++c)
      for (int64_t i = 0; i < n; ++i) {
        x_out[2 * (c * n + i)] = hrow[(size_t)i * L + c].x;
        x_out[2 * (c * n + i) + 1] = hrow[(size_t)i * L + c].y;
      }
  });
}

sssvd_status sssvd_gpu_moments(sssvd_gpu_ctx* ctx, int64_t h, const double* shifts, const double* weights,
                               const double* nodes, const double* s0, int64_t L, int64_t ell, int64_t M,
                               double* s_out) {
  return guarded(ctx, [&]() {
    if (h < 1 || L < 1 || ell < 1 || M < 0) throw std::invalid_argument("moments: bad counts");
    if (!ctx->has_gram) throw Status(SSSVD_E_INVALID_ARGUMENT, "moments: call sssvd_gpu_form_gram first");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const int64_t n = ctx->n;
    std::vector<std::complex<double>> z(h), w(h), t(h);
    for (int64_t j = 0; j < h; ++j) {
      z[j] = {shifts[2 * j], shifts[2 * j + 1]};
      w[j] = {weights[2 * j], weights[2 * j + 1]};
      t[j] = {nodes[2 * j], nodes[2 * j + 1]};
    }
    int64_t jb = 0, je = h;
    shard_range(h, ctx->nranks, ctx->rank, &jb, &je);
    double* Vd = ctx->V.as<double>((size_t)n * L);
    ctx->fact_valid = false;   // the cache lives inside one accumulator call
    CK(cudaMemcpyAsync(Vd, s0, sizeof(double) * n * L, cudaMemcpyHostToDevice, s));
    double* S = ctx->S.as<double>((size_t)(M + 1) * n * L);
    for (int64_t nu = 1; nu < ell; ++nu) {
      moment_pass_agreed(ctx, z, w, h, jb, je, Vd, (int)L, 0, S);
      allreduce_S(ctx, S, (size_t)n * L);
      CK(blocks_to_colmajor(S, (int)n, (int)L, 1, Vd, s));
    }
    auto coef = moment_coefficients(w, t, h, M);
    moment_pass_agreed(ctx, z, coef, h, jb, je, Vd, (int)L, (int)M, S);
    allreduce_S(ctx, S, (size_t)(M + 1) * n * L);
    double* Sc = ctx->t0.as<double>((size_t)(M + 1) * n * L);
    CK(blocks_to_colmajor(S, (int)n, (int)L, (int)M + 1, Sc, s));
    CK(cudaMemcpyAsync(s_out, Sc, sizeof(double) * (M + 1) * n * L, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  });
}

sssvd_status sssvd_gpu_run_solve(sssvd_gpu_ctx* ctx, const sssvd_config* cfg, sssvd_gpu_result** out) {
  *out = nullptr;
  auto* res = new sssvd_gpu_result();
  sssvd_status st;
  {
    auto body = [&]() {
      CK(cudaSetDevice(ctx->device));
      run_solve_impl(ctx, *cfg, res);
    };
    try {
      body();
      st = SSSVD_OK;
    } catch (const Status& e) {
      ctx->err = e.what();
      st = e.code;
    } catch (const std::domain_error& e) {
      ctx->err = e.what();
      st = SSSVD_E_DOMAIN;
    } catch (const std::length_error& e) {
      ctx->err = e.what();
      st = SSSVD_E_LENGTH;
    } catch (const std::invalid_argument& e) {
      ctx->err = e.what();
      st = SSSVD_E_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
      ctx->err = e.what();
      st = SSSVD_E_CUDA;
    }
  }
  if (st != SSSVD_OK) {
    delete res;
    return st;
  }
  *out = res;
  return SSSVD_OK;
}

sssvd_status sssvd_result_info_get(const sssvd_gpu_result* res, sssvd_result_info* info) {
  *info = res->info;
  return SSSVD_OK;
}

sssvd_status sssvd_result_copy(const sssvd_gpu_result* res, int field, void* dst) {
  auto cp = [&](const auto& v) {
    if (!v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(*v.data()));
  };
  switch (field) {
    case SSSVD_FIELD_SIGMA: cp(res->sigma); break;
    case SSSVD_FIELD_TAU: cp(res->tau); break;
    case SSSVD_FIELD_ESTIMATED: cp(res->estimated); break;
    case SSSVD_FIELD_EXACT: cp(res->exact); break;
    case SSSVD_FIELD_GALERKIN: cp(res->galerkin); break;
    case SSSVD_FIELD_IN_INTERVAL: cp(res->in_interval); break;
    case SSSVD_FIELD_SPURIOUS: cp(res->spurious); break;
    case SSSVD_FIELD_LEFT: cp(res->left); break;
    case SSSVD_FIELD_RIGHT: cp(res->right); break;
    case SSSVD_FIELD_BASIS_SV: cp(res->basis_sv); break;
    case SSSVD_FIELD_BLOCKS: cp(res->blocks); break;
    case SSSVD_FIELD_Q: cp(res->q); break;
    case SSSVD_FIELD_INVALID: cp(res->invalid); break;
    default: return SSSVD_E_INVALID_ARGUMENT;
  }
  return SSSVD_OK;
}

const char* sssvd_result_note(const sssvd_gpu_result* res) { return res->note.c_str(); }
void sssvd_result_free(sssvd_gpu_result* res) { delete res; }

}  // extern "C"
