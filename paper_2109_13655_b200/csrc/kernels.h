// Launchers for the sm_100a kernels of the shifted-solve path (internal C++ interface).
#pragma once
#include <cstddef>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

namespace sssvd_gpu {

cudaError_t cuda_fail(cudaError_t e, const char* expr, const char* file, int line);
// per-(kernel, device) dynamic shared-memory / non-portable cluster attributes (zgemm.cu)
cudaError_t set_kernel_smem(const void* fn, size_t bytes, bool nonportable_cluster);

// instrumentation: every launcher bumps the launch counter; when profiling is on, zgemm_sub
// brackets each launch with CUDA events on its stream (the dominant kernel's live timing)
void note_launch(unsigned long long count = 1);
unsigned long long launch_count();
void unnote_launch(unsigned long long count);   // captured into a graph, not executed
void zgemm_profile_enable(bool on);
void zgemm_profile_collect(double* ms, double* flops, double* algorithmic, unsigned long long* launches);
// GEMM stamps of one shifted-solve pass (zgemm.cu): begin resets the slots (stream-ordered, so it
// is captured with a graph), end returns the per-slot flops, harvest folds a finished pass in
cudaError_t zgemm_stamp_pass_begin(cudaStream_t s);
std::vector<double> zgemm_stamp_pass_end();
void zgemm_stamp_harvest(const std::vector<double>& flops);

// K0 Gram (gram.cu): G = A^T A, A column-major (lda even, K = rows incl. zero padding)
cudaError_t gram(const double* A, int lda, int K, int n, double* G, int ldg, int part, int nparts, cudaStream_t s);
// max |a_i| (lu.cu)
cudaError_t absmax(const double* a, long long count, double* out, cudaStream_t s);

// K1 assembly (lu.cu): mats[b] = [z_b I - G | V]  row-major, pitch ld
cudaError_t assemble(const double* G, int n, int ldg, const double* V, int L, const double2* shifts,
                     double2* out, int ld, long long stride, int batch, cudaStream_t s);
cudaError_t load_rhs(const double* V, int n, int L, double2* out, int ld, long long stride, int batch, cudaStream_t s);
// K2 leaf panel LU (lu.cu): rows [r0, n) x cols [r0, r0+w), W in {8,16,32}
size_t leaf_smem_bytes(int n, int W, int cluster);
// K2 (lu.cu): cluster leaf LU; cb < r0: the leaf also applies its interchanges to columns [cb, r0)
cudaError_t leaf_lu(double2* mats, int ld, long long stride, int n, int r0, int w, int W, int cluster, int* ipiv,
                       int batch, cudaStream_t s, int cb);
cudaError_t pivot_floor(const double2* mats, int ld, long long stride, int n, const double2* shifts,
                        const double* gmax, int* status, double* minpiv, int batch, cudaStream_t s);
// K5 (zgemm.cu): C -= A B, row-major complex, batched
cudaError_t zgemm_sub(int M, int N, int K, const double2* A, int lda, long long sA, const double2* B,
                      int ldb, long long sB, double2* C, int ldc, long long sC, int batch,
                      cudaStream_t stream);
// debug: route zgemm_sub to 1 = the cp.async kernel, 2 = the TMA kernel, 0 = the default (zgemm.cu)
void zgemm_force(int kernel);
// allocates the current device's arrival counters of the first-wave CTA offset (zgemm.cu)
void zgemm_init_device();
// C = A B[brow[k], :] (row-gathered B), row-major complex, batched (zgemm.cu)
cudaError_t zgemm_set_gather(int M, int N, int K, const double2* A, int lda, long long sA, const double2* B,
                             int ldb, long long sB, const int* brow, int sR, double2* C, int ldc, long long sC,
                             int batch, cudaStream_t stream);
// K3/K4 (lu.cu): the panel's interchange map + L11^{-1} in one launch
cudaError_t panel_prep(const double2* mats, int ld, long long stride, int r0, int np, double2* linv, long long lstride,
                       const int* ipiv, int n, int* src, int* disp, int dstride, int batch, cudaStream_t s);
cudaError_t scatter_copy(double2* mats, int ld, long long stride, int r0, int np, int c0, int c1, const int* disp,
                         int dstride, const double2* T, int ldt, long long tstride, int batch, cudaStream_t s);
// K6 (lu.cu): rows r0..r0+np of columns [c0, c1) <- U11^{-1} (.), shared-memory staged
cudaError_t trsm_upper_blocks(double2* mats, int ld, long long stride, int r0, int np, int c0, int c1, int batch,
                            cudaStream_t s);
// Tail GEMMs on DMMA (dgemm.cu), column-major: C (m x n) = alpha op(A) B + beta C with op(A) = A
// (m x k) or A^T (A stored k x m). Deep-K skinny outputs split K into `work` (reduced in fixed order)
// when work_elems allows; deterministic.
int dgemm_split_count(int m, int n, int k, size_t work_elems);
cudaError_t dgemm(bool ta, int m, int n, int k, double alpha, const double* A, int lda, const double* B, int ldb,
                  double beta, double* C, int ldc, double* work, size_t work_elems, cudaStream_t s);
// out[j] = || op(A) B[:, j] - d[j] V[:, j] ||_2, fused epilogue; part: dgemm_norm_scratch(m, n) doubles
size_t dgemm_norm_scratch(int m, int n);
cudaError_t dgemm_colnorm_diff(bool ta, int m, int n, int k, const double* A, int lda, const double* B, int ldb,
                               const double* d, const double* V, int ldv, double* out, double* part, cudaStream_t s);
// out (cols x rows) = in^T, column-major (dgemm.cu)
cudaError_t transpose(const double* in, int rows, int cols, int ldi, double* out, int ldo, cudaStream_t s);
// sgn[j] = sign(U[:, j] . V[:, j]) for rows x cols column-major U, V (dgemm.cu)
cudaError_t col_dot_sign(const double* U, const double* V, int rows, int cols, double* sgn, cudaStream_t s);
// h <- (h + h^T) / 2 in place (dgemm.cu)
cudaError_t symmetrize(double* h, int k, int ldh, cudaStream_t s);
// one-sided Jacobi SVD (jacobi_svd.cu): W (k x k, in) -> W = U (unsorted), V, S = sigma
cudaError_t jacobi_svd(double* W, double* V, int k, int ldw, double* S, double tol, int max_sweeps,
                       unsigned int* scratch, int* sweeps_out, cudaStream_t s);
// 64 <= k <= 2048: block Jacobi over the whole GPU (one block pair per SM per outer round)
cudaError_t jacobi_svd_grid_block(double* W, double* V, int k, int ldw, double* S, double tol, int max_sweeps,
                                  unsigned int* scratch, int* sweeps_out, cudaStream_t s);
bool jacobi_grid_block_plan(int k, int sms, int* b, int* nbe, int* rpl, size_t* smem);
// K7 (moments.cu)
cudaError_t moments(const double2* mats, int ld, long long stride, int xcol, int n, int L, int nb,
                    const double2* coef, int M, double* S, cudaStream_t s);
cudaError_t blocks_to_colmajor(const double* S, int n, int L, int nblk, double* out, cudaStream_t s);
// part: colnorm_scratch(rows, cols) doubles of per-chunk partial sums
size_t colnorm_scratch(int rows, int cols);
cudaError_t colnorm_diff(const double* X, int ldx, const double* Y, int ldy, const double* s, int rows,
                         int cols, double* out, double* part, cudaStream_t st);
cudaError_t tau_scale(const double* q, int rank, int tcount, const double* sv, const double* inv, double* tau,
                      double* qsc, cudaStream_t st);
cudaError_t gather_cols(const double* src, int lds, const int* perm, const double* scale, int rows,
                        int cols, double* dst, int ldd, cudaStream_t st);
cudaError_t sumsq(const double* a, long long count, double* scratch, double* out, cudaStream_t s);
cudaError_t pad_copy(const double* src, int rows, int cols, int lds, double* dst, int ldd, cudaStream_t s);
// sparse ingest (sparse.cu): CSC validation (sets *bad) and densify into a zeroed operator
cudaError_t csc_check(const int64_t* colptr, const int64_t* rowind, int64_t rows, int64_t cols, int64_t nnz,
                      int* bad, cudaStream_t s);
cudaError_t csc_scatter(const int64_t* colptr, const int64_t* rowind, const double* vals, int64_t cols,
                        bool transposed, double* Ad, int64_t ldp, cudaStream_t s);
// Householder QR of the tail (householder_qr.cu): cluster panel factorisation of A[j:m, j:j+w]
// (w <= 32) writing R/v in place, explicit Y (rows j..m, ldy) and T (32 x 32 column-major)
size_t qr_panel_smem(int rp, int w);
int qr_panel_plan(int mp, int w, int* cluster);
cudaError_t qr_panel(double* A, int lda, int m, int j, int w, double* Y, int ldy, double* T, double* tau,
                     cudaStream_t s);
// register-resident panel (householder_qr.cu): W in {8, 16, 32}, up to 16 x qr_panel_reg_rows(W) rows
int qr_panel_reg_rows(int W);
cudaError_t qr_panel_reg(double* A, int lda, int m, int j, int w, int W, double* Y, int ldy, double* T, double* tau,
                         cudaStream_t s);
cudaError_t eye(double* Q, int m, int k, int ldq, cudaStream_t s);
// T (kb x kb) of the block reflector H_0..H_{kb-1} = I - Y T Y^T from G = Y^T Y and tau (kb <= 128)
cudaError_t larft(const double* G, int kb, const double* tau, double* T, cudaStream_t s);
cudaError_t copy_r(const double* A, int lda, int k, double* R, cudaStream_t s);
// *bad |= 1 if any of a[0..count) is NaN / Inf (sparse.cu)
cudaError_t any_nonfinite(const double* a, long long count, int* bad, cudaStream_t s);

}  // namespace sssvd_gpu
