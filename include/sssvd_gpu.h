/* sssvd_gpu.h - C ABI of the B200-native block SS-SVD shifted-solve path.
 *
 * Drop-in boundary for the reference C++ library `sssvd` (header-only, Eigen 3;
 * /root/reference/proj/include/sssvd). The reference's plugin point is the Backend template
 * parameter of MomentAccumulator<Scalar, Backend> (moments.hpp:101) and, above it, the entry
 * point run_solve(ProblemMatrix, RunConfig) -> RunResult (pipeline.hpp:112). Because a
 * per-shift solve() returning a host matrix would force h device->host copies and host-side
 * accumulation, the boundary sits one level up: the accumulator (refine + accumulate) and the
 * whole run_solve. Every entry point below names the reference interface it replaces.
 *
 * Conventions: plain pointers and sizes; all matrices column-major (Eigen's default);
 * complex arrays interleaved (re, im). The caller owns every host buffer; the context owns all
 * device memory, the stream and the (optional) NCCL communicator. A context is not re-entrant.
 * There is NO CPU fallback: every compute entry point runs sm_100a kernels and fails with
 * SSSVD_E_CUDA if no B200 is present.
 */
#ifndef SSSVD_GPU_H
#define SSSVD_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sssvd_gpu_ctx sssvd_gpu_ctx;
typedef struct sssvd_gpu_result sssvd_gpu_result;

/* Error taxonomy of the reference mapped onto status codes (core.hpp:29-39; CLI exit codes
 * sssvd.cpp:390-408: 2 for the first three, 3 for NUMERICAL / EMPTY_SUBSPACE). */
typedef enum {
  SSSVD_OK = 0,
  SSSVD_E_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  SSSVD_E_DOMAIN = 2,           /* std::domain_error (Exp transform with a = 0, g^{-1}(<=0)) */
  SSSVD_E_LENGTH = 3,           /* std::length_error (form_gram cap, problem.hpp:84-85) */
  SSSVD_E_NUMERICAL = 4,        /* NumericalError: min|U_ii| <= 1e-30 (max|G| + |z|) */
  SSSVD_E_EMPTY_SUBSPACE = 5,   /* EmptySubspaceError (moments.hpp:201-203) */
  SSSVD_E_CUDA = 6,
  SSSVD_E_NCCL = 7,
  SSSVD_E_OOM = 8,
  SSSVD_E_FORMAT = 9,           /* MatrixMarketError (matrix_market.hpp:17-21): "path:line: what" */
  SSSVD_E_IO = 10               /* std::runtime_error: cannot open / write failed */
} sssvd_status;

/* SolveMode (pipeline.hpp:24) */
typedef enum {
  SSSVD_MODE_SS_SVD = 0,
  SSSVD_MODE_SS_SVD_NT = 1,
  SSSVD_MODE_NAIVE = 2,
  SSSVD_MODE_NAIVE_NT = 3
} sssvd_mode;

/* SpectralTransform kind (transform.hpp:14) */
typedef enum { SSSVD_TRANSFORM_IDENTITY = 0, SSSVD_TRANSFORM_EXP = 1 } sssvd_transform;

/* SsParams (moments.hpp:23-31) */
typedef struct {
  int64_t block_size;       /* L   (default 20) */
  int64_t moment_degree;    /* M   (default 4)  */
  int64_t quadrature_count; /* N   (default 32) */
  int64_t refinement_steps; /* ell (default 1)  */
  double lowrank_threshold; /* delta   (1e-20) */
  double spurious_threshold;/* epsilon (1e-8)  */
  uint64_t seed;            /* 42 */
} sssvd_params;

/* RunConfig (pipeline.hpp:43-58) + the form_gram cap (problem.hpp:82) */
typedef struct {
  double interval_a;
  double interval_b;
  int32_t mode; /* sssvd_mode */
  double aspect;
  sssvd_params params;
  int32_t threads; /* accepted for API parity; the GPU path has no worker pool */
  double estimator_rcond_identity;
  double estimator_rcond_exp;
  int64_t gram_cap; /* 8192 in the reference; BASELINE config 5 lifts it */
} sssvd_config;

/* Fills the reference defaults (RunConfig{} / SsParams{}). */
void sssvd_default_config(sssvd_config* cfg);

/* ---- context ---------------------------------------------------------------------------- */
sssvd_status sssvd_gpu_create(int device, sssvd_gpu_ctx** out);
void sssvd_gpu_destroy(sssvd_gpu_ctx* ctx);
const char* sssvd_gpu_last_error(const sssvd_gpu_ctx* ctx);
/* Cap on shifts factored concurrently (memory budget); 0 = automatic. */
sssvd_status sssvd_gpu_set_batch(sssvd_gpu_ctx* ctx, int max_shifts_in_flight);

/* ---- multi-GPU (one process per GPU) ------------------------------------------------------ *
 * Replaces parallel_for over quadrature points (parallel.hpp:26-52). Rank r factors the
 * contiguous shift range sssvd_shard_range(h, nranks, r); the partial moment blocks are summed
 * with one ncclAllReduce. unique_id is NCCL's 128-byte ncclUniqueId made by rank 0. */
sssvd_status sssvd_gpu_nccl_unique_id(void* out128);
sssvd_status sssvd_gpu_init_comm(sssvd_gpu_ctx* ctx, const void* unique_id128, int nranks, int rank);
void sssvd_shard_range(int64_t h, int nranks, int rank, int64_t* begin, int64_t* end);
/* The lower-triangle Gram tiles (kGramTile = 64 square, csrc/partition.h) rank `part` of `nparts`
 * computes in the multi-GPU form_gram: writes up to `cap` (ti, tj) pairs into ij (tile-row, tile-col,
 * ti >= tj) and returns their count (-1 for bad arguments). Host only; the same decode as the kernel. */
int64_t sssvd_gram_tiles(int64_t n, int part, int nparts, int32_t* ij, int64_t cap);

/* ---- operator ------------------------------------------------------------------------------ *
 * ProblemMatrix::from_dense (problem.hpp:20-25 auto-transpose when rows < cols, :56-58 NaN
 * check) + upload. `a` is column-major rows x cols with leading dimension lda; on_device != 0
 * means `a` is a device pointer on the context's GPU. */
sssvd_status sssvd_gpu_set_operator(sssvd_gpu_ctx* ctx, const double* a, int64_t rows, int64_t cols,
                                    int64_t lda, int on_device);
/* Multi-GPU form of set_operator: collective over the context's communicator. Only rank `root`
 * reads `a` (host or device as on_device says; others may pass NULL); the padded operator is then
 * sent to every rank with ONE ncclBroadcast over NVLink ("A is broadcast once").
 * rows/cols must be given on every rank. Without a communicator it is set_operator. */
sssvd_status sssvd_gpu_set_operator_root(sssvd_gpu_ctx* ctx, const double* a, int64_t rows, int64_t cols,
                                         int64_t lda, int on_device, int root);
/* Number of ranks of the context's NCCL communicator (ncclCommCount); 1 without one. */
sssvd_status sssvd_gpu_comm_size(sssvd_gpu_ctx* ctx, int* nranks);
/* ProblemMatrix::from_sparse (problem.hpp:27-35) + upload: A given as compressed sparse column
 * (Eigen's SparseMatrix layout) in the user orientation, colptr[cols+1], rowind[nnz] strictly
 * increasing inside each column, values[nnz]; all three are device pointers if on_device != 0.
 * The operator is densified in HBM; wide inputs are stored transposed
 * exactly as from_sparse does. INVALID_ARGUMENT for a malformed CSC or a NaN/Inf value. */
sssvd_status sssvd_gpu_set_operator_csc(sssvd_gpu_ctx* ctx, int64_t rows, int64_t cols, int64_t nnz,
                                        const int64_t* colptr, const int64_t* rowind, const double* values,
                                        int on_device);
/* form_gram (problem.hpp:81-95) of the current operator; G_out (cols x cols, column-major) may
 * be NULL to keep G on the device only. */
sssvd_status sssvd_gpu_form_gram(sssvd_gpu_ctx* ctx, int64_t size_cap, double* g_out);

/* ---- DenseShiftedSolver / ShiftedFactorization (shifted_solver.hpp:20-75) ------------------ *
 * x = (z I - G)^{-1} rhs for one shift; G column-major n x n (symmetric), rhs/x complex
 * interleaved n x L column-major. Status NUMERICAL for the pivot floor, INVALID_ARGUMENT for a
 * dimension mismatch. */
sssvd_status sssvd_gpu_shifted_solve(sssvd_gpu_ctx* ctx, const double* g, int64_t n, double shift_re,
                                     double shift_im, const double* rhs, int64_t rhs_rows, int64_t L,
                                     double* x_out);

/* ---- MomentAccumulator (moments.hpp:101-169) ------------------------------------------------ *
 * Uses the Gram of the current operator (sssvd_gpu_form_gram must have run). Over the h
 * upper-half nodes: (ell-1) refinement passes S0 <- 2 sum_j Re(w_j X_j), then the moment pass
 * S_k = 2 sum_j Re(w_j t_j^k X_j), k = 0..M. shifts/weights/nodes are complex interleaved (2h
 * doubles each, shift_j = g(t_j)); S0 is n x L column-major; S_out receives (M+1) column-major
 * n x L blocks, block k at offset k*n*L. */
sssvd_status sssvd_gpu_moments(sssvd_gpu_ctx* ctx, int64_t h, const double* shifts, const double* weights,
                               const double* nodes, const double* s0, int64_t L, int64_t ell, int64_t M,
                               double* s_out);

/* ---- run_solve (pipeline.hpp:112-231) -------------------------------------------------------- */
sssvd_status sssvd_gpu_run_solve(sssvd_gpu_ctx* ctx, const sssvd_config* cfg, sssvd_gpu_result** out);

typedef struct {
  int64_t count;         /* candidate triplets (TripletSet::count) */
  int64_t rows, cols;    /* user orientation: left is rows x count, right cols x count */
  int64_t retained_rank; /* basis.rank() */
  int64_t n_internal;    /* operator columns after auto-transpose */
  int64_t block_size, moment_degree;
  int32_t empty, input_transposed, rank_deficient_qr;
  int64_t count_in_interval, count_nonspurious_in_interval, count_interior, count_boundary;
  int64_t calibration_index; /* -1 if none */
  double mu, spurious_threshold;
  /* StepTimings (pipeline.hpp:65-72), seconds, host wall clock around synchronised phases */
  double steps_1_2, step_3, step_4, step_5, postprocess;
  /* device-event breakdown of steps 1-2 (seconds) */
  double t_gram, t_shifted_solves, t_allreduce;
  double shifted_solve_flops; /* h_local (8n^3/3 + 8n^2 L) summed over passes, this rank */
} sssvd_result_info;

typedef enum {
  SSSVD_FIELD_SIGMA = 0,      /* double[count] ascending */
  SSSVD_FIELD_TAU = 1,        /* double[count] */
  SSSVD_FIELD_ESTIMATED = 2,  /* double[count] */
  SSSVD_FIELD_EXACT = 3,      /* double[count]  (after the orientation swap) */
  SSSVD_FIELD_GALERKIN = 4,   /* double[count]  (after the orientation swap) */
  SSSVD_FIELD_IN_INTERVAL = 5,/* int32[count] */
  SSSVD_FIELD_SPURIOUS = 6,   /* int32[count] */
  SSSVD_FIELD_LEFT = 7,       /* double[rows*count] column-major */
  SSSVD_FIELD_RIGHT = 8,      /* double[cols*count] column-major */
  SSSVD_FIELD_BASIS_SV = 9,   /* double[retained_rank] Sigma_S1 */
  SSSVD_FIELD_BLOCKS = 10,    /* double[(M+1)*n_internal*L] moment blocks, column-major */
  SSSVD_FIELD_Q = 11,         /* double[retained_rank*count] column-major */
  SSSVD_FIELD_INVALID = 12    /* int32[count] TripletSet::invalid (naive route: theta <= 0) */
} sssvd_field;

sssvd_status sssvd_result_info_get(const sssvd_gpu_result* res, sssvd_result_info* info);
sssvd_status sssvd_result_copy(const sssvd_gpu_result* res, int field, void* dst);
const char* sssvd_result_note(const sssvd_gpu_result* res);
void sssvd_result_free(sssvd_gpu_result* res);

/* ---- host-side mirrors (no GPU needed) ------------------------------------------------------ */
/* ContourRule (contour.hpp:27-62): nodes/weights complex interleaved, N entries each (slot
 * j + N/2 is the conjugate of slot j); center_radius[0..1]. */
sssvd_status sssvd_contour(double a, double b, int64_t count, double aspect, int transform,
                           double* nodes, double* weights, double* center_radius);
/* random_start (moments.hpp:84-94): n x L column-major */
sssvd_status sssvd_random_start(int64_t n, int64_t block_size, uint64_t seed, double* out);
/* SsParams::validate (moments.hpp:35-46) */
sssvd_status sssvd_validate_params(const sssvd_params* p, int64_t n);
/* Moment coefficient table c[k][j] = w_j t_j^k, k = 0..M, j < h (the reference's power chain,
 * moments.hpp:138-144), complex interleaved, row k at offset 2*k*h. */
sssvd_status sssvd_moment_coefficients(int64_t h, const double* weights, const double* nodes, int64_t M,
                                       double* coef_out);
/* Model problems (problems.hpp:50-70): A = U diag(sigma) V^T from the model-seeded libstdc++ normal
 * stream, Householder Q factors; which = 1 (sigma_i = 0.005 + 0.01 i) or 2 (10^(-10 + 0.05 i)).
 * a_out rows x cols column-major, sigma_out[cols] ascending (may be NULL). rows >= cols. */
sssvd_status sssvd_build_model(int which, int64_t rows, int64_t cols, uint64_t seed, double* a_out,
                               double* sigma_out);
/* filter_profile (filter.hpp:36-55): grid[points] and |f(sigma)| values[points] of the rational
 * filter of the quadrature rule; log_spacing != 0 for a log grid. */
sssvd_status sssvd_filter_profile(double a, double b, int64_t count, double aspect, int transform,
                                  double sigma_min, double sigma_max, int64_t points, int log_spacing,
                                  double* grid, double* values);
/* Instrumentation: number of kernels this library launched so far (process-wide), and live
 * CUDA-event timing of the dominant kernel (the DMMA trailing update) while enabled: `ms` is the
 * GEMM-busy time (union of the launch intervals; the shift groups overlap their GEMMs), `flops`
 * the EXECUTED tensor flops of those launches (6 M N K for a 3-product complex update, 8 M N K for a
 * 4-product one); collect2 also returns the same work in the conventional 8 M N K unit. */
uint64_t sssvd_gpu_launch_count(void);
void sssvd_gpu_profile_gemm(int enable);
void sssvd_gpu_profile_gemm_collect(double* ms, double* flops, uint64_t* launches);
void sssvd_gpu_profile_gemm_collect2(double* ms, double* executed_flops, double* algorithmic_flops, uint64_t* launches);
/* Debug: tile share `part` of `nparts` of form_gram (the multi-GPU Gram sharding), zeros
 * elsewhere; n x n column-major. */
sssvd_status sssvd_debug_gram_part(sssvd_gpu_ctx* ctx, int part, int nparts, double* g_out);
/* Debug: the tail's hand-written Householder QR (HouseholderQR, moments.hpp:195-198 / extract.hpp:
 * 43-57) on host data: a (m x k column-major, m >= k) -> thin q_out (m x k) and upper r_out (k x k). */
sssvd_status sssvd_debug_thin_qr(sssvd_gpu_ctx* ctx, const double* a, int64_t m, int64_t k, double* q_out,
                                 double* r_out);
/* Debug: the tail's one-sided Jacobi SVD of a square k x k matrix b (svd_small, extract.hpp:66-70):
 * u_out, v_out (k x k column-major), s_out[k] descending. */
sssvd_status sssvd_debug_svd_square(sssvd_gpu_ctx* ctx, const double* b, int64_t k, double* u_out, double* s_out,
                                    double* v_out);
/* Debug: the trailing-update GEMM (C -= A B, complex, row-major, batched; zgemm.cu) on seeded device
 * data, timed over `reps` launches -> ms_out (mean per launch). variant 0 = the cp.async kernel (the
 * product default), 1 = the TMA + mbarrier persistent kernel; mismatches_out = entries of C that
 * differ BITWISE from the cp.async kernel's result on the same inputs. */
sssvd_status sssvd_debug_zgemm(sssvd_gpu_ctx* ctx, int variant, int64_t m, int64_t n, int64_t k, int64_t batch,
                               int reps, double* ms_out, int64_t* mismatches_out);
/* Debug: the tail GEMM (dgemm.cu) on host column-major data. mode 0: c_io (m x n, ldc) <- alpha
 * op(a) b + beta c_io, op(a) = a (m x k, lda) or a^T (ta != 0: a is k x m); mode 1: c_io[j] <-
 * ||op(a) b[:, j] - d[j] v[:, j]|| (v m x n with leading dimension ldc), the fused residual form. */
sssvd_status sssvd_debug_dgemm(sssvd_gpu_ctx* ctx, int mode, int ta, int64_t m, int64_t n, int64_t k, double alpha,
                               const double* a, int64_t lda, const double* b, int64_t ldb, double beta,
                               const double* d, const double* v, double* c_io, int64_t ldc);
/* ---- Matrix Market ingest (matrix_market.hpp:34-149; host only) ---------------------------- *
 * sssvd_mm_read mirrors read_matrix_market: real/integer/double `array` (dense) and `coordinate`
 * (sparse, duplicates summed in file order, (skew-)symmetric expanded) formats; `complex` and
 * `pattern` are rejected. Data are in the FILE's orientation (the caller's ProblemMatrix applies
 * the rows >= cols normalisation): dense = rows x cols column-major values; sparse = CSC colptr /
 * rowind / values. Errors: SSSVD_E_IO (cannot open), SSSVD_E_FORMAT ("path:line: what"); the
 * message is sssvd_host_last_error(). */
typedef struct sssvd_mm_matrix sssvd_mm_matrix;
typedef struct {
  int64_t rows, cols, nnz; /* nnz = rows*cols for dense */
  int sparse;
} sssvd_mm_info;
sssvd_status sssvd_mm_read(const char* path, sssvd_mm_matrix** out);
void sssvd_mm_info_get(const sssvd_mm_matrix* mm, sssvd_mm_info* info);
const double* sssvd_mm_values(const sssvd_mm_matrix* mm);
const int64_t* sssvd_mm_colptr(const sssvd_mm_matrix* mm); /* NULL for dense */
const int64_t* sssvd_mm_rowind(const sssvd_mm_matrix* mm); /* NULL for dense */
void sssvd_mm_free(sssvd_mm_matrix* mm);
/* write_matrix_market (matrix_market.hpp:121-149), given the USER orientation: colptr == NULL
 * writes `values` (rows x cols column-major) in array format, else the CSC in coordinate format;
 * 17 significant digits; `comment` (may be NULL/empty) becomes a "% comment" line. */
sssvd_status sssvd_mm_write(const char* path, int64_t rows, int64_t cols, int64_t nnz, const int64_t* colptr,
                            const int64_t* rowind, const double* values, const char* comment);
/* Message of the last failing host-only call on this thread. */
const char* sssvd_host_last_error(void);

/* Build provenance for the loaded library ("sm_100a ..."). */
const char* sssvd_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* SSSVD_GPU_H */
