// sssvd_gpu.hpp - the reference-side C++ binding over the C ABI (include/sssvd_gpu.h).
//
// This is the adapter a maintainer of the reference library (proj/include/sssvd, header-only
// C++20 on Eigen 3) adds to route its hot path to the B200. It keeps the
// reference's names, types and error behaviour:
//   * errors: status codes are rethrown as the reference's own exception types
//     (core.hpp:29-39: sssvd::NumericalError, sssvd::EmptySubspaceError; std::invalid_argument,
//     std::domain_error, std::length_error). When the reference's <sssvd/core.hpp> is on the include
//     path those ARE the reference's classes (catch (const sssvd::NumericalError&) at
//     pipeline.hpp:151 and sssvd.cpp:389 catches them); otherwise this header defines identical
//     classes under the same names;
//   * GpuMomentAccumulator has the MomentAccumulator surface (moments.hpp:101-147: refine,
//     accumulate);
//   * run_solve(ProblemMatrix, RunConfig) -> RunResult (pipeline.hpp:74-95, :112) with the
//     reference's field names. Eigen is not required: the mirror types below hold std::vector
//     column-major data (Matrix<double>::data() plugs in directly; INTEGRATION.md 2 shows the
//     Eigen::Map copy into the reference's own RunResult).
#pragma once

#include <complex>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "sssvd_gpu.h"

#if __has_include(<sssvd/core.hpp>)
#include <sssvd/core.hpp>
#define SSSVD_GPU_REFERENCE_ERRORS 1
#else
namespace sssvd {
// core.hpp:29-39, restated for builds without the reference tree (same names and hierarchy)
class NumericalError : public std::runtime_error {
 public:
  explicit NumericalError(const std::string& what) : std::runtime_error(what) {}
};
class EmptySubspaceError : public NumericalError {
 public:
  explicit EmptySubspaceError(const std::string& what) : NumericalError(what) {}
};
}  // namespace sssvd
#endif

namespace sssvd::gpu {

using NumericalError = ::sssvd::NumericalError;
using EmptySubspaceError = ::sssvd::EmptySubspaceError;
// device / NCCL failures: not part of the reference's taxonomy (no device there), a runtime_error
class DeviceError : public std::runtime_error {
 public:
  explicit DeviceError(const std::string& w) : std::runtime_error(w) {}
};
// matrix_market.hpp:17-21 ("path:line: what")
class MatrixMarketError : public std::runtime_error {
 public:
  explicit MatrixMarketError(const std::string& w) : std::runtime_error(w) {}
};

inline void check(sssvd_status st, const sssvd_gpu_ctx* ctx) {
  if (st == SSSVD_OK) return;
  const std::string msg = ctx ? sssvd_gpu_last_error(ctx) : "sssvd_gpu";
  switch (st) {
    case SSSVD_E_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case SSSVD_E_DOMAIN: throw std::domain_error(msg);
    case SSSVD_E_LENGTH: throw std::length_error(msg);
    case SSSVD_E_NUMERICAL: throw NumericalError(msg);
    case SSSVD_E_EMPTY_SUBSPACE: throw EmptySubspaceError(msg);
    case SSSVD_E_FORMAT: throw MatrixMarketError(msg);
    case SSSVD_E_IO: throw std::runtime_error(msg);
    default: throw DeviceError(msg + " (status " + std::to_string(int(st)) + ")");
  }
}

// RAII owner of one B200 context (one per process / GPU).
class Device {
 public:
  explicit Device(int device = 0) { check(sssvd_gpu_create(device, &ctx_), nullptr); }
  ~Device() { sssvd_gpu_destroy(ctx_); }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  sssvd_gpu_ctx* get() const { return ctx_; }

  // multi-GPU: rank 0 calls unique_id() and shares the 128 bytes (MPI, torch.distributed, ...)
  static std::vector<char> unique_id() {
    std::vector<char> id(128);
    check(sssvd_gpu_nccl_unique_id(id.data()), nullptr);
    return id;
  }
  void init_comm(const std::vector<char>& id, int nranks, int rank) {
    check(sssvd_gpu_init_comm(ctx_, id.data(), nranks, rank), ctx_);
  }

  // ProblemMatrix::from_dense + upload (problem.hpp:20-25): column-major rows x cols
  void set_operator(const double* a, int64_t rows, int64_t cols, int64_t lda) {
    check(sssvd_gpu_set_operator(ctx_, a, rows, cols, lda, 0), ctx_);
  }
  // collective upload: rank `root` passes `a`, the others nullptr; one ncclBroadcast
  void set_operator_root(const double* a, int64_t rows, int64_t cols, int64_t lda, int root = 0) {
    check(sssvd_gpu_set_operator_root(ctx_, a, rows, cols, lda, 0, root), ctx_);
  }
  // ProblemMatrix::from_sparse + upload (problem.hpp:27-35): compressed CSC, user orientation
  void set_operator_csc(int64_t rows, int64_t cols, const int64_t* colptr, const int64_t* rowind,
                        const double* values, int64_t nnz) {
    check(sssvd_gpu_set_operator_csc(ctx_, rows, cols, nnz, colptr, rowind, values, 0), ctx_);
  }
  // form_gram (problem.hpp:81-95); g_out may be nullptr
  void form_gram(int64_t cap = 8192, double* g_out = nullptr) {
    check(sssvd_gpu_form_gram(ctx_, cap, g_out), ctx_);
  }

 private:
  sssvd_gpu_ctx* ctx_ = nullptr;
};

// Drop-in for MomentAccumulator<double, DenseShiftedSolver<double>> (moments.hpp:101-169),
// constructed from the reference's ContourRule data (nodes, weights, shifts of the h upper-half
// points). Operates on the Gram resident on `dev` (Device::form_gram).
class GpuMomentAccumulator {
 public:
  GpuMomentAccumulator(Device& dev, const std::vector<std::complex<double>>& shifts,
                       const std::vector<std::complex<double>>& weights,
                       const std::vector<std::complex<double>>& nodes)
      : dev_(dev), shifts_(shifts), weights_(weights), nodes_(nodes) {}

  // refine (moments.hpp:121-128): out = 2 sum_j Re(w_j X_j), n x L column-major
  void refine(const double* s0, int64_t n, int64_t L, double* out) const {
    run(s0, n, L, 1, 0, out);
  }
  // accumulate (moments.hpp:132-147): out holds (degree+1) column-major n x L blocks
  void accumulate(const double* s0, int64_t n, int64_t L, int64_t degree, double* out) const {
    run(s0, n, L, 1, degree, out);
  }

 private:
  void run(const double* s0, int64_t, int64_t L, int64_t ell, int64_t degree, double* out) const {
    const int64_t h = static_cast<int64_t>(shifts_.size());
    check(sssvd_gpu_moments(dev_.get(), h, reinterpret_cast<const double*>(shifts_.data()),
                            reinterpret_cast<const double*>(weights_.data()),
                            reinterpret_cast<const double*>(nodes_.data()), s0, L, ell, degree, out),
          dev_.get());
  }
  Device& dev_;
  std::vector<std::complex<double>> shifts_, weights_, nodes_;
};

// ---- the reference's parameter / result contract, Eigen-free (pipeline.hpp:43-95) -----------
enum class SolveMode { SsSvd = SSSVD_MODE_SS_SVD, SsSvdNT = SSSVD_MODE_SS_SVD_NT, Naive = SSSVD_MODE_NAIVE,
                       NaiveNT = SSSVD_MODE_NAIVE_NT };

struct SsParams {   // moments.hpp:23-47 (defaults from sssvd_default_config)
  int64_t block_size = 20, moment_degree = 4, quadrature_count = 32, refinement_steps = 1;
  double lowrank_threshold = 1e-20, spurious_threshold = 1e-8;
  uint64_t seed = 42;
};

struct RunConfig {   // pipeline.hpp:43-58
  double interval_a = 0.0, interval_b = 1.0;
  SolveMode mode = SolveMode::SsSvd;
  double aspect = 0.1;
  SsParams params;
  int threads = 0;
  double estimator_rcond_identity = 2e-15, estimator_rcond_exp = 1e-14;
  int64_t gram_cap = 8192;   // problem.hpp:82 (BASELINE config 5 lifts it)

  sssvd_config to_c() const {
    sssvd_config c;
    sssvd_default_config(&c);
    c.interval_a = interval_a;
    c.interval_b = interval_b;
    c.mode = static_cast<int32_t>(mode);
    c.aspect = aspect;
    c.params.block_size = params.block_size;
    c.params.moment_degree = params.moment_degree;
    c.params.quadrature_count = params.quadrature_count;
    c.params.refinement_steps = params.refinement_steps;
    c.params.lowrank_threshold = params.lowrank_threshold;
    c.params.spurious_threshold = params.spurious_threshold;
    c.params.seed = params.seed;
    c.threads = threads;
    c.estimator_rcond_identity = estimator_rcond_identity;
    c.estimator_rcond_exp = estimator_rcond_exp;
    c.gram_cap = gram_cap;
    return c;
  }
};

// ProblemMatrix (problem.hpp:14-60) in the user orientation: dense column-major, or compressed CSC
struct ProblemMatrix {
  int64_t rows = 0, cols = 0;
  std::vector<double> dense;                 // rows x cols column-major (dense form)
  std::vector<int64_t> colptr, rowind;       // CSC (sparse form), values in `values`
  std::vector<double> values;
  bool sparse() const { return !colptr.empty(); }
  static ProblemMatrix from_dense(const double* a, int64_t rows, int64_t cols) {
    ProblemMatrix p;
    p.rows = rows;
    p.cols = cols;
    p.dense.assign(a, a + rows * cols);
    return p;
  }
};

struct TripletSet {   // extract.hpp:21-31, user orientation
  std::vector<double> sigma;
  std::vector<double> left, right, q;   // rows x t, cols x t, r x t column-major
  std::vector<bool> in_interval, invalid;
  int64_t count() const { return static_cast<int64_t>(sigma.size()); }
};
struct SpuriousVerdict {   // postprocess.hpp:47-62
  std::vector<double> tau;
  double threshold = 0;
  std::vector<bool> spurious;
};
struct ResidualReport {   // postprocess.hpp:100-156
  std::vector<double> estimated, exact;
  int64_t calibration_index = -1;   // std::optional in the reference: -1 = none
  double mu = 0;
};
struct StepTimings {   // pipeline.hpp:65-72
  double steps_1_2 = 0, step_3 = 0, step_4 = 0, step_5 = 0, postprocess = 0;
  double total() const { return steps_1_2 + step_3 + step_4 + step_5; }
};
struct RunResult {   // pipeline.hpp:74-95
  TripletSet triplets;
  SpuriousVerdict verdict;
  ResidualReport residuals;
  std::vector<double> galerkin;
  std::vector<double> basis_singular_values;   // ReducedBasis::singular_values (Sigma_S1)
  std::vector<double> blocks;                  // MomentBlocks: (M+1) column-major n x L blocks
  bool rank_deficient_qr = false;
  StepTimings timings;
  bool empty = false;
  std::string note;
  bool input_transposed = false;
  int64_t count_in_interval = 0, count_nonspurious_in_interval = 0, count_interior = 0, count_boundary = 0;
  int64_t retained_rank_ = 0;
  int64_t retained_rank() const { return retained_rank_; }
};

// the raw result handle (sssvd_result_copy reads the fields; see sssvd_gpu.h for the layouts)
class Result {
 public:
  explicit Result(sssvd_gpu_result* r) : r_(r) { sssvd_result_info_get(r_, &info_); }
  ~Result() { sssvd_result_free(r_); }
  Result(const Result&) = delete;
  Result& operator=(const Result&) = delete;
  const sssvd_result_info& info() const { return info_; }
  std::vector<double> field(sssvd_field f, size_t count) const {
    std::vector<double> out(count);
    if (count) check(sssvd_result_copy(r_, f, out.data()), nullptr);
    return out;
  }
  std::vector<bool> flags(sssvd_field f, size_t count) const {
    std::vector<int32_t> raw(count);
    if (count) check(sssvd_result_copy(r_, f, raw.data()), nullptr);
    return std::vector<bool>(raw.begin(), raw.end());
  }
  std::string note() const { return sssvd_result_note(r_); }
  sssvd_gpu_result* raw() const { return r_; }

  RunResult to_run_result() const {
    const auto& i = info_;
    RunResult out;
    const size_t t = static_cast<size_t>(i.count);
    out.triplets.sigma = field(SSSVD_FIELD_SIGMA, t);
    out.triplets.left = field(SSSVD_FIELD_LEFT, static_cast<size_t>(i.rows) * t);
    out.triplets.right = field(SSSVD_FIELD_RIGHT, static_cast<size_t>(i.cols) * t);
    out.triplets.q = field(SSSVD_FIELD_Q, static_cast<size_t>(i.retained_rank) * t);
    out.triplets.in_interval = flags(SSSVD_FIELD_IN_INTERVAL, t);
    out.triplets.invalid = flags(SSSVD_FIELD_INVALID, t);
    out.verdict.tau = field(SSSVD_FIELD_TAU, t);
    out.verdict.threshold = i.spurious_threshold;
    out.verdict.spurious = flags(SSSVD_FIELD_SPURIOUS, t);
    out.residuals.estimated = field(SSSVD_FIELD_ESTIMATED, t);
    out.residuals.exact = field(SSSVD_FIELD_EXACT, t);
    out.residuals.calibration_index = i.calibration_index;
    out.residuals.mu = i.mu;
    out.galerkin = field(SSSVD_FIELD_GALERKIN, t);
    out.basis_singular_values = field(SSSVD_FIELD_BASIS_SV, static_cast<size_t>(i.retained_rank));
    out.blocks = field(SSSVD_FIELD_BLOCKS, static_cast<size_t>((i.moment_degree + 1) * i.n_internal * i.block_size));
    out.rank_deficient_qr = i.rank_deficient_qr != 0;
    out.timings = {i.steps_1_2, i.step_3, i.step_4, i.step_5, i.postprocess};
    out.empty = i.empty != 0;
    out.note = note();
    out.input_transposed = i.input_transposed != 0;
    out.count_in_interval = i.count_in_interval;
    out.count_nonspurious_in_interval = i.count_nonspurious_in_interval;
    out.count_interior = i.count_interior;
    out.count_boundary = i.count_boundary;
    out.retained_rank_ = i.retained_rank;
    return out;
  }

 private:
  sssvd_gpu_result* r_;
  sssvd_result_info info_{};
};

// Host-only calls report through sssvd_host_last_error().
inline void check_host(sssvd_status st) {
  if (st == SSSVD_OK) return;
  const std::string msg = sssvd_host_last_error();
  switch (st) {
    case SSSVD_E_FORMAT: throw MatrixMarketError(msg);
    case SSSVD_E_IO: throw std::runtime_error(msg);
    case SSSVD_E_DOMAIN: throw std::domain_error(msg);
    default: throw std::invalid_argument(msg);
  }
}

// read_matrix_market (matrix_market.hpp:34-119) in the file's orientation: dense column-major
// `values` (colptr/rowind empty) or compressed CSC.
struct MarketMatrix {
  int64_t rows = 0, cols = 0;
  bool sparse = false;
  std::vector<double> values;
  std::vector<int64_t> colptr, rowind;
};

inline MarketMatrix read_matrix_market(const std::string& path) {
  sssvd_mm_matrix* h = nullptr;
  check_host(sssvd_mm_read(path.c_str(), &h));
  sssvd_mm_info info{};
  sssvd_mm_info_get(h, &info);
  MarketMatrix m;
  m.rows = info.rows;
  m.cols = info.cols;
  m.sparse = info.sparse != 0;
  m.values.assign(sssvd_mm_values(h), sssvd_mm_values(h) + info.nnz);
  if (m.sparse) {
    m.colptr.assign(sssvd_mm_colptr(h), sssvd_mm_colptr(h) + info.cols + 1);
    m.rowind.assign(sssvd_mm_rowind(h), sssvd_mm_rowind(h) + info.nnz);
  }
  sssvd_mm_free(h);
  return m;
}

inline void write_matrix_market(const std::string& path, const MarketMatrix& m, const std::string& comment = {}) {
  check_host(sssvd_mm_write(path.c_str(), m.rows, m.cols, (int64_t)m.values.size(),
                            m.sparse ? m.colptr.data() : nullptr, m.sparse ? m.rowind.data() : nullptr,
                            m.values.data(), comment.c_str()));
}

// run_solve on the operator already uploaded to `dev` (raw handle)
inline Result run_solve(Device& dev, const sssvd_config& cfg) {
  sssvd_gpu_result* r = nullptr;
  check(sssvd_gpu_run_solve(dev.get(), &cfg, &r), dev.get());
  return Result(r);
}

// run_solve(ProblemMatrix, RunConfig) -> RunResult (pipeline.hpp:112): upload + solve + results.
// EmptySubspaceError / an all-annihilated filter come back as RunResult::empty with the note, as
// in the reference (pipeline.hpp:142-156); NumericalError propagates (pipeline.hpp:151).
inline RunResult run_solve(Device& dev, const ProblemMatrix& a, const RunConfig& config) {
  if (a.sparse())
    dev.set_operator_csc(a.rows, a.cols, a.colptr.data(), a.rowind.data(), a.values.data(),
                         static_cast<int64_t>(a.values.size()));
  else
    dev.set_operator(a.dense.data(), a.rows, a.cols, a.rows);
  return run_solve(dev, config.to_c()).to_run_result();
}

}  // namespace sssvd::gpu
