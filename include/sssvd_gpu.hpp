// sssvd_gpu.hpp - the reference-side C++ binding over the C ABI (include/sssvd_gpu.h).
//
// This is the adapter a maintainer of the reference library (proj/include/sssvd, header-only
// C++20 on Eigen 3) adds to route its hot path to the B200. It keeps the reference's types and
// error behaviour: status codes are rethrown as the reference's exceptions (core.hpp:29-39,
// std::invalid_argument / std::domain_error / std::length_error), and the accumulator has the
// MomentAccumulator surface (moments.hpp:101-147: refine, accumulate). Eigen is not required:
// every call takes plain column-major pointers, so Matrix<double>::data() plugs in directly.
#pragma once

#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "sssvd_gpu.h"

namespace sssvd::gpu {

// Same names as the reference's error taxonomy (core.hpp:29-39).
class NumericalError : public std::runtime_error {
 public:
  explicit NumericalError(const std::string& w) : std::runtime_error(w) {}
};
class EmptySubspaceError : public NumericalError {
 public:
  explicit EmptySubspaceError(const std::string& w) : NumericalError(w) {}
};
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

// run_solve (pipeline.hpp:112-231) returning the raw result handle; copy fields with
// sssvd_result_copy (see sssvd_gpu.h for the layout of each field).
class Result {
 public:
  explicit Result(sssvd_gpu_result* r) : r_(r) { sssvd_result_info_get(r_, &info_); }
  ~Result() { sssvd_result_free(r_); }
  Result(const Result&) = delete;
  Result& operator=(const Result&) = delete;
  const sssvd_result_info& info() const { return info_; }
  std::vector<double> field(sssvd_field f, size_t count) const {
    std::vector<double> out(count);
    check(sssvd_result_copy(r_, f, out.data()), nullptr);
    return out;
  }
  std::string note() const { return sssvd_result_note(r_); }
  sssvd_gpu_result* raw() const { return r_; }

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

inline Result run_solve(Device& dev, const sssvd_config& cfg) {
  sssvd_gpu_result* r = nullptr;
  check(sssvd_gpu_run_solve(dev.get(), &cfg, &r), dev.get());
  return Result(r);
}

}  // namespace sssvd::gpu
