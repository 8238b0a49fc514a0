// Host-side generators behind the CLI (no GPU): the model problems and the filter profile.
//
//   build_model    problems.hpp:50-70 - the same libstdc++ normal stream (mt19937_64 seeded with
//                  the model seed, column-major U draws then V draws), Householder QR of each
//                  Gaussian block (LAPACK/Eigen sign convention beta = -sign(alpha)||x||, no sign
//                  fix), A = U diag(sigma) V^T. The QR and the product are this file's own loops,
//                  so A matches the reference to rounding and sigma (the truth) exactly.
//   filter_profile filter.hpp:19-55 - |f(sigma)| = |2 Re sum_j w_j / (g(t_j) - sigma^2)| on a
//                  linear or log grid.
#include <cmath>
#include <complex>
#include <cstdint>
#include <random>
#include <stdexcept>
#include <vector>

#include "host_mirror.h"

namespace sssvd_gpu {

namespace {

// In-place Householder QR of the m x n column-major block `a` (m >= n); on return `a` holds the
// explicit thin Q (m x n). Unblocked: the generator sizes are small (the CLI's default 1000 x 200).
void householder_thin_q(std::vector<double>& a, int64_t m, int64_t n) {
  std::vector<double> tau(n, 0.0);
  auto col = [&](int64_t j) { return a.data() + (size_t)j * m; };
  for (int64_t k = 0; k < n; ++k) {
    double* x = col(k) + k;
    const int64_t len = m - k;
    double tail = 0.0;
    for (int64_t i = 1; i < len; ++i) tail += x[i] * x[i];
    const double alpha = x[0];
    if (tail == 0.0) {            // already upper triangular in this column: H = I
      tau[k] = 0.0;
      continue;
    }
    double beta = std::sqrt(alpha * alpha + tail);
    if (alpha >= 0.0) beta = -beta;
    const double scale = 1.0 / (alpha - beta);
    for (int64_t i = 1; i < len; ++i) x[i] *= scale;
    tau[k] = (beta - alpha) / beta;
    x[0] = beta;
    // apply H_k = I - tau v v^T (v = [1; x[1:]]) to the trailing columns
    for (int64_t j = k + 1; j < n; ++j) {
      double* y = col(j) + k;
      double d = y[0];
      for (int64_t i = 1; i < len; ++i) d += x[i] * y[i];
      d *= tau[k];
      y[0] -= d;
      for (int64_t i = 1; i < len; ++i) y[i] -= d * x[i];
    }
  }
  // backward accumulation Q = H_0 ... H_{n-1} I[:, :n], reusing the reflector storage
  std::vector<double> v(m);
  for (int64_t k = n - 1; k >= 0; --k) {
    double* x = col(k) + k;
    const int64_t len = m - k;
    v[0] = 1.0;
    for (int64_t i = 1; i < len; ++i) v[i] = x[i];
    // column k of Q starts as e_k; columns j > k already hold H_{k+1..} e_j (zero in row k)
    for (int64_t i = 0; i < len; ++i) x[i] = (i == 0 ? 1.0 : 0.0) - tau[k] * v[i];
    for (int64_t j = k + 1; j < n; ++j) {
      double* y = col(j) + k;
      double d = 0.0;
      for (int64_t i = 0; i < len; ++i) d += v[i] * y[i];
      d *= tau[k];
      for (int64_t i = 0; i < len; ++i) y[i] -= d * v[i];
    }
    for (int64_t i = 0; i < k; ++i) col(k)[i] = 0.0;
  }
}

}  // namespace

// problems.hpp:38-48
std::vector<double> model_spectrum(int which, int64_t n) {
  std::vector<double> s(n);
  for (int64_t i = 0; i < n; ++i)
    s[i] = which == 1 ? 0.005 + 0.01 * double(i) : std::pow(10.0, -10.0 + 0.05 * double(i));
  return s;
}

void build_model(int which, int64_t rows, int64_t cols, uint64_t seed, double* a_out, double* sigma_out) {
  if (which != 1 && which != 2) throw std::invalid_argument("build_model: model must be 1 or 2");
  if (cols < 1 || rows < cols) throw std::invalid_argument("build_model: needs rows >= cols");
  std::mt19937_64 gen(seed);
  std::normal_distribution<double> dist(0.0, 1.0);
  std::vector<double> u((size_t)rows * cols), v((size_t)cols * cols);
  for (auto& x : u) x = dist(gen);   // column-major, the reference's (j outer, i inner) order
  for (auto& x : v) x = dist(gen);
  householder_thin_q(u, rows, cols);
  householder_thin_q(v, cols, cols);
  const std::vector<double> s = model_spectrum(which, cols);
  // A = (U diag(s)) V^T, column by column
  for (int64_t j = 0; j < cols; ++j) {
    double* aj = a_out + (size_t)j * rows;
    for (int64_t i = 0; i < rows; ++i) aj[i] = 0.0;
    for (int64_t k = 0; k < cols; ++k) {
      const double c = s[k] * v[(size_t)k * cols + j];
      const double* uk = u.data() + (size_t)k * rows;
      for (int64_t i = 0; i < rows; ++i) aj[i] += uk[i] * c;
    }
  }
  if (sigma_out)
    for (int64_t k = 0; k < cols; ++k) sigma_out[k] = s[k];
}

// filter.hpp:19-28
double eval_filter_abs(const Contour& rule, double sigma) {
  const std::complex<double> s2(sigma * sigma, 0.0);
  std::complex<double> half_sum(0.0);
  const int64_t half = rule.count() / 2;
  for (int64_t j = 0; j < half; ++j) half_sum += rule.weights[j] / (rule.shift(j) - s2);
  return std::abs(std::complex<double>(2.0 * half_sum.real(), 0.0));
}

}  // namespace sssvd_gpu

using namespace sssvd_gpu;

extern "C" {

sssvd_status sssvd_build_model(int which, int64_t rows, int64_t cols, uint64_t seed, double* a_out,
                               double* sigma_out) {
  try {
    if (!a_out) return SSSVD_E_INVALID_ARGUMENT;
    build_model(which, rows, cols, seed, a_out, sigma_out);
    return SSSVD_OK;
  } catch (const std::invalid_argument&) {
    return SSSVD_E_INVALID_ARGUMENT;
  } catch (const std::bad_alloc&) {
    return SSSVD_E_OOM;
  }
}

// filter.hpp:36-55
sssvd_status sssvd_filter_profile(double a, double b, int64_t count, double aspect, int transform, double sigma_min,
                                  double sigma_max, int64_t points, int log_spacing, double* grid, double* values) {
  try {
    const Contour rule = make_contour(a, b, count, aspect, transform == SSSVD_TRANSFORM_EXP);
    if (!(sigma_min > 0.0) || !(sigma_min < sigma_max))
      throw std::invalid_argument("filter_profile: need 0 < sigma_min < sigma_max");
    if (points < 1) throw std::invalid_argument("filter_profile: need at least one point");
    for (int64_t i = 0; i < points; ++i) {
      const double frac = points == 1 ? 0.0 : double(i) / double(points - 1);
      const double sigma =
          log_spacing ? std::exp(std::log(sigma_min) + frac * (std::log(sigma_max) - std::log(sigma_min)))
                      : sigma_min + frac * (sigma_max - sigma_min);
      grid[i] = sigma;
      values[i] = eval_filter_abs(rule, sigma);
    }
    return SSSVD_OK;
  } catch (const std::domain_error&) {
    return SSSVD_E_DOMAIN;
  } catch (const std::invalid_argument&) {
    return SSSVD_E_INVALID_ARGUMENT;
  }
}

}  // extern "C"
