// Host-side C++ mirror of the reference's O(N) control logic: ContourRule, SpectralTransform,
// SsParams::validate, random_start and the moment power chain. These run on the host (as in
// the reference) and upload O(N) scalars; they are compiled with the same g++/libstdc++
// semantics as the reference headers so the nodes, weights, starting block and coefficient
// table are bit-identical to the reference's.
#include <cmath>
#include <complex>
#include <cstdint>
#include <numbers>
#include <random>
#include <stdexcept>
#include <vector>

#include "host_mirror.h"
#include "partition.h"
#include "../../include/sssvd_gpu.h"

namespace sssvd_gpu {

// contour.hpp:27-62
Contour make_contour(double a, double b, int64_t count, double aspect, bool exp_transform) {
  if (!(a >= 0.0) || !(a < b)) throw std::invalid_argument("ContourRule: need 0 <= a < b");
  if (count < 4 || count % 2 != 0)
    throw std::invalid_argument("ContourRule: quadrature count must be even and >= 4");
  if (!(aspect > 0.0) || aspect > 1.0)
    throw std::invalid_argument("ContourRule: aspect ratio must lie in (0,1]");
  if (exp_transform && a == 0.0)
    throw std::domain_error("ContourRule: Exp transform requires a > 0 (g^{-1}(0) diverges)");
  Contour r;
  r.exp_transform = exp_transform;
  if (!exp_transform) {
    r.center = (a * a + b * b) / 2.0;
    r.radius = (b * b - a * a) / 2.0;
  } else {
    r.center = std::log(a) + std::log(b);
    r.radius = std::log(b) - std::log(a);
  }
  const int64_t half = count / 2;
  r.nodes.resize(count);
  r.weights.resize(count);
  const double two_pi = 2.0 * std::numbers::pi_v<double>;
  for (int64_t j = 0; j < half; ++j) {
    const double theta = (two_pi / double(count)) * (double(j) + 0.5);
    const double c = std::cos(theta), s = std::sin(theta);
    const std::complex<double> t(r.center + r.radius * c, r.radius * aspect * s);
    std::complex<double> w(r.radius / double(count) * aspect * c, r.radius / double(count) * s);
    if (exp_transform) w *= std::exp(t);
    r.nodes[j] = t;
    r.weights[j] = w;
    r.nodes[j + half] = std::conj(t);
    r.weights[j + half] = std::conj(w);
  }
  return r;
}

// contour.hpp:76 + transform.hpp:26-31
std::complex<double> Contour::shift(int64_t j) const {
  return exp_transform ? std::exp(nodes[j]) : nodes[j];
}

// moments.hpp:35-46
void validate_params(const sssvd_params& p, int64_t n) {
  if (p.block_size < 1 || p.moment_degree < 1 || p.quadrature_count < 4 || p.refinement_steps < 1)
    throw std::invalid_argument("SsParams: counts must be positive (N >= 4)");
  if (p.quadrature_count % 2 != 0) throw std::invalid_argument("SsParams: quadrature count must be even");
  if (p.block_size * p.moment_degree > n)
    throw std::invalid_argument("SsParams: L*M must not exceed the column count");
  if (!(p.lowrank_threshold > 0.0) || !(p.lowrank_threshold < 1.0))
    throw std::invalid_argument("SsParams: delta must lie in (0,1)");
  if (!(p.spurious_threshold > 0.0)) throw std::invalid_argument("SsParams: epsilon must be positive");
}

// moments.hpp:84-94
std::vector<double> random_start(int64_t n, int64_t block_size, uint64_t seed) {
  if (n < block_size) throw std::invalid_argument("random_start: block size exceeds dimension");
  std::mt19937_64 gen(seed);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  std::vector<double> v((size_t)n * block_size);
  for (int64_t j = 0; j < block_size; ++j)
    for (int64_t i = 0; i < n; ++i) v[(size_t)j * n + i] = dist(gen);
  return v;
}

// moments.hpp:138-144: w = weights[j] * power[j]; power[j] *= nodes[j]  (k outer, j inner)
std::vector<std::complex<double>> moment_coefficients(const std::vector<std::complex<double>>& weights,
                                                      const std::vector<std::complex<double>>& nodes,
                                                      int64_t h, int64_t degree) {
  std::vector<std::complex<double>> coef((size_t)(degree + 1) * h);
  std::vector<std::complex<double>> power(h, std::complex<double>(1.0));
  for (int64_t k = 0; k <= degree; ++k)
    for (int64_t j = 0; j < h; ++j) {
      coef[(size_t)k * h + j] = weights[j] * power[j];
      power[j] *= nodes[j];
    }
  return coef;
}

// contiguous shard of the h upper-half nodes for one rank (ascending j within each rank)
void shard_range(int64_t h, int nranks, int rank, int64_t* begin, int64_t* end) {
  if (nranks < 1) nranks = 1;
  const int64_t base = h / nranks, rem = h % nranks;
  *begin = rank * base + std::min<int64_t>(rank, rem);
  *end = *begin + base + (rank < rem ? 1 : 0);
}

}  // namespace sssvd_gpu

using namespace sssvd_gpu;

extern "C" {

void sssvd_default_config(sssvd_config* cfg) {
  cfg->interval_a = 0.0;
  cfg->interval_b = 1.0;
  cfg->mode = SSSVD_MODE_SS_SVD;
  cfg->aspect = 0.1;
  cfg->params.block_size = 20;
  cfg->params.moment_degree = 4;
  cfg->params.quadrature_count = 32;
  cfg->params.refinement_steps = 1;
  cfg->params.lowrank_threshold = 1e-20;
  cfg->params.spurious_threshold = 1e-8;
  cfg->params.seed = 42;
  cfg->threads = 0;
  cfg->estimator_rcond_identity = 2e-15;
  cfg->estimator_rcond_exp = 1e-14;
  cfg->gram_cap = 8192;
}

sssvd_status sssvd_contour(double a, double b, int64_t count, double aspect, int transform, double* nodes,
                           double* weights, double* center_radius) {
  try {
    Contour r = make_contour(a, b, count, aspect, transform == SSSVD_TRANSFORM_EXP);
    for (int64_t j = 0; j < count; ++j) {
      if (nodes) { nodes[2 * j] = r.nodes[j].real(); nodes[2 * j + 1] = r.nodes[j].imag(); }
      if (weights) { weights[2 * j] = r.weights[j].real(); weights[2 * j + 1] = r.weights[j].imag(); }
    }
    if (center_radius) { center_radius[0] = r.center; center_radius[1] = r.radius; }
    return SSSVD_OK;
  } catch (const std::domain_error&) {
    return SSSVD_E_DOMAIN;
  } catch (const std::invalid_argument&) {
    return SSSVD_E_INVALID_ARGUMENT;
  }
}

sssvd_status sssvd_random_start(int64_t n, int64_t block_size, uint64_t seed, double* out) {
  try {
    auto v = random_start(n, block_size, seed);
    std::copy(v.begin(), v.end(), out);
    return SSSVD_OK;
  } catch (const std::invalid_argument&) {
    return SSSVD_E_INVALID_ARGUMENT;
  }
}

sssvd_status sssvd_validate_params(const sssvd_params* p, int64_t n) {
  try {
    validate_params(*p, n);
    return SSSVD_OK;
  } catch (const std::invalid_argument&) {
    return SSSVD_E_INVALID_ARGUMENT;
  }
}

sssvd_status sssvd_moment_coefficients(int64_t h, const double* weights, const double* nodes, int64_t M,
                                       double* coef_out) {
  if (h < 1 || M < 0) return SSSVD_E_INVALID_ARGUMENT;
  std::vector<std::complex<double>> w(h), t(h);
  for (int64_t j = 0; j < h; ++j) {
    w[j] = {weights[2 * j], weights[2 * j + 1]};
    t[j] = {nodes[2 * j], nodes[2 * j + 1]};
  }
  auto c = moment_coefficients(w, t, h, M);
  for (size_t i = 0; i < c.size(); ++i) { coef_out[2 * i] = c[i].real(); coef_out[2 * i + 1] = c[i].imag(); }
  return SSSVD_OK;
}

void sssvd_shard_range(int64_t h, int nranks, int rank, int64_t* begin, int64_t* end) {
  shard_range(h, nranks, rank, begin, end);
}

int64_t sssvd_gram_tiles(int64_t n, int part, int nparts, int32_t* ij, int64_t cap) {
  if (n <= 0 || nparts < 1 || part < 0 || part >= nparts) return -1;
  const long long total = sssvd_gpu::gram_tile_total(n);
  int64_t cnt = 0;
  for (long long t = part; t < total; t += nparts, ++cnt) {
    if (cnt < cap && ij) {
      int ti, tj;
      sssvd_gpu::gram_tile_decode(t, &ti, &tj);
      ij[2 * cnt] = ti;
      ij[2 * cnt + 1] = tj;
    }
  }
  return cnt;
}

}  // extern "C"
