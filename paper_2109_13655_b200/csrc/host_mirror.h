// Host-side mirror of the reference's contour / params / PRNG logic (host_mirror.cpp).
#pragma once
#include <complex>
#include <cstdint>
#include <vector>

#include "../../include/sssvd_gpu.h"

namespace sssvd_gpu {

struct Contour {
  bool exp_transform = false;
  double center = 0, radius = 0;
  std::vector<std::complex<double>> nodes, weights;
  std::complex<double> shift(int64_t j) const;
  int64_t count() const { return (int64_t)nodes.size(); }
};

Contour make_contour(double a, double b, int64_t count, double aspect, bool exp_transform);
void validate_params(const sssvd_params& p, int64_t n);
std::vector<double> random_start(int64_t n, int64_t block_size, uint64_t seed);
std::vector<std::complex<double>> moment_coefficients(const std::vector<std::complex<double>>& weights,
                                                      const std::vector<std::complex<double>>& nodes,
                                                      int64_t h, int64_t degree);
void shard_range(int64_t h, int nranks, int rank, int64_t* begin, int64_t* end);

}  // namespace sssvd_gpu
