// Compile-and-link check of the reference-side C++ binding (include/sssvd_gpu.hpp) against
// libsssvd_gpu.so. Without a GPU it exercises the host mirrors and the error mapping only.
#include <cmath>
#include <cstdio>
#include <vector>

#include "sssvd_gpu.hpp"

int main(int argc, char** argv) {
  sssvd_config cfg;
  sssvd_default_config(&cfg);
  if (cfg.params.block_size != 20 || cfg.params.quadrature_count != 32) return 1;
  std::vector<double> nodes(64), weights(64), cr(2);
  sssvd::gpu::check(sssvd_contour(0.8, 1.2, 32, 0.1, SSSVD_TRANSFORM_IDENTITY, nodes.data(), weights.data(), cr.data()), nullptr);
  if (std::fabs(cr[0] - 1.04) > 1e-15) return 2;
  try {
    sssvd::gpu::check(sssvd_contour(0.0, 1.2, 32, 0.1, SSSVD_TRANSFORM_EXP, nodes.data(), weights.data(), cr.data()), nullptr);
    return 3;
  } catch (const std::domain_error&) {
  }
  bool gpu = argc > 1;
  if (!gpu) {
    try {
      sssvd::gpu::Device d(0);
      return 4;  // no GPU expected here
    } catch (const sssvd::gpu::DeviceError&) {
    }
  }
  std::printf("abi_smoke ok\n");
  return 0;
}
