// Work partition of the multi-GPU path, shared by the device kernels and the host mirror (so the
// gloo tests drive exactly the decode the GPU uses).
//   * quadrature points: contiguous shift ranges per rank (sssvd_shard_range, host_mirror.cpp);
//   * form_gram: the lower-triangle tiles t = 0 .. T(T+1)/2 - 1 of G (T = ceil(n / kGramTile)),
//     row-major over (ti >= tj); rank r of G computes t = r, r + G, r + 2G, ... and one all-reduce
//     assembles G (every entry has exactly one writer, so the sum is exact).
#pragma once

#ifdef __CUDACC__
#define SSSVD_HD __host__ __device__
#else
#define SSSVD_HD
#endif
#include <cmath>

namespace sssvd_gpu {

constexpr int kGramTile = 64;

SSSVD_HD inline long long gram_tile_total(long long n) {
  const long long T = (n + kGramTile - 1) / kGramTile;
  return T * (T + 1) / 2;
}

// linear lower-triangle tile index -> (ti, tj), ti >= tj
SSSVD_HD inline void gram_tile_decode(long long t, int* ti_out, int* tj_out) {
  int ti = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while ((long long)(ti + 1) * (ti + 2) / 2 <= t) ++ti;
  while ((long long)ti * (ti + 1) / 2 > t) --ti;
  *ti_out = ti;
  *tj_out = (int)(t - (long long)ti * (ti + 1) / 2);
}

}  // namespace sssvd_gpu
