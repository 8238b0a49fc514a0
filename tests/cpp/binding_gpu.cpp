// GPU check of the reference-side C++ binding (include/sssvd_gpu.hpp), driven by
// tests/test_gpu_binding.py: GpuMomentAccumulator::accumulate and run_solve(ProblemMatrix,
// RunConfig) -> RunResult on a seeded operator, plus the reference's error behaviour (a shift on
// the spectrum throws sssvd::NumericalError; an interval without spectrum returns empty).
//   binding_gpu in.bin out.bin
//   in : int64 rows, cols; double a, b; int64 L, M, N; rows*cols doubles (column-major A)
//   out: int64 nb; nb doubles (moment blocks); int64 t; t doubles each of sigma, tau, spurious,
//        exact, galerkin; int64 count_in_interval, count_nonspurious, retained_rank, empty(far),
//        numerical_error_caught
#include <complex>
#include <cstdio>
#include <vector>

#include "sssvd_gpu.hpp"

namespace g = sssvd::gpu;

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  FILE* f = std::fopen(argv[1], "rb");
  if (!f) return 2;
  int64_t rows, cols, L, M, N;
  double a, b;
  std::fread(&rows, 8, 1, f);
  std::fread(&cols, 8, 1, f);
  std::fread(&a, 8, 1, f);
  std::fread(&b, 8, 1, f);
  std::fread(&L, 8, 1, f);
  std::fread(&M, 8, 1, f);
  std::fread(&N, 8, 1, f);
  std::vector<double> A(rows * cols);
  if (std::fread(A.data(), 8, A.size(), f) != A.size()) return 2;
  std::fclose(f);
  const int64_t n = std::min(rows, cols), h = N / 2;

  g::Device dev(0);
  // MomentAccumulator path (moments.hpp:101-147) on the uploaded operator's Gram
  dev.set_operator(A.data(), rows, cols, rows);
  dev.form_gram(1 << 30);
  std::vector<double> nodes(2 * N), weights(2 * N), cr(2), v0(n * L);
  g::check(sssvd_contour(a, b, N, 0.1, SSSVD_TRANSFORM_IDENTITY, nodes.data(), weights.data(), cr.data()), nullptr);
  g::check(sssvd_random_start(n, L, 42, v0.data()), nullptr);
  std::vector<std::complex<double>> z(h), w(h), t(h);
  for (int64_t j = 0; j < h; ++j) {
    t[j] = {nodes[2 * j], nodes[2 * j + 1]};
    w[j] = {weights[2 * j], weights[2 * j + 1]};
    z[j] = t[j];   // identity transform: shift = node (transform.hpp:26-31)
  }
  g::GpuMomentAccumulator acc(dev, z, w, t);
  std::vector<double> blocks((M + 1) * n * L);
  acc.accumulate(v0.data(), n, L, M, blocks.data());

  // run_solve(ProblemMatrix, RunConfig) -> RunResult (pipeline.hpp:112)
  g::RunConfig cfg;
  cfg.interval_a = a;
  cfg.interval_b = b;
  cfg.params.block_size = L;
  cfg.params.moment_degree = M;
  cfg.params.quadrature_count = N;
  const g::ProblemMatrix pm = g::ProblemMatrix::from_dense(A.data(), rows, cols);
  const g::RunResult res = g::run_solve(dev, pm, cfg);

  // an interval without spectrum: the filter annihilates the block -> empty (pipeline.hpp:142-156)
  g::RunConfig far = cfg;
  far.interval_a = 5.0;
  far.interval_b = 6.0;
  const g::RunResult empty = g::run_solve(dev, pm, far);

  // a shift exactly on the spectrum: ShiftedFactorization throws sssvd::NumericalError
  // (shifted_solver.hpp:29-30); A = diag(1..8) so G = diag(1, 4, ..); z = 4 is an eigenvalue
  int64_t caught = 0;
  {
    std::vector<double> D(64, 0.0);
    for (int i = 0; i < 8; ++i) D[i * 8 + i] = i + 1.0;
    dev.set_operator(D.data(), 8, 8, 8);
    dev.form_gram();
    std::vector<std::complex<double>> zs = {{4.0, 0.0}}, ws = {{1.0, 0.0}}, ts = {{4.0, 0.0}};
    g::GpuMomentAccumulator bad(dev, zs, ws, ts);
    std::vector<double> s0(8, 1.0), out(8);
    try {
      bad.refine(s0.data(), 8, 1, out.data());
    } catch (const sssvd::NumericalError& e) {
      caught = 1;
    }
  }

  FILE* o = std::fopen(argv[2], "wb");
  const int64_t nb = (int64_t)blocks.size(), tc = res.triplets.count();
  std::fwrite(&nb, 8, 1, o);
  std::fwrite(blocks.data(), 8, nb, o);
  std::fwrite(&tc, 8, 1, o);
  std::fwrite(res.triplets.sigma.data(), 8, tc, o);
  std::fwrite(res.verdict.tau.data(), 8, tc, o);
  for (int64_t i = 0; i < tc; ++i) {
    const double s = res.verdict.spurious[i] ? 1.0 : 0.0;
    std::fwrite(&s, 8, 1, o);
  }
  std::fwrite(res.residuals.exact.data(), 8, tc, o);
  std::fwrite(res.galerkin.data(), 8, tc, o);
  const int64_t tail[5] = {res.count_in_interval, res.count_nonspurious_in_interval, res.retained_rank(),
                           empty.empty ? 1 : 0, caught};
  std::fwrite(tail, 8, 5, o);
  std::fclose(o);
  std::printf("binding_gpu ok: %lld triplets, %lld non-spurious in interval\n", (long long)tc,
              (long long)res.count_nonspurious_in_interval);
  return 0;
}
