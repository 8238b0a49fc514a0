"""A/B of the tail QR on config 1: per matched triplet, GPU exact residual vs the oracle's."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from paper_2109_13655_b200 import sssvd, workloads
from oracle import sssvd_oracle as orc
a, sigma = workloads.make_operator(1)
cfg = sssvd.RunConfig(0.45, 0.55, mode=sssvd.SolveMode.SsSvdNT, params=sssvd.SsParams(block_size=16, moment_degree=8, quadrature_count=32))
res = sssvd.run_solve(a, cfg, sssvd.Device(0))
ocfg = orc.RunConfig(0.45, 0.55, mode=orc.SS_SVD_NT, params=orc.SsParams(block_size=16, moment_degree=8, quadrature_count=32))
ores = orc.run_solve(orc.ProblemMatrix(a), ocfg)
gs, os_ = res.triplets.sigma, ores.triplets.sigma
worst = []
for i in range(ores.triplets.count()):
    if not ores.triplets.in_interval[i] or ores.verdict.spurious[i]:
        continue
    j = int(np.argmin(np.abs(gs - os_[i])))
    worst.append((res.exact[j] / max(ores.residuals.exact[i], 1e-300), os_[i], res.exact[j], ores.residuals.exact[i],
                  res.tau[j] / res.spurious_threshold, ores.verdict.tau[i] / ores.verdict.threshold))
worst.sort(reverse=True)
print(os.environ.get("SSSVD_QR", "hand"), "ns", res.count_nonspurious_in_interval, ores.count_nonspurious_in_interval,
      "basis_sv_min", res.basis_singular_values.min(), "worst ratio rows (ratio, sigma, gpu_res, cpu_res, tau/thr gpu, cpu):")
for w in worst[:5]:
    print("  ", " ".join("%.3e" % x for x in w))
