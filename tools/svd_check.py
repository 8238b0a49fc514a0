"""Check the hand-written Jacobi SVD inside run_solve against LAPACK on the same tail inputs."""
import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2109_13655_b200 import sssvd, workloads
for c in [int(x) for x in sys.argv[1:]]:
    w = workloads.CONFIGS[c]
    a, sigma = workloads.make_operator(c)
    dev = sssvd.Device(0)
    for mode in w.modes:
        cfg = sssvd.RunConfig(w.a, w.b, mode=mode, params=sssvd.SsParams(block_size=w.L, moment_degree=w.M, quadrature_count=w.N), gram_cap=1 << 30)
        r = sssvd.run_solve(a, cfg, dev); r = sssvd.run_solve(a, cfg, dev)
        S = r.blocks.stacked()
        q, R = np.linalg.qr(S)
        sv = np.linalg.svd(R, compute_uv=False)
        g = r.basis_singular_values
        print(json.dumps({"cfg": c, "mode": mode, "step3_ms": r.timings.step_3 * 1e3, "step5_ms": r.timings.step_5 * 1e3,
                          "ns": r.count_nonspurious_in_interval, "in": r.count_in_interval,
                          "sv_rel_err_top": float(np.max(np.abs(g[:64] - sv[:64]) / sv[:64])),
                          "sv_min_gpu": float(g.min()), "sv_min_lapack": float(sv.min())}), flush=True)
