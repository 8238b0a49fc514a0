"""Run one BASELINE config end to end on the GPU and check size-independent properties:
moment identity on a column sample (S_{k+1} = G S_k for the identity transform), exact residuals
of the non-spurious triplets, and their sigma against the constructed truth."""
import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2109_13655_b200 import sssvd, workloads
c = int(sys.argv[1]); modes = [int(x) for x in sys.argv[2:]] or None
w = workloads.CONFIGS[c]
t0 = time.time(); a, sigma = workloads.make_operator(c); tg = time.time() - t0
dev = sssvd.Device(0)
for mode in (modes or w.modes):
    cfg = sssvd.RunConfig(w.a, w.b, mode=mode, params=sssvd.SsParams(block_size=w.L, moment_degree=w.M, quadrature_count=w.N), gram_cap=1 << 30)
    t0 = time.time(); r = sssvd.run_solve(a, cfg, dev); wall = time.time() - t0
    out = {"cfg": c, "mode": mode, "wall_s": wall, "gen_s": tg, "timings": r.timings.__dict__, **r.device_times,
           "solve_tflops": r.device_times["shifted_solve_flops"] / r.device_times["shifted_solves_s"] / 1e12,
           "rank": r.retained_rank(), "ns": r.count_nonspurious_in_interval, "in": r.count_in_interval,
           "boundary": r.count_boundary, "truth_in": int(np.sum((sigma >= w.a) & (sigma <= w.b)))}
    if mode == 0:
        # moment identity on 8 sampled columns: S_{k+1} = (A^T A) S_k
        cols = np.linspace(0, w.L - 1, 8).astype(int)
        errs = []
        for k in (0, w.M // 2, w.M - 1):
            sk, sk1 = r.blocks.blocks[k][:, cols], r.blocks.blocks[k + 1][:, cols]
            gs = a.T @ (a @ sk)
            errs.append(float(np.linalg.norm(sk1 - gs) / np.linalg.norm(gs)))
        out["moment_identity_relerr"] = errs
    ns = [i for i in range(r.triplets.count()) if r.triplets.in_interval[i] and not r.spurious[i]]
    if ns:
        s = r.triplets.sigma[ns]
        out["max_rel_err_vs_truth"] = float(max(np.min(np.abs(sigma - x) / sigma) for x in s))
        out["max_exact_residual"] = float(np.max(r.exact[ns]))
        out["max_galerkin"] = float(np.max(r.galerkin[ns]))
    print(json.dumps(out), flush=True)
