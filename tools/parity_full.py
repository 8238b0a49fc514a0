"""Full-size GPU-vs-oracle parity for one BASELINE config, same seeded input.
Writes gpurun_out/parity_cfg<c>_mode<m>.json with the robust matching of
tests/test_gpu_pipeline.py::compare_with_oracle (firm triplets, endpoint and tau-borderline
slack) plus raw counts."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2109_13655_b200 import sssvd, workloads
from oracle import sssvd_oracle as orc

DELTA = float(os.environ.get('PARITY_DELTA', '1e-20'))   # diagnostic: delta (moments.hpp:27) on both sides
c = int(sys.argv[1]); modes = [int(x) for x in sys.argv[2:]] or list(workloads.CONFIGS[c].modes)
w = workloads.CONFIGS[c]
a, sigma = workloads.make_operator(c)
dev = sssvd.Device(0)
for mode in modes:
    cfg = sssvd.RunConfig(w.a, w.b, mode=mode, params=sssvd.SsParams(block_size=w.L, moment_degree=w.M, quadrature_count=w.N, lowrank_threshold=DELTA), gram_cap=1 << 30)
    t0 = time.time(); g = sssvd.run_solve(a, cfg, dev); tg = time.time() - t0
    ocfg = orc.RunConfig(w.a, w.b, mode=[orc.SS_SVD, orc.SS_SVD_NT][mode], params=orc.SsParams(block_size=w.L, moment_degree=w.M, quadrature_count=w.N, lowrank_threshold=DELTA))
    t0 = time.time(); o = orc.run_solve(orc.ProblemMatrix(a), ocfg, gram_cap=1 << 30); to = time.time() - t0
    blk = max(float(np.linalg.norm(g.blocks.blocks[k] - o.blocks.blocks[k]) / np.linalg.norm(o.blocks.blocks[k])) for k in range(w.M + 1))
    gs, os_ = g.triplets.sigma, o.triplets.sigma
    gthr, othr = g.spurious_threshold, o.verdict.threshold
    def near(s): return any(abs(s - e) <= 1e-9 * max(abs(e), s) for e in (w.a, w.b))
    def firm(s, tau, thr): return not near(s) and not (0.5 <= tau / thr <= 2.0)
    matched, worst_sigma, worst_res_ratio, mism, worst_vec = 0, 0.0, 0.0, [], 0.0
    res_cases = []
    for i in range(o.triplets.count()):
        if not o.triplets.in_interval[i] or o.verdict.spurious[i] or not firm(os_[i], o.verdict.tau[i], othr):
            continue
        j = int(np.argmin(np.abs(gs - os_[i])))
        rel = abs(gs[j] - os_[i]) / os_[i]
        ok = rel <= 1e-10 and g.triplets.in_interval[j] and not g.spurious[j]
        if ok:
            matched += 1
            worst_sigma = max(worst_sigma, rel)
            for gv, ov in ((g.triplets.left[:, j], o.triplets.left[:, i]), (g.triplets.right[:, j], o.triplets.right[:, i])):
                worst_vec = max(worst_vec, min(np.linalg.norm(gv - ov), np.linalg.norm(gv + ov)))
            ratio = g.exact[j] / max(1e-9 * sigma.max(), 10 * o.residuals.exact[i])
            worst_res_ratio = max(worst_res_ratio, ratio)
            res_cases.append({"sigma": float(os_[i]), "ratio": float(ratio), "gpu_exact": float(g.exact[j]),
                              "oracle_exact": float(o.residuals.exact[i]), "gpu_tau_ratio": float(g.tau[j] / gthr),
                              "oracle_tau_ratio": float(o.verdict.tau[i] / othr)})
        else:
            mism.append({"oracle_sigma": float(os_[i]), "gpu_sigma": float(gs[j]), "rel": float(rel),
                         "gpu_tau_ratio": float(g.tau[j] / gthr), "oracle_tau_ratio": float(o.verdict.tau[i] / othr)})
    # every oracle candidate inside [a, b] (converged or not): relative distance to the nearest GPU value
    cand = [abs(gs[int(np.argmin(np.abs(gs - x)))] - x) / x for x, f in zip(os_, o.triplets.in_interval) if f]
    out = {"cfg": c, "mode": mode, "delta": DELTA, "gpu_s": tg, "oracle_s": to, "cores": os.cpu_count(),
           "in_interval_sigma_reldiff_median": float(np.median(cand)) if cand else None,
           "in_interval_sigma_reldiff_max": float(np.max(cand)) if cand else None,
           "firm_matched_vector_max_diff": worst_vec,
           "gpu_nonspurious": g.count_nonspurious_in_interval, "oracle_nonspurious": o.count_nonspurious_in_interval,
           "gpu_in_interval": g.count_in_interval, "oracle_in_interval": o.count_in_interval,
           "gpu_boundary": g.count_boundary, "oracle_boundary": o.count_boundary,
           "truth_in_interval": int(np.sum((sigma >= w.a) & (sigma <= w.b))),
           "moment_blocks_max_relerr": blk, "firm_matched": matched, "firm_mismatches": mism[:20],
           "n_firm_mismatches": len(mism), "worst_matched_sigma_relerr": worst_sigma,
           "worst_residual_over_bound": worst_res_ratio,
           "n_residual_over_bound": sum(1 for x in res_cases if x["ratio"] > 1),
           "residual_cases_worst": sorted(res_cases, key=lambda x: -x["ratio"])[:12],
           "matched_exact_residual_quantiles": {q: [float(np.quantile([x[k] for x in res_cases], q)) for k in ("gpu_exact", "oracle_exact")]
                                                for q in (0.5, 0.9, 1.0)} if res_cases else None}
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open(f"gpurun_out/parity_cfg{c}_mode{mode}" + ("" if DELTA == 1e-20 else f"_delta{DELTA:g}") + ".json", "w"), indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "firm_mismatches"}), flush=True)
