"""GPU vs oracle side-by-side on one config (prints per-candidate tau/threshold, residuals)."""
import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2109_13655_b200 import sssvd, workloads
from oracle import sssvd_oracle as orc
c = int(sys.argv[1]); mode = int(sys.argv[2]) if len(sys.argv) > 2 else workloads.CONFIGS[c].modes[0]
w = workloads.CONFIGS[c]
a, sigma = workloads.make_operator(c)
cfg = sssvd.RunConfig(w.a, w.b, mode=mode, params=sssvd.SsParams(block_size=w.L, moment_degree=w.M, quadrature_count=w.N), gram_cap=1<<30)
g = sssvd.run_solve(a, cfg, sssvd.Device(0))
ocfg = orc.RunConfig(w.a, w.b, mode=[orc.SS_SVD, orc.SS_SVD_NT][mode], params=orc.SsParams(block_size=w.L, moment_degree=w.M, quadrature_count=w.N))
t = time.time(); o = orc.run_solve(orc.ProblemMatrix(a), ocfg, gram_cap=1<<30); to = time.time() - t
print(json.dumps({"cfg": c, "mode": mode, "gpu_ns": g.count_nonspurious_in_interval, "orc_ns": o.count_nonspurious_in_interval,
                  "gpu_in": g.count_in_interval, "orc_in": o.count_in_interval, "oracle_s": to,
                  "blocks_relerr": max(float(np.linalg.norm(g.blocks.blocks[k] - o.blocks.blocks[k]) / np.linalg.norm(o.blocks.blocks[k])) for k in range(len(o.blocks.blocks)))}))
gi = np.where(g.triplets.in_interval)[0]; oi = np.where(o.triplets.in_interval)[0]
print("gpu: sigma tau/thr exact"); 
for i in gi: print(f"  {g.triplets.sigma[i]:.15f} {g.tau[i]/g.spurious_threshold:10.3e} {g.exact[i]:9.2e} {'S' if g.spurious[i] else ''}")
print("orc:")
for i in oi: print(f"  {o.triplets.sigma[i]:.15f} {o.verdict.tau[i]/o.verdict.threshold:10.3e} {o.residuals.exact[i]:9.2e} {'S' if o.verdict.spurious[i] else ''}")
