"""Median shifted-solve phase time (config 2, both modes, graph replay) for the current env."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_13655_b200 import sssvd, workloads
w = workloads.CONFIGS[2]
a, _ = workloads.make_operator(2)
dev = sssvd.Device(0)
dev.set_operator(a)
t = []
for it in range(10):
    for mode in w.modes:
        cfg = sssvd.RunConfig(w.a, w.b, mode=mode, params=sssvd.SsParams(block_size=w.L, moment_degree=w.M, quadrature_count=w.N))
        r = dev.run_solve(cfg)
        if it >= 2:
            t.append(r.device_times["shifted_solves_s"] * 1e3)
tag = " ".join(f"{k}={os.environ[k]}" for k in ("SSSVD_GROUPS", "SSSVD_LEAF_W", "SSSVD_LEAF_C", "SSSVD_NB") if k in os.environ)
print(f"{tag or 'default'}: median {statistics.median(t):.1f} ms  min {min(t):.1f}  max {max(t):.1f}", flush=True)
