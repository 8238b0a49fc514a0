"""Shifted-solve phase time per run_solve call, repeated in one process (config 2, both modes)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_13655_b200 import sssvd, workloads
w = workloads.CONFIGS[2]
a, _ = workloads.make_operator(2)
dev = sssvd.Device(0)
dev.set_operator(a)
out = {0: [], 1: []}
for it in range(8):
    for mode in w.modes:
        cfg = sssvd.RunConfig(w.a, w.b, mode=mode, params=sssvd.SsParams(block_size=w.L, moment_degree=w.M, quadrature_count=w.N))
        r = dev.run_solve(cfg)
        out[mode].append(round(r.device_times["shifted_solves_s"] * 1e3, 1))
print("groups", os.environ.get("SSSVD_GROUPS", "default"), out)
