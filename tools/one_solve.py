"""One run_solve of a BASELINE config (for ncu captures): python tools/one_solve.py <config> [mode]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_13655_b200 import sssvd, workloads
c = int(sys.argv[1])
w = workloads.CONFIGS[c]
mode = int(sys.argv[2]) if len(sys.argv) > 2 else w.modes[0]
a, _ = workloads.make_operator(c)
dev = sssvd.Device(0)
cfg = sssvd.RunConfig(w.a, w.b, mode=mode, params=sssvd.SsParams(block_size=w.L, moment_degree=w.M,
                                                                 quadrature_count=w.N), gram_cap=1 << 30)
r = dev.run_solve(cfg) if False else sssvd.run_solve(a, cfg, dev)
print("count_in_interval", r.count_in_interval)
