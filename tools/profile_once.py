"""One run_solve of a config (for ncu launch lists / single-kernel captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_13655_b200 import sssvd, workloads
c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 1
w = workloads.CONFIGS[c]
a, _ = workloads.make_operator(c)
dev = sssvd.Device(0)
cfg = sssvd.RunConfig(w.a, w.b, mode=mode, params=sssvd.SsParams(block_size=w.L, moment_degree=w.M, quadrature_count=w.N), gram_cap=1 << 30)
r = dev.run_solve(cfg) if False else sssvd.run_solve(a, cfg, dev)
print("ok", r.count_nonspurious_in_interval, r.device_times)
