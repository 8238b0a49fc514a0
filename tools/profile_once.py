"""One run_solve of a config (for ncu launch lists / single-kernel captures). The operator is
generated (torch on the GPU, workloads.py) and two warm-up run_solve calls run BEFORE
cudaProfilerStart, so with `ncu --profile-from-start off` the capture holds exactly one
steady-state run_solve (the shifted-solve pass replayed from its CUDA graph) and only the
library's own kernels.
    python tools/profile_once.py [cfg] [mode] [warmups]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2109_13655_b200 import sssvd, workloads  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 1
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 2
w = workloads.CONFIGS[c]
a, _ = workloads.make_operator(c)
dev = sssvd.Device(0)
cfg = sssvd.RunConfig(w.a, w.b, mode=mode, params=sssvd.SsParams(block_size=w.L, moment_degree=w.M, quadrature_count=w.N), gram_cap=1 << 30)
for _ in range(warm):
    sssvd.run_solve(a, cfg, dev)
torch.cuda.synchronize()
torch.cuda.profiler.start()
r = sssvd.run_solve(a, cfg, dev)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok", r.count_nonspurious_in_interval, r.device_times)
