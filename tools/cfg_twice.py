"""Three run_solve calls of one config in one process: first call (eager), second (captures the
shifted-solve pass as a CUDA graph) and steady state (graph replay)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_13655_b200 import sssvd, workloads
c = int(sys.argv[1])
w = workloads.CONFIGS[c]
a, _ = workloads.make_operator(c)
dev = sssvd.Device(0)
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
for it in range(iters):
    for mode in w.modes:
        cfg = sssvd.RunConfig(w.a, w.b, mode=mode, params=sssvd.SsParams(block_size=w.L, moment_degree=w.M, quadrature_count=w.N), gram_cap=1 << 30)
        t0 = time.time(); r = sssvd.run_solve(a, cfg, dev); wall = time.time() - t0
        t = r.timings
        print(f"cfg{c} mode{mode} call{it}: wall {wall:.3f} s12 {t.steps_1_2:.3f} s3 {t.step_3:.3f} s4 {t.step_4:.3f} "
              f"s5 {t.step_5:.3f} post {t.postprocess:.3f} solves {r.device_times['shifted_solves_s']:.3f}", flush=True)
