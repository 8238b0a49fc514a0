"""Time run_solve phases on configs (device events inside the library). Usage:
    python tools/time_phase.py 1 2 [--reps 2]"""
import json, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2109_13655_b200 import sssvd, workloads

def main():
    cfgs = [int(x) for x in sys.argv[1:] if x.isdigit()]
    reps = 2
    dev = sssvd.Device(0)
    for c in cfgs:
        w = workloads.CONFIGS[c]
        t0 = time.time(); a, sigma = workloads.make_operator(c); tg = time.time() - t0
        for mode in w.modes:
            cfg = sssvd.RunConfig(w.a, w.b, mode=mode, params=sssvd.SsParams(block_size=w.L, moment_degree=w.M, quadrature_count=w.N), gram_cap=1 << 30)
            for r in range(reps):
                t0 = time.time(); res = sssvd.run_solve(a, cfg, dev); wall = time.time() - t0
                d = res.device_times
                out = {"cfg": c, "mode": mode, "rep": r, "wall_s": wall, "gen_s": tg,
                       "steps_1_2": res.timings.steps_1_2, "step3": res.timings.step_3, "step4": res.timings.step_4,
                       "step5": res.timings.step_5, "post": res.timings.postprocess, **d,
                       "solve_tflops": d["shifted_solve_flops"] / max(d["shifted_solves_s"], 1e-12) / 1e12,
                       "count_ns": res.count_nonspurious_in_interval, "truth": int(np.sum((sigma >= w.a) & (sigma <= w.b)))}
                print(json.dumps(out), flush=True)

if __name__ == "__main__":
    main()
