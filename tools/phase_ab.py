"""Steady-state shifted-solve phase of one config (after 2 warm-up calls per mode: eager, then
graph capture), median over --reps calls. Usage: python tools/phase_ab.py 2 [--reps 5]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2109_13655_b200 import sssvd, workloads

c = int(sys.argv[1])
reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 5
w = workloads.CONFIGS[c]
a, _ = workloads.make_operator(c)
dev = sssvd.Device(0)
for mode in w.modes:
    cfg = sssvd.RunConfig(w.a, w.b, mode=mode, params=sssvd.SsParams(block_size=w.L, moment_degree=w.M,
                                                                      quadrature_count=w.N), gram_cap=1 << 30)
    ph, tot = [], []
    for it in range(reps + 2):
        r = sssvd.run_solve(a, cfg, dev)
        if it >= 2:
            ph.append(r.device_times["shifted_solves_s"] * 1e3)
            t = r.timings
            tot.append((t.steps_1_2 + t.step_3 + t.step_4 + t.step_5 + t.postprocess) * 1e3)
    print(json.dumps({"cfg": c, "mode": mode, "env": {k: v for k, v in os.environ.items() if k.startswith("SSSVD_")},
                      "phase_ms_median": float(np.median(ph)), "phase_ms": [round(x, 1) for x in ph],
                      "run_ms_median": float(np.median(tot))}), flush=True)
