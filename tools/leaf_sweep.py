"""Shifted-solve phase time (steady state: graph replay) of configs 1/2 for leaf shapes (W, C)
and GEMM kernels, each in its own process (the library reads SSSVD_LEAF_W / SSSVD_LEAF_C /
SSSVD_ZGEMM once). Measurement tool; prints one JSON line per setting."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json
sys.path.insert(0, ROOT)
from paper_2109_13655_b200 import sssvd, workloads
c = CFG
w = workloads.CONFIGS[c]
a, _ = workloads.make_operator(c)
dev = sssvd.Device(0)
dev.set_operator(a)
out = []
for it in range(4):
    cfg = sssvd.RunConfig(w.a, w.b, mode=w.modes[0], params=sssvd.SsParams(block_size=w.L, moment_degree=w.M,
                          quadrature_count=w.N), gram_cap=1 << 30)
    r = dev.run_solve(cfg)
    out.append(r.device_times["shifted_solves_s"])
flops = r.device_times["shifted_solve_flops"]
print(json.dumps({"phase_s": min(out[2:]), "tflops": flops / min(out[2:]) / 1e12, "all": out}))
'''

def run(cfg, env):
    code = CHILD.replace("ROOT", repr(ROOT)).replace("CFG", str(cfg))
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=dict(os.environ, **env),
                       timeout=900)
    try:
        return json.loads(p.stdout.strip().splitlines()[-1])
    except Exception:
        return {"error": (p.stderr or p.stdout)[-400:]}


if __name__ == "__main__":
    cfgs = [int(x) for x in sys.argv[1].split(",")]
    settings = [s for s in sys.argv[2:]] or ["default"]
    for c in cfgs:
        for s in settings:
            env = {}
            if s != "default":
                for kv in s.split("+"):
                    k, v = kv.split("=")
                    env[k] = v
            print(json.dumps({"cfg": c, "setting": s, **run(c, env)}), flush=True)
