"""Multi-GPU scaling estimate from one B200 (the pool gives one GPU per call).

Every rank of a G-GPU run does: its contiguous shard of the h shifts (shifted solves + partial
moments), its 1/G share of the Gram tiles, one all-reduce of G (n^2 f64) and one of the moment
blocks ((M+1) n L f64), then the replicated tail (steps 3-5 + postprocess, identical on every
rank). This tool measures on one GPU:
  * the full N=1 run_solve (operator resident in HBM, like bench.py's `value`), three times,
    keeping the third (steady state: the first run is eager, the second captures the
    shifted-solve pass as a CUDA graph, the third replays it);
  * for each G and for the first and the last rank, the shard's shifted-solve phase alone
    (SSSVD_SIM_RANKS=G:r: the library factors just that shard; no collective, partial moments);
and prints T_G = T_1 - solves_1 - gram_1 (1 - 1/G) + max_r solves_shard(G, r) + allreduce_G, with
the all-reduces costed at a ring's 2 (G-1)/G bytes over NVLink at --nvlink-gbs (bus bandwidth),
and the strong-scaling efficiency T_1 / (G T_G).

    python tools/scale_estimate.py [--config 5] [--gpus 2 4 8] [--nvlink-gbs 350]
"""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(cfg_id, reps=3):
    import numpy as np
    import torch
    from paper_2109_13655_b200 import sssvd, workloads
    w = workloads.CONFIGS[cfg_id]
    a, _ = workloads.make_operator(cfg_id)
    a_dev = torch.from_numpy(np.ascontiguousarray(a.T)).cuda()
    dev = sssvd.Device(0)
    mode = w.modes[0]
    cfg = sssvd.RunConfig(w.a, w.b, mode=mode, params=sssvd.SsParams(block_size=w.L, moment_degree=w.M,
                                                                     quadrature_count=w.N), gram_cap=1 << 30)
    out = None
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev.set_operator_device(a_dev.data_ptr(), w.m, w.n, w.m)
        r = dev.run_solve(cfg)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        t = r.timings
        out = {"wall_s": wall, "gram_s": r.device_times["gram_s"], "solves_s": r.device_times["shifted_solves_s"],
               "steps_1_2": t.steps_1_2, "step_3": t.step_3, "step_4": t.step_4, "step_5": t.step_5,
               "postprocess": t.postprocess, "m": w.m, "n": w.n, "L": w.L, "M": w.M, "N": w.N}
        del r
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--gpus", type=int, nargs="*", default=[2, 4, 8])
    ap.add_argument("--nvlink-gbs", type=float, default=350.0)
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.child:
        print(json.dumps(run(a.config)), flush=True)
        return
    def child(env_extra):
        env = dict(os.environ, **env_extra)
        p = subprocess.run([sys.executable, __file__, "--child", "--config", str(a.config)], env=env,
                           capture_output=True, text=True)
        if p.returncode:
            sys.stderr.write(p.stderr)
            raise SystemExit(p.returncode)
        return json.loads(p.stdout.strip().splitlines()[-1])
    base = child({})
    print(json.dumps({"config": a.config, "n_gpus": 1, "measured": base}), flush=True)
    t1 = base["wall_s"]
    n, m, L, M = base["n"], base["m"], base["L"], base["M"]
    for g in a.gpus:
        shards = [child({"SSSVD_SIM_RANKS": f"{g}:{r}"}) for r in sorted({0, g - 1})]   # steady state too
        solve_g = max(s["solves_s"] for s in shards)
        ring = 2.0 * (g - 1) / g / (a.nvlink_gbs * 1e9)
        ar = ring * 8.0 * (n * n + (M + 1) * n * L)
        tg = t1 - base["solves_s"] - base["gram_s"] * (1 - 1 / g) + solve_g + ar
        print(json.dumps({"config": a.config, "n_gpus": g, "estimate_s": tg, "efficiency": t1 / (g * tg),
                          "shard_solves_s": [s["solves_s"] for s in shards], "allreduce_s_est": ar,
                          "serial_s": t1 - base["solves_s"] - base["gram_s"],
                          "basis": "one-GPU measurement of the rank shards; tail replicated; ring all-reduce model"}),
              flush=True)


if __name__ == "__main__":
    main()
