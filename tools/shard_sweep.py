"""Shifted-solve phase time of one rank's shard (SSSVD_SIM_RANKS=G:r) per shift-group count
(SSSVD_GROUPS). The LU work does not depend on the entries of A, so a seeded Gaussian operator of
the config's shape (scaled to sigma_max ~ 2) stands in for the generated one (fast to build).

    python tools/shard_sweep.py --config 5 --sim 8:0 --groups 2 4 8
"""
import argparse, json, os, subprocess, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(cfg_id):
    import torch
    from paper_2109_13655_b200 import sssvd, workloads
    w = workloads.CONFIGS[cfg_id]
    g = torch.Generator(device="cuda").manual_seed(7)
    a_dev = torch.randn((w.n, w.m), generator=g, device="cuda", dtype=torch.float64) / (w.m ** 0.5)
    dev = sssvd.Device(0)
    cfg = sssvd.RunConfig(w.a, w.b, mode=w.modes[0], params=sssvd.SsParams(block_size=w.L, moment_degree=w.M,
                                                                           quadrature_count=w.N), gram_cap=1 << 30)
    out = []
    for _ in range(3):
        dev.set_operator_device(a_dev.data_ptr(), w.m, w.n, w.m)
        r = dev.run_solve(cfg)
        out.append(r.device_times["shifted_solves_s"])
        flops = r.device_times["shifted_solve_flops"]
        del r
    print(json.dumps({"solves_s": out, "tflops": flops / min(out[1:]) / 1e12}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--sim", default="")
    ap.add_argument("--groups", type=int, nargs="*", default=[4])
    ap.add_argument("--env", nargs="*", default=[""], help="extra VAR=value settings, one run each")
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.child:
        child(a.config)
        return
    for extra in a.env:
        for grp in a.groups:
            env = dict(os.environ, SSSVD_GROUPS=str(grp))
            if a.sim:
                env["SSSVD_SIM_RANKS"] = a.sim
            for kv in extra.split(","):
                if "=" in kv:
                    k, v = kv.split("=", 1)
                    env[k] = v
            p = subprocess.run([sys.executable, __file__, "--child", "--config", str(a.config)], env=env,
                               capture_output=True, text=True)
            line = p.stdout.strip().splitlines()[-1] if p.stdout.strip() else p.stderr[-400:]
            print(f"config {a.config} sim {a.sim or '1:0'} groups {grp} {extra}: {line}", flush=True)


if __name__ == "__main__":
    main()
