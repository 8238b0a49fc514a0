"""Benchmark: time-to-triplets of the block SS-SVD shifted-solve path on B200 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

The workload is BASELINE config 5 by default (16384 x 16384, L=128, M=16, N=128: the largest
configuration and the one the north-star targets name); --config 1..4 selects the others.

One step = one end-to-end solve through the public C ABI, per solve mode of the config:
  sssvd_gpu_set_operator(_root) from pinned HOST memory (H2D + pad + NaN check), then
  sssvd_gpu_run_solve (Gram, shifted solves + moments, tail, postprocess), whose results (sigma,
  tau, residuals, triplet vectors, moment blocks) are copied to host memory before it returns.
CUDA events on the current stream bracket each step (the library calls return synchronised):
  e2e   : from before the operator upload to the end of run_solve (H2D and D2H included);
  value : from the end of the upload (the operator is resident in HBM) to the end of run_solve.
Multi-GPU (one rank per GPU, NCCL): the h = N/2 quadrature points are sharded contiguously over
the ranks, rank 0 uploads A and ONE ncclBroadcast sends it to the others, the partial moment
blocks are summed with one ncclAllReduce inside the library; total work is fixed ("strong"). The
step time is the max over ranks. `--gpus N` without torchrun re-launches itself under
torch.distributed.run with N ranks.

--impl reference times the reference algorithm on the host cores: the CPU restatement of
run_solve (oracle/, numpy + LAPACK over all host threads; the reference itself needs Eigen, absent
here), as a bounded sample per step (see cpu_sample()).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "time-to-triplets (s)"
FP64_PEAK_TFLOPS = 37.1   # measured DMMA probe, profiles/r01_fp64_peaks.json (MEASURED_PEAKS.json has no FP64 entry)
ZGEMM_PROFILE = os.path.join(ROOT, "profiles", "r02_ncu_zgemm3m_cfg5.json")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


def relaunch_distributed(args):
    """`bench.py --gpus N` outside torchrun: run N ranks under torch.distributed.run (127.0.0.1)."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")   # keep stdout to the one JSON line
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd, env=env))


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index=0):
        self.samples, self.proc = [], None
        self.index = index

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw",
                 "--format=csv,noheader,nounits", "-lms", os.environ.get("BENCH_CLOCK_MS", "200")],
                stdout=subprocess.PIPE, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(s[0]) for s in self.samples if s and num(s[0]) is not None]
        mx = [num(s[1]) for s in self.samples if len(s) > 1 and num(s[1]) is not None]
        pw = [num(s[7]) for s in self.samples if len(s) > 7 and num(s[7]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 3 + i and s[3 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm), "power_w_max": max(pw) if pw else None}


# ----------------------------------------------------------------------------- CPU sample
def cpu_sample(w, a, steps, warmup, log=None):
    """The reference algorithm on the host cores (oracle/: the CPU restatement of run_solve with
    numpy + LAPACK over all host threads), as a bounded sample of the config's run_solve:
      * once (first warm-up step): form_gram (problem.hpp:81-95) and the tail (steps 3-5 +
        postprocess, pipeline.hpp:141-231) on stacked blocks [V, G V, .., G^M V] of the moment
        blocks' shapes (the tail's cost is set by the shapes, not the values);
      * every step: ONE full-size shifted factorisation + block solve + its moment update
        (shifted_solver.hpp:20-40, moments.hpp:132-147) at shift j = step mod h.
    Per-step estimate of run_solve = h * t_shift + t_gram + t_tail (summed over the modes)."""
    from oracle import sssvd_oracle as orc
    A = orc.ProblemMatrix(a)
    h = w.N // 2
    t0 = time.perf_counter()
    gram = orc.form_gram(A, 1 << 30)
    t_gram = time.perf_counter() - t0
    absmax = float(np.abs(gram).max())
    v0 = orc.random_start(w.n, w.L, 42)
    t_tail = {}
    rules = {}
    for mode in w.modes:
        rules[mode] = orc.ContourRule(w.a, w.b, w.N, 0.1, orc.SpectralTransform(orc.EXP if mode == 1 else orc.IDENTITY))
    for mode in w.modes:
        blocks, x = [], v0.copy()
        for _ in range(w.M + 1):
            blocks.append(x / np.linalg.norm(x))
            x = gram @ blocks[-1]
        res = orc.RunResult(input_transposed=A.transposed)
        res.blocks, res.starting_norm = orc.MomentBlocks(blocks), float(np.linalg.norm(v0))
        cfg = orc.RunConfig(w.a, w.b, mode=[orc.SS_SVD, orc.SS_SVD_NT][mode],
                            params=orc.SsParams(block_size=w.L, moment_degree=w.M, quadrature_count=w.N))
        t0 = time.perf_counter()
        orc.finish_solve(A, cfg, res, gram)
        t_tail[mode] = time.perf_counter() - t0
    per_step = []
    for i in range(warmup + steps):
        dt = 0.0
        for mode in w.modes:
            rule = rules[mode]
            j = i % h
            t0 = time.perf_counter()
            x = orc.ShiftedFactorization(gram, rule.shift(j), absmax).solve(v0)
            s = np.zeros_like(v0)
            p = complex(1.0)
            for _ in range(w.M + 1):
                s += 2.0 * (complex(rule.weights[j]) * p * x).real
                p *= complex(rule.nodes[j])
            dt_shift = time.perf_counter() - t0
            dt += h * dt_shift + t_gram + t_tail[mode]
        if i >= warmup:
            per_step.append(dt)
        if log:
            log(f"[cpu] step {i}: estimate {dt:.1f} s (shift sample {dt_shift:.2f} s)")
    cores = os.cpu_count()
    sample = (f"{w.name}: per step one full-size shifted LU + block solve + moment update "
              f"(n={w.n}, L={w.L}) at shift j = step mod {h}, per mode; form_gram ({t_gram:.2f} s) and the tail "
              f"({', '.join(f'{v:.2f} s' for v in t_tail.values())}) timed once on blocks of the moment shapes; "
              f"value = sum over modes of {h} * t_shift + t_gram + t_tail; numpy/OpenBLAS on {cores} host threads")
    return float(np.mean(per_step)), cores, sample


def run_reference(args, rank, world):
    """CPU arm (rank 0 only; other ranks exit without work)."""
    if rank != 0:
        return
    from paper_2109_13655_b200 import workloads
    w = workloads.CONFIGS[args.config]
    a, _ = workloads.make_operator(args.config)
    sha = workloads.sha256(a)
    v, cores, sample = cpu_sample(w, a, args.steps, args.warmup, log=lambda s: print(s, file=sys.stderr, flush=True))
    print(json.dumps({"impl": "reference", "metric": METRIC, "value": v, "unit": "s", "n_gpus": world,
                      "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
                      "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                      "config": config_block(w, world), "input_sha256": sha,
                      "cpu_baseline": {"value": v, "unit": "s", "cores": cores, "kind": "port", "sample": sample},
                      "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
          flush=True)


def config_block(w, world):
    return {"workload": w.description, "m": w.m, "n": w.n, "L": w.L, "M": w.M, "N": w.N,
            "modes": ["ss-svd" if m == 0 else "ss-svd-nt" for m in w.modes],
            "parallelism": f"quadrature points sharded over {world} GPU(s), A broadcast once, 1 NCCL all-reduce",
            "l2": "inputs larger than L2 (A and every shifted factor exceed the 126 MB L2)"}


# ----------------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_distributed(args)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2109_13655_b200 import sssvd, workloads
    w = workloads.CONFIGS[args.config]
    dev = sssvd.Device(local)
    if world > 1:
        uid = [sssvd.Device.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        dev.init_comm(uid[0], world, rank)
    comm_nranks = dev.comm_size()

    # the operator in pinned host memory on rank 0 (column-major A == row-major A^T)
    a_pin = a = sha = sigma = None
    if rank == 0:
        a_pin = torch.empty((w.n, w.m), dtype=torch.float64).pin_memory()
        a, sigma = workloads.make_operator(args.config, out=a_pin.numpy())
        sha = workloads.sha256(a)
    cfgs = [sssvd.RunConfig(w.a, w.b, mode=m, params=sssvd.SsParams(block_size=w.L, moment_degree=w.M,
                                                                     quadrature_count=w.N), gram_cap=1 << 30)
            for m in w.modes]
    a_ptr = a_pin.data_ptr() if a_pin is not None else None

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    def step(evs):
        evs[0].record()
        if world > 1:
            dev.set_operator_root(a_ptr, w.m, w.n, w.m, on_device=False, root=0)
        else:
            dev.check(sssvd.lib().sssvd_gpu_set_operator(dev.h, sssvd.ctypes.c_void_p(a_ptr), w.m, w.n, w.m, 0))
        evs[1].record()
        out = [dev.run_solve(c) for c in cfgs]
        for r in out:   # results are in host memory when run_solve returns; read the small fields
            _ = (r.triplets.sigma[:1], r.tau[:1], r.exact[:1])
        evs[2].record()
        return out

    # GEMM stamps on from the first warm-up step: the library captures the shifted-solve pass into
    # a CUDA graph on its second run, keyed (among others) by the profiling state
    sssvd.profile_gemm(True)
    res = None
    for _ in range(args.warmup):
        res = None   # return the previous step's pinned result buffers to the library's pool first
        res = step([torch.cuda.Event(enable_timing=True) for _ in range(3)])
    barrier()
    sssvd.profile_gemm_collect()   # discard the warm-up timings
    launches0 = sssvd.launch_count()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    phases = []
    with Clocks(local) as clk:
        t_wait = time.perf_counter()
        while not clk.samples and time.perf_counter() - t_wait < 3.0:
            time.sleep(0.05)
        time.sleep(0.2)
        barrier()
        # BENCH_PROFILER_RANGE=1 (launch-list captures: ncu --profile-from-start off): the capture
        # holds exactly the timed steps. A number printed by a run under ncu is never a bench value.
        prof_range = os.environ.get("BENCH_PROFILER_RANGE") == "1"
        if prof_range:
            torch.cuda.profiler.start()
        for i in range(args.steps):
            # only the last step's results are kept: holding every step's (pinned) result arrays would
            # make the library page-lock ~1 GB of new host memory per step at config 5 instead of
            # reusing its pool, inside the timed region
            res = None
            res = step(evs[i])
        phases.append(res)
        barrier()
        if prof_range:
            torch.cuda.profiler.stop()
    launches = sssvd.launch_count() - launches0
    gemm_ms, gemm_flops, gemm_alg_flops, gemm_launches = sssvd.profile_gemm_collect2()
    sssvd.profile_gemm(False)
    e2e_steps = [e[0].elapsed_time(e[2]) / 1e3 for e in evs]
    val_steps = [e[1].elapsed_time(e[2]) / 1e3 for e in evs]
    t, te = float(np.mean(val_steps)), float(np.mean(e2e_steps))
    if dist:
        tt = torch.tensor([t, te], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t, te = float(tt[0]), float(tt[1])
    last = phases[-1]
    h2d = (a.nbytes if a is not None else 0)
    d2h = sum(r.triplets.left.nbytes + r.triplets.right.nbytes + 6 * r.triplets.sigma.nbytes + r.triplets.q.nbytes +
              sum(b.nbytes for b in r.blocks.blocks) for r in last)
    solve_s = sum(r.device_times["shifted_solves_s"] for r in last)
    solve_flops = sum(r.device_times["shifted_solve_flops"] for r in last)
    gemm_tflops = gemm_flops / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else None
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            v, cores, sample = cpu_sample(w, a, 1, 0)
            cpu = {"value": v, "unit": "s", "cores": cores, "kind": "port", "sample": sample}
        except Exception as e:  # reported, never required
            cpu = {"value": None, "unit": "s", "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {e}"}
    traffic = None
    prof = {}
    if os.path.exists(ZGEMM_PROFILE):
        prof = json.load(open(ZGEMM_PROFILE))
        traffic = prof.get("dram_bytes_per_launch")
    if rank == 0:
        line = {
            "metric": METRIC, "value": t, "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded A = U diag(sigma) V^T, GPU-generated)",
            "config": config_block(w, world),
            "e2e": {"value": te, "unit": "s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "step_s": [round(x, 4) for x in e2e_steps]},
            "roofline": {"bound": "tensor",
                         "kernel": "zgemm3m_kernel (DMMA trailing update of the blocked LU, 3 real products per "
                                   "complex multiply-add)",
                         "achieved": gemm_tflops, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": (gemm_tflops / FP64_PEAK_TFLOPS) if gemm_tflops else None,
                         # the same GEMM work in the conventional unit (8 M N K per complex launch, SURVEY 8d's
                         # algorithmic unit) over the same busy time: above `achieved` by the share of 3M launches,
                         # and allowed to pass the peak (a 4-product kernel would need this rate for the same time)
                         "achieved_algorithmic": gemm_alg_flops / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else None,
                         "frac_algorithmic": gemm_alg_flops / (gemm_ms / 1e3) / 1e12 / FP64_PEAK_TFLOPS if gemm_ms > 0 else None,
                         "traffic": traffic,
                         "traffic_launch": prof or None,
                         "achieved_basis": "EXECUTED tensor flops of the DMMA GEMMs (6 M N K per 3M launch, 8 M N K per "
                                           "4-product launch) / GEMM-busy time (union of the launch intervals from "
                                           "%globaltimer stamps; the shift groups overlap their GEMMs), rank 0",
                         "peak_source": "measured FP64 DMMA probe (tools/fp64_peak.cu, profiles/r01_fp64_peaks.json); "
                                        "MEASURED_PEAKS.json has no FP64 entry",
                         "gemm_launches": gemm_launches, "gemm_busy_s_per_step": gemm_ms / 1e3 / args.steps,
                         # the whole phase (assembly + LU + substitution + moments): executed tensor flops / phase time
                         "phase_tflops": gemm_flops / args.steps / solve_s / 1e12 if solve_s > 0 else None,
                         "phase_frac": (gemm_flops / args.steps / solve_s / 1e12 / FP64_PEAK_TFLOPS) if solve_s > 0 else None,
                         # the north-star unit h (8 n^3 / 3 + 8 n^2 L) / t: it counts 8 real flops per complex
                         # multiply-add, the 3M updates execute 6, so this rate may exceed the 4-product roofline
                         "phase_algorithmic_tflops": solve_flops / solve_s / 1e12 if solve_s > 0 else None,
                         "phase_flops_per_step": solve_flops, "phase_s_per_step": solve_s},
            "phases_s": {"steps_1_2": sum(r.timings.steps_1_2 for r in last),
                         "step_3": sum(r.timings.step_3 for r in last), "step_4": sum(r.timings.step_4 for r in last),
                         "step_5": sum(r.timings.step_5 for r in last),
                         "postprocess": sum(r.timings.postprocess for r in last),
                         "gram": last[0].device_times["gram_s"],
                         "allreduce": sum(r.device_times["allreduce_s"] for r in last)},
            "counts": [{"mode": c.mode, "nonspurious_in_interval": r.count_nonspurious_in_interval,
                        "in_interval": r.count_in_interval, "boundary": r.count_boundary} for c, r in zip(cfgs, last)],
            "truth_in_interval": int(np.sum((sigma >= w.a) & (sigma <= w.b))),
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "step_s": [round(x, 4) for x in val_steps],
            "gpu_launches": int(launches // max(1, args.steps)),
            "gpu_launches_timed_region": int(launches),
            "comm_nranks": comm_nranks, "comm_nranks_ok": comm_nranks == world,
            "input_sha256": sha,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
