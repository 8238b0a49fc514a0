"""Runs the CPU oracle (the reference restatement, oracle/sssvd_oracle.py) on one BASELINE config
and stores the compact parity fixture that tests/test_gpu_parity_configs.py compares the GPU
library against (tests/golden/oracle_cfg<N>.npz).

    python tools/make_oracle_fixture.py 5 [--out gpurun_out/oracle_cfg5.npz]

It must run on a B200 box: the operator comes from workloads.make_operator (generated on the GPU,
bit-reproducible across boxes of this image) and its SHA-256 is stored, so the test can assert it
compares the same matrix. For each solve mode of the config the oracle runs run_solve at the
reference default delta = 1e-20, then finish_solve from the same moment blocks at delta = 1e-12
(moments.hpp:205); both runs are reduced to tests/parity_contract.Summary arrays (sigma, verdicts,
tau, residuals, and projections of the triplet vectors on fixed random vectors) plus the true
spectrum. Config 5 takes ~15-20 min on 16 host threads (64 complex LUs of n = 16384).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from oracle import sssvd_oracle as orc  # noqa: E402
from paper_2109_13655_b200 import workloads  # noqa: E402
from parity_contract import summarize_oracle  # noqa: E402


def oracle_runs(a, w, mode, gram_cap=1 << 30):
    prm = dict(block_size=w.L, moment_degree=w.M, quadrature_count=w.N)
    A = orc.ProblemMatrix(a)
    cfg20 = orc.RunConfig(w.a, w.b, mode=[orc.SS_SVD, orc.SS_SVD_NT][mode], params=orc.SsParams(**prm))
    t0 = time.perf_counter()
    r20 = orc.run_solve(A, cfg20, gram_cap=gram_cap)
    t20 = time.perf_counter() - t0
    cfg12 = orc.RunConfig(w.a, w.b, mode=cfg20.mode, params=orc.SsParams(lowrank_threshold=1e-12, **prm))
    r12 = orc.RunResult(input_transposed=A.transposed)
    r12.blocks, r12.starting_norm = r20.blocks, r20.starting_norm
    t0 = time.perf_counter()
    orc.finish_solve(A, cfg12, r12)
    t12 = time.perf_counter() - t0
    return r20, r12, {"run_solve_s": t20, "finish_delta12_s": t12, "steps_1_2_s": r20.timings.steps_1_2,
                      "tail_s": r20.timings.step_3 + r20.timings.step_4 + r20.timings.step_5 + r20.timings.postprocess}


def main():
    p = argparse.ArgumentParser()
    p.add_argument("cfg", type=int)
    p.add_argument("--out", default=None)
    args = p.parse_args()
    w = workloads.CONFIGS[args.cfg]
    t0 = time.perf_counter()
    a, truth = workloads.make_operator(args.cfg)
    sha = workloads.sha256(a)
    gen_s = time.perf_counter() - t0
    print(f"cfg{args.cfg}: A {a.shape} sha256 {sha} ({gen_s:.1f} s)", flush=True)
    arrays = {"truth": truth}
    meta = {"cfg": args.cfg, "sha256": sha, "modes": list(w.modes), "threads": os.cpu_count(), "timings": {}}
    for mode in w.modes:
        r20, r12, tm = oracle_runs(a, w, mode)
        print(f"  mode {mode}: {json.dumps(tm)}; non-spurious {r20.count_nonspurious_in_interval} "
              f"(delta 1e-12: {r12.count_nonspurious_in_interval}), in-interval {r20.count_in_interval}", flush=True)
        arrays.update(summarize_oracle(r20, keep_vectors=False).arrays(f"m{mode}_d20_"))
        arrays.update(summarize_oracle(r12, keep_vectors=False).arrays(f"m{mode}_d12_"))
        meta["timings"][str(mode)] = tm
    arrays["meta"] = np.array(json.dumps(meta))
    out = args.out or os.path.join(ROOT, "gpurun_out", f"oracle_cfg{args.cfg}.npz")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    np.savez_compressed(out, **arrays)
    print(f"wrote {out} ({os.path.getsize(out) / 1e6:.2f} MB)", flush=True)


if __name__ == "__main__":
    main()
