"""Dumps the parity Summaries (tests/parity_contract.py) of the GPU library and the oracle at both
truncation levels (delta 1e-20 / 1e-12) for BASELINE configs, for offline analysis of the contract:
    python tools/parity_dump.py 1,2,3,4,5 [--out gpurun_out/parity_dump]
Config 5 takes the oracle side from tests/golden/oracle_cfg5.npz (SHA-checked)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402

from paper_2109_13655_b200 import sssvd, workloads  # noqa: E402
from parity_contract import Summary, summarize_gpu, summarize_oracle  # noqa: E402
from make_oracle_fixture import oracle_runs  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("cfgs")
    p.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "parity_dump"))
    args = p.parse_args()
    os.makedirs(args.out, exist_ok=True)
    dev = sssvd.Device(0)
    for c in [int(x) for x in args.cfgs.split(",")]:
        w = workloads.CONFIGS[c]
        a, truth = workloads.make_operator(c)
        sha = workloads.sha256(a)
        arrays = {"truth": truth}
        meta = {"cfg": c, "sha256": sha}
        for mode in w.modes:
            prm = dict(block_size=w.L, moment_degree=w.M, quadrature_count=w.N)
            for tag, delta in (("d20", 1e-20), ("d12", 1e-12)):
                cfg = sssvd.RunConfig(w.a, w.b, mode=mode, gram_cap=1 << 30,
                                      params=sssvd.SsParams(lowrank_threshold=delta, **prm))
                arrays.update(summarize_gpu(sssvd.run_solve(a, cfg, dev), keep_vectors=False).arrays(f"g{mode}_{tag}_"))
            if c == 5:
                fx = np.load(os.path.join(ROOT, "tests", "golden", "oracle_cfg5.npz"))
                meta["fixture_sha_ok"] = json.loads(str(fx["meta"]))["sha256"] == sha
                for tag in ("d20", "d12"):
                    arrays.update(Summary.from_arrays(fx, f"m{mode}_{tag}_").arrays(f"o{mode}_{tag}_"))
            else:
                r20, r12, tm = oracle_runs(a, w, mode)
                arrays.update(summarize_oracle(r20, keep_vectors=False).arrays(f"o{mode}_d20_"))
                arrays.update(summarize_oracle(r12, keep_vectors=False).arrays(f"o{mode}_d12_"))
                meta[f"oracle_timings_{mode}"] = tm
        arrays["meta"] = np.array(json.dumps(meta))
        np.savez_compressed(os.path.join(args.out, f"cfg{c}.npz"), **arrays)
        print(f"cfg{c}: {json.dumps(meta)}", flush=True)


if __name__ == "__main__":
    main()
