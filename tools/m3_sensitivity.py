"""Sensitivity of the parity contract to the trailing-update kernel (SSSVD_ZGEMM = 4m | 3m): moment-block
errors against the oracle, counts, and the candidates whose verdicts differ at delta = 1e-20.
    SSSVD_ZGEMM=3m python tools/m3_sensitivity.py <config> [out.npz]"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2109_13655_b200 import sssvd, workloads  # noqa: E402
import test_gpu_parity_configs as T  # noqa: E402
from parity_contract import match  # noqa: E402

cfg = int(sys.argv[1])
w = workloads.CONFIGS[cfg]
a, truth = workloads.make_operator(cfg)
dev = sssvd.Device(0)
for mode in w.modes:
    g = T.gpu_runs(dev, a, w, mode)
    o = T.oracle_runs(a, w, mode)
    ob = o["blocks"].blocks if hasattr(o["blocks"], "blocks") else o["blocks"]
    errs = [float(np.linalg.norm(np.asarray(gb) - np.asarray(b)) / np.linalg.norm(b)) for gb, b in zip(g["blocks"], ob)]
    out = {"kernel": os.environ.get("SSSVD_ZGEMM", "default"), "config": cfg, "mode": mode,
           "block_err_max": max(errs), "block_err": errs[:4] + errs[-2:]}
    for tag in ("d20", "d12"):
        gs, os_ = g[tag], o[tag]
        out[tag] = {"gpu_in": gs.count_in_interval, "orc_in": os_.count_in_interval,
                    "gpu_nonspurious": gs.count_nonspurious, "orc_nonspurious": os_.count_nonspurious}
        diff = []
        for i in np.flatnonzero(os_.in_interval):
            if os_.exact[i] > 1e-2 * truth.max():
                continue
            j = match(os_.sigma[i], os_.exact[i], gs, 1e-2 * truth.max())
            if j is None:
                diff.append((float(os_.sigma[i]), None, float(os_.tau[i] / os_.threshold)))
            elif gs.spurious[j] != os_.spurious[i]:
                diff.append((float(os_.sigma[i]), float(gs.tau[j] / gs.threshold), float(os_.tau[i] / os_.threshold),
                             float(gs.exact[j]), float(os_.exact[i])))
        out[tag]["verdict_diffs"] = diff
    print(json.dumps(out), flush=True)
    if len(sys.argv) > 2:
        np.savez(sys.argv[2] + f"_m{mode}.npz", *g["blocks"])
    try:
        s, r = T.contract(g, o, w, truth)
        print("contract ok", s, r, flush=True)
    except AssertionError as e:
        print("contract FAILED", str(e)[:300], flush=True)
