"""Full-size parity of the GPU library with the CPU oracle on BASELINE configs 1-5,
through the C ABI. Configs 1-4 run the oracle live (numpy/LAPACK on the host cores, ~1-2 min
each); config 5 (~15-20 min of oracle time) compares against the committed fixture
tests/golden/oracle_cfg5.npz made by tools/make_oracle_fixture.py on a B200 box, keyed by the
SHA-256 of the generated operator. The contract itself lives in tests/parity_contract.py."""
import json
import os

import numpy as np
import pytest

from oracle import sssvd_oracle as orc
from parity_contract import (Summary, check_robust, check_strict, principal_angle_sine, summarize_gpu,
                             summarize_oracle)

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def gpu_runs(dev, a, w, mode):
    from paper_2109_13655_b200 import sssvd
    prm = dict(block_size=w.L, moment_degree=w.M, quadrature_count=w.N)
    out = {}
    for tag, delta in (("d20", 1e-20), ("d12", 1e-12)):
        cfg = sssvd.RunConfig(w.a, w.b, mode=mode, gram_cap=1 << 30,
                              params=sssvd.SsParams(lowrank_threshold=delta, **prm))
        out[tag] = summarize_gpu(sssvd.run_solve(a, cfg, dev))
    return out


def oracle_runs(a, w, mode):
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(GOLDEN), "..", "tools"))
    from make_oracle_fixture import oracle_runs as runs
    r20, r12, _ = runs(a, w, mode)
    return {"d20": summarize_oracle(r20), "d12": summarize_oracle(r12)}


def contract(g, o, w, truth):
    smax = float(truth.max())
    strict = check_strict(g["d12"], o["d12"], w.a, w.b, smax, truth)
    robust = check_robust(g["d20"], o["d20"], g["d12"], o["d12"], w.a, w.b, smax, truth)
    return strict, robust


MIN_CHECKED = {1: 90, 2: 250, 3: 150, 4: 100, 5: 800}


def check_counts(cfg, strict, robust, o):
    # the comparisons must not be vacuous: most in-interval candidates are compared at both levels,
    # and only a few verdicts at delta = 1e-20 are set by roundoff
    assert strict.checked >= MIN_CHECKED[cfg]
    assert robust.checked + robust.junk >= 0.5 * o["d20"].count_in_interval
    assert robust.undetermined <= max(2, 0.02 * o["d20"].count_in_interval)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_config_parity_with_live_oracle(dev, cfg):
    from paper_2109_13655_b200 import workloads
    w = workloads.CONFIGS[cfg]
    a, truth = workloads.make_operator(cfg)
    for mode in w.modes:
        g = gpu_runs(dev, a, w, mode)
        o = oracle_runs(a, w, mode)
        strict, robust = contract(g, o, w, truth)
        print(f"cfg{cfg} mode{mode}: strict {strict}; robust {robust}")
        check_counts(cfg, strict, robust, o)
        if cfg == 4:
            # the clustered config: the right Ritz vectors of the in-interval candidates span the
            # same subspace on both sides (delta = 1e-12, same count)
            gi, oi = np.flatnonzero(g["d12"].in_interval), np.flatnonzero(o["d12"].in_interval)
            assert gi.size == oi.size
            s = principal_angle_sine(g["d12"].right[:, gi], o["d12"].right[:, oi])
            print(f"cfg4 cluster subspace: {gi.size} vectors, largest principal-angle sine {s:.3e}")
            assert s <= 1e-8


def test_config5_parity_with_oracle_fixture(dev):
    from paper_2109_13655_b200 import workloads
    path = os.path.join(GOLDEN, "oracle_cfg5.npz")
    fx = np.load(path)
    meta = json.loads(str(fx["meta"]))
    w = workloads.CONFIGS[5]
    a, truth = workloads.make_operator(5)
    assert workloads.sha256(a) == meta["sha256"], "operator differs from the one the fixture was made from"
    assert np.array_equal(truth, fx["truth"])
    for mode in w.modes:
        g = gpu_runs(dev, a, w, mode)
        o = {t: Summary.from_arrays(fx, f"m{mode}_{t}_") for t in ("d20", "d12")}
        strict, robust = contract(g, o, w, truth)
        print(f"cfg5 mode{mode}: strict {strict}; robust {robust}")
        check_counts(cfg=5, strict=strict, robust=robust, o=o)
