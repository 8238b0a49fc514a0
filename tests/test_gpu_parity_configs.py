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
        res = sssvd.run_solve(a, cfg, dev)
        out[tag] = summarize_gpu(res)
        out["blocks"] = [np.array(b) for b in res.blocks.blocks]   # the same moment blocks at either delta
    return out


def oracle_runs(a, w, mode):
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(GOLDEN), "..", "tools"))
    from make_oracle_fixture import oracle_runs as runs
    r20, r12, _ = runs(a, w, mode)
    return {"d20": summarize_oracle(r20), "d12": summarize_oracle(r12), "blocks": r20.blocks,
            "starting_norm": r20.starting_norm}


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
            cluster_subspace_check(dev, a, w, mode, g, o)


def cluster_subspace_check(dev, a, w, mode, g, o):
    """Config 4 (the clustered spectrum): the right Ritz vectors of the in-interval candidates span
    the same subspace on both sides (criterion 4: largest principal-angle sine below 1e-8).

    Measured on this config (tools/cfg4_subspace.py, profiles/r02_cfg4_subspace.jsonl): at
    delta = 1e-12 the reduced subspace itself is not determined to 1e-8 by the data. Feeding the
    GPU's moment blocks (7.9e-12 relative from the oracle's, i.e. roundoff) to the ORACLE's own tail
    moves the oracle's in-interval subspace by 4.9e-7, because the truncation keeps directions whose
    singular values sit at the roundoff level of the blocks. So the criterion is applied
      (a) as written, 1e-8, at delta = 1e-8, where the kept directions are data-determined
          (measured 3.7e-10, the oracle's self-sensitivity 3.6e-10);
      (b) at delta = 1e-12 relative to that self-sensitivity: the GPU library may differ from the
          oracle by no more than 3x what the oracle differs from itself under a roundoff-level
          change of its input (and by no more than 1e-8 where the self-sensitivity is below it)."""
    from paper_2109_13655_b200 import sssvd
    A = orc.ProblemMatrix(a)
    omode = [orc.SS_SVD, orc.SS_SVD_NT][mode]
    prm = dict(block_size=w.L, moment_degree=w.M, quadrature_count=w.N)

    def oracle_tail(blocks, delta):
        r = orc.RunResult(input_transposed=A.transposed)
        r.blocks, r.starting_norm = blocks, o["starting_norm"]
        orc.finish_solve(A, orc.RunConfig(w.a, w.b, mode=omode, params=orc.SsParams(lowrank_threshold=delta, **prm)), r)
        return r.triplets.right[:, np.flatnonzero(r.triplets.in_interval)]

    gpu_blocks = orc.MomentBlocks([np.array(b) for b in g["blocks"]])
    # (b) delta = 1e-12
    gd, od = g["d12"], o["d12"]
    vg, vo = gd.right[:, np.flatnonzero(gd.in_interval)], od.right[:, np.flatnonzero(od.in_interval)]
    vx = oracle_tail(gpu_blocks, 1e-12)   # X: the oracle's tail on the GPU's moment blocks
    assert vg.shape[1] == vo.shape[1] == vx.shape[1]
    s_go, s_gx, s_ox = principal_angle_sine(vg, vo), principal_angle_sine(vg, vx), principal_angle_sine(vo, vx)
    print(f"cfg4 cluster subspace, delta 1e-12 ({vg.shape[1]} vectors): sin(GPU, oracle) {s_go:.3e}, sin(GPU, oracle "
          f"tail on GPU blocks) {s_gx:.3e}, oracle self-sensitivity {s_ox:.3e}")
    bound = max(1e-8, 3.0 * s_ox)
    assert s_go <= bound, (s_go, s_ox)
    assert s_gx <= bound, (s_gx, s_ox)
    # (a) delta = 1e-8: the criterion as written
    cfg8 = sssvd.RunConfig(w.a, w.b, mode=mode, gram_cap=1 << 30, params=sssvd.SsParams(lowrank_threshold=1e-8, **prm))
    r8 = sssvd.run_solve(a, cfg8, dev)
    vg8 = r8.triplets.right[:, np.flatnonzero(r8.triplets.in_interval)]
    vo8 = oracle_tail(o["blocks"], 1e-8)
    assert vg8.shape[1] == vo8.shape[1] and vg8.shape[1] >= 64
    s8 = principal_angle_sine(vg8, vo8)
    print(f"cfg4 cluster subspace, delta 1e-8 ({vg8.shape[1]} vectors): sin(GPU, oracle) {s8:.3e}")
    assert s8 <= 1e-8


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
