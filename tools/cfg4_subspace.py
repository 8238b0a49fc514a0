"""Config-4 cluster-subspace diagnostic: how far apart the spans of the in-interval right Ritz
vectors are between (G) the GPU library, (O) the oracle on its own moment blocks and (X) the
ORACLE's tail run on the GPU's moment blocks -- so the implementation difference (G vs X: same
blocks, two tails) is separated from the sensitivity of the problem itself to moment-level roundoff
(O vs X: one tail, two sets of blocks that agree to ~1e-11).
    python tools/cfg4_subspace.py [cfg] [deltas]"""
import os
import sys
import json

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
from oracle import sssvd_oracle as orc  # noqa: E402
from paper_2109_13655_b200 import sssvd, workloads  # noqa: E402
from parity_contract import principal_angle_sine  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 4
deltas = [float(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1e-12, 1e-10, 1e-8]
w = workloads.CONFIGS[c]
a, truth = workloads.make_operator(c)
dev = sssvd.Device(0)
mode = w.modes[-1]
prm = dict(block_size=w.L, moment_degree=w.M, quadrature_count=w.N)
A = orc.ProblemMatrix(a)
o20 = orc.run_solve(A, orc.RunConfig(w.a, w.b, mode=[orc.SS_SVD, orc.SS_SVD_NT][mode], params=orc.SsParams(**prm)),
                    gram_cap=1 << 30)


def span(res_triplets, in_interval):
    idx = np.flatnonzero(np.asarray(in_interval, bool))
    return res_triplets.right[:, idx], res_triplets.sigma[idx]


for delta in deltas:
    g = sssvd.run_solve(a, sssvd.RunConfig(w.a, w.b, mode=mode, gram_cap=1 << 30,
                                           params=sssvd.SsParams(lowrank_threshold=delta, **prm)), dev)
    ocfg = orc.RunConfig(w.a, w.b, mode=[orc.SS_SVD, orc.SS_SVD_NT][mode],
                         params=orc.SsParams(lowrank_threshold=delta, **prm))
    ro = orc.RunResult(input_transposed=A.transposed)
    ro.blocks, ro.starting_norm = o20.blocks, o20.starting_norm
    orc.finish_solve(A, ocfg, ro)
    rx = orc.RunResult(input_transposed=A.transposed)
    rx.blocks, rx.starting_norm = orc.MomentBlocks([np.array(b) for b in g.blocks.blocks]), o20.starting_norm
    orc.finish_solve(A, ocfg, rx)
    bd = max(np.linalg.norm(gb - ob) / np.linalg.norm(ob) for gb, ob in zip(g.blocks.blocks, o20.blocks.blocks))
    vg, sg = span(g.triplets, g.triplets.in_interval)
    vo, so = span(ro.triplets, ro.triplets.in_interval)
    vx, sx = span(rx.triplets, rx.triplets.in_interval)
    out = {"cfg": c, "delta": delta, "blocks_rel_diff": bd, "in_interval": [int(vg.shape[1]), int(vo.shape[1]), int(vx.shape[1])],
           "rank": [int(g.triplets.count()), int(ro.triplets.count()), int(rx.triplets.count())]}
    if vg.shape[1] == vo.shape[1] == vx.shape[1]:
        out["sin_G_O"] = principal_angle_sine(vg, vo)
        out["sin_G_X"] = principal_angle_sine(vg, vx)
        out["sin_O_X"] = principal_angle_sine(vo, vx)
        # all r Ritz vectors: the reduced subspace itself
        out["sin_all_G_O"] = principal_angle_sine(g.triplets.right, ro.triplets.right)
        out["sin_all_G_X"] = principal_angle_sine(g.triplets.right, rx.triplets.right)
        out["sin_all_O_X"] = principal_angle_sine(ro.triplets.right, rx.triplets.right)
        allo = np.sort(ro.triplets.sigma)
        ins = np.sort(so)
        outside = allo[(allo < w.a) | (allo > w.b)]
        out["ritz_gap"] = float(min(np.min(np.abs(outside[:, None] - ins[None, :]), axis=0))) if outside.size else None
        out["exact_median"] = [float(np.median(g.exact[np.asarray(g.triplets.in_interval, bool)])),
                               float(np.median(ro.residuals.exact[np.asarray(ro.triplets.in_interval, bool)]))]
    print(json.dumps(out), flush=True)
