"""The reference-side C++ binding (include/sssvd_gpu.hpp) compiled and run on the GPU:
GpuMomentAccumulator::accumulate and run_solve(ProblemMatrix, RunConfig) -> RunResult against the
oracle (acceptance model 1, problems.hpp:50-70; acceptance.cpp:108-121), and the reference's error
behaviour through the binding (sssvd::NumericalError, empty result)."""
import os
import subprocess

import numpy as np
import pytest

from oracle import sssvd_oracle as orc

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_binding_accumulate_and_run_solve(tmp_path):
    from paper_2109_13655_b200 import build
    build.build()
    exe = tmp_path / "binding_gpu"
    libdir = os.path.join(ROOT, "paper_2109_13655_b200")
    subprocess.run(["g++", "-O2", "-std=c++20", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "binding_gpu.cpp"), "-o", str(exe), "-L", libdir,
                    "-lsssvd_gpu", f"-Wl,-rpath,{libdir}"], check=True)
    am, _, sigma, _ = orc.build_model(1)
    a = am.dense
    lo, hi, L, M, N = 0.8, 1.2, 20, 4, 32
    inp, out = tmp_path / "in.bin", tmp_path / "out.bin"
    with open(inp, "wb") as f:
        np.array(a.shape, dtype=np.int64).tofile(f)
        np.array([lo, hi]).tofile(f)
        np.array([L, M, N], dtype=np.int64).tofile(f)
        np.asfortranarray(a).T.astype(np.float64).tofile(f)
    r = subprocess.run([str(exe), str(inp), str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    raw = np.fromfile(out, dtype=np.float64)
    ints = raw.view(np.int64)
    nb = int(ints[0])
    blocks = raw[1:1 + nb]
    p = 1 + nb
    t = int(ints[p]); p += 1
    sig, tau, spur, exact, gal = (raw[p + k * t:p + (k + 1) * t] for k in range(5))
    p += 5 * t
    cin, cns, rank, far_empty, caught = (int(x) for x in ints[p:p + 5])
    # accumulate vs the oracle's MomentAccumulator (moments.hpp:132-147)
    g = orc.form_gram(am)
    rule = orc.ContourRule(lo, hi, N, 0.1, orc.SpectralTransform(orc.IDENTITY))
    ref = orc.MomentAccumulator(g, rule).accumulate(orc.random_start(a.shape[1], L, 42), M).blocks
    n = a.shape[1]
    for k in range(M + 1):
        blk = blocks[k * n * L:(k + 1) * n * L].reshape((L, n)).T
        assert np.linalg.norm(blk - ref[k]) <= 1e-11 * np.linalg.norm(ref[k])
    # run_solve: acceptance criterion 1 (exactly 40 non-spurious, error <= 1e-10, residual <= 1e-9)
    assert cns == 40 and cin >= 40 and rank == L * M
    ns = [i for i in range(t) if lo <= sig[i] <= hi and spur[i] == 0.0]
    assert len(ns) == 40
    assert max(np.min(np.abs(sigma - s)) / s for s in sig[ns]) <= 1e-10
    assert max(exact[ns]) <= 1e-9 and max(gal[ns]) <= 1e-9
    # [5, 6] lies far above sigma_max = 1.195: the oracle's filter annihilates the block there too
    far = orc.run_solve(am, orc.RunConfig(5.0, 6.0, params=orc.SsParams(block_size=L, moment_degree=M, quadrature_count=N)))
    assert far.empty and far_empty == 1
    assert caught == 1
