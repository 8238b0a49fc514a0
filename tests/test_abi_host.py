"""CPU-side checks of the drop-in boundary: libsssvd_gpu.so loads, exports every symbol that
include/sssvd_gpu.h declares, its host mirrors of the reference's O(N) logic are bit-identical
to the oracle, and compute entry points fail loudly (no CPU fallback) without a B200."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import sssvd_oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "sssvd_gpu.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sssvd_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2109_13655_b200 import sssvd
    lib = sssvd.lib()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(sssvd.EXPORTED_SYMBOLS)
    assert b"sm_100a" in lib.sssvd_build_info()


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_2109_13655_b200", "libsssvd_gpu.so")
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {so} 2>/dev/null").read()
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_sass_uses_fp64_tensor_cores():
    so = os.path.join(ROOT, "paper_2109_13655_b200", "libsssvd_gpu.so")
    sass = os.popen(f"/usr/local/cuda/bin/cuobjdump -sass {so} 2>/dev/null").read()
    funcs = sass.split("Function : ")
    zg = [f for f in funcs if "zgemm_kernel" in f[:60]]
    z3 = [f for f in funcs if "zgemm3m_kernel" in f[:60]]
    tm = [f for f in funcs if "zgemm_tma_kernel" in f[:60]]
    gr = [f for f in funcs if f.startswith("_ZN9sssvd_gpu11gram_kernel")]
    assert z3 and z3[0].count("DMMA.8x8x4") >= 144   # 3M trailing update: 36 DMMAs per k-quad, 4 k-quads per stage
    assert "LDGSTS" in z3[0] and "LDL" not in z3[0]  # cp.async staging, no register spill
    assert zg and "DMMA.8x8x4" in zg[0]        # 4-product kernel (gather-GEMM, A/B comparator)
    assert tm and "UTMALDG" in tm[0]           # its TMA form
    assert gr and "DMMA.8x8x4" in gr[0]        # Gram on the FP64 tensor pipe


@pytest.mark.parametrize("a,b,N,aspect,kind", [(0.8, 1.2, 32, 0.1, 0), (1e-3, 1e-1, 32, 0.1, 1),
                                               (0.45, 0.55, 32, 0.1, 1), (0.8, 0.9, 128, 0.1, 0),
                                               (0.5, 0.501, 64, 0.1, 1), (0.5, 1.5, 4, 1.0, 0)])
def test_contour_bit_identical_to_oracle(a, b, N, aspect, kind):
    from paper_2109_13655_b200 import sssvd
    r = sssvd.ContourRule(a, b, N, aspect, sssvd.SpectralTransform(kind))
    o = orc.ContourRule(a, b, N, aspect, orc.SpectralTransform(orc.EXP if kind else orc.IDENTITY))
    assert np.array_equal(r.nodes(), o.nodes) and np.array_equal(r.weights(), o.weights)
    assert r.center() == o.center and r.radius() == o.radius
    for j in range(N // 2):
        assert r.shift(j) == o.shift(j)


def test_contour_errors():
    from paper_2109_13655_b200 import sssvd
    with pytest.raises(ValueError):
        sssvd.ContourRule(0.8, 1.2, 31, 0.1, sssvd.SpectralTransform.identity())
    with pytest.raises(sssvd.DomainError):
        sssvd.ContourRule(0.0, 1.2, 32, 0.1, sssvd.SpectralTransform.exponential())


@pytest.mark.parametrize("n,L,seed", [(200, 20, 3141), (1000, 16, 42), (4096, 32, 42), (17, 3, 1)])
def test_random_start_bit_identical(n, L, seed):
    from paper_2109_13655_b200 import sssvd
    assert np.array_equal(sssvd.random_start(n, L, seed), orc.random_start(n, L, seed))


def test_moment_coefficients_bit_identical():
    from paper_2109_13655_b200 import sssvd
    o = orc.ContourRule(1e-3, 1e-1, 64, 0.1, orc.SpectralTransform(orc.EXP))
    h = 32
    c = sssvd.moment_coefficients(o.weights[:h], o.nodes[:h], 16)
    power = [1 + 0j] * h
    for k in range(17):                                     # moments.hpp:138-144
        for j in range(h):
            assert c[k, j] == complex(o.weights[j]) * power[j]
            power[j] *= complex(o.nodes[j])


def test_params_validation_mirror():
    from paper_2109_13655_b200 import sssvd
    sssvd.SsParams().validate(200)
    for bad, n in ((sssvd.SsParams(), 50), (sssvd.SsParams(lowrank_threshold=0.0), 200),
                   (sssvd.SsParams(quadrature_count=31), 200), (sssvd.SsParams(block_size=0), 200)):
        with pytest.raises(ValueError):
            bad.validate(n)


@pytest.mark.parametrize("h,G", [(16, 1), (16, 2), (16, 8), (64, 8), (17, 4), (3, 8)])
def test_shard_ranges_partition(h, G):
    from paper_2109_13655_b200 import sssvd
    spans = [sssvd.shard_range(h, G, r) for r in range(G)]
    assert spans[0][0] == 0 and spans[-1][1] == h
    for (b0, e0), (b1, _) in zip(spans, spans[1:]):
        assert e0 == b1
    sizes = [e - b for b, e in spans]
    assert max(sizes) - min(sizes) <= 1


def test_default_config_matches_reference():
    from paper_2109_13655_b200 import sssvd
    c = sssvd._Config()
    sssvd.lib().sssvd_default_config(ctypes.byref(c))
    assert (c.params.block_size, c.params.moment_degree, c.params.quadrature_count) == (20, 4, 32)
    assert c.params.lowrank_threshold == 1e-20 and c.params.spurious_threshold == 1e-8
    assert c.params.seed == 42 and c.aspect == 0.1 and c.gram_cap == 8192
    assert c.estimator_rcond_identity == 2e-15 and c.estimator_rcond_exp == 1e-14


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2109_13655_b200 import sssvd
    with pytest.raises(sssvd.CudaError):
        sssvd.Device(0)


def test_cpp_binding_compiles_and_maps_errors(tmp_path):
    """include/sssvd_gpu.hpp (the reference-side binding) builds with g++ -std=c++20
    against the library and maps status codes onto the reference's exception types."""
    import subprocess
    import torch
    exe = tmp_path / "abi_smoke"
    lib = os.path.join(ROOT, "paper_2109_13655_b200")
    subprocess.check_call(["g++", "-std=c++20", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cpp", "abi_smoke.cpp"), "-L", lib, "-lsssvd_gpu",
                           f"-Wl,-rpath,{lib}", "-o", str(exe)])
    args = [str(exe)] + (["gpu"] if torch.cuda.is_available() else [])
    out = subprocess.run(args, capture_output=True, text=True)
    assert out.returncode == 0 and "abi_smoke ok" in out.stdout, out.stdout + out.stderr
