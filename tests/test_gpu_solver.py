"""GPU parity for the shifted solves, re-expressing proj/tests/test_solver.cpp against the
sm_100a library (Gram kernel, batched blocked LU, back substitution) through the C ABI."""
import numpy as np
import pytest

from oracle import sssvd_oracle as orc

pytestmark = pytest.mark.gpu


def sym(n, seed):
    g = orc.random_matrix(n, n, seed)
    return (g + g.T) / 2


def test_gram_identity_and_orthogonal_columns(dev):
    from paper_2109_13655_b200 import sssvd
    g = sssvd.form_gram(sssvd.ProblemMatrix.from_dense(np.eye(3)))
    assert np.linalg.norm(g - np.eye(3)) == 0.0                     # test_solver.cpp:31-33
    a = np.array([[1, 0], [0, 2], [0, 0]], dtype=float)
    g = sssvd.form_gram(sssvd.ProblemMatrix.from_dense(a))
    assert np.linalg.norm(g - np.diag([1.0, 4.0])) == 0.0


@pytest.mark.parametrize("m,n", [(50, 20), (300, 200), (2000, 1000), (1037, 517)])
def test_gram_matches_triple_loop_product(dev, m, n):
    from paper_2109_13655_b200 import sssvd
    a = orc.random_matrix(m, n, 123)
    g = sssvd.form_gram(sssvd.ProblemMatrix.from_dense(a))
    ref = a.T @ a                                                     # test_solver.cpp:38-48
    assert np.linalg.norm(g - ref) / np.linalg.norm(ref) <= 1e-15 * max(1, m / 50) ** 0.5
    assert np.linalg.norm(g - g.T) == 0.0


def test_gram_cap(dev):
    from paper_2109_13655_b200 import sssvd
    with pytest.raises(sssvd.LengthError):                            # test_solver.cpp:50-53
        sssvd.form_gram(sssvd.ProblemMatrix.from_dense(np.eye(10)), size_cap=8)


def test_diagonal_closed_form(dev):
    from paper_2109_13655_b200 import sssvd
    g = np.diag([1.0, 4.0])
    fact = sssvd.factor_shift(g, complex(2, 1))
    x = sssvd.solve_block(fact, np.eye(2, dtype=complex))            # test_solver.cpp:55-67
    assert abs(x[0, 0] - complex(0.5, -0.5)) <= 1e-15
    assert abs(x[1, 0]) <= 1e-15
    assert abs(x[1, 1] - complex(-0.4, -0.2)) <= 1e-15


@pytest.mark.parametrize("n,L", [(20, 5), (100, 7), (600, 16), (1500, 32), (3000, 20), (8192, 4)])   # 8192: NB = 256
def test_residual_bound_random_symmetric(dev, n, L):
    from paper_2109_13655_b200 import sssvd
    g = sym(n, 7)
    z = complex(1.04, 0.4)
    x = sssvd.solve_block(sssvd.factor_shift(g, z), orc.random_matrix(n, L, 8).astype(complex))
    rhs = orc.random_matrix(n, L, 8)
    shifted = -g.astype(complex) + z * np.eye(n)
    for c in range(L):                                                # test_solver.cpp:69-82
        res = np.linalg.norm(shifted @ x[:, c] - rhs[:, c]) / np.linalg.norm(rhs[:, c])
        assert res <= 1e-12 * max(1.0, n / 100)


def test_matches_lapack_zgetrs(dev):
    """GPU LU+solve against the oracle's zgetrf/zgetrs (the restated PartialPivLU)."""
    from paper_2109_13655_b200 import sssvd
    n, L = 700, 12
    a = orc.random_matrix(900, n, 3)
    g = a.T @ a
    g = (g + g.T) / 2
    z = complex(0.9, 0.05)
    v = orc.random_start(n, L, 42)
    x = sssvd.solve_block(sssvd.factor_shift(g, z), v.astype(complex))
    xo = orc.ShiftedFactorization(g, z).solve(v)
    assert np.linalg.norm(x - xo) / np.linalg.norm(xo) <= 1e-11


def test_zero_rhs(dev):
    from paper_2109_13655_b200 import sssvd
    x = sssvd.solve_block(sssvd.factor_shift(np.eye(4), complex(2, 0.5)), np.zeros((4, 3), complex))
    assert np.linalg.norm(x) == 0.0                                   # test_solver.cpp:84-89


def test_eigenvector_rhs(dev):
    from paper_2109_13655_b200 import sssvd
    g = sym(12, 3)
    lam, vec = np.linalg.eigh(g)
    z = complex(0.7, 0.3)
    fact = sssvd.factor_shift(g, z)
    for k in (0, 5, 11):                                              # test_solver.cpp:91-104
        x = sssvd.solve_block(fact, vec[:, k].astype(complex))[:, 0]
        expected = vec[:, k] / (z - lam[k])
        assert np.linalg.norm(x - expected) <= 1e-10 * np.linalg.norm(expected)


def test_block_equals_columns(dev):
    from paper_2109_13655_b200 import sssvd
    g = sym(15, 5)
    fact = sssvd.factor_shift(g, complex(0.2, 0.9))
    rhs = orc.random_matrix(15, 20, 6).astype(complex)
    block = sssvd.solve_block(fact, rhs)
    for c in range(20):                                               # test_solver.cpp:106-116
        single = sssvd.solve_block(fact, rhs[:, c])[:, 0]
        assert np.linalg.norm(block[:, c] - single) <= 1e-14 * np.linalg.norm(single)


def test_conjugate_shift(dev):
    from paper_2109_13655_b200 import sssvd
    g = sym(10, 9)
    rhs = orc.random_matrix(10, 4, 10).astype(complex)
    z = complex(0.5, 0.25)
    x = sssvd.solve_block(sssvd.factor_shift(g, z), rhs)
    xc = sssvd.solve_block(sssvd.factor_shift(g, z.conjugate()), rhs)
    assert np.linalg.norm(x - xc.conj()) <= 1e-13 * np.linalg.norm(x)  # test_solver.cpp:118-126


def test_shift_on_spectrum_rejected(dev):
    from paper_2109_13655_b200 import sssvd
    with pytest.raises(sssvd.NumericalError):                         # test_solver.cpp:128-132
        sssvd.factor_shift(np.diag([1.0, 4.0]), complex(1.0, 0.0))


def test_dimension_mismatch(dev):
    from paper_2109_13655_b200 import sssvd
    fact = sssvd.factor_shift(np.eye(4), complex(2, 1))
    with pytest.raises(ValueError):                                   # test_solver.cpp:134-138
        sssvd.solve_block(fact, np.zeros((5, 2), complex))


def test_pivoting_is_exercised(dev):
    """A matrix whose natural pivots are tiny: without row interchanges the LU would blow up."""
    from paper_2109_13655_b200 import sssvd
    n = 257
    rng = np.random.default_rng(5)
    u, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.linspace(0.0, 2.0, n)
    g = (u * lam) @ u.T
    g = (g + g.T) / 2
    z = complex(1.0, 1e-6)     # tiny imaginary part: ill-conditioned and pivot-hungry
    rhs = rng.standard_normal((n, 3)).astype(complex)
    x = sssvd.solve_block(sssvd.factor_shift(g, z), rhs)
    xo = orc.ShiftedFactorization(g, z).solve(rhs.real)
    assert np.linalg.norm(x - xo) / np.linalg.norm(xo) <= 1e-6
    shifted = -g + z * np.eye(n)
    # normwise backward error of GEPP, no worse than 10x LAPACK's on the same system
    berr = np.linalg.norm(shifted @ x - rhs) / (np.linalg.norm(shifted, 2) * np.linalg.norm(x) + np.linalg.norm(rhs))
    berr_o = np.linalg.norm(shifted @ xo - rhs) / (np.linalg.norm(shifted, 2) * np.linalg.norm(xo) + np.linalg.norm(rhs))
    assert berr <= max(1e-15, 10 * berr_o)


def test_gram_sharding_is_exact(dev):
    """Multi-GPU form_gram: the round-robin tile shares of 3 ranks sum to the single-GPU G bitwise
    (every entry is written by exactly one share)."""
    from paper_2109_13655_b200 import sssvd
    a = orc.random_matrix(700, 333, 77)
    g = sssvd.form_gram(sssvd.ProblemMatrix.from_dense(a), device=dev)
    parts = []
    for p in range(3):
        out = np.empty((333, 333), order="F")
        dev.check(sssvd.lib().sssvd_debug_gram_part(dev.h, p, 3, sssvd._ptr(out)))
        parts.append(out)
    assert np.array_equal(parts[0] + parts[1] + parts[2], g)
    assert all(np.count_nonzero(p) > 0 for p in parts)


@pytest.mark.parametrize("variant", [0, 1, 2])
@pytest.mark.parametrize("m,n,k,batch", [(200, 136, 128, 3), (64, 64, 16, 1), (77, 35, 9, 2), (1000, 1016, 64, 2),
                                         (3968, 4000, 128, 2), (513, 129, 256, 1), (1, 1, 1, 1), (65, 49, 33, 2)])
def test_zgemm_kernels_agree(dev, variant, m, n, k, batch):
    """The TMA + mbarrier trailing-update GEMM (variant 1) issues the same DMMA chain per entry of C
    as the 4-product cp.async kernel (variant 0): bitwise-equal C, ragged edges and K not a
    multiple of 16 included (TMA zero-fills out-of-bounds boxes). The 3-product (3M) kernel
    (variant 2, the product default, 64 x 48 tiles) agrees with it within the 3M rounding bound
    (K * 1e-15 on operands in [-0.5, 0.5]; the library counts the entries beyond it)."""
    import ctypes
    from paper_2109_13655_b200 import sssvd
    ms, mism = ctypes.c_double(), ctypes.c_int64()
    dev.check(sssvd.lib().sssvd_debug_zgemm(dev.h, variant, m, n, k, batch, 1, ctypes.byref(ms), ctypes.byref(mism)))
    assert mism.value == 0


@pytest.mark.parametrize("trans_a", [False, True])
@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (64, 64, 16), (77, 35, 9), (130, 67, 301), (33, 96, 5000),
                                   (128, 128, 16384), (1000, 513, 64), (5, 3, 0)])
def test_dgemm_matches_numpy(dev, trans_a, m, n, k):
    """Tail GEMM (dgemm.cu) vs numpy float64: NN and TN, ragged tiles, the split-K path (deep K,
    few tiles), K = 0, alpha/beta, and odd leading dimensions (8-byte staging)."""
    rng = np.random.default_rng(m * 7 + n * 3 + k)
    a = rng.standard_normal((k, m) if trans_a else (m, k))
    b = rng.standard_normal((k, n))
    c = rng.standard_normal((m, n))
    ref = 0.5 * ((a.T if trans_a else a) @ b) - 1.25 * c
    scale = np.sqrt(max(k, 1)) * 4
    for pads in [(None, None, None), (a.shape[0] + 1, k + 3, m + 1)]:
        got = dev.dgemm(a, b, c, alpha=0.5, beta=-1.25, trans_a=trans_a, lda=pads[0], ldb=pads[1], ldc=pads[2])
        assert np.max(np.abs(got - ref)) <= 1e-14 * scale * max(1.0, np.max(np.abs(ref)))
    # beta = 0 never reads C (NaN in C must not leak)
    cn = np.full((m, n), np.nan)
    got = dev.dgemm(a, b, cn, trans_a=trans_a)
    assert np.all(np.isfinite(got))
    assert np.max(np.abs(got - (a.T if trans_a else a) @ b), initial=0.0) <= 1e-14 * scale * 4


@pytest.mark.parametrize("trans_a", [False, True])
@pytest.mark.parametrize("m,n,k", [(300, 70, 45), (64, 1, 128), (1025, 130, 77)])
def test_dgemm_fused_residual_norms(dev, trans_a, m, n, k):
    """The fused residual epilogue ||op(A) B_j - d_j V_j|| (exact / Galerkin / transformed
    residuals, postprocess.hpp:34-41, :91-95; pipeline.hpp:203-208) against numpy."""
    rng = np.random.default_rng(m + n + k)
    a = rng.standard_normal((k, m) if trans_a else (m, k))
    b = rng.standard_normal((k, n))
    d = rng.standard_normal(n)
    v = rng.standard_normal((m, n))
    ref = np.linalg.norm((a.T if trans_a else a) @ b - v * d[None, :], axis=0)
    got = dev.dgemm_colnorm_diff(a, b, d, v, trans_a=trans_a)
    assert np.allclose(got, ref, rtol=1e-12, atol=0)
