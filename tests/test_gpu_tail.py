"""GPU parity of the small dense tail's hand-written kernels against LAPACK (numpy): the blocked
Householder QR (HouseholderQR in low_rank, moments.hpp:195-198, and project_qr, extract.hpp:43-57)
and the one-sided Jacobi SVD (JacobiSVD in low_rank and svd_small, extract.hpp:66-70)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def graded(m, k, seed, decades=17.0):
    """Columns scaled over `decades` orders of magnitude (the stacked-moment structure)."""
    rng = np.random.default_rng(seed)
    u, _ = np.linalg.qr(rng.standard_normal((m, k)))
    v, _ = np.linalg.qr(rng.standard_normal((k, k)))
    s = 10.0 ** (-decades * np.arange(k) / max(k - 1, 1))
    return (u * s) @ v.T


@pytest.mark.parametrize("m,k", [(700, 300), (4096, 512), (512, 512), (2000, 33), (13000, 64), (40, 1),
                                 (32768, 40), (2500, 1030), (1100, 1100)])
def test_thin_qr_matches_lapack(dev, m, k):
    rng = np.random.default_rng(m + k)
    a = rng.standard_normal((m, k))
    q, r = dev.thin_qr(a)
    _, r_ref = np.linalg.qr(a)
    scale = np.linalg.norm(a)
    assert np.linalg.norm(q @ r - a) <= 1e-14 * scale * np.sqrt(k)
    assert np.linalg.norm(q.T @ q - np.eye(k)) <= 1e-14 * np.sqrt(m * k)
    assert np.allclose(np.tril(r, -1), 0.0)
    # same reflector convention as LAPACK / Eigen: R agrees to rounding, signs included
    assert np.linalg.norm(r - r_ref) <= 1e-13 * np.linalg.norm(r_ref)


@pytest.mark.parametrize("m,k", [(70000, 48), (400000, 12), (33000, 700)])
def test_thin_qr_tall_tsqr(dev, m, k):
    """Above 32768 rows thin_qr runs one level of TSQR (the reference's HouseholderQR has no row
    limit; 60000 x 784 is the paper's MNIST shape): Q R = A, Q^T Q = I, R upper triangular and equal
    to LAPACK's up to the signs of its rows."""
    rng = np.random.default_rng(m + k)
    a = rng.standard_normal((m, k))
    q, r = dev.thin_qr(a)
    _, r_ref = np.linalg.qr(a)
    assert np.linalg.norm(q @ r - a) <= 1e-14 * np.linalg.norm(a) * np.sqrt(k)
    assert np.linalg.norm(q.T @ q - np.eye(k)) <= 1e-14 * np.sqrt(m * k)
    assert np.allclose(np.tril(r, -1), 0.0)
    sg = np.sign(np.diag(r)) * np.sign(np.diag(r_ref))
    assert np.linalg.norm(sg[:, None] * r - r_ref) <= 1e-13 * np.linalg.norm(r_ref)


def test_thin_qr_graded_and_rank_deficient(dev):
    a = graded(1500, 256, 3)
    a[:, 100] = a[:, 7]          # exact duplicate column
    a[:, 200] = 0.0              # zero column
    q, r = dev.thin_qr(a)
    assert np.linalg.norm(q @ r - a) <= 1e-15 * np.linalg.norm(a) * 16
    assert np.linalg.norm(q.T @ q - np.eye(256)) <= 1e-13
    _, r_ref = np.linalg.qr(a)
    d, d_ref = np.abs(np.diag(r)), np.abs(np.diag(r_ref))
    # the leading (well-determined) part of R's diagonal matches LAPACK; the dependent columns are
    # roundoff-level in both (project_qr's rank flag |R_ii| <= 1e-14 |R_00|)
    assert np.max(np.abs(d[:64] - d_ref[:64]) / d_ref[:64]) <= 1e-12
    assert d[200] <= 1e-14 * d[0] and d_ref[200] <= 1e-14 * d_ref[0]


@pytest.mark.parametrize("k", [64, 300, 512])
def test_svd_square_matches_lapack(dev, k):
    b = np.triu(graded(k, k, k, decades=12.0))
    u, s, v = dev.svd_square(b)
    s_ref = np.linalg.svd(b, compute_uv=False)
    assert np.all(np.diff(s) <= 0)
    # LAPACK's gesdd is only absolutely accurate (~eps sigma_max) on the tiny values
    assert np.all(np.abs(s - s_ref) <= 1e-9 * s_ref + 1e-14 * s_ref[0])
    assert np.linalg.norm(u * s @ v.T - b) <= 1e-13 * np.linalg.norm(b)
    assert np.linalg.norm(v.T @ v - np.eye(k)) <= 1e-12


@pytest.mark.parametrize("k", [777, 1024, 1500, 2048])
def test_svd_square_large_grid_kernel(dev, k):
    """k > 512: the whole-GPU block Jacobi (configs 3 and 5 have k = 1024 and 2048).
    Rounding grows with the k - 1 rotations per column per sweep: bounds scale with k eps."""
    b = np.triu(graded(k, k, k, decades=10.0))
    u, s, v = dev.svd_square(b)
    s_ref = np.linalg.svd(b, compute_uv=False)
    assert np.all(np.diff(s) <= 0)
    assert np.all(np.abs(s - s_ref) <= 1e-9 * s_ref + 1e-14 * s_ref[0])
    assert np.linalg.norm(u * s @ v.T - b) <= 4e-15 * k * np.linalg.norm(b)
    assert np.linalg.norm(v.T @ v - np.eye(k)) <= 2e-14 * k   # Frobenius: ~1e-14 per entry
