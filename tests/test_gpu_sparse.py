"""GPU parity of the sparse operator path: ProblemMatrix::from_sparse
(problem.hpp:27-35), the sparse Gram (problem.hpp:87-89) and run_solve on sparse input, through
sssvd_gpu_set_operator_csc, against the CPU oracle's scipy-sparse restatement."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import sssvd_oracle as orc
from test_gpu_pipeline import compare_with_oracle

pytestmark = pytest.mark.gpu


def sparse_matrix(m, n, density, seed):
    rng = np.random.default_rng(seed)
    a = sp.random(m, n, density=density, random_state=rng, data_rvs=rng.standard_normal, format="csc")
    a = a + sp.eye(m, n, format="csc") * 0.5       # no empty columns
    return sp.csc_matrix(a)


def interval_with_gaps(sigma, lo_idx, hi_idx):
    """[a, b] around sigma[lo_idx..hi_idx] (ascending), endpoints mid-gap."""
    s = np.sort(sigma)
    return 0.5 * (s[lo_idx - 1] + s[lo_idx]), 0.5 * (s[hi_idx] + s[hi_idx + 1])


def test_sparse_gram_matches_oracle_and_dense_upload(dev):
    from paper_2109_13655_b200 import sssvd
    a = sparse_matrix(3000, 500, 0.02, 1)
    g_sp = sssvd.form_gram(sssvd.ProblemMatrix.from_sparse(a), device=dev)
    g_dn = sssvd.form_gram(sssvd.ProblemMatrix.from_dense(a.toarray()), device=dev)
    assert np.array_equal(g_sp, g_dn)          # densified in HBM: the same operator bit for bit
    ref = orc.form_gram(orc.ProblemMatrix(a))  # sparse product, then (G + G^T)/2
    assert np.linalg.norm(g_sp - ref) / np.linalg.norm(ref) <= 1e-14
    assert np.array_equal(g_sp, g_sp.T)


@pytest.mark.parametrize("shape", [(1200, 400), (300, 900)])
def test_sparse_run_solve_equals_dense_bitwise(dev, shape):
    """Same matrix uploaded sparse and dense (tall, and wide -> stored transposed): identical
    triplets, verdicts and residuals."""
    from paper_2109_13655_b200 import sssvd
    a = sparse_matrix(*shape, 0.03, 2)
    sigma = np.linalg.svd(a.toarray(), compute_uv=False)
    lo, hi = interval_with_gaps(sigma, 150, 165)
    cfg = sssvd.RunConfig(lo, hi, params=sssvd.SsParams(block_size=12, moment_degree=4, quadrature_count=32))
    rs = sssvd.run_solve(sssvd.ProblemMatrix.from_sparse(a), cfg, dev)
    rd = sssvd.run_solve(a.toarray(), cfg, dev)
    assert rs.input_transposed == (shape[0] < shape[1]) == rd.input_transposed
    assert rs.triplets.count() == rd.triplets.count() > 0
    assert np.array_equal(rs.triplets.sigma, rd.triplets.sigma)
    assert np.array_equal(rs.tau, rd.tau) and np.array_equal(rs.exact, rd.exact)
    assert np.array_equal(rs.triplets.left, rd.triplets.left)
    assert rs.triplets.left.shape[0] == shape[0] and rs.triplets.right.shape[0] == shape[1]


@pytest.mark.parametrize("mode", ["ss-svd", "ss-svd-nt"])
def test_sparse_run_solve_parity_with_oracle(dev, mode):
    from paper_2109_13655_b200 import sssvd
    a = sparse_matrix(2000, 600, 0.01, 3)
    sigma = np.linalg.svd(a.toarray(), compute_uv=False)
    lo, hi = interval_with_gaps(sigma, 300, 312)
    nt = mode == "ss-svd-nt"
    cfg = sssvd.RunConfig(lo, hi, mode=sssvd.SolveMode.SsSvdNT if nt else sssvd.SolveMode.SsSvd,
                          params=sssvd.SsParams(block_size=16, moment_degree=4, quadrature_count=32))
    res = sssvd.run_solve(sssvd.ProblemMatrix.from_sparse(a), cfg, dev)
    ocfg = orc.RunConfig(lo, hi, mode=orc.SS_SVD_NT if nt else orc.SS_SVD,
                         params=orc.SsParams(block_size=16, moment_degree=4, quadrature_count=32))
    ores = orc.run_solve(orc.ProblemMatrix(a), ocfg)
    compare_with_oracle(res, ores, sigma.max(), lo, hi)
    for k in range(5):
        ref = ores.blocks.blocks[k]
        assert np.linalg.norm(res.blocks.blocks[k] - ref) / np.linalg.norm(ref) <= 1e-10


def test_permuted_diagonal_exact_spectrum(dev):
    """A = P diag(s) Q (P, Q permutations): singular values known exactly; acceptance-style
    accuracy bounds (acceptance.cpp:108-121)."""
    from paper_2109_13655_b200 import sssvd
    m, n = 900, 300
    rng = np.random.default_rng(4)
    s = 0.005 + 0.01 * np.arange(n)
    rows = rng.permutation(m)[:n]
    cols = rng.permutation(n)
    a = sp.csc_matrix((s, (rows, cols)), shape=(m, n))
    lo, hi = 0.8, 1.2
    cfg = sssvd.RunConfig(lo, hi, params=sssvd.SsParams(block_size=16, moment_degree=4, quadrature_count=32))
    res = sssvd.run_solve(sssvd.ProblemMatrix.from_sparse(a), cfg, dev)
    inside = s[(s >= lo) & (s <= hi)]
    idx = [i for i in range(res.triplets.count()) if res.triplets.in_interval[i] and not res.spurious[i]]
    assert res.count_nonspurious_in_interval == inside.size == 40
    got = np.sort(res.triplets.sigma[idx])
    assert np.max(np.abs(got - inside) / inside) <= 1e-10
    assert np.all(res.exact[idx] <= 1e-9)


def test_malformed_csc_rejected(dev):
    from paper_2109_13655_b200 import sssvd
    cp = np.array([0, 2, 3])
    with pytest.raises(ValueError, match="compressed CSC"):          # unsorted rows in column 0
        dev.set_operator_csc(4, 2, cp, np.array([2, 1, 0]), np.ones(3))
    with pytest.raises(ValueError, match="compressed CSC"):          # duplicate row
        dev.set_operator_csc(4, 2, cp, np.array([1, 1, 0]), np.ones(3))
    with pytest.raises(ValueError, match="compressed CSC"):          # row out of range
        dev.set_operator_csc(4, 2, cp, np.array([0, 4, 0]), np.ones(3))
    with pytest.raises(ValueError, match="compressed CSC"):          # colptr not ending at nnz
        dev.set_operator_csc(4, 2, np.array([0, 2, 2]), np.array([0, 1, 0]), np.ones(3))
    with pytest.raises(ValueError, match="compressed CSC"):          # decreasing colptr
        dev.set_operator_csc(4, 2, np.array([0, 3, 2]), np.array([0, 1, 2]), np.ones(3))
    with pytest.raises(ValueError, match="NaN/Inf"):
        dev.set_operator_csc(4, 2, cp, np.array([0, 1, 0]), np.array([1.0, np.inf, 2.0]))
    dev.set_operator_csc(4, 2, cp, np.array([0, 3, 1]), np.array([1.0, 2.0, 3.0]))   # well-formed
    g = dev.form_gram()
    assert np.array_equal(g, np.array([[5.0, 0.0], [0.0, 9.0]]))


def test_matrix_market_file_through_run_solve(dev, tmp_path):
    """.mtx (coordinate) -> read_matrix_market -> run_solve equals the in-memory sparse run."""
    from paper_2109_13655_b200 import sssvd
    a = sparse_matrix(800, 250, 0.03, 5)
    pm = sssvd.ProblemMatrix.from_sparse(a)
    path = str(tmp_path / "a.mtx")
    sssvd.write_matrix_market(path, pm, "test")
    back = sssvd.read_matrix_market(path)
    assert back.is_sparse() and np.array_equal(back.to_dense(), pm.to_dense())
    sigma = np.linalg.svd(a.toarray(), compute_uv=False)
    lo, hi = interval_with_gaps(sigma, 100, 110)
    cfg = sssvd.RunConfig(lo, hi, params=sssvd.SsParams(block_size=12, moment_degree=4, quadrature_count=16))
    r1, r2 = sssvd.run_solve(back, cfg, dev), sssvd.run_solve(pm, cfg, dev)
    assert np.array_equal(r1.triplets.sigma, r2.triplets.sigma) and r1.count_nonspurious_in_interval > 0
