"""GPU parity for the moment accumulation (MomentAccumulator, moments.hpp:101-169), re-expressing
proj/tests/test_moments.cpp against the sm_100a path and comparing with the CPU oracle."""
import numpy as np
import pytest

from oracle import sssvd_oracle as orc

pytestmark = pytest.mark.gpu


def constructed(m, n, sigma, su, sv):
    u, _ = np.linalg.qr(orc.random_matrix(m, n, su))
    v, _ = np.linalg.qr(orc.random_matrix(n, n, sv))
    return (u * sigma[None, :]) @ v.T


def gpu_blocks(dev, a, rule, s0, degree, ell=1):
    from paper_2109_13655_b200 import sssvd
    dev.set_operator(a)
    dev.form_gram(1 << 30, copy_out=False)
    acc = sssvd.MomentAccumulator(rule, dev)
    if ell == 1:
        return acc.accumulate(s0, degree).blocks
    return acc._run(s0, ell, degree)


def rules(a, b, N, aspect, exp=False):
    from paper_2109_13655_b200 import sssvd
    tf = sssvd.SpectralTransform.exponential() if exp else sssvd.SpectralTransform.identity()
    return (sssvd.ContourRule(a, b, N, aspect, tf),
            orc.ContourRule(a, b, N, aspect, orc.SpectralTransform("exp" if exp else "identity")))


def test_moment_identity_identity_transform(dev):
    n = 40
    a = constructed(80, n, 0.2 + 0.04 * np.arange(n), 51, 52)
    g = a.T @ a
    rg, _ = rules(0.8, 1.2, 32, 0.1)
    s0 = orc.random_start(n, 10, 7)
    blocks = gpu_blocks(dev, a, rg, s0, 4)
    assert len(blocks) == 5
    power = blocks[0]
    for k in range(1, 5):                                             # test_moments.cpp:116-139
        power = g @ power
        assert np.linalg.norm(blocks[k] - power) / np.linalg.norm(power) <= 1e-8
    splus, stacked = np.hstack(blocks[1:]), np.hstack(blocks[:4])
    assert np.linalg.norm(splus - g @ stacked) / np.linalg.norm(g @ stacked) <= 1e-8


@pytest.mark.parametrize("m,n,L,M,N,exp", [(80, 40, 10, 4, 32, False), (300, 200, 8, 3, 16, True),
                                            (2000, 1000, 16, 8, 32, True), (1500, 1100, 20, 4, 32, False)])
def test_moments_match_oracle(dev, m, n, L, M, N, exp):
    a = constructed(m, n, np.linspace(0.01, 1.0, n), 11, 12)
    lo, hi = (0.45, 0.55)
    rg, ro = rules(lo, hi, N, 0.1, exp)
    s0 = orc.random_start(n, L, 42)
    blocks = gpu_blocks(dev, a, rg, s0, M)
    ref = orc.MomentAccumulator(orc.form_gram(orc.ProblemMatrix(a), 1 << 30), ro).accumulate(s0, M).blocks
    for k in range(M + 1):
        err = np.linalg.norm(blocks[k] - ref[k]) / np.linalg.norm(ref[k])
        assert err <= 1e-10, (k, err)


def test_three_product_update_matches_four_product(monkeypatch):
    """The LU's trailing updates use the 3-product (3M) complex GEMM by default; SSSVD_ZGEMM=4m
    selects the 4-product kernel. Both paths' moment blocks agree with each other to roundoff times
    the conditioning of the shifted solves, and each is as close to the oracle as the other
    (profiles/r02_3m_sensitivity.txt has the full-size configs)."""
    from paper_2109_13655_b200 import sssvd
    m, n, L, M, N = 2000, 1000, 16, 8, 32
    a = constructed(m, n, np.linspace(0.01, 1.0, n), 11, 12)
    rg, ro = rules(0.45, 0.55, N, 0.1, True)
    s0 = orc.random_start(n, L, 42)
    ref = orc.MomentAccumulator(orc.form_gram(orc.ProblemMatrix(a), 1 << 30), ro).accumulate(s0, M).blocks
    out = {}
    for kernel in ("3m", "4m"):
        monkeypatch.setenv("SSSVD_ZGEMM", kernel)
        out[kernel] = gpu_blocks(sssvd.Device(0), a, rg, s0, M)   # a fresh context: no captured pass is replayed
    monkeypatch.delenv("SSSVD_ZGEMM")
    e3 = max(np.linalg.norm(out["3m"][k] - ref[k]) / np.linalg.norm(ref[k]) for k in range(M + 1))
    e4 = max(np.linalg.norm(out["4m"][k] - ref[k]) / np.linalg.norm(ref[k]) for k in range(M + 1))
    d34 = max(np.linalg.norm(out["3m"][k] - out["4m"][k]) / np.linalg.norm(ref[k]) for k in range(M + 1))
    assert d34 > 0                       # the two kernels really are different arithmetic
    assert e3 <= 1e-10 and e4 <= 1e-10 and d34 <= 1e-10
    assert e3 <= 5 * e4 + 1e-13, (e3, e4)   # 3M is not measurably further from the oracle


def test_batching_does_not_change_result(dev):
    """test_moments.cpp:205-215 (worker count) -> shifts-in-flight count: bitwise identical."""
    a = orc.random_matrix(300, 160, 91)
    rg, _ = rules(0.5, 2.0, 32, 0.1)
    s0 = orc.random_start(160, 5, 11)
    dev.set_batch(16)
    b16 = gpu_blocks(dev, a, rg, s0, 3)
    dev.set_batch(1)
    b1 = gpu_blocks(dev, a, rg, s0, 3)
    dev.set_batch(5)
    b5 = gpu_blocks(dev, a, rg, s0, 3)
    dev.set_batch(0)
    for k in range(4):
        assert np.array_equal(b16[k], b1[k]) and np.array_equal(b16[k], b5[k])


def test_refinement_fixed_map_on_invariant_block(dev):
    from paper_2109_13655_b200 import sssvd
    n = 40
    sigma = 0.3 + 0.05 * np.arange(n)
    u, _ = np.linalg.qr(orc.random_matrix(60, n, 21))
    v, _ = np.linalg.qr(orc.random_matrix(n, n, 22))
    a = (u * sigma) @ v.T
    rg, _ = rules(0.8, 1.2, 32, 0.1)
    inside = [i for i in range(n) if 0.8 <= sigma[i] <= 1.2]
    vsel = v[:, inside]
    dev.set_operator(a)
    dev.form_gram(1 << 30, copy_out=False)
    refined = sssvd.MomentAccumulator(rg, dev).refine(vsel)
    qx, _ = np.linalg.qr(refined)
    qy, _ = np.linalg.qr(vsel)
    assert np.linalg.svd(qx - qy @ (qy.T @ qx), compute_uv=False)[0] <= 1e-8   # test_moments.cpp:61-82


def test_refinement_annihilates_far_spectrum(dev):
    from paper_2109_13655_b200 import sssvd
    n = 30
    a = constructed(50, n, 5.0 + 0.03 * np.arange(n), 41, 42)
    rg, _ = rules(0.8, 1.2, 32, 0.1)
    s0 = orc.random_start(n, 8, 6)
    dev.set_operator(a)
    dev.form_gram(1 << 30, copy_out=False)
    refined = sssvd.MomentAccumulator(rg, dev).refine(s0)
    assert np.linalg.norm(refined) / np.linalg.norm(s0) <= 1e-6      # test_moments.cpp:102-114


def test_exp_transform_approximates_log_g(dev):
    n = 40
    a = constructed(80, n, 10.0 ** (-6.0 + 6.0 * np.arange(n) / (n - 1)), 61, 62)
    g = a.T @ a
    g = (g + g.T) / 2
    rg, _ = rules(1e-4, 1e-1, 32, 0.1, exp=True)
    s0 = orc.random_start(n, 10, 8)
    blocks = gpu_blocks(dev, a, rg, s0, 2)
    lam, vec = np.linalg.eigh(g)
    logg = (vec * np.log(np.maximum(lam, 1e-300))) @ vec.T
    expected = logg @ blocks[0]
    assert np.linalg.norm(blocks[1] - expected) / np.linalg.norm(expected) <= 1e-4   # :141-163


def test_rank_one_filter_gain(dev):
    m, n = 50, 20
    u = orc.random_matrix(m, 1, 101)[:, 0]
    u /= np.linalg.norm(u)
    v = orc.random_matrix(n, 1, 102)[:, 0]
    v /= np.linalg.norm(v)
    s = 1.03
    a = s * np.outer(u, v)
    rg, ro = rules(0.8, 1.2, 32, 0.1)
    vin = orc.random_start(n, 6, 12)
    blocks = gpu_blocks(dev, a, rg, vin, 1)
    gain = np.linalg.norm(blocks[0]) / np.linalg.norm(v @ vin)
    assert abs(gain - abs(orc.eval_filter(ro, s))) <= 1e-10 * abs(orc.eval_filter(ro, s))  # :217-231


def test_ell2_matches_oracle(dev):
    a = constructed(120, 60, np.linspace(0.05, 1.5, 60), 7, 8)
    rg, ro = rules(0.6, 0.9, 16, 0.1)
    s0 = orc.random_start(60, 6, 42)
    blocks = gpu_blocks(dev, a, rg, s0, 3, ell=2)
    acc = orc.MomentAccumulator(orc.form_gram(orc.ProblemMatrix(a)), ro)
    ref = acc.accumulate(acc.refine(s0), 3).blocks
    for k in range(4):
        assert np.linalg.norm(blocks[k] - ref[k]) / np.linalg.norm(ref[k]) <= 1e-10


def test_nccl_single_rank_comm_path(dev):
    """The multi-GPU code path (dlopen'ed NCCL, shard range, ncclAllReduce of the partial
    moments) run with a 1-rank communicator: results must be bitwise those without a comm."""
    from paper_2109_13655_b200 import sssvd
    a = constructed(300, 150, np.linspace(0.05, 1.5, 150), 3, 4)
    rg, _ = rules(0.6, 0.9, 16, 0.1)
    s0 = orc.random_start(150, 6, 42)
    ref = gpu_blocks(dev, a, rg, s0, 3)
    d2 = sssvd.Device(0)
    d2.init_comm(sssvd.Device.nccl_unique_id(), 1, 0)
    got = gpu_blocks(d2, a, rg, s0, 3)
    d2.close()
    for k in range(4):
        assert np.array_equal(ref[k], got[k])


def test_nccl_single_rank_operator_broadcast_and_failure_agreement(dev):
    """With a (1-rank) communicator: set_operator_root uploads on the root and broadcasts the padded
    operator with ncclBroadcast (the multi-GPU upload), and run_solve through it is bitwise the plain
    upload's; a shift on the spectrum goes through the failure agreement (one int all-reduce before
    the moment all-reduce) and surfaces as NumericalError (shifted_solver.hpp:29-30)."""
    from paper_2109_13655_b200 import sssvd
    am, _, _, _ = orc.build_model(1, 400, 120, 7)
    a = np.asfortranarray(am.dense)
    cfg = sssvd.RunConfig(0.8, 1.2, params=sssvd.SsParams(block_size=8, moment_degree=4, quadrature_count=16))
    d1 = sssvd.Device(0)
    d1.set_operator(a)
    ref = d1.run_solve(cfg)
    d1.close()
    d2 = sssvd.Device(0)
    d2.init_comm(sssvd.Device.nccl_unique_id(), 1, 0)
    assert d2.comm_size() == 1
    d2.set_operator_root(a.ctypes.data, a.shape[0], a.shape[1], a.shape[0], on_device=False, root=0)
    got = d2.run_solve(cfg)
    assert np.array_equal(ref.triplets.sigma, got.triplets.sigma)
    assert np.array_equal(ref.triplets.left, got.triplets.left) and np.array_equal(ref.exact, got.exact)
    # G = diag(1, 4, ...) and a shift exactly at 4: the pivot floor trips on the (only) rank
    diag = np.diag(np.arange(1.0, 9.0))
    d2.set_operator(diag)
    d2.form_gram(copy_out=False)
    with pytest.raises(sssvd.NumericalError):
        d2.check(sssvd.lib().sssvd_gpu_moments(
            d2.h, 1, sssvd._ptr(np.array([4.0, 0.0])), sssvd._ptr(np.array([1.0, 0.0])),
            sssvd._ptr(np.array([4.0, 0.0])), sssvd._ptr(np.ones(8)), 1, 1, 0, sssvd._ptr(np.empty(8))))
    d2.close()


def test_ell3_factor_cache_matches_oracle(dev):
    """ell > 1 with resident factors (moments.hpp:106-128): the refinement passes replay only the
    forward/back substitution of the new block; results must equal the oracle's to rounding."""
    a = constructed(400, 300, np.linspace(0.05, 1.5, 300), 17, 18)
    rg, ro = rules(0.6, 0.9, 32, 0.1)
    s0 = orc.random_start(300, 8, 42)
    blocks = gpu_blocks(dev, a, rg, s0, 3, ell=3)
    acc = orc.MomentAccumulator(orc.form_gram(orc.ProblemMatrix(a)), ro)
    ref = acc.accumulate(acc.refine(acc.refine(s0)), 3).blocks
    for k in range(4):
        assert np.linalg.norm(blocks[k] - ref[k]) / np.linalg.norm(ref[k]) <= 1e-10


def test_graph_replay_is_bitwise_eager(dev):
    """The shifted-solve pass runs eagerly on the first call of a plan, is captured into a CUDA
    graph on the second and replayed afterwards: all three give bitwise-identical moments, and
    the grouped path (>= 8 shifts -> 4 groups) is covered."""
    a = constructed(600, 400, np.linspace(0.05, 1.5, 400), 21, 22)
    rg, ro = rules(0.6, 0.9, 32, 0.1)
    s0 = orc.random_start(400, 8, 42)
    runs = [gpu_blocks(dev, a, rg, s0, 4) for _ in range(4)]
    for r in runs[1:]:
        for k in range(5):
            assert np.array_equal(runs[0][k], r[k])
    ref = orc.MomentAccumulator(orc.form_gram(orc.ProblemMatrix(a)), ro).accumulate(s0, 4).blocks
    for k in range(5):
        assert np.linalg.norm(runs[-1][k] - ref[k]) / np.linalg.norm(ref[k]) <= 1e-10


def test_lookahead_schedule_is_bitwise_plain_schedule(dev, monkeypatch):
    """The depth-1 look-ahead LU schedule (next block's columns on the panel stream, far columns on
    the GEMM stream) applies every update to every column in the same order with the same
    kernels, so its moments must equal the plain grouped schedule's bit for bit (n = 700: five full
    128-wide blocks and a ragged one)."""
    a = constructed(900, 700, np.linspace(0.05, 1.5, 700), 31, 32)
    rg, ro = rules(0.6, 0.9, 32, 0.1)
    s0 = orc.random_start(700, 8, 42)
    monkeypatch.setenv("SSSVD_LOOKAHEAD", "0")
    plain = gpu_blocks(dev, a, rg, s0, 3)
    monkeypatch.setenv("SSSVD_LOOKAHEAD", "1")
    look = [gpu_blocks(dev, a, rg, s0, 3) for _ in range(3)]   # eager, captured, replayed
    for r in look:
        for k in range(4):
            assert np.array_equal(plain[k], r[k])
    ref = orc.MomentAccumulator(orc.form_gram(orc.ProblemMatrix(a)), ro).accumulate(s0, 3).blocks
    for k in range(4):
        assert np.linalg.norm(look[-1][k] - ref[k]) / np.linalg.norm(ref[k]) <= 1e-10


def test_graph_capture_and_replay_are_bitwise_eager(dev):
    """The shifted-solve pass runs eagerly on its first sighting, is captured into a CUDA graph on
    the second and replayed afterwards: all three must give the same moments bit for bit, and match
    the oracle (n = 700: a ragged last block; a pivot-hungry interval inside the spectrum; L = 12
    leaves idle warps in the back substitution)."""
    a = constructed(900, 700, np.linspace(0.05, 1.5, 700), 41, 42)
    rg, ro = rules(0.6, 0.9, 32, 0.1)
    s0 = orc.random_start(700, 12, 42)
    runs = [gpu_blocks(dev, a, rg, s0, 3) for _ in range(3)]   # eager, captured, replayed
    for r in runs[1:]:
        for k in range(4):
            assert np.array_equal(runs[0][k], r[k])
    ref = orc.MomentAccumulator(orc.form_gram(orc.ProblemMatrix(a)), ro).accumulate(s0, 3).blocks
    for k in range(4):
        assert np.linalg.norm(runs[0][k] - ref[k]) / np.linalg.norm(ref[k]) <= 1e-10


def test_high_moment_degree_chunks(dev):
    """M = 40 > 32 register-resident accumulators: the moment kernel runs in degree chunks of 33
    (any M with L M <= n is valid, moments.hpp:35-46); blocks match the oracle's power chain."""
    a = constructed(160, 120, np.linspace(0.3, 1.6, 120), 71, 72)
    rg, ro = rules(0.7, 1.1, 16, 0.1)
    s0 = orc.random_start(120, 2, 42)
    got = gpu_blocks(dev, a, rg, s0, 40)
    ref = orc.MomentAccumulator(orc.form_gram(orc.ProblemMatrix(a)), ro).accumulate(s0, 40).blocks
    assert len(got) == 41
    for k in range(41):
        assert np.linalg.norm(got[k] - ref[k]) <= 1e-10 * np.linalg.norm(ref[k]) + 1e-300
