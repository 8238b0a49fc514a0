"""Pins the CPU oracle (oracle/sssvd_oracle.py) to every known-answer constant and tolerance
test the reference holds for this path. The reference (proj/, Eigen) cannot be built here, so
these are the parity anchors. Each test cites the reference test it restates;
tests/golden/reference_pins.json carries the constants with their file:line."""
import json
import math
import os

import numpy as np
import pytest

from oracle import sssvd_oracle as orc

PINS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_pins.json")))


def idt():
    return orc.SpectralTransform(orc.IDENTITY)


def ext():
    return orc.SpectralTransform(orc.EXP)


def test_ellipse_constants():
    r = orc.ContourRule(0.8, 1.2, 32, 0.1, idt())
    assert r.center == pytest.approx(PINS["center_identity_0.8_1.2"], rel=1e-15)   # test_contour.cpp:21-22
    assert r.radius == pytest.approx(PINS["radius_identity_0.8_1.2"], rel=1e-15)
    e = orc.ContourRule(1e-3, 1e-1, 32, 0.1, ext())
    assert e.center == pytest.approx(PINS["center_exp_1e-3_1e-1"], rel=1e-12)      # test_contour.cpp:31-32
    assert e.radius == pytest.approx(PINS["radius_exp_1e-3_1e-1"], rel=1e-12)
    assert e.transform.g_inverse(1e-6) == pytest.approx(e.center - e.radius, rel=1e-14)
    assert e.transform.g_inverse(1e-2) == pytest.approx(e.center + e.radius, rel=1e-14)


def test_nodes_and_weights_parameterisation():
    r = orc.ContourRule(0.8, 1.2, 32, 0.1, idt())
    for j in range(16):                                              # test_contour.cpp:37-47
        th = (2 * math.pi / 32) * (j + 0.5)
        assert abs(r.nodes[j] - complex(1.04 + 0.4 * math.cos(th), 0.04 * math.sin(th))) <= 1e-15
        assert abs(r.weights[j] - complex(0.4 / 32 * 0.1 * math.cos(th), 0.4 / 32 * math.sin(th))) <= 1e-17


def test_conjugate_mirror_bit_exact():
    for tf in (idt(), ext()):                                        # test_contour.cpp:49-59
        r = orc.ContourRule(0.5, 2.0, 32, 0.1, tf)
        for j in range(16):
            assert r.nodes[j] == np.conj(r.nodes[j + 16])
            assert r.weights[j] == np.conj(r.weights[j + 16])


def test_argument_validation():
    with pytest.raises(ValueError):
        orc.ContourRule(0.8, 1.2, 31, 0.1, idt())                    # test_contour.cpp:88-99
    with pytest.raises(ValueError):
        orc.ContourRule(0.8, 1.2, 32, 1.5, idt())
    with pytest.raises(ValueError):
        orc.ContourRule(1.2, 0.8, 32, 0.1, idt())
    with pytest.raises(orc.DomainError):
        orc.ContourRule(0.0, 1.2, 32, 0.1, ext())
    orc.ContourRule(0.0, 1.2, 32, 0.1, idt())


def test_vanishing_moment_sums():
    for a, b in ((0.8, 1.2), (1e-3, 1e-1)):                          # test_contour.cpp:101-110
        sums = orc.moment_condition_check(orc.ContourRule(a, b, 32, 0.1, idt()), 30)
        assert max(sums) <= 1e-12


def test_cauchy_defect():
    def cauchy(r):
        return sum(r.weights[j] / (r.nodes[j] - r.center) for j in range(r.count))
    assert abs(cauchy(orc.ContourRule(0.8, 1.2, 32, 1.0, idt())) - 1) <= 1e-13     # test_contour.cpp:118-133
    d32 = abs(cauchy(orc.ContourRule(0.8, 1.2, 32, 0.1, idt())) - 1)
    d64 = abs(cauchy(orc.ContourRule(0.8, 1.2, 64, 0.1, idt())) - 1)
    assert d32 == pytest.approx(PINS["cauchy_defect_N32_aspect0.1"], rel=0.01)
    assert d64 < 0.05 * d32


def test_filter_reference_value():
    r = orc.ContourRule(0.8, 1.2, 32, 0.1, idt())
    assert abs(orc.eval_filter(r, math.sqrt(1.04))) == pytest.approx(PINS["filter_center_0.8_1.2"], rel=1e-9)
    c = orc.ContourRule(0.8, 1.2, 32, 1.0, idt())                    # test_filter.cpp:42-57
    assert abs(orc.eval_filter(c, math.sqrt(1.04))) == pytest.approx(1.0, rel=1e-13)
    assert abs(orc.eval_filter(r, 12.0)) <= 1e-4                     # test_filter.cpp:59-69


def test_filter_contrast_log_interval():
    fid = abs(orc.eval_filter(orc.ContourRule(1e-3, 1e-1, 32, 0.1, idt()), 1e-5))
    fex = abs(orc.eval_filter(orc.ContourRule(1e-3, 1e-1, 32, 0.1, ext()), 1e-5))
    assert 0.4 < fid < 0.6 and fex <= 1e-4                           # test_filter.cpp:71-79


def test_random_start_determinism():
    v1 = orc.random_start(200, 20, 3141)                              # test_moments.cpp:49-59
    assert np.array_equal(v1, orc.random_start(200, 20, 3141))
    assert not np.array_equal(v1, orc.random_start(200, 20, 3142))
    assert np.abs(v1).max() <= 1.0
    assert np.linalg.svd(v1, compute_uv=False).min() > 0
    with pytest.raises(ValueError):
        orc.random_start(10, 20, 1)
    # libstdc++ mt19937_64 + uniform_real_distribution(-1,1): first draws of seed 42
    v = orc.random_start(4, 1, 42)[:, 0]
    assert np.array_equal(v, np.array(PINS["random_start_seed42_first4"]))


def test_model_counts():
    _, _, s1, _ = orc.build_model(1)
    _, _, s2, _ = orc.build_model(2)
    assert int(np.sum((s1 >= 0.8) & (s1 <= 1.2))) == PINS["model1_count_0.8_1.2"]   # test_problems.cpp:18
    assert int(np.sum((s2 >= 1e-3) & (s2 <= 1e-1))) == PINS["model2_count_1e-3_1e-1"]  # test_problems.cpp:30


def constructed(m, n, sigma, su, sv):
    u, _ = np.linalg.qr(orc.random_matrix(m, n, su))
    v, _ = np.linalg.qr(orc.random_matrix(n, n, sv))
    return (u * sigma[None, :]) @ v.T


def test_moment_identity_oracle():
    n = 40
    a = constructed(80, n, 0.2 + 0.04 * np.arange(n), 51, 52)
    g = orc.form_gram(orc.ProblemMatrix(a))
    rule = orc.ContourRule(0.8, 1.2, 32, 0.1, idt())
    b = orc.MomentAccumulator(g, rule).accumulate(orc.random_start(n, 10, 7), 4).blocks
    p = b[0]
    for k in range(1, 5):                                            # test_moments.cpp:116-139
        p = g @ p
        assert np.linalg.norm(b[k] - p) / np.linalg.norm(p) <= 1e-8


def test_half_rule_equals_full_rule():
    a = constructed(50, 20, 0.7 + 0.06 * np.arange(20), 81, 82)
    g = orc.form_gram(orc.ProblemMatrix(a))
    rule = orc.ContourRule(0.5, 2.0, 16, 0.1, idt())
    s0 = orc.random_start(20, 6, 10)
    b = orc.MomentAccumulator(g, rule).accumulate(s0, 2).blocks
    for k in range(3):                                               # test_moments.cpp:176-203
        full = np.zeros((20, 6), complex)
        for j in range(16):
            f = orc.ShiftedFactorization(g, rule.shift(j))
            full += rule.weights[j] * rule.nodes[j] ** k * f.solve(s0)
        assert np.abs(full.imag).max() <= 1e-13 * np.linalg.norm(full.real)
        assert np.linalg.norm(b[k] - full.real) <= 1e-13 * np.linalg.norm(full.real)


def test_shard_sum_equals_full_sum():
    """moments.hpp:96-100: per-shard partial sums add up to the ascending-j total (tolerance;
    bitwise only when the shard boundaries are merged in ascending order)."""
    a = orc.random_matrix(40, 16, 91)
    g = orc.form_gram(orc.ProblemMatrix(a))
    rule = orc.ContourRule(0.5, 2.0, 32, 0.1, idt())
    s0 = orc.random_start(16, 5, 11)
    acc = orc.MomentAccumulator(g, rule)
    full = acc.accumulate(s0, 3).blocks
    p1 = acc.accumulate(s0, 3, shifts=range(0, 8)).blocks
    p2 = acc.accumulate(s0, 3, shifts=range(8, 16)).blocks
    for k in range(4):
        assert np.linalg.norm(p1[k] + p2[k] - full[k]) <= 1e-14 * (np.linalg.norm(p1[k]) + np.linalg.norm(p2[k]))


def test_low_rank_semantics():
    q, _ = np.linalg.qr(orc.random_matrix(30, 8, 111))
    b = orc.low_rank(q, 1e-12)                                        # test_moments.cpp:233-258
    assert b.rank() == 8 and np.abs(b.singular_values - 1).max() <= 1e-12
    dup = np.repeat(orc.random_matrix(20, 1, 112), 2, axis=1)
    assert orc.low_rank(dup, 1e-12).rank() == 1
    with pytest.raises(orc.EmptySubspaceError):
        orc.low_rank(np.zeros((10, 4)), 1e-12)


def test_params_validation():
    p = orc.SsParams()
    p.validate(200)                                                  # test_moments.cpp:260-269
    with pytest.raises(ValueError):
        p.validate(50)
    with pytest.raises(ValueError):
        orc.SsParams(lowrank_threshold=0.0).validate(200)
    with pytest.raises(ValueError):
        orc.SsParams(quadrature_count=31).validate(200)


def test_solver_pins_oracle():
    g = np.diag([1.0, 4.0])                                          # test_solver.cpp:55-67
    x = orc.ShiftedFactorization(g, complex(2, 1)).solve(np.eye(2))
    assert abs(x[0, 0] - complex(0.5, -0.5)) <= 1e-15 and abs(x[1, 1] - complex(-0.4, -0.2)) <= 1e-15
    with pytest.raises(orc.NumericalError):                          # test_solver.cpp:128-132
        orc.ShiftedFactorization(g, complex(1.0, 0.0))
    with pytest.raises(orc.LengthError):                             # test_solver.cpp:50-53
        orc.form_gram(orc.ProblemMatrix(np.eye(10)), 8)


def test_pipeline_smoke_oracle():
    a, _, sigma, _ = orc.build_model(1, 80, 48, 7)
    cfg = orc.RunConfig(0.2, 0.33, params=orc.SsParams(block_size=8, moment_degree=3, quadrature_count=16))
    res = orc.run_solve(a, cfg)
    assert res.count_nonspurious_in_interval == int(np.sum((sigma >= 0.2) & (sigma <= 0.33)))  # test_pipeline.cpp:48-74
    st = orc.accuracy_vs_truth(sigma, res)
    assert st.max_rel_error_nonspurious <= 1e-9


def test_acceptance_model1_oracle():
    """acceptance.cpp:108-121, the headline pin of the oracle."""
    a, _, sigma, _ = orc.build_model(1)
    res = orc.run_solve(a, orc.RunConfig(0.8, 1.2))
    assert res.count_nonspurious_in_interval == 40
    st = orc.accuracy_vs_truth(sigma, res)
    assert st.max_rel_error_nonspurious <= 1e-10
    ns = [i for i in range(res.triplets.count()) if res.triplets.in_interval[i] and not res.verdict.spurious[i]]
    assert max(res.residuals.exact[ns]) <= 1e-9
    assert res.galerkin.max() <= 1e-10 * sigma.max()                 # criterion 7


def test_empty_interval_oracle():
    a, _, _, _ = orc.build_model(1, 80, 48, 7)
    res = orc.run_solve(a, orc.RunConfig(17.0, 18.0, params=orc.SsParams(block_size=8, moment_degree=3,
                                                                        quadrature_count=16)))
    assert res.empty and "no singular values inside" in res.note    # test_pipeline.cpp:76-86
