"""The SURVEY.md 8(d) parity contract between the GPU library and the CPU oracle, shared by the
-m gpu parity tests and the fixture generator (tools/make_oracle_fixture.py).

A run is reduced to a `Summary` (plain arrays: sigma, verdicts, tau, residuals, vector projections)
so that a live oracle run and a committed fixture are compared by the same code.

The contract (criteria 1-4 of SURVEY.md 8d) is applied at two truncation levels of the stacked
moment matrix (delta, moments.hpp:27, :205):

* delta = 1e-12 (`check_strict`): the roundoff-level directions of S are cut off, every kept
  direction is determined by the data, and the two implementations must agree on everything:
  in-interval and non-spurious counts, sigma within 1e-10, the same verdict, residuals within 2x,
  vectors up to sign.

* delta = 1e-20, the reference default (`check_robust`): S keeps directions whose singular values
  are ~1e-17 sigma_0, i.e. pure roundoff, different in every implementation (Eigen's, LAPACK's,
  this library's). They produce junk candidates (Ritz pairs of random directions, residual ~ 1,
  tau ~ 1e-9 of the threshold), and they can move tau (postprocess.hpp:56-60) and the residual of an
  unconverged Ritz pair. So: junk must be spurious on both sides; every other candidate is matched
  on the other side; verdicts must agree wherever they are data-determined (tau firmly on one side of
  the threshold, or unchanged by truncating to delta = 1e-12, on both sides: VERDICT round 1, "next
  round" item 1); found triplets agree in sigma; residuals are compared where truncation leaves them
  unchanged; the non-spurious counts may differ by at most the candidates whose verdict is not
  data-determined.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

N_PROJ = 4   # fixed random unit vectors the triplet vectors are projected on (fixture checksums)


def _proj_vectors(rows: int, seed: int) -> np.ndarray:
    z = np.random.default_rng(seed).standard_normal((rows, N_PROJ))
    return z / np.linalg.norm(z, axis=0)


@dataclass
class Summary:
    sigma: np.ndarray
    in_interval: np.ndarray
    spurious: np.ndarray
    tau: np.ndarray
    threshold: float
    exact: np.ndarray
    galerkin: np.ndarray
    count_in_interval: int
    count_nonspurious: int
    count_boundary: int
    proj_u: np.ndarray            # N_PROJ x t: z_k . u_i
    proj_v: np.ndarray            # N_PROJ x t: z_k . v_i
    left: Optional[np.ndarray] = None
    right: Optional[np.ndarray] = None

    def arrays(self, prefix: str) -> dict:
        out = {}
        for k in ("sigma", "in_interval", "spurious", "tau", "exact", "galerkin", "proj_u", "proj_v"):
            out[prefix + k] = getattr(self, k)
        out[prefix + "scalars"] = np.array([self.threshold, self.count_in_interval, self.count_nonspurious,
                                            self.count_boundary], dtype=np.float64)
        return out

    @staticmethod
    def from_arrays(d, prefix: str) -> "Summary":
        sc = d[prefix + "scalars"]
        return Summary(np.asarray(d[prefix + "sigma"]), np.asarray(d[prefix + "in_interval"]).astype(bool),
                       np.asarray(d[prefix + "spurious"]).astype(bool), np.asarray(d[prefix + "tau"]), float(sc[0]),
                       np.asarray(d[prefix + "exact"]), np.asarray(d[prefix + "galerkin"]), int(sc[1]), int(sc[2]),
                       int(sc[3]), np.asarray(d[prefix + "proj_u"]), np.asarray(d[prefix + "proj_v"]))


def summarize_gpu(res, keep_vectors: bool = True) -> Summary:
    t = res.triplets
    m, n = t.left.shape[0], t.right.shape[0]
    return Summary(t.sigma.copy(), np.asarray(t.in_interval, bool), np.asarray(res.spurious, bool), res.tau.copy(),
                   res.spurious_threshold, res.exact.copy(), res.galerkin.copy(), res.count_in_interval,
                   res.count_nonspurious_in_interval, res.count_boundary,
                   _proj_vectors(m, 1).T @ t.left, _proj_vectors(n, 2).T @ t.right,
                   t.left if keep_vectors else None, t.right if keep_vectors else None)


def summarize_oracle(ores, keep_vectors: bool = True) -> Summary:
    t = ores.triplets
    m, n = t.left.shape[0], t.right.shape[0]
    return Summary(t.sigma.copy(), np.asarray(t.in_interval, bool), np.asarray(ores.verdict.spurious, bool),
                   ores.verdict.tau.copy(), ores.verdict.threshold, ores.residuals.exact.copy(), ores.galerkin.copy(),
                   ores.count_in_interval, ores.count_nonspurious_in_interval, ores.count_boundary,
                   _proj_vectors(m, 1).T @ t.left, _proj_vectors(n, 2).T @ t.right,
                   t.left if keep_vectors else None, t.right if keep_vectors else None)


def near_endpoint(s: float, a: float, b: float) -> bool:
    """pipeline.hpp:103-106: within 1e-9 (relative) of an endpoint."""
    return abs(s - a) <= 1e-9 * max(abs(a), s) or abs(s - b) <= 1e-9 * max(abs(b), s)


def match(s: float, rho: float, other: Summary, junk_abs: float = np.inf, tol: float = 1e-6,
          class_slack: float = 3.0) -> Optional[int]:
    """The candidate of `other` that approximates the same singular value as (sigma s, residual
    rho): the nearest sigma among the candidates of the same class (meaningful: residual <=
    junk_abs; junk: a Ritz pair built from roundoff directions, residual ~ 1) within
    max(tol, min(2 rho / s, 1e-3)) relative of s (two implementations' Ritz values of one singular
    value differ by at most their residuals), so a junk candidate is never paired with a converged one
    that happens to sit close by. The class boundary itself is soft: a residual within class_slack
    of junk_abs counts for either class (config 2's unconverged candidates have residuals right at
    1e-2 sigma_max, and the two sides land on either side of it by roundoff)."""
    t = max(tol, min(2.0 * rho / max(s, 1e-300), 1e-3))
    if rho > junk_abs:
        same = other.exact > junk_abs / class_slack
    else:
        same = other.exact <= junk_abs * class_slack
    cand = np.flatnonzero((np.abs(other.sigma - s) <= t * s) & same)
    if cand.size == 0:
        return None
    return int(cand[int(np.argmin(np.abs(other.sigma[cand] - s)))])


def _nearest(s: float, other: Summary, k: int = 3):
    """(sigma, exact residual, in_interval) of the k candidates of `other` nearest to s (failure messages)."""
    idx = np.argsort(np.abs(other.sigma - s))[:k]
    return [(float(other.sigma[i]), float(other.exact[i]), bool(other.in_interval[i])) for i in idx]


def _borderline(tau: float, thr: float, factor: float) -> bool:
    return thr > 0 and 1.0 / factor <= tau / thr <= factor


def _gap(s: float, truth: np.ndarray) -> float:
    """Distance from s to the second-nearest true singular value (the nearest is its own)."""
    d = np.sort(np.abs(truth - s))
    return float(d[1]) if d.size > 1 else 1.0


def _vector_dist(g: Summary, j: int, o: Summary, i: int) -> float:
    """Sign-invariant distance of the right (and left) vectors; from the full vectors when both
    sides carry them, else from the N_PROJ projections (a lower bound of the same distance)."""
    if g.right is not None and o.right is not None:
        dv = min(np.linalg.norm(g.right[:, j] - o.right[:, i]), np.linalg.norm(g.right[:, j] + o.right[:, i]))
        du = min(np.linalg.norm(g.left[:, j] - o.left[:, i]), np.linalg.norm(g.left[:, j] + o.left[:, i]))
        return max(dv, du)
    dv = min(np.max(np.abs(g.proj_v[:, j] - o.proj_v[:, i])), np.max(np.abs(g.proj_v[:, j] + o.proj_v[:, i])))
    du = min(np.max(np.abs(g.proj_u[:, j] - o.proj_u[:, i])), np.max(np.abs(g.proj_u[:, j] + o.proj_u[:, i])))
    return max(dv, du)


@dataclass
class Report:
    checked: int = 0
    verdicts: int = 0
    sigmas: int = 0
    residuals: int = 0
    vectors: int = 0
    junk: int = 0
    undetermined: int = 0
    worst_sigma: float = 0.0
    worst_residual_ratio: float = 0.0
    notes: list = field(default_factory=list)


def _vectors(rep, g, j, o, i, truth):
    if truth is None:
        return
    bound = max(1e-8, 10.0 * (g.exact[j] + o.exact[i] + g.galerkin[j] + o.galerkin[i]) / _gap(o.sigma[i], truth))
    if bound < 1.0:
        d = _vector_dist(g, j, o, i)
        assert d <= bound, ("vectors differ", o.sigma[i], d, bound)
        rep.vectors += 1


def check_strict(g: Summary, o: Summary, a: float, b: float, sigma_max: float, truth: Optional[np.ndarray] = None,
                 tol_sigma: float = 1e-10, res_factor: float = 2.0, tau_eps: float = 1e-6) -> Report:
    """delta = 1e-12 on both sides: every kept direction is data-determined, so the contract holds
    without exceptions other than exact ties (a Ritz value within 1e-9 of an endpoint, tau within
    1e-6 of the threshold): every in-interval candidate of either side is matched on the other side
    with the same verdict; found (non-spurious) triplets agree in sigma within tol_sigma, in the
    exact and Galerkin residuals within res_factor, and in their vectors up to sign."""
    rep = Report()
    floor = 1e-9 * sigma_max
    ties = sum(1 for s in o.sigma if near_endpoint(s, a, b)) + sum(1 for s in g.sigma if near_endpoint(s, a, b))
    assert abs(g.count_in_interval - o.count_in_interval) <= ties, (g.count_in_interval, o.count_in_interval)
    tau_ties = 0
    for i in np.flatnonzero(o.in_interval):
        if near_endpoint(o.sigma[i], a, b):
            continue
        j = match(o.sigma[i], o.exact[i], g)
        assert j is not None, ("unmatched oracle candidate", o.sigma[i], o.exact[i])
        rep.checked += 1
        assert g.in_interval[j]
        if _borderline(o.tau[i], o.threshold, 1 + tau_eps) or _borderline(g.tau[j], g.threshold, 1 + tau_eps):
            tau_ties += 1
            continue
        assert g.spurious[j] == o.spurious[i], (o.sigma[i], g.tau[j] / g.threshold, o.tau[i] / o.threshold)
        rep.verdicts += 1
        if o.spurious[i]:
            continue
        dev = abs(g.sigma[j] - o.sigma[i]) / o.sigma[i]
        assert dev <= tol_sigma, ("sigma", o.sigma[i], g.sigma[j])
        rep.worst_sigma = max(rep.worst_sigma, dev)
        rep.sigmas += 1
        for gr, orr in ((g.exact[j], o.exact[i]), (g.galerkin[j], o.galerkin[i])):
            assert gr <= max(floor, res_factor * orr) and orr <= max(floor, res_factor * gr), (o.sigma[i], gr, orr)
            rep.worst_residual_ratio = max(rep.worst_residual_ratio, gr / max(orr, floor))
        rep.residuals += 1
        _vectors(rep, g, j, o, i, truth)
    for j in np.flatnonzero(g.in_interval):
        if not near_endpoint(g.sigma[j], a, b):
            assert match(g.sigma[j], g.exact[j], o) is not None, ("unmatched GPU candidate", g.sigma[j])
    assert abs(g.count_nonspurious - o.count_nonspurious) <= ties + tau_ties, (g.count_nonspurious, o.count_nonspurious)
    return rep


def check_robust(g20: Summary, o20: Summary, g12: Summary, o12: Summary, a: float, b: float, sigma_max: float,
                 truth: Optional[np.ndarray] = None, tol_sigma: float = 1e-10, res_factor: float = 10.0,
                 junk: float = 1e-2, firm: float = 10.0) -> Report:
    """delta = 1e-20 (the reference default), the contract on every data-determined candidate:
      * junk candidates (residual > junk * sigma_max: Ritz pairs built from roundoff directions)
        must be spurious on both sides;
      * every other in-interval candidate is matched on the other side (`match`);
      * its verdict must agree where it is data-determined: tau firm (outside [1/firm, firm] x the
        threshold) on both sides, or the verdict unchanged by truncating to delta = 1e-12 on both
        sides. firm = 10: config 1 has an unconverged pair (sigma 0.542) whose residual moves
        1.3e-6 -> 6e-5 and whose tau moves 2.1 -> 0.3 of the threshold between two implementations
        whose moment blocks differ by 1e-13, the same distance each has from the oracle's
        (profiles/r02_3m_sensitivity.txt), so a tau within a decade of the threshold is not firm ("every candidate whose verdict does not change when directions below
        1e-12 sigma_0 are truncated");
      * found triplets: sigma within max(tol_sigma sigma, rho_gpu + rho_oracle) (two Ritz values of
        one singular value differ by at most their residuals), within tol_sigma where the residual is
        data-determined; the exact residual <= max(1e-9 sigma_max, res_factor x oracle) where the
        residual is data-determined (unchanged within 2x by the truncation, on both sides);
      * the non-spurious counts differ by at most the candidates whose verdict is not
        data-determined."""
    rep = Report()
    floor = 1e-9 * sigma_max
    jabs = junk * sigma_max

    def cross(s20: Summary, s12: Summary, i: int):
        """(verdict stable, residual stable) of candidate i of s20 under truncation to s12."""
        k = match(s20.sigma[i], s20.exact[i], s12, jabs)
        if k is None or not s12.in_interval[k]:
            return False, False
        v = bool(s20.spurious[i]) == bool(s12.spurious[k])
        r = max(s20.exact[i], floor) <= 2 * max(s12.exact[k], floor) and \
            max(s12.exact[k], floor) <= 2 * max(s20.exact[i], floor)
        return v, r

    undetermined = 0
    for side, other in ((o20, g20), (g20, o20)):
        for i in np.flatnonzero(side.in_interval):
            if side.exact[i] > junk * sigma_max:
                assert side.spurious[i], ("junk candidate accepted", side.sigma[i], side.tau[i] / side.threshold)
                rep.junk += 1
            elif not near_endpoint(side.sigma[i], a, b):
                assert match(side.sigma[i], side.exact[i], other, jabs) is not None, \
                    ("unmatched candidate", side.sigma[i], side.exact[i], _nearest(side.sigma[i], other))
    for i in np.flatnonzero(o20.in_interval):
        if o20.exact[i] > junk * sigma_max or near_endpoint(o20.sigma[i], a, b):
            continue
        j = match(o20.sigma[i], o20.exact[i], g20, jabs)
        rep.checked += 1
        vo, ro = cross(o20, o12, i)
        vg, rg = cross(g20, g12, j)
        firm_both = not _borderline(o20.tau[i], o20.threshold, firm) and not _borderline(g20.tau[j], g20.threshold, firm)
        if not (firm_both or (vo and vg)):
            undetermined += 1
            continue
        assert g20.spurious[j] == o20.spurious[i], (o20.sigma[i], g20.tau[j] / g20.threshold, o20.tau[i] / o20.threshold)
        rep.verdicts += 1
        if o20.spurious[i]:
            continue
        dev = abs(g20.sigma[j] - o20.sigma[i])
        tol = tol_sigma * o20.sigma[i] if (ro and rg) else max(tol_sigma * o20.sigma[i], g20.exact[j] + o20.exact[i])
        assert dev <= tol, ("sigma", o20.sigma[i], g20.sigma[j], o20.exact[i], g20.exact[j])
        rep.sigmas += 1
        rep.worst_sigma = max(rep.worst_sigma, dev / o20.sigma[i])
        if ro and rg:
            assert g20.exact[j] <= max(floor, res_factor * o20.exact[i]), (o20.sigma[i], g20.exact[j], o20.exact[i])
            rep.worst_residual_ratio = max(rep.worst_residual_ratio, g20.exact[j] / max(o20.exact[i], floor))
            rep.residuals += 1
            _vectors(rep, g20, j, o20, i, truth)
    rep.undetermined = undetermined
    for j in np.flatnonzero(g20.in_interval):   # GPU-side candidates whose verdict is undetermined
        if g20.exact[j] > junk * sigma_max or near_endpoint(g20.sigma[j], a, b):
            continue
        i = match(g20.sigma[j], g20.exact[j], o20, jabs)
        if _borderline(g20.tau[j], g20.threshold, firm) or _borderline(o20.tau[i], o20.threshold, firm):
            if not (cross(g20, g12, j)[0] and cross(o20, o12, i)[0]):
                undetermined += 1
    ties = sum(1 for x in o20.sigma if near_endpoint(x, a, b)) + sum(1 for x in g20.sigma if near_endpoint(x, a, b))
    diff = abs(g20.count_nonspurious - o20.count_nonspurious)
    assert diff <= undetermined + ties, (g20.count_nonspurious, o20.count_nonspurious, undetermined, ties)
    rep.notes.append(f"non-spurious GPU {g20.count_nonspurious} / oracle {o20.count_nonspurious}; "
                     f"verdict not data-determined: {rep.undetermined} (oracle side)")
    return rep


def principal_angle_sine(x: np.ndarray, y: np.ndarray) -> float:
    """Largest principal-angle sine between span(x) and span(y) (equal dimensions, orthonormalised
    first), as the norm of the part of span(y) outside span(x): || (I - Qx Qx^T) Qy ||_2. (The
    cosine form sqrt(1 - c_min^2) cannot resolve sines below ~sqrt(eps) = 1.5e-8.)"""
    if x.shape[1] == 0 or y.shape[1] == 0:
        return 0.0
    qx, _ = np.linalg.qr(x)
    qy, _ = np.linalg.qr(y)
    r = qy - qx @ (qx.T @ qy)
    r -= qx @ (qx.T @ r)   # second projection pass: keeps the residual accurate at the 1e-16 level
    return float(np.linalg.svd(r, compute_uv=False)[0])
