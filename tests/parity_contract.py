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
  this library's). tau (postprocess.hpp:56-60) and the residual of an unconverged Ritz pair can be
  driven by those directions. A quantity is data-determined when it does not change once those
  directions are truncated, so for every candidate whose verdict (resp. residual, within 2x) is the
  same at delta = 1e-20 and at delta = 1e-12 on BOTH sides, the two sides must agree exactly as in
  the contract; the non-spurious counts may differ by at most the number of candidates that are not
  ("next round" item 1).
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


def _match(s: float, sigmas: np.ndarray, tol: float) -> Optional[int]:
    j = int(np.argmin(np.abs(sigmas - s)))
    return j if abs(sigmas[j] - s) <= tol * max(s, 1e-300) else None


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
    residuals: int = 0
    vectors: int = 0
    nonrobust: int = 0
    worst_sigma: float = 0.0
    worst_residual_ratio: float = 0.0
    notes: list = field(default_factory=list)


def check_strict(g: Summary, o: Summary, a: float, b: float, sigma_max: float, truth: Optional[np.ndarray] = None,
                 tol_sigma: float = 1e-10, res_factor: float = 2.0, tau_eps: float = 1e-6) -> Report:
    """delta = 1e-12 on both sides: the contract without exceptions other than exact ties (a Ritz
    value within 1e-9 of an endpoint, tau within 1e-6 of the threshold)."""
    rep = Report()
    ties = sum(1 for s in o.sigma if near_endpoint(s, a, b)) + sum(1 for s in g.sigma if near_endpoint(s, a, b))
    assert abs(g.count_in_interval - o.count_in_interval) <= ties, (g.count_in_interval, o.count_in_interval)
    tau_ties = 0
    for i in np.flatnonzero(o.in_interval):
        j = _match(o.sigma[i], g.sigma, tol_sigma)
        assert j is not None, ("unmatched oracle candidate", o.sigma[i])
        rep.checked += 1
        rep.worst_sigma = max(rep.worst_sigma, abs(g.sigma[j] - o.sigma[i]) / o.sigma[i])
        if near_endpoint(o.sigma[i], a, b):
            continue
        assert g.in_interval[j]
        if _borderline(o.tau[i], o.threshold, 1 + tau_eps) or _borderline(g.tau[j], g.threshold, 1 + tau_eps):
            tau_ties += 1
        else:
            assert g.spurious[j] == o.spurious[i], (o.sigma[i], g.tau[j] / g.threshold, o.tau[i] / o.threshold)
            rep.verdicts += 1
        floor = 1e-9 * sigma_max
        for gr, orr in ((g.exact[j], o.exact[i]), (g.galerkin[j], o.galerkin[i])):
            assert gr <= max(floor, res_factor * orr) and orr <= max(floor, res_factor * gr), (o.sigma[i], gr, orr)
            rep.worst_residual_ratio = max(rep.worst_residual_ratio, gr / max(orr, floor))
        rep.residuals += 1
        if truth is not None:
            bound = max(1e-8, 10.0 * (g.exact[j] + o.exact[i] + g.galerkin[j] + o.galerkin[i]) / _gap(o.sigma[i], truth))
            if bound < 1.0:
                assert _vector_dist(g, j, o, i) <= bound, (o.sigma[i], _vector_dist(g, j, o, i), bound)
                rep.vectors += 1
    assert abs(g.count_nonspurious - o.count_nonspurious) <= ties + tau_ties, (g.count_nonspurious, o.count_nonspurious)
    return rep


def check_robust(g20: Summary, o20: Summary, g12: Summary, o12: Summary, a: float, b: float, sigma_max: float,
                 truth: Optional[np.ndarray] = None, tol_sigma: float = 1e-10, res_factor: float = 10.0) -> Report:
    """delta = 1e-20 (reference default): the contract on every data-determined candidate (see the
    module docstring); counts may differ by at most the number of candidates that are not."""
    rep = Report()
    floor = 1e-9 * sigma_max

    def stable(s20: Summary, s12: Summary, i: int):
        """(verdict stable, residual stable) of candidate i of s20 under truncation to s12."""
        k = _match(s20.sigma[i], s12.sigma, tol_sigma)
        if k is None or near_endpoint(s20.sigma[i], a, b):
            return False, False
        v = bool(s20.spurious[i]) == bool(s12.spurious[k]) and s12.in_interval[k]
        r = (s20.exact[i] <= max(floor, 2 * s12.exact[k]) and s12.exact[k] <= max(floor, 2 * s20.exact[i]))
        return v, r

    nonrobust_o = nonrobust_g = 0
    for i in np.flatnonzero(o20.in_interval):
        vo, ro = stable(o20, o12, i)
        j = _match(o20.sigma[i], g20.sigma, tol_sigma)
        vg, rg = stable(g20, g12, j) if j is not None else (False, False)
        if not (vo and vg):
            nonrobust_o += 1
            continue
        rep.checked += 1
        rep.worst_sigma = max(rep.worst_sigma, abs(g20.sigma[j] - o20.sigma[i]) / o20.sigma[i])
        assert g20.in_interval[j]
        assert g20.spurious[j] == o20.spurious[i], (o20.sigma[i], g20.tau[j] / g20.threshold, o20.tau[i] / o20.threshold)
        rep.verdicts += 1
        if ro and rg:
            assert g20.exact[j] <= max(floor, res_factor * o20.exact[i]), (o20.sigma[i], g20.exact[j], o20.exact[i])
            rep.worst_residual_ratio = max(rep.worst_residual_ratio, g20.exact[j] / max(o20.exact[i], floor))
            rep.residuals += 1
            if truth is not None:
                bound = max(1e-8, 10.0 * (g20.exact[j] + o20.exact[i] + g20.galerkin[j] + o20.galerkin[i]) /
                            _gap(o20.sigma[i], truth))
                if bound < 1.0:
                    assert _vector_dist(g20, j, o20, i) <= bound
                    rep.vectors += 1
    for j in np.flatnonzero(g20.in_interval):
        vg, _ = stable(g20, g12, j)
        i = _match(g20.sigma[j], o20.sigma, tol_sigma)
        vo = stable(o20, o12, i)[0] if i is not None else False
        if not (vg and vo):
            nonrobust_g += 1
    rep.nonrobust = max(nonrobust_o, nonrobust_g)
    diff = abs(g20.count_nonspurious - o20.count_nonspurious)
    assert diff <= nonrobust_o + nonrobust_g, (g20.count_nonspurious, o20.count_nonspurious, nonrobust_o, nonrobust_g)
    rep.notes.append(f"non-spurious GPU {g20.count_nonspurious} / oracle {o20.count_nonspurious}; "
                     f"non-robust candidates oracle-side {nonrobust_o}, GPU-side {nonrobust_g}")
    return rep


def principal_angle_sine(x: np.ndarray, y: np.ndarray) -> float:
    """Largest principal-angle sine between span(x) and span(y) (orthonormalised first)."""
    qx, _ = np.linalg.qr(x)
    qy, _ = np.linalg.qr(y)
    c = np.linalg.svd(qx.T @ qy, compute_uv=False)
    return float(np.sqrt(max(0.0, 1.0 - np.min(c) ** 2))) if c.size else 0.0
