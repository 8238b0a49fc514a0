"""CPU oracle: a numpy/scipy restatement of the reference block SS-SVD solver.

TEST INFRASTRUCTURE ONLY. Only tests/, bench.py's cpu_baseline / --impl reference leg and
__graft_entry__.smoke() may import this module; the product path
(paper_2109_13655_b200/) never does and fails loudly without its CUDA library.

The reference (proj/include/sssvd/*.hpp) is header-only C++ on Eigen 3, which is absent
here, so it cannot be compiled. This module restates its
algorithm line by line; each function cites the reference lines it follows. Dense kernels
come from LAPACK through scipy (OpenBLAS): zgetrf/zgetrs in place of Eigen::PartialPivLU,
dgeqrf/dorgqr in place of Eigen::HouseholderQR, and the preconditioned one-sided Jacobi
SVD dgejsv (JOBA='C': no rank truncation) in place of Eigen::JacobiSVD. Seeded inputs are bit-identical to the reference's because they are drawn
by the same libstdc++ code (oracle/rng.cpp).

Pinning: parity of this oracle is pinned against every known-answer constant and tolerance
test the reference holds for this path (tests/test_oracle_pins.py lists them with the
reference file:line of each pin), plus acceptance criterion 1 (model 1: exactly 40
non-spurious triplets, error <= 1e-10, residual <= 1e-9; proj/tests/acceptance.cpp:108-121).
"""
from __future__ import annotations

import ctypes
import math
import os
import time
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np
import scipy.linalg as sla

_HERE = os.path.dirname(os.path.abspath(__file__))

# ----------------------------------------------------------------------------- errors
# proj/include/sssvd/core.hpp:29-39


class NumericalError(RuntimeError):
    """core.hpp:29-32 (CLI exit 3)."""


class EmptySubspaceError(NumericalError):
    """core.hpp:36-39."""


class LengthError(ValueError):
    """std::length_error (problem.hpp:84-85, the dense Gram cap)."""


class DomainError(ValueError):
    """std::domain_error (transform.hpp:75-76, contour.hpp:128-129)."""


# ----------------------------------------------------------------------------- RNG (libstdc++)
_rng = None


def _rng_lib():
    global _rng
    if _rng is None:
        path = os.path.join(_HERE, "liboracle_rng.so")
        if not os.path.exists(path):
            build_rng()
        _rng = ctypes.CDLL(path)
        _rng.oracle_random_start.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                             ctypes.c_void_p]
        _rng.oracle_random_start.restype = ctypes.c_int
        _rng.oracle_normal_stream.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p]
        _rng.oracle_uniform_stream.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_double,
                                               ctypes.c_double, ctypes.c_void_p]
    return _rng


def build_rng():
    import subprocess
    subprocess.check_call(["g++", "-O2", "-shared", "-fPIC", "-o",
                           os.path.join(_HERE, "liboracle_rng.so"), os.path.join(_HERE, "rng.cpp")])


def random_start(n: int, block_size: int, seed: int) -> np.ndarray:
    """moments.hpp:84-94: mt19937_64 + uniform_real_distribution(-1,1), j-outer fill."""
    if n < block_size:
        raise ValueError("random_start: block size exceeds dimension")
    out = np.empty((n, block_size), dtype=np.float64, order="F")
    _rng_lib().oracle_random_start(seed, n, block_size, out.ctypes.data)
    return out


def normal_stream(seed: int, count: int) -> np.ndarray:
    """One std::normal_distribution<double> drawn `count` times (problems.hpp:53-59)."""
    out = np.empty(count, dtype=np.float64)
    _rng_lib().oracle_normal_stream(seed, count, out.ctypes.data)
    return out


def uniform_stream(seed: int, count: int, lo: float, hi: float) -> np.ndarray:
    out = np.empty(count, dtype=np.float64)
    _rng_lib().oracle_uniform_stream(seed, count, lo, hi, out.ctypes.data)
    return out


def random_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    """The tests' random_matrix fixture (test_solver.cpp:16-23): column-major normal fill."""
    return normal_stream(seed, rows * cols).reshape((cols, rows)).T.copy(order="F")


# ----------------------------------------------------------------------------- transform / contour
IDENTITY, EXP = "identity", "exp"


class SpectralTransform:
    """transform.hpp:16-45."""

    def __init__(self, kind: str):
        self.kind = kind

    def g(self, t):
        return t if self.kind == IDENTITY else np.exp(t)

    def g_inverse(self, z: float) -> float:
        if self.kind == IDENTITY:
            return z
        if not z > 0:
            raise DomainError("SpectralTransform: g_inverse of non-positive value under Exp")
        return math.log(z)

    def g_prime(self, t: float) -> float:
        return 1.0 if self.kind == IDENTITY else math.exp(t)


class ContourRule:
    """contour.hpp:27-62 (nodes, weights, bit-exact conjugate mirror) and :76 shift(j)."""

    def __init__(self, a: float, b: float, count: int, aspect: float, transform: SpectralTransform):
        if not (a >= 0) or not (a < b):
            raise ValueError("ContourRule: need 0 <= a < b")
        if count < 4 or count % 2 != 0:
            raise ValueError("ContourRule: quadrature count must be even and >= 4")
        if not (aspect > 0) or aspect > 1:
            raise ValueError("ContourRule: aspect ratio must lie in (0,1]")
        if transform.kind == EXP and a == 0:
            raise DomainError("ContourRule: Exp transform requires a > 0 (g^{-1}(0) diverges)")
        self.a, self.b, self.count, self.aspect, self.transform = a, b, count, aspect, transform
        if transform.kind == IDENTITY:
            self.center = (a * a + b * b) / 2.0
            self.radius = (b * b - a * a) / 2.0
        else:
            self.center = math.log(a) + math.log(b)
            self.radius = math.log(b) - math.log(a)
        half = count // 2
        self.nodes = np.empty(count, dtype=np.complex128)
        self.weights = np.empty(count, dtype=np.complex128)
        two_pi = 2.0 * math.pi
        for j in range(half):
            theta = (two_pi / float(count)) * (float(j) + 0.5)
            c, s = math.cos(theta), math.sin(theta)
            t = complex(self.center + self.radius * c, self.radius * aspect * s)
            w = complex(self.radius / float(count) * aspect * c, self.radius / float(count) * s)
            if transform.kind == EXP:
                w = w * _cexp(t)
            self.nodes[j] = t
            self.weights[j] = w
            self.nodes[j + half] = t.conjugate()
            self.weights[j + half] = w.conjugate()

    def shift(self, j: int) -> complex:
        t = complex(self.nodes[j])
        return t if self.transform.kind == IDENTITY else _cexp(t)


def _cexp(t: complex) -> complex:
    # std::exp(complex): exp(re) * (cos(im), sin(im))
    e = math.exp(t.real)
    return complex(e * math.cos(t.imag), e * math.sin(t.imag))


def moment_condition_check(rule: ContourRule, kmax: int) -> List[float]:
    """contour.hpp:116-136 (long double accumulation; numpy longdouble is x87 80-bit here)."""
    if rule.transform.kind != IDENTITY:
        raise ValueError("moment_condition_check: defined for Identity rules")
    re_n = np.array(rule.nodes.real, dtype=np.longdouble)
    im_n = np.array(rule.nodes.imag, dtype=np.longdouble)
    re_p = np.ones(rule.count, dtype=np.longdouble)
    im_p = np.zeros(rule.count, dtype=np.longdouble)
    re_w = np.array(rule.weights.real, dtype=np.longdouble)
    im_w = np.array(rule.weights.imag, dtype=np.longdouble)
    out = []
    for _ in range(kmax + 1):
        sr = np.longdouble(0)
        si = np.longdouble(0)
        for j in range(rule.count):
            sr += re_w[j] * re_p[j] - im_w[j] * im_p[j]
            si += re_w[j] * im_p[j] + im_w[j] * re_p[j]
            nr = re_p[j] * re_n[j] - im_p[j] * im_n[j]
            ni = re_p[j] * im_n[j] + im_p[j] * re_n[j]
            re_p[j], im_p[j] = nr, ni
        out.append(float(np.sqrt(sr * sr + si * si)))
    return out


def eval_filter(rule: ContourRule, sigma: float) -> float:
    """filter.hpp:18-28: f(sigma) = 2 Re sum_{j<N/2} w_j / (g(t_j) - sigma^2)."""
    s2 = sigma * sigma
    half_sum = 0j
    for j in range(rule.count // 2):
        half_sum += complex(rule.weights[j]) / (rule.shift(j) - s2)
    return 2.0 * half_sum.real


# ----------------------------------------------------------------------------- params
@dataclass
class SsParams:
    """moments.hpp:23-47."""
    block_size: int = 20          # L
    moment_degree: int = 4        # M
    quadrature_count: int = 32    # N
    refinement_steps: int = 1     # ell
    lowrank_threshold: float = 1e-20   # delta
    spurious_threshold: float = 1e-8   # epsilon
    seed: int = 42

    def subspace_dim(self) -> int:
        return self.block_size * self.moment_degree

    def validate(self, n: int) -> None:
        if (self.block_size < 1 or self.moment_degree < 1 or self.quadrature_count < 4
                or self.refinement_steps < 1):
            raise ValueError("SsParams: counts must be positive (N >= 4)")
        if self.quadrature_count % 2 != 0:
            raise ValueError("SsParams: quadrature count must be even")
        if self.subspace_dim() > n:
            raise ValueError("SsParams: L*M must not exceed the column count")
        if not (self.lowrank_threshold > 0) or not (self.lowrank_threshold < 1):
            raise ValueError("SsParams: delta must lie in (0,1)")
        if not (self.spurious_threshold > 0):
            raise ValueError("SsParams: epsilon must be positive")


SS_SVD, SS_SVD_NT, NAIVE, NAIVE_NT = "ss-svd", "ss-svd-nt", "naive", "naive-nt"
K_RCOND_IDENTITY = 2e-15   # postprocess.hpp:101
K_RCOND_EXP = 1e-14        # postprocess.hpp:102


@dataclass
class RunConfig:
    """pipeline.hpp:43-58."""
    interval_a: float = 0.0
    interval_b: float = 1.0
    mode: str = SS_SVD
    aspect: float = 0.1
    params: SsParams = field(default_factory=SsParams)
    threads: int = 0
    estimator_rcond_identity: float = K_RCOND_IDENTITY
    estimator_rcond_exp: float = K_RCOND_EXP

    def transform(self) -> SpectralTransform:
        return SpectralTransform(EXP if self.mode in (SS_SVD_NT, NAIVE_NT) else IDENTITY)


# ----------------------------------------------------------------------------- problem / Gram
class ProblemMatrix:
    """problem.hpp:14-77: dense (numpy) or sparse (scipy CSC) storage; auto-transpose when
    rows < cols; NaN check (:20-35, :56-58)."""

    def __init__(self, a):
        import scipy.sparse as sp
        self.is_sparse = sp.issparse(a)
        if self.is_sparse:
            a = sp.csc_matrix(a, dtype=np.float64)
            self.transposed = a.shape[0] < a.shape[1]
            if self.transposed:
                a = a.T.tocsc()
            a.sum_duplicates()
            a.sort_indices()
            if not np.all(np.isfinite(a.data)):
                raise ValueError("ProblemMatrix: NaN/Inf entry")
            self.sparse = a
            return
        a = np.asarray(a, dtype=np.float64)
        self.transposed = a.shape[0] < a.shape[1]
        if self.transposed:
            a = a.T
        if not np.all(np.isfinite(a)):
            raise ValueError("ProblemMatrix: NaN/Inf entry")
        self.dense = np.asfortranarray(a)

    @property
    def shape(self):
        return self.sparse.shape if self.is_sparse else self.dense.shape

    @property
    def rows(self):
        return self.shape[0]

    @property
    def cols(self):
        return self.shape[1]

    def to_dense(self):
        return np.asfortranarray(self.sparse.toarray()) if self.is_sparse else self.dense

    def apply(self, x):
        return np.asarray(self.sparse @ x) if self.is_sparse else self.dense @ x

    def apply_adjoint(self, x):
        return np.asarray(self.sparse.T @ x) if self.is_sparse else self.dense.T @ x


def form_gram(a: ProblemMatrix, size_cap: int = 8192) -> np.ndarray:
    """problem.hpp:81-95: G = A^T A (sparse product for sparse storage, :87-89) then
    (G + G^T)/2; length_error above the cap.

    The BASELINE config 5 (n = 16384) lifts the cap (documented deviation)."""
    if a.cols > size_cap:
        raise LengthError("form_gram: column count exceeds the dense Gram cap")
    if a.is_sparse:
        g = (a.sparse.T @ a.sparse).toarray()
    else:
        g = a.dense.T @ a.dense
    return np.asfortranarray((g + g.T) / 2.0)


class MatrixMarketError(RuntimeError):
    """matrix_market.hpp:17-21."""


def read_matrix_market(path: str) -> ProblemMatrix:
    """matrix_market.hpp:34-119 restated in Python (checker for the library's C++ reader).
    Numbers are parsed with the same acceptance rules as std::istream >> for the inputs the tests
    use (plain decimal / exponent notation); duplicates are summed in file order."""
    import scipy.sparse as sp

    def err(line, what):
        return MatrixMarketError(f"{path}:{line}: {what}")

    try:
        f = open(path, "r")
    except OSError:
        raise RuntimeError("read_matrix_market: cannot open " + path)
    with f:
        lines = f.read().split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    if not lines:
        raise err(1, "empty file")
    tok = lines[0].split() + [""] * 5
    banner, obj, fmt, field_, sym = tok[:5]
    if banner != "%%MatrixMarket" or obj.lower() != "matrix":
        raise err(1, "not a MatrixMarket matrix header")
    fmt, field_, sym = fmt.lower(), field_.lower(), sym.lower()
    if field_ in ("complex", "pattern"):
        raise err(1, f"unsupported field '{field_}' (real data required)")
    if field_ not in ("real", "integer", "double"):
        raise err(1, f"unknown field '{field_}'")
    if sym not in ("general", "symmetric", "skew-symmetric"):
        raise err(1, f"unsupported symmetry '{sym}'")
    state = {"line": 1, "pos": 1}

    def next_data():
        while state["pos"] < len(lines):
            ln = lines[state["pos"]]
            state["pos"] += 1
            state["line"] += 1
            st = ln.lstrip(" \t\r")
            if st == "" or st.startswith("%"):
                continue
            return ln
        return None

    def ints(ln, k):
        parts = ln.split()
        return [int(x) for x in parts[:k]] if len(parts) >= k else None

    ln = next_data()
    if ln is None:
        raise err(state["line"], "missing size line")
    if fmt == "array":
        try:
            rows, cols = ints(ln, 2)
        except (TypeError, ValueError):
            raise err(state["line"], "bad array size line")
        if rows < 1 or cols < 1:
            raise err(state["line"], "bad array size line")
        a = np.zeros((rows, cols))
        for j in range(cols):
            for i in range(0 if sym == "general" else j, rows):
                ln = next_data()
                if ln is None:
                    raise err(state["line"], "unexpected end of array data")
                try:
                    v = float(ln.split()[0])
                except (IndexError, ValueError):
                    raise err(state["line"], "bad array value")
                a[i, j] = v
                if sym == "symmetric":
                    a[j, i] = v
                if sym == "skew-symmetric":
                    a[j, i] = -v
        return ProblemMatrix(a)
    if fmt != "coordinate":
        raise err(1, f"unknown format '{fmt}'")
    try:
        rows, cols, nnz = ints(ln, 3)
    except (TypeError, ValueError):
        raise err(state["line"], "bad coordinate size line")
    if rows < 1 or cols < 1 or nnz < 0:
        raise err(state["line"], "bad coordinate size line")
    trip = []
    for _ in range(nnz):
        ln = next_data()
        if ln is None:
            raise err(state["line"], "unexpected end of coordinate data")
        parts = ln.split()
        try:
            i, j, v = int(parts[0]), int(parts[1]), float(parts[2])
        except (IndexError, ValueError):
            raise err(state["line"], "bad coordinate entry")
        if i < 1 or i > rows or j < 1 or j > cols:
            raise err(state["line"], "index out of range")
        trip.append((i - 1, j - 1, v))
        if sym != "general" and i != j:
            trip.append((j - 1, i - 1, v if sym == "symmetric" else -v))
    acc = {}
    for i, j, v in trip:                       # setFromTriplets: duplicates summed in file order
        acc[(i, j)] = acc[(i, j)] + v if (i, j) in acc else v
    keys = sorted(acc, key=lambda ij: (ij[1], ij[0]))
    data = np.array([acc[k] for k in keys], dtype=np.float64)
    ri = np.array([k[0] for k in keys], dtype=np.int64)
    ci = np.array([k[1] for k in keys], dtype=np.int64)
    colptr = np.zeros(cols + 1, dtype=np.int64)
    np.add.at(colptr, ci + 1, 1)
    return ProblemMatrix(sp.csc_matrix((data, ri, np.cumsum(colptr)), shape=(rows, cols)))


# ----------------------------------------------------------------------------- shifted solves
class ShiftedFactorization:
    """shifted_solver.hpp:20-40: LU of (z I - G) with partial pivoting + the pivot floor."""

    def __init__(self, gram: np.ndarray, shift: complex, gram_absmax: Optional[float] = None):
        if gram.shape[0] != gram.shape[1]:
            raise ValueError("ShiftedFactorization: Gram matrix must be square")
        self.shift = shift
        self.n = gram.shape[0]
        shifted = (-gram).astype(np.complex128)
        shifted[np.diag_indices(self.n)] += shift
        self.lu, self.piv = sla.lu_factor(shifted, overwrite_a=True, check_finite=False)
        scale = (np.abs(gram).max() if gram_absmax is None else gram_absmax) + abs(shift)
        floor = 1e-30 * scale
        if np.abs(np.diag(self.lu)).min() <= floor:
            raise NumericalError("ShiftedFactorization: shift numerically on the spectrum")

    def solve(self, rhs: np.ndarray) -> np.ndarray:
        if rhs.shape[0] != self.n:
            raise ValueError("ShiftedFactorization: right-hand side dimension mismatch")
        return sla.lu_solve((self.lu, self.piv), rhs.astype(np.complex128), check_finite=False)


def factor_bytes(n: int) -> int:
    """shifted_solver.hpp:68-71."""
    return n * n * 16


@dataclass
class MomentBlocks:
    """moments.hpp:51-71."""
    blocks: List[np.ndarray]

    def degree(self):
        return len(self.blocks) - 1

    def stacked(self):
        return np.hstack(self.blocks[:self.degree()])

    def stacked_plus(self):
        return np.hstack(self.blocks[1:self.degree() + 1])


class MomentAccumulator:
    """moments.hpp:101-169: factor cache (<= 4 GiB), refine, accumulate (ascending j)."""

    def __init__(self, gram: np.ndarray, rule: ContourRule, threads: int = 0,
                 cache_budget_bytes: int = 4 << 30):
        self.gram, self.rule = gram, rule
        self.half = rule.count // 2
        self.absmax = float(np.abs(gram).max())
        self.cache_factors = self.half * factor_bytes(gram.shape[0]) <= cache_budget_bytes
        self.cache = None
        if self.cache_factors:
            self.cache = [ShiftedFactorization(gram, rule.shift(j), self.absmax)
                          for j in range(self.half)]

    def solve_all(self, s0: np.ndarray, shifts=None) -> List[np.ndarray]:
        rhs = s0.astype(np.complex128)
        out = []
        for j in (range(self.half) if shifts is None else shifts):
            if self.cache_factors:
                out.append(self.cache[j].solve(rhs))
            else:
                out.append(ShiftedFactorization(self.gram, self.rule.shift(j), self.absmax).solve(rhs))
        return out

    def refine(self, s0: np.ndarray) -> np.ndarray:
        """moments.hpp:121-128."""
        sols = self.solve_all(s0)
        acc = np.zeros(s0.shape)
        for j in range(self.half):
            acc += 2.0 * (self.rule.weights[j] * sols[j]).real
        return acc

    def accumulate(self, s0: np.ndarray, degree: int, shifts=None) -> MomentBlocks:
        """moments.hpp:132-147: k outer, j ascending, power_j *= t_j (untransformed node).

        `shifts` restricts the sum to a subset of j (the multi-GPU shard restatement)."""
        js = list(range(self.half)) if shifts is None else list(shifts)
        sols = self.solve_all(s0, js)
        blocks = [np.zeros(s0.shape) for _ in range(degree + 1)]
        power = [1 + 0j for _ in js]
        for k in range(degree + 1):
            for idx, j in enumerate(js):
                w = complex(self.rule.weights[j]) * power[idx]
                blocks[k] += 2.0 * (w * sols[idx]).real
                power[idx] *= complex(self.rule.nodes[j])
        return MomentBlocks(blocks)


@dataclass
class ReducedBasis:
    """moments.hpp:74-80."""
    left: np.ndarray
    singular_values: np.ndarray
    right: np.ndarray

    def rank(self):
        return self.singular_values.size


def _svd(mat: np.ndarray):
    """Jacobi SVD standing in for Eigen::JacobiSVD (moments.hpp:199, extract.hpp:68).

    The reference picks a Jacobi method on purpose: it never deflates roundoff-level singular values
    to zero, so delta = 1e-20 keeps the full direction set (moments.hpp:183-189). LAPACK dgejsv
    (preconditioned one-sided Jacobi, Drmac-Veselic) with JOBA = 'C' keeps every value above
    underflow as well (no rank truncation), like the library's QR-preconditioned one-sided Jacobi
    (csrc/jacobi_svd.cu). Returns (U, sigma nonincreasing, V) with mat = U diag(sigma) V^T; a
    matrix with fewer rows than columns is decomposed through its transpose (dgejsv needs m >= n).
    """
    a = np.asfortranarray(mat, dtype=np.float64)
    m, n = a.shape
    if m < n:
        v, s, u = _svd(a.T)
        return u, s, v
    if n == 0:
        return np.zeros((m, 0)), np.zeros(0), np.zeros((0, 0))
    sva, u, v, work, _, info = sla.lapack.dgejsv(a, joba=0, jobu=0, jobv=0)
    if info < 0:
        raise ValueError(f"dgejsv: illegal argument {-info}")
    if info > 0:   # no convergence in the Jacobi sweeps: fall back to the bidiagonal SVD
        u2, s2, vt2 = sla.svd(a, full_matrices=False, lapack_driver="gesvd", check_finite=False)
        return u2, s2, vt2.T
    s = sva * (work[1] / work[0])
    return u[:, :n], s, v[:, :n]


def low_rank(stacked: np.ndarray, delta: float) -> ReducedBasis:
    """moments.hpp:190-211: HouseholderQR -> thin Q, SVD(R), keep sigma >= delta sigma_0."""
    q, r = np.linalg.qr(stacked, mode="reduced")
    u, sv, v = _svd(r)
    if sv.size == 0 or not (sv[0] > 0):
        raise EmptySubspaceError(
            "low_rank: stacked moment matrix vanished (no spectrum inside the interval)")
    rank = 0
    while rank < sv.size and sv[rank] >= delta * sv[0]:
        rank += 1
    return ReducedBasis(q @ u[:, :rank], sv[:rank].copy(), v[:, :rank].copy())


# ----------------------------------------------------------------------------- extraction
@dataclass
class TripletSet:
    """extract.hpp:21-31."""
    sigma: np.ndarray
    left: np.ndarray
    right: np.ndarray
    q: np.ndarray
    in_interval: np.ndarray
    invalid: np.ndarray

    def count(self):
        return self.sigma.size


def project_qr(a: ProblemMatrix, basis: ReducedBasis):
    """extract.hpp:43-57: economy QR of A U_S1; rank flag |B_ii| <= 1e-14 |B_11|."""
    au = a.apply(basis.left)
    qmat, b = np.linalg.qr(au, mode="reduced")
    lead = abs(b[0, 0])
    rank_def = bool(np.any(np.abs(np.diag(b)) <= 1e-14 * lead))
    return qmat, b, rank_def


def svd_small(b: np.ndarray):
    """extract.hpp:66-70: B = P diag(phi) Q^T, phi nonincreasing."""
    return _svd(b)


def assemble_triplets(orthonormal, basis: ReducedBasis, p, phi, qm, lo, hi) -> TripletSet:
    """extract.hpp:76-102: stable ascending sort; u = Utilde p, v = U_S1 q; closed interval."""
    order = np.argsort(phi, kind="stable")
    sigma = phi[order].copy()
    left = orthonormal @ p[:, order]
    right = basis.left @ qm[:, order]
    q = qm[:, order].copy()
    in_int = (sigma >= lo) & (sigma <= hi)
    return TripletSet(sigma, left, right, q, in_int, np.zeros(sigma.size, dtype=bool))


def naive_eigen_route(a: ProblemMatrix, gram, basis: ReducedBasis, lo, hi) -> TripletSet:
    """extract.hpp:108-139 (comparator mode)."""
    h = basis.left.T @ gram @ basis.left
    h = (h + h.T) / 2.0
    theta, vecs = np.linalg.eigh(h)
    t = theta.size
    sigma = np.sqrt(np.maximum(theta, 0.0))
    right = basis.left @ vecs
    left = np.zeros((a.rows, t))
    invalid = np.zeros(t, dtype=bool)
    for i in range(t):
        if theta[i] > 0:
            left[:, i] = a.apply(right[:, i]) / sigma[i]
        else:
            invalid[i] = True
    in_int = (sigma >= lo) & (sigma <= hi)
    return TripletSet(sigma, left, right, vecs.copy(), in_int, invalid)


# ----------------------------------------------------------------------------- postprocess
@dataclass
class SpuriousVerdict:
    tau: np.ndarray
    threshold: float
    spurious: np.ndarray


def detect_spurious(ts: TripletSet, sigma_s1: np.ndarray, epsilon: float) -> SpuriousVerdict:
    """postprocess.hpp:47-62."""
    if np.any(sigma_s1 <= 0):
        raise ValueError("detect_spurious: Sigma_S1 must be positive")
    threshold = epsilon * sigma_s1.max()
    q2 = ts.q ** 2
    tau = q2.sum(axis=0) / (q2 / sigma_s1[:, None]).sum(axis=0)
    spurious = (tau < threshold) | ts.invalid
    return SpuriousVerdict(tau, threshold, spurious)


def exact_residual(a: ProblemMatrix, ts: TripletSet) -> np.ndarray:
    """postprocess.hpp:34-41: ||A^T u_i - sigma_i v_i||."""
    atu = a.apply_adjoint(ts.left)
    return np.linalg.norm(atu - ts.right * ts.sigma[None, :], axis=0)


def stabilized_inverse(sigma: np.ndarray, rcond: float) -> np.ndarray:
    """postprocess.hpp:70-74."""
    cutoff = rcond * sigma.max()
    return np.where(sigma >= cutoff, 1.0 / sigma, 0.0)


def transformed_residual_norms(blocks: MomentBlocks, basis: ReducedBasis, ts: TripletSet,
                               images, rcond: float) -> np.ndarray:
    """postprocess.hpp:76-97 (all triplets at once: the columns are independent)."""
    splus = blocks.stacked_plus()
    inv = stabilized_inverse(basis.singular_values, rcond)
    coeff = basis.right @ (inv[:, None] * ts.q)
    res = splus @ coeff - (basis.left @ ts.q) * np.asarray(images)[None, :]
    out = np.linalg.norm(res, axis=0) / np.where(ts.sigma > 1e-30, ts.sigma, 1.0)
    out[ts.sigma <= 1e-30] = np.inf
    return out


def estimate_residual_linear(blocks, basis, ts, rcond=K_RCOND_IDENTITY):
    """postprocess.hpp:107-115."""
    return transformed_residual_norms(blocks, basis, ts, ts.sigma * ts.sigma, rcond)


@dataclass
class ResidualReport:
    exact: Optional[np.ndarray] = None
    estimated: Optional[np.ndarray] = None
    calibration_index: Optional[int] = None
    mu: Optional[float] = None


def estimate_residual_nonlinear(blocks, basis, ts, a: ProblemMatrix, transform, verdict,
                                rcond=K_RCOND_EXP) -> ResidualReport:
    """postprocess.hpp:121-156: images g^{-1}(sigma^2); calibrate at argmax tau."""
    images = [transform.g_inverse(s * s) if s > 1e-30 else 0.0 for s in ts.sigma]
    tilde = transformed_residual_norms(blocks, basis, ts, images, rcond)
    best = -1
    for i in range(ts.count()):
        if not ts.in_interval[i] or verdict.spurious[i]:
            continue
        if best < 0 or verdict.tau[i] > verdict.tau[best]:
            best = i
    if best < 0:
        raise NumericalError(
            "estimate_residual_nonlinear: no non-spurious in-interval triplet to calibrate with")
    exact_at_best = float(np.linalg.norm(a.apply_adjoint(ts.left[:, best])
                                         - ts.sigma[best] * ts.right[:, best]))
    mu = exact_at_best / tilde[best]
    est = mu * tilde
    est[best] = exact_at_best
    return ResidualReport(None, est, best, mu)


# ----------------------------------------------------------------------------- pipeline
@dataclass
class StepTimings:
    """pipeline.hpp:65-72."""
    steps_1_2: float = 0.0
    step_3: float = 0.0
    step_4: float = 0.0
    step_5: float = 0.0
    postprocess: float = 0.0

    def total(self):
        return self.steps_1_2 + self.step_3 + self.step_4 + self.step_5


@dataclass
class RunResult:
    """pipeline.hpp:74-95."""
    triplets: Optional[TripletSet] = None
    verdict: Optional[SpuriousVerdict] = None
    residuals: ResidualReport = field(default_factory=ResidualReport)
    galerkin: Optional[np.ndarray] = None
    basis: Optional[ReducedBasis] = None
    blocks: Optional[MomentBlocks] = None
    left_projection_basis: Optional[np.ndarray] = None
    rank_deficient_qr: bool = False
    timings: StepTimings = field(default_factory=StepTimings)
    empty: bool = False
    note: str = ""
    input_transposed: bool = False
    count_in_interval: int = 0
    count_nonspurious_in_interval: int = 0
    count_interior: int = 0
    count_boundary: int = 0
    starting_norm: float = 0.0

    def retained_rank(self):
        return 0 if self.basis is None else self.basis.rank()


def near_endpoint(sigma: float, endpoint: float) -> bool:
    """pipeline.hpp:103-106."""
    return abs(sigma - endpoint) <= 1e-9 * max(abs(endpoint), sigma)


EMPTY_NOTE = "filter annihilated the starting block: no singular values inside the interval"


def run_solve(a: ProblemMatrix, config: RunConfig, gram_cap: int = 8192) -> RunResult:
    """pipeline.hpp:112-231, step for step (timers in the same StepTimings buckets)."""
    config.params.validate(a.cols)
    transform = config.transform()
    rule = ContourRule(config.interval_a, config.interval_b, config.params.quadrature_count,
                       config.aspect, transform)
    result = RunResult(input_transposed=a.transposed)

    t0 = time.perf_counter()
    gram = form_gram(a, gram_cap)
    acc = MomentAccumulator(gram, rule, config.threads)
    block = random_start(a.cols, config.params.block_size, config.params.seed)
    starting_norm = float(np.linalg.norm(block))
    result.starting_norm = starting_norm
    for _ in range(1, config.params.refinement_steps):
        block = acc.refine(block)
    result.blocks = acc.accumulate(block, config.params.moment_degree)
    result.timings.steps_1_2 = time.perf_counter() - t0
    return finish_solve(a, config, result, gram)


def finish_solve(a: ProblemMatrix, config: RunConfig, result: RunResult, gram=None) -> RunResult:
    """Steps 3-5 + postprocess of run_solve (pipeline.hpp:141-231) from result.blocks."""
    transform = config.transform()
    t0 = time.perf_counter()
    stacked = result.blocks.stacked()
    if np.linalg.norm(stacked) <= 1e-12 * result.starting_norm:
        result.empty = True
        result.note = EMPTY_NOTE
        result.timings.step_3 = time.perf_counter() - t0
        return result
    try:
        result.basis = low_rank(stacked, config.params.lowrank_threshold)
    except EmptySubspaceError:
        result.empty = True
        result.note = EMPTY_NOTE
        result.timings.step_3 = time.perf_counter() - t0
        return result
    result.timings.step_3 = time.perf_counter() - t0

    if config.mode not in (NAIVE, NAIVE_NT):
        t0 = time.perf_counter()
        orth, b, rank_def = project_qr(a, result.basis)
        result.timings.step_4 = time.perf_counter() - t0
        t0 = time.perf_counter()
        p, phi, qm = svd_small(b)
        result.triplets = assemble_triplets(orth, result.basis, p, phi, qm,
                                            config.interval_a, config.interval_b)
        result.timings.step_5 = time.perf_counter() - t0
        result.rank_deficient_qr = rank_def
        result.left_projection_basis = orth
    else:
        t0 = time.perf_counter()
        if gram is None:
            gram = form_gram(a, 1 << 30)
        result.triplets = naive_eigen_route(a, gram, result.basis, config.interval_a,
                                            config.interval_b)
        result.timings.step_5 = time.perf_counter() - t0

    t0 = time.perf_counter()
    ts = result.triplets
    result.verdict = detect_spurious(ts, result.basis.singular_values,
                                     config.params.spurious_threshold)
    if transform.kind == EXP:
        try:
            result.residuals = estimate_residual_nonlinear(result.blocks, result.basis, ts, a,
                                                           transform, result.verdict,
                                                           config.estimator_rcond_exp)
        except NumericalError:
            result.residuals = ResidualReport(None, np.full(ts.count(), np.nan), None, None)
            result.note = "nonlinear residual calibration impossible: all candidates spurious"
    else:
        result.residuals = ResidualReport(
            None, estimate_residual_linear(result.blocks, result.basis, ts,
                                           config.estimator_rcond_identity), None, None)
    result.residuals.exact = exact_residual(a, ts)
    if result.residuals.calibration_index is not None:
        ci = result.residuals.calibration_index
        result.residuals.estimated[ci] = result.residuals.exact[ci]
    av = a.apply(ts.right)
    result.galerkin = np.linalg.norm(av - ts.left * ts.sigma[None, :], axis=0)
    result.timings.postprocess = time.perf_counter() - t0

    if a.transposed:
        ts.left, ts.right = ts.right, ts.left
        result.residuals.exact, result.galerkin = result.galerkin, result.residuals.exact

    for i in range(ts.count()):
        if not ts.in_interval[i]:
            continue
        result.count_in_interval += 1
        if not result.verdict.spurious[i]:
            result.count_nonspurious_in_interval += 1
        if near_endpoint(ts.sigma[i], config.interval_a) or near_endpoint(ts.sigma[i], config.interval_b):
            result.count_boundary += 1
        else:
            result.count_interior += 1
    return result


@dataclass
class AccuracyStats:
    max_rel_error_nonspurious: float = 0.0
    median_rel_error_nonspurious: float = 0.0
    max_rel_error_all: float = 0.0
    median_rel_error_all: float = 0.0
    matched_nonspurious: int = 0
    matched_all: int = 0


def accuracy_vs_truth(truth: np.ndarray, result: RunResult) -> AccuracyStats:
    """pipeline.hpp:245-273."""
    rel_all, rel_ns = [], []
    ts = result.triplets
    if ts is not None:
        for i in range(ts.count()):
            if not ts.in_interval[i]:
                continue
            s = ts.sigma[i]
            best = float(np.min(np.abs(truth - s) / truth))
            rel_all.append(best)
            if not result.verdict.spurious[i]:
                rel_ns.append(best)
    st = AccuracyStats()
    st.matched_all, st.matched_nonspurious = len(rel_all), len(rel_ns)
    st.max_rel_error_all = max(rel_all) if rel_all else 0.0
    st.max_rel_error_nonspurious = max(rel_ns) if rel_ns else 0.0
    st.median_rel_error_all = float(np.median(rel_all)) if rel_all else 0.0
    st.median_rel_error_nonspurious = float(np.median(rel_ns)) if rel_ns else 0.0
    return st


# ----------------------------------------------------------------------------- model problems
def model_spectrum(which: int, n: int) -> np.ndarray:
    """problems.hpp:38-48."""
    i = np.arange(n, dtype=np.float64)
    if which == 1:
        return 0.005 + 0.01 * i
    return np.array([math.pow(10.0, -10.0 + 0.05 * float(k)) for k in range(n)])


def build_model(which: int = 1, rows: int = 1000, cols: int = 200, seed: int = 7):
    """problems.hpp:50-70: same normal stream, Householder Q (no sign fix), A = U S V^T."""
    if rows < cols:
        raise ValueError("build_model: needs rows >= cols")
    draws = normal_stream(seed, rows * cols + cols * cols)
    gu = draws[:rows * cols].reshape((cols, rows)).T
    gv = draws[rows * cols:].reshape((cols, cols)).T
    u, _ = np.linalg.qr(gu, mode="reduced")
    v, _ = np.linalg.qr(gv, mode="reduced")
    sigma = model_spectrum(which, cols)
    a = (u * sigma[None, :]) @ v.T
    return ProblemMatrix(a), u, sigma, v
