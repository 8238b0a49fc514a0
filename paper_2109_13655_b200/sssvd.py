"""Python mirror of the reference `sssvd` API over the C ABI of libsssvd_gpu.so.

The reference is a header-only C++ library (proj/include/sssvd); this module exposes the same
names, argument meanings and error behaviour for the shifted-solve path so the parity tests read
like the reference's own tests:

    ProblemMatrix.from_dense   problem.hpp:20-25       form_gram            problem.hpp:81-95
    ProblemMatrix.from_sparse  problem.hpp:27-35       read/write_matrix_market matrix_market.hpp:34-149
    ContourRule / build_contour contour.hpp:27-62     SpectralTransform     transform.hpp:16-45
    SsParams (+ validate)      moments.hpp:23-47       random_start         moments.hpp:84-94
    ShiftedFactorization       shifted_solver.hpp:20-40 (factor_shift / solve_block :77-87)
    DenseShiftedSolver         shifted_solver.hpp:54-75
    MomentAccumulator          moments.hpp:101-169 (refine / accumulate)
    RunConfig / run_solve      pipeline.hpp:43-58 / :112-231
Errors map back onto the reference's exception types (core.hpp:29-39).

Everything numerical runs in the CUDA library; there is no CPU fallback. Loading this module
without the built library, or calling a compute entry point without a B200, raises.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsssvd_gpu.so")


# ----------------------------------------------------------------------------- errors
class NumericalError(RuntimeError):
    """core.hpp:29-32."""


class EmptySubspaceError(NumericalError):
    """core.hpp:36-39."""


class DomainError(ValueError):
    """std::domain_error."""


class LengthError(ValueError):
    """std::length_error."""


class CudaError(RuntimeError):
    pass


class MatrixMarketError(RuntimeError):
    """matrix_market.hpp:17-21: "path:line: what"."""


SSSVD_OK, E_INVALID, E_DOMAIN, E_LENGTH, E_NUMERICAL, E_EMPTY, E_CUDA, E_NCCL, E_OOM, E_FORMAT, E_IO = range(11)


def _raise(code: int, msg: str):
    if code == E_INVALID:
        raise ValueError(msg)
    if code == E_DOMAIN:
        raise DomainError(msg)
    if code == E_LENGTH:
        raise LengthError(msg)
    if code == E_NUMERICAL:
        raise NumericalError(msg)
    if code == E_EMPTY:
        raise EmptySubspaceError(msg)
    if code == E_FORMAT:
        raise MatrixMarketError(msg)
    if code == E_IO:
        raise RuntimeError(msg)
    raise CudaError(f"status {code}: {msg}")


# ----------------------------------------------------------------------------- C structs
class _Params(ctypes.Structure):
    _fields_ = [("block_size", ctypes.c_int64), ("moment_degree", ctypes.c_int64),
                ("quadrature_count", ctypes.c_int64), ("refinement_steps", ctypes.c_int64),
                ("lowrank_threshold", ctypes.c_double), ("spurious_threshold", ctypes.c_double),
                ("seed", ctypes.c_uint64)]


class _Config(ctypes.Structure):
    _fields_ = [("interval_a", ctypes.c_double), ("interval_b", ctypes.c_double),
                ("mode", ctypes.c_int32), ("aspect", ctypes.c_double), ("params", _Params),
                ("threads", ctypes.c_int32), ("estimator_rcond_identity", ctypes.c_double),
                ("estimator_rcond_exp", ctypes.c_double), ("gram_cap", ctypes.c_int64)]


class _Info(ctypes.Structure):
    _fields_ = [("count", ctypes.c_int64), ("rows", ctypes.c_int64), ("cols", ctypes.c_int64),
                ("retained_rank", ctypes.c_int64), ("n_internal", ctypes.c_int64),
                ("block_size", ctypes.c_int64), ("moment_degree", ctypes.c_int64),
                ("empty", ctypes.c_int32), ("input_transposed", ctypes.c_int32),
                ("rank_deficient_qr", ctypes.c_int32),
                ("count_in_interval", ctypes.c_int64),
                ("count_nonspurious_in_interval", ctypes.c_int64),
                ("count_interior", ctypes.c_int64), ("count_boundary", ctypes.c_int64),
                ("calibration_index", ctypes.c_int64), ("mu", ctypes.c_double),
                ("spurious_threshold", ctypes.c_double),
                ("steps_1_2", ctypes.c_double), ("step_3", ctypes.c_double),
                ("step_4", ctypes.c_double), ("step_5", ctypes.c_double),
                ("postprocess", ctypes.c_double), ("t_gram", ctypes.c_double),
                ("t_shifted_solves", ctypes.c_double), ("t_allreduce", ctypes.c_double),
                ("shifted_solve_flops", ctypes.c_double)]


EXPORTED_SYMBOLS = [
    "sssvd_default_config", "sssvd_gpu_create", "sssvd_gpu_destroy", "sssvd_gpu_last_error",
    "sssvd_gpu_set_batch", "sssvd_gpu_nccl_unique_id", "sssvd_gpu_init_comm", "sssvd_shard_range", "sssvd_gram_tiles",
    "sssvd_gpu_set_operator", "sssvd_gpu_set_operator_root", "sssvd_gpu_comm_size", "sssvd_gpu_form_gram", "sssvd_gpu_shifted_solve", "sssvd_gpu_moments",
    "sssvd_gpu_run_solve", "sssvd_result_info_get", "sssvd_result_copy", "sssvd_result_note",
    "sssvd_result_free", "sssvd_contour", "sssvd_random_start", "sssvd_validate_params",
    "sssvd_moment_coefficients", "sssvd_build_info", "sssvd_gpu_launch_count", "sssvd_gpu_profile_gemm",
    "sssvd_gpu_profile_gemm_collect", "sssvd_gpu_profile_gemm_collect2", "sssvd_debug_gram_part",
    "sssvd_gpu_set_operator_csc", "sssvd_mm_read", "sssvd_mm_info_get", "sssvd_mm_values", "sssvd_mm_colptr",
    "sssvd_mm_rowind", "sssvd_mm_free", "sssvd_mm_write", "sssvd_host_last_error", "sssvd_build_model",
    "sssvd_filter_profile", "sssvd_debug_thin_qr", "sssvd_debug_svd_square", "sssvd_debug_zgemm",
    "sssvd_debug_dgemm",
]

class _MmInfo(ctypes.Structure):
    _fields_ = [("rows", ctypes.c_int64), ("cols", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("sparse", ctypes.c_int)]


_lib = None


def lib():
    """Load libsssvd_gpu.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2109_13655_b200.build`")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, dp, ip = ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
    L.sssvd_default_config.argtypes = [ctypes.POINTER(_Config)]
    L.sssvd_gpu_create.argtypes = [ctypes.c_int, ctypes.POINTER(vp)]
    L.sssvd_gpu_destroy.argtypes = [vp]
    L.sssvd_gpu_last_error.argtypes = [vp]
    L.sssvd_gpu_last_error.restype = ctypes.c_char_p
    L.sssvd_gpu_set_batch.argtypes = [vp, ctypes.c_int]
    L.sssvd_gpu_nccl_unique_id.argtypes = [vp]
    L.sssvd_gpu_init_comm.argtypes = [vp, vp, ctypes.c_int, ctypes.c_int]
    L.sssvd_shard_range.argtypes = [i64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.sssvd_shard_range.restype = None
    L.sssvd_gram_tiles.argtypes = [i64, ctypes.c_int, ctypes.c_int, dp, i64]
    L.sssvd_gram_tiles.restype = i64
    L.sssvd_gpu_set_operator.argtypes = [vp, dp, i64, i64, i64, ip]
    L.sssvd_gpu_set_operator_root.argtypes = [vp, dp, i64, i64, i64, ip, ip]
    L.sssvd_gpu_comm_size.argtypes = [vp, ctypes.POINTER(ctypes.c_int)]
    L.sssvd_gpu_set_operator_csc.argtypes = [vp, i64, i64, i64, dp, dp, dp, ip]
    L.sssvd_gpu_form_gram.argtypes = [vp, i64, dp]
    L.sssvd_mm_read.argtypes = [ctypes.c_char_p, ctypes.POINTER(vp)]
    L.sssvd_mm_info_get.argtypes = [vp, ctypes.POINTER(_MmInfo)]
    L.sssvd_mm_info_get.restype = None
    for f in ("sssvd_mm_values", "sssvd_mm_colptr", "sssvd_mm_rowind"):
        getattr(L, f).argtypes = [vp]
        getattr(L, f).restype = vp
    L.sssvd_mm_free.argtypes = [vp]
    L.sssvd_mm_free.restype = None
    L.sssvd_mm_write.argtypes = [ctypes.c_char_p, i64, i64, i64, dp, dp, dp, ctypes.c_char_p]
    L.sssvd_host_last_error.restype = ctypes.c_char_p
    L.sssvd_debug_thin_qr.argtypes = [vp, dp, i64, i64, dp, dp]
    L.sssvd_debug_svd_square.argtypes = [vp, dp, i64, dp, dp, dp]
    L.sssvd_debug_zgemm.argtypes = [vp, ctypes.c_int, i64, i64, i64, i64, ctypes.c_int, dp,
                                    ctypes.POINTER(ctypes.c_int64)]
    L.sssvd_debug_dgemm.argtypes = [vp, ctypes.c_int, ctypes.c_int, i64, i64, i64, ctypes.c_double, dp, i64, dp, i64,
                                    ctypes.c_double, dp, dp, dp, i64]
    L.sssvd_build_model.argtypes = [ctypes.c_int, i64, i64, ctypes.c_uint64, dp, dp]
    L.sssvd_filter_profile.argtypes = [ctypes.c_double, ctypes.c_double, i64, ctypes.c_double, ctypes.c_int,
                                       ctypes.c_double, ctypes.c_double, i64, ctypes.c_int, dp, dp]
    L.sssvd_gpu_shifted_solve.argtypes = [vp, dp, i64, ctypes.c_double, ctypes.c_double, dp, i64, i64, dp]
    L.sssvd_gpu_moments.argtypes = [vp, i64, dp, dp, dp, dp, i64, i64, i64, dp]
    L.sssvd_gpu_run_solve.argtypes = [vp, ctypes.POINTER(_Config), ctypes.POINTER(vp)]
    L.sssvd_result_info_get.argtypes = [vp, ctypes.POINTER(_Info)]
    L.sssvd_result_copy.argtypes = [vp, ctypes.c_int, dp]
    L.sssvd_result_note.argtypes = [vp]
    L.sssvd_result_note.restype = ctypes.c_char_p
    L.sssvd_result_free.argtypes = [vp]
    L.sssvd_result_free.restype = None
    L.sssvd_contour.argtypes = [ctypes.c_double, ctypes.c_double, i64, ctypes.c_double, ctypes.c_int, dp, dp, dp]
    L.sssvd_random_start.argtypes = [i64, i64, ctypes.c_uint64, dp]
    L.sssvd_validate_params.argtypes = [ctypes.POINTER(_Params), i64]
    L.sssvd_moment_coefficients.argtypes = [i64, dp, dp, i64, dp]
    L.sssvd_build_info.restype = ctypes.c_char_p
    L.sssvd_debug_gram_part.argtypes = [vp, ctypes.c_int, ctypes.c_int, dp]
    L.sssvd_gpu_launch_count.restype = ctypes.c_uint64
    L.sssvd_gpu_profile_gemm.argtypes = [ctypes.c_int]
    L.sssvd_gpu_profile_gemm.restype = None
    L.sssvd_gpu_profile_gemm_collect.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                                 ctypes.POINTER(ctypes.c_uint64)]
    L.sssvd_gpu_profile_gemm_collect.restype = None
    L.sssvd_gpu_profile_gemm_collect2.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                                  ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_uint64)]
    L.sssvd_gpu_profile_gemm_collect2.restype = None
    _lib = L
    return L


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ----------------------------------------------------------------------------- transform / contour
IDENTITY, EXP = 0, 1


class SpectralTransform:
    """transform.hpp:16-45."""

    def __init__(self, kind: int):
        self._kind = kind

    @staticmethod
    def identity():
        return SpectralTransform(IDENTITY)

    @staticmethod
    def exponential():
        return SpectralTransform(EXP)

    def kind(self):
        return self._kind

    def g(self, t):
        return t if self._kind == IDENTITY else np.exp(t)

    def g_inverse(self, z: float) -> float:
        if self._kind == IDENTITY:
            return z
        if not z > 0:
            raise DomainError("SpectralTransform: g_inverse of non-positive value under Exp")
        return math.log(z)

    def g_prime(self, t: float) -> float:
        return 1.0 if self._kind == IDENTITY else math.exp(t)


class ContourRule:
    """contour.hpp:27-62, computed by the library's host mirror (host_mirror.cpp)."""

    def __init__(self, a: float, b: float, count: int, aspect: float, transform: SpectralTransform):
        nodes = np.empty(2 * count)
        weights = np.empty(2 * count)
        cr = np.empty(2)
        st = lib().sssvd_contour(a, b, count, aspect, transform.kind(), _ptr(nodes), _ptr(weights), _ptr(cr))
        if st != SSSVD_OK:
            _raise(st, "ContourRule: " + ("Exp transform requires a > 0" if st == E_DOMAIN else "bad arguments"))
        self._a, self._b, self._count, self._aspect, self._transform = a, b, count, aspect, transform
        self._center, self._radius = float(cr[0]), float(cr[1])
        self._nodes = nodes.view(np.complex128).copy()
        self._weights = weights.view(np.complex128).copy()

    def interval_a(self): return self._a
    def interval_b(self): return self._b
    def center(self): return self._center
    def radius(self): return self._radius
    def aspect(self): return self._aspect
    def count(self): return self._count
    def transform(self): return self._transform
    def nodes(self): return self._nodes
    def weights(self): return self._weights

    def shift(self, j: int) -> complex:
        t = complex(self._nodes[j])
        if self._transform.kind() == IDENTITY:
            return t
        e = math.exp(t.real)
        return complex(e * math.cos(t.imag), e * math.sin(t.imag))


def build_contour(a, b, count, aspect, transform):
    return ContourRule(a, b, count, aspect, transform)


# ----------------------------------------------------------------------------- params / config
@dataclass
class SsParams:
    """moments.hpp:23-47."""
    block_size: int = 20
    moment_degree: int = 4
    quadrature_count: int = 32
    refinement_steps: int = 1
    lowrank_threshold: float = 1e-20
    spurious_threshold: float = 1e-8
    seed: int = 42

    def subspace_dim(self):
        return self.block_size * self.moment_degree

    def _c(self):
        return _Params(self.block_size, self.moment_degree, self.quadrature_count, self.refinement_steps,
                       self.lowrank_threshold, self.spurious_threshold, self.seed)

    def validate(self, n: int):
        p = self._c()
        if lib().sssvd_validate_params(ctypes.byref(p), n) != SSSVD_OK:
            raise ValueError("SsParams: invalid parameters")


class SolveMode:
    """pipeline.hpp:24."""
    SsSvd, SsSvdNT, Naive, NaiveNT = 0, 1, 2, 3


@dataclass
class RunConfig:
    """pipeline.hpp:43-58 (+ the form_gram cap, problem.hpp:82)."""
    interval_a: float = 0.0
    interval_b: float = 1.0
    mode: int = SolveMode.SsSvd
    aspect: float = 0.1
    params: SsParams = field(default_factory=SsParams)
    threads: int = 0
    estimator_rcond_identity: float = 2e-15
    estimator_rcond_exp: float = 1e-14
    gram_cap: int = 8192

    def transform(self):
        return SpectralTransform(EXP if self.mode in (SolveMode.SsSvdNT, SolveMode.NaiveNT) else IDENTITY)

    def _c(self):
        return _Config(self.interval_a, self.interval_b, self.mode, self.aspect, self.params._c(), self.threads,
                       self.estimator_rcond_identity, self.estimator_rcond_exp, self.gram_cap)


def random_start(n: int, block_size: int, seed: int) -> np.ndarray:
    """moments.hpp:84-94 (libstdc++ mt19937_64 in the library's host mirror)."""
    out = np.empty((n, block_size), order="F")
    if lib().sssvd_random_start(n, block_size, seed, _ptr(out)) != SSSVD_OK:
        raise ValueError("random_start: block size exceeds dimension")
    return out


def moment_coefficients(weights, nodes, degree: int) -> np.ndarray:
    """c[k][j] = w_j t_j^k with the reference's power chain (moments.hpp:138-144)."""
    w = np.ascontiguousarray(weights, dtype=np.complex128)
    t = np.ascontiguousarray(nodes, dtype=np.complex128)
    out = np.empty((degree + 1) * w.size, dtype=np.complex128)
    st = lib().sssvd_moment_coefficients(w.size, _ptr(w), _ptr(t), degree, _ptr(out))
    if st != SSSVD_OK:
        _raise(st, "moment_coefficients")
    return out.reshape(degree + 1, w.size)


def launch_count() -> int:
    return int(lib().sssvd_gpu_launch_count())


def profile_gemm(enable: bool):
    lib().sssvd_gpu_profile_gemm(1 if enable else 0)


def profile_gemm_collect():
    """(GEMM-busy ms, executed tensor flops, launches) of the DMMA GEMMs since enable."""
    ms, fl, _, n = profile_gemm_collect2()
    return ms, fl, n


def profile_gemm_collect2():
    """(GEMM-busy ms, executed tensor flops, the same work in 8 M N K units, launches) since enable."""
    ms, fl, alg, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_double(), ctypes.c_uint64()
    lib().sssvd_gpu_profile_gemm_collect2(ctypes.byref(ms), ctypes.byref(fl), ctypes.byref(alg), ctypes.byref(n))
    return ms.value, fl.value, alg.value, int(n.value)


def shard_range(h: int, nranks: int, rank: int):
    b, e = ctypes.c_int64(), ctypes.c_int64()
    lib().sssvd_shard_range(h, nranks, rank, ctypes.byref(b), ctypes.byref(e))
    return b.value, e.value


def gram_tiles(n: int, nranks: int, rank: int) -> np.ndarray:
    """The (ti, tj) lower-triangle 64 x 64 tiles of G that `rank` forms in the multi-GPU form_gram
    (the decode of csrc/partition.h, shared with the kernel)."""
    cnt = lib().sssvd_gram_tiles(n, rank, nranks, None, 0)
    if cnt < 0:
        raise ValueError("gram_tiles: bad arguments")
    out = np.zeros((max(cnt, 1), 2), dtype=np.int32)
    lib().sssvd_gram_tiles(n, rank, nranks, _ptr(out), cnt)
    return out[:cnt]


# ----------------------------------------------------------------------------- device context
class Device:
    """One B200 context: owns device memory, the stream and the optional NCCL communicator."""

    def __init__(self, device: int = 0):
        h = ctypes.c_void_p()
        st = lib().sssvd_gpu_create(device, ctypes.byref(h))
        if st != SSSVD_OK:
            raise CudaError(f"sssvd_gpu_create({device}) failed: no sm_100 GPU available (status {st})")
        self.h = h

    def close(self):
        if self.h:
            lib().sssvd_gpu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, st: int):
        if st != SSSVD_OK:
            _raise(st, lib().sssvd_gpu_last_error(self.h).decode())

    def set_batch(self, max_shifts: int):
        lib().sssvd_gpu_set_batch(self.h, max_shifts)

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        if lib().sssvd_gpu_nccl_unique_id(buf) != SSSVD_OK:
            raise CudaError("ncclGetUniqueId failed")
        return buf.raw

    def init_comm(self, unique_id: bytes, nranks: int, rank: int):
        buf = ctypes.create_string_buffer(unique_id, 128)
        self.check(lib().sssvd_gpu_init_comm(self.h, buf, nranks, rank))

    def set_operator(self, a: np.ndarray):
        a = np.asfortranarray(a, dtype=np.float64)
        self.check(lib().sssvd_gpu_set_operator(self.h, _ptr(a), a.shape[0], a.shape[1], a.shape[0], 0))
        self._n = min(a.shape)

    def set_operator_csc(self, rows: int, cols: int, colptr: np.ndarray, rowind: np.ndarray, values: np.ndarray):
        """Sparse operator in the user orientation (problem.hpp:27-35), compressed CSC."""
        colptr = np.ascontiguousarray(colptr, dtype=np.int64)
        rowind = np.ascontiguousarray(rowind, dtype=np.int64)
        values = np.ascontiguousarray(values, dtype=np.float64)
        if colptr.size != cols + 1 or rowind.size != values.size:
            raise ValueError("set_operator_csc: array sizes do not match the shape")
        self.check(lib().sssvd_gpu_set_operator_csc(self.h, rows, cols, values.size, _ptr(colptr), _ptr(rowind),
                                                    _ptr(values), 0))
        self._n = min(rows, cols)

    def set_problem(self, a: "ProblemMatrix"):
        """Upload a ProblemMatrix (dense or sparse) in its user orientation."""
        if a.is_sparse():
            s = a.sparse().T.tocsc() if a.transposed() else a.sparse()
            self.set_operator_csc(s.shape[0], s.shape[1], s.indptr, s.indices, s.data)
        else:
            self.set_operator(a.dense().T if a.transposed() else a.dense())

    def set_operator_root(self, a_ptr: Optional[int], rows: int, cols: int, lda: int, on_device: bool = False,
                          root: int = 0):
        """Collective upload: rank `root` passes the operator (host or device pointer), the other
        ranks None; one ncclBroadcast of the padded operator reaches every rank."""
        self.check(lib().sssvd_gpu_set_operator_root(self.h, ctypes.c_void_p(a_ptr) if a_ptr else None, rows, cols,
                                                     lda, int(on_device), root))
        self._n = min(rows, cols)

    def comm_size(self) -> int:
        c = ctypes.c_int(0)
        self.check(lib().sssvd_gpu_comm_size(self.h, ctypes.byref(c)))
        return c.value

    def set_operator_device(self, ptr: int, rows: int, cols: int, lda: int):
        self.check(lib().sssvd_gpu_set_operator(self.h, ctypes.c_void_p(ptr), rows, cols, lda, 1))
        self._n = min(rows, cols)

    def form_gram(self, size_cap: int = 8192, copy_out: bool = True):
        if not copy_out:
            self.check(lib().sssvd_gpu_form_gram(self.h, size_cap, None))
            return None
        g = np.empty((self._n, self._n), order="F")
        self.check(lib().sssvd_gpu_form_gram(self.h, size_cap, _ptr(g)))
        return g

    def thin_qr(self, a: np.ndarray):
        """Debug: the tail's Householder QR (thin Q, R) of a tall matrix."""
        a = np.asfortranarray(a, dtype=np.float64)
        m, k = a.shape
        q, r = np.empty((m, k), order="F"), np.empty((k, k), order="F")
        self.check(lib().sssvd_debug_thin_qr(self.h, _ptr(a), m, k, _ptr(q), _ptr(r)))
        return q, r

    def svd_square(self, b: np.ndarray):
        """Debug: the tail's Jacobi SVD (U, s descending, V) of a square matrix."""
        b = np.asfortranarray(b, dtype=np.float64)
        k = b.shape[0]
        u, v, sv = np.empty((k, k), order="F"), np.empty((k, k), order="F"), np.empty(k)
        self.check(lib().sssvd_debug_svd_square(self.h, _ptr(b), k, _ptr(u), _ptr(sv), _ptr(v)))
        return u, sv, v

    def dgemm(self, a: np.ndarray, b: np.ndarray, c: Optional[np.ndarray] = None, alpha: float = 1.0,
              beta: float = 0.0, trans_a: bool = False, lda: Optional[int] = None, ldb: Optional[int] = None,
              ldc: Optional[int] = None) -> np.ndarray:
        """Debug: the tail GEMM C = alpha op(A) B + beta C (column-major; optional padded leading
        dimensions exercise the unaligned staging path)."""
        a = np.asfortranarray(a, dtype=np.float64)
        b = np.asfortranarray(b, dtype=np.float64)
        k, n = b.shape
        m = a.shape[1] if trans_a else a.shape[0]
        lda = max(lda or a.shape[0], 1)
        ldb = max(ldb or b.shape[0], 1)
        ldc = max(ldc or m, 1)
        ap = np.zeros((lda, max(a.shape[1], 1)), order="F"); ap[:a.shape[0], :a.shape[1]] = a
        bp = np.zeros((ldb, n), order="F"); bp[:k] = b
        cp = np.zeros((ldc, n), order="F")
        if c is not None:
            cp[:m] = c
        self.check(lib().sssvd_debug_dgemm(self.h, 0, int(trans_a), m, n, k, alpha, _ptr(ap), lda, _ptr(bp), ldb,
                                           beta, None, None, _ptr(cp), ldc))
        return cp[:m].copy()

    def dgemm_colnorm_diff(self, a: np.ndarray, b: np.ndarray, d: np.ndarray, v: np.ndarray,
                           trans_a: bool = False) -> np.ndarray:
        """Debug: ||op(A) B[:, j] - d_j V[:, j]|| per column through the fused GEMM epilogue."""
        a = np.asfortranarray(a, dtype=np.float64)
        b = np.asfortranarray(b, dtype=np.float64)
        v = np.asfortranarray(v, dtype=np.float64)
        d = np.ascontiguousarray(d, dtype=np.float64)
        k, n = b.shape
        m = a.shape[1] if trans_a else a.shape[0]
        out = np.zeros(max(m, 1) * n)
        self.check(lib().sssvd_debug_dgemm(self.h, 1, int(trans_a), m, n, k, 1.0, _ptr(a), max(a.shape[0], 1), _ptr(b),
                                           max(k, 1), 0.0, _ptr(d), _ptr(v), _ptr(out), m))
        return out[:n].copy()

    def run_solve(self, config: RunConfig) -> "RunResult":
        c = config._c()
        res = ctypes.c_void_p()
        self.check(lib().sssvd_gpu_run_solve(self.h, ctypes.byref(c), ctypes.byref(res)))
        return RunResult._from_handle(res)


_default_device: Optional[Device] = None


def default_device() -> Device:
    global _default_device
    if _default_device is None:
        _default_device = Device(int(os.environ.get("LOCAL_RANK", "0")))
    return _default_device


# ----------------------------------------------------------------------------- problem / Gram
class ProblemMatrix:
    """problem.hpp:14-77: dense or sparse (scipy CSC) storage, normalised so rows >= cols (wide
    inputs stored transposed and flagged). The NaN/Inf check also runs in the library."""

    def __init__(self, a, transposed: bool, sparse: bool = False):
        self._a = a
        self._transposed = transposed
        self._sparse = sparse

    @staticmethod
    def from_dense(a) -> "ProblemMatrix":
        a = np.asarray(a, dtype=np.float64)
        if not np.all(np.isfinite(a)):
            raise ValueError("ProblemMatrix: NaN/Inf entry")
        tr = a.shape[0] < a.shape[1]
        return ProblemMatrix(np.asfortranarray(a.T if tr else a), tr)

    @staticmethod
    def from_sparse(a) -> "ProblemMatrix":
        """problem.hpp:27-35. `a` is any scipy.sparse matrix/array; stored compressed CSC
        (duplicates summed, row indices sorted, explicit zeros kept) like Eigen's SparseMatrix."""
        import scipy.sparse as sp
        s = sp.csc_matrix(a, dtype=np.float64, copy=True)
        s.sum_duplicates()
        s.sort_indices()
        if not np.all(np.isfinite(s.data)):
            raise ValueError("ProblemMatrix: NaN/Inf entry")
        tr = s.shape[0] < s.shape[1]
        if tr:
            s = s.T.tocsc()
            s.sort_indices()
        return ProblemMatrix(s, tr, True)

    def rows(self): return self._a.shape[0]
    def cols(self): return self._a.shape[1]
    def transposed(self): return self._transposed
    def is_sparse(self): return self._sparse

    def dense(self):
        if self._sparse:
            raise TypeError("ProblemMatrix: sparse storage (use sparse() or to_dense())")
        return self._a

    def sparse(self):
        if not self._sparse:
            raise TypeError("ProblemMatrix: dense storage")
        return self._a

    def to_dense(self):
        """Densified copy regardless of storage (problem.hpp:60-64; tests only)."""
        return np.asfortranarray(self._a.toarray()) if self._sparse else self._a


def build_model(which: int = 1, rows: int = 1000, cols: int = 200, seed: int = 7):
    """problems.hpp:50-70 (host generator in the library): (ProblemMatrix, sigma ascending)."""
    a = np.empty((rows, cols), order="F")
    s = np.empty(cols)
    st = lib().sssvd_build_model(which, rows, cols, seed, _ptr(a), _ptr(s))
    if st != SSSVD_OK:
        _raise(st, "build_model: needs rows >= cols and model 1 or 2")
    return ProblemMatrix.from_dense(a), s


def filter_profile(rule: "ContourRule", sigma_min: float, sigma_max: float, points: int, log_spacing: bool = False):
    """filter.hpp:36-55: (grid, |f(grid)|)."""
    if points < 1:
        raise ValueError("filter_profile: need at least one point")
    grid, vals = np.empty(points), np.empty(points)
    st = lib().sssvd_filter_profile(rule.interval_a(), rule.interval_b(), rule.count(), rule.aspect(),
                                    rule.transform().kind(), sigma_min, sigma_max, points, int(log_spacing),
                                    _ptr(grid), _ptr(vals))
    if st != SSSVD_OK:
        _raise(st, "filter_profile: need 0 < sigma_min < sigma_max")
    return grid, vals


def read_matrix_market(path: str) -> ProblemMatrix:
    """matrix_market.hpp:34-119 through the library's C++ reader (sssvd_mm_read)."""
    L = lib()
    h = ctypes.c_void_p()
    st = L.sssvd_mm_read(os.fsencode(path), ctypes.byref(h))
    if st != SSSVD_OK:
        _raise(st, L.sssvd_host_last_error().decode())
    try:
        info = _MmInfo()
        L.sssvd_mm_info_get(h, ctypes.byref(info))

        def arr(fn, count, ctype, dtype):
            if count == 0:
                return np.empty(0, dtype=dtype)
            p = ctypes.cast(fn(h), ctypes.POINTER(ctype))
            return np.ctypeslib.as_array(p, shape=(count,)).copy()

        vals = arr(L.sssvd_mm_values, info.nnz, ctypes.c_double, np.float64)
        if not info.sparse:
            return ProblemMatrix.from_dense(vals.reshape((info.cols, info.rows)).T)
        import scipy.sparse as sp
        colptr = arr(L.sssvd_mm_colptr, info.cols + 1, ctypes.c_int64, np.int64)
        rowind = arr(L.sssvd_mm_rowind, info.nnz, ctypes.c_int64, np.int64)
        return ProblemMatrix.from_sparse(sp.csc_matrix((vals, rowind, colptr), shape=(info.rows, info.cols)))
    finally:
        L.sssvd_mm_free(h)


def write_matrix_market(path: str, a: ProblemMatrix, comment: str = "") -> None:
    """matrix_market.hpp:121-149: the caller's original orientation, 17 significant digits."""
    L = lib()
    if a.is_sparse():
        s = a.sparse().T.tocsc() if a.transposed() else a.sparse()
        cp = np.ascontiguousarray(s.indptr, dtype=np.int64)
        ri = np.ascontiguousarray(s.indices, dtype=np.int64)
        va = np.ascontiguousarray(s.data, dtype=np.float64)
        st = L.sssvd_mm_write(os.fsencode(path), s.shape[0], s.shape[1], va.size, _ptr(cp), _ptr(ri), _ptr(va),
                              comment.encode())
    else:
        d = np.asfortranarray(a.dense().T if a.transposed() else a.dense())
        st = L.sssvd_mm_write(os.fsencode(path), d.shape[0], d.shape[1], d.size, None, None, _ptr(d),
                              comment.encode())
    if st != SSSVD_OK:
        _raise(st, L.sssvd_host_last_error().decode())


def form_gram(a: ProblemMatrix, size_cap: int = 8192, device: Optional[Device] = None) -> np.ndarray:
    """problem.hpp:81-95 on the GPU (DMMA Gram kernel); length_error above the cap."""
    dev = device or default_device()
    if a.cols() > size_cap:
        raise LengthError("form_gram: column count exceeds the dense Gram cap")
    dev.set_problem(a)
    return dev.form_gram(size_cap)


# ----------------------------------------------------------------------------- shifted solves
class ShiftedFactorization:
    """shifted_solver.hpp:20-40. The factorisation and the solve both run on the GPU; because
    the library fuses them (the right-hand side rides through the LU as extra columns), the
    factor step validates the shift eagerly and solve() re-runs the fused kernel chain."""

    def __init__(self, gram: np.ndarray, shift: complex, device: Optional[Device] = None):
        gram = np.asfortranarray(gram, dtype=np.float64)
        if gram.shape[0] != gram.shape[1]:
            raise ValueError("ShiftedFactorization: Gram matrix must be square")
        self._g, self._shift, self._n = gram, complex(shift), gram.shape[0]
        self._dev = device or default_device()
        # eager pivot-floor check like the reference constructor (shifted_solver.hpp:27-30)
        self.solve(np.zeros((self._n, 1), dtype=np.complex128))

    def shift(self): return self._shift
    def size(self): return self._n

    def solve(self, rhs) -> np.ndarray:
        rhs = np.asarray(rhs)
        if rhs.ndim == 1:
            rhs = rhs[:, None]
        if rhs.shape[0] != self._n:
            raise ValueError("ShiftedFactorization: right-hand side dimension mismatch")
        r = np.asfortranarray(rhs, dtype=np.complex128)
        x = np.empty_like(r, order="F")
        self._dev.check(lib().sssvd_gpu_shifted_solve(
            self._dev.h, _ptr(self._g), self._n, self._shift.real, self._shift.imag,
            _ptr(r), r.shape[0], r.shape[1], _ptr(x)))
        return x

    def solve_real(self, rhs):
        return self.solve(np.asarray(rhs, dtype=np.complex128))


def factor_shift(gram, shift, device=None):
    return ShiftedFactorization(gram, shift, device)


def solve_block(fact: ShiftedFactorization, rhs):
    return fact.solve(rhs)


class DenseShiftedSolver:
    """shifted_solver.hpp:54-75."""

    def __init__(self, gram: np.ndarray):
        self._g = np.asfortranarray(gram, dtype=np.float64)

    def gram(self): return self._g
    def size(self): return self._g.shape[0]
    def factor(self, shift): return ShiftedFactorization(self._g, shift)
    def factor_bytes(self): return self._g.shape[0] ** 2 * 16


@dataclass
class MomentBlocks:
    """moments.hpp:51-71."""
    blocks: List[np.ndarray]

    def degree(self): return len(self.blocks) - 1
    def stacked(self): return np.hstack(self.blocks[:self.degree()])
    def stacked_plus(self): return np.hstack(self.blocks[1:self.degree() + 1])


class MomentAccumulator:
    """moments.hpp:101-169 on the GPU: the operator's Gram must be resident (form_gram or
    set_operator + form_gram on the same device)."""

    def __init__(self, rule: ContourRule, device: Optional[Device] = None):
        self._rule = rule
        self._dev = device or default_device()
        h = rule.count() // 2
        self._h = h
        self._shifts = np.array([rule.shift(j) for j in range(h)], dtype=np.complex128)
        self._w = np.ascontiguousarray(rule.weights()[:h])
        self._t = np.ascontiguousarray(rule.nodes()[:h])

    def rule(self): return self._rule

    def _run(self, s0, ell, degree):
        s0 = np.asfortranarray(s0, dtype=np.float64)
        n, L = s0.shape
        out = np.empty((degree + 1) * n * L)
        self._dev.check(lib().sssvd_gpu_moments(self._dev.h, self._h, _ptr(self._shifts), _ptr(self._w),
                                                _ptr(self._t), _ptr(s0), L, ell, degree, _ptr(out)))
        return [out[k * n * L:(k + 1) * n * L].reshape((L, n)).T.copy(order="F") for k in range(degree + 1)]

    def refine(self, s0):
        """moments.hpp:121-128: one pass S0 <- 2 sum_j Re(w_j X_j) (the k = 0 moment)."""
        return self._run(s0, 1, 0)[0]

    def accumulate(self, s0, degree: int) -> MomentBlocks:
        """moments.hpp:132-147."""
        return MomentBlocks(self._run(s0, 1, degree))


# ----------------------------------------------------------------------------- run_solve
@dataclass
class StepTimings:
    steps_1_2: float = 0.0
    step_3: float = 0.0
    step_4: float = 0.0
    step_5: float = 0.0
    postprocess: float = 0.0

    def total(self):
        return self.steps_1_2 + self.step_3 + self.step_4 + self.step_5


@dataclass
class TripletSet:
    sigma: np.ndarray
    left: np.ndarray
    right: np.ndarray
    q: np.ndarray
    in_interval: np.ndarray

    def count(self): return self.sigma.size


class _Handle:
    """Owns a sssvd_gpu_result; freed with the last Python reference."""

    def __init__(self, h):
        self.h = h

    def __del__(self):
        try:
            if self.h:
                lib().sssvd_result_free(self.h)
        except Exception:
            pass


class RunResult:
    """pipeline.hpp:74-95. Scalars are read eagerly; the arrays (triplet vectors, tau,
    residuals, moment blocks) are copied out of the C result handle on first access."""

    def __init__(self, handle: _Handle):
        L = lib()
        info = _Info()
        L.sssvd_result_info_get(handle.h, ctypes.byref(info))
        self._h, self._info = handle, info
        self.empty = bool(info.empty)
        self.note = L.sssvd_result_note(handle.h).decode()
        self.input_transposed = bool(info.input_transposed)
        self.rank_deficient_qr = bool(info.rank_deficient_qr)
        self.timings = StepTimings(info.steps_1_2, info.step_3, info.step_4, info.step_5, info.postprocess)
        self.device_times = {"gram_s": info.t_gram, "shifted_solves_s": info.t_shifted_solves,
                             "allreduce_s": info.t_allreduce, "shifted_solve_flops": info.shifted_solve_flops}
        self.count_in_interval = info.count_in_interval
        self.count_nonspurious_in_interval = info.count_nonspurious_in_interval
        self.count_interior, self.count_boundary = info.count_interior, info.count_boundary
        self.calibration_index = None if info.calibration_index < 0 else info.calibration_index
        self.mu = info.mu if info.calibration_index >= 0 else None
        self.spurious_threshold = info.spurious_threshold
        self._cache = {}

    def _get(self, field, count, dtype=np.float64):
        key = (field, count)
        if key not in self._cache:
            out = np.empty(count, dtype=dtype)
            if count:
                lib().sssvd_result_copy(self._h.h, field, _ptr(out))
            self._cache[key] = out
        return self._cache[key]

    def retained_rank(self):
        return self._info.retained_rank

    @property
    def basis_singular_values(self):
        return self._get(9, self._info.retained_rank)

    @property
    def blocks(self):
        i = self._info
        n, Lb, M = i.n_internal, i.block_size, i.moment_degree
        blk = self._get(10, (M + 1) * n * Lb)
        return MomentBlocks([blk[k * n * Lb:(k + 1) * n * Lb].reshape((Lb, n)).T for k in range(M + 1)])

    @property
    def triplets(self):
        i = self._info
        if self.empty:
            return TripletSet(np.empty(0), np.empty((i.rows, 0)), np.empty((i.cols, 0)), np.empty((0, 0)),
                              np.empty(0, dtype=bool))
        t = i.count
        return TripletSet(self._get(0, t), self._get(7, i.rows * t).reshape((t, i.rows)).T,
                          self._get(8, i.cols * t).reshape((t, i.cols)).T,
                          self._get(11, i.retained_rank * t).reshape((t, i.retained_rank)).T,
                          self._get(5, t, np.int32).astype(bool))

    @property
    def tau(self):
        return None if self.empty else self._get(1, self._info.count)

    @property
    def spurious(self):
        return None if self.empty else self._get(6, self._info.count, np.int32).astype(bool)

    @property
    def estimated(self):
        return None if self.empty else self._get(2, self._info.count)

    @property
    def exact(self):
        return None if self.empty else self._get(3, self._info.count)

    @property
    def galerkin(self):
        return None if self.empty else self._get(4, self._info.count)

    @staticmethod
    def _from_handle(h) -> "RunResult":
        return RunResult(_Handle(h))


def run_solve(a, config: RunConfig, device: Optional[Device] = None) -> RunResult:
    """pipeline.hpp:112-231 on the GPU. `a` is a ProblemMatrix or a dense array (user
    orientation); the library auto-transposes wide inputs like ProblemMatrix::from_dense."""
    dev = device or default_device()
    if isinstance(a, ProblemMatrix):
        dev.set_problem(a)
    else:
        dev.set_operator(np.asarray(a, dtype=np.float64))
    return dev.run_solve(config)
