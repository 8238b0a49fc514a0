"""Synthetic inputs for the five BASELINE.json configurations (and small variants).

BASELINE.json names no dataset: each config is A = U diag(sigma) V^T with Haar U, V (QR of a
seeded standard-Gaussian matrix, columns sign-fixed by diag(R)) and a stated spectrum.

Host portability. A LAPACK QR on the CPU is not bit-reproducible across hosts (OpenBLAS picks its
kernels by CPU model), and the round-1 config-2 matrix hashed differently on two hosts. So the
operator is generated on the GPU whenever one is present, by one fixed recipe:
  * Gaussian factors: torch's Philox generator on cuda:0, seeded (seed 7 = the reference's model
    seed, problems.hpp:27; U from `seed`, V from `seed + 1`);
  * QR: torch.linalg.qr on the device (cuSOLVER), columns sign-fixed by diag(R);
  * spectrum: numpy PCG64 (seed) with the transcendental parts in Python's math module (numpy's
    SIMD float64 math differs in the last bit between CPU generations);
  * A = (U diag sigma) V^T on the device.
Every B200 box with this image produces the same bits; the bench, the tests and the committed
fixtures record and assert SHA-256(A). The CPU fallback (numpy) exists for small CPU-side cases
only and is flagged as such (its hash is host-dependent).

This module is input generation, not the measured path.
"""
from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass
from typing import Optional

import numpy as np

SS_SVD, SS_SVD_NT = 0, 1


@dataclass
class Workload:
    name: str
    m: int
    n: int
    a: float
    b: float
    L: int
    M: int
    N: int
    modes: tuple
    description: str


CONFIGS = {
    1: Workload("cfg1", 2000, 1000, 0.45, 0.55, 16, 8, 32, (SS_SVD_NT,),
                "2000x1000, sigma_i = i/n, [0.45,0.55], L=16 M=8 N=32, NT on"),
    2: Workload("cfg2", 4096, 4096, 0.9, 1.0, 32, 16, 32, (SS_SVD, SS_SVD_NT),
                "4096^2, sigma ~ U(0,1) sorted, [0.9,1.0], L=32 M=16 N=32, NT off and on"),
    3: Workload("cfg3", 32768, 8192, 0.01, 0.02, 64, 16, 64, (SS_SVD,),
                "32768x8192, log-spaced sigma in [1e-3,1], [0.01,0.02], L=64 M=16 N=64"),
    4: Workload("cfg4", 8192, 8192, 0.5, 0.501, 32, 16, 64, (SS_SVD_NT,),
                "8192^2 clustered: 200 in [0.5,0.501] + 200 just outside, L=32 M=16 N=64, NT on"),
    5: Workload("cfg5", 16384, 16384, 0.8, 0.9, 128, 16, 128, (SS_SVD,),
                "16384^2 quarter-circle spectrum on [0,2], [0.8,0.9], L=128 M=16 N=128"),
}


def _quarter_circle_cdf_grid(points: int = 200001):
    grid = [2.0 * i / (points - 1) for i in range(points)]
    cdf = [(s * math.sqrt(max(4.0 - s * s, 0.0)) / 2.0 + 2.0 * math.asin(min(s / 2.0, 1.0))) / math.pi for s in grid]
    return np.array(grid), np.array(cdf)


def spectrum(cfg: int, n: int, rng: np.random.Generator) -> np.ndarray:
    if cfg == 1:
        return np.arange(1, n + 1, dtype=np.float64) / n
    if cfg == 2:
        return np.sort(rng.uniform(0.0, 1.0, n))
    if cfg == 3:
        return np.array([math.pow(10.0, -3.0 * i / (n - 1)) for i in range(n)])
    if cfg == 4:
        k = 200
        bg = 1.0 + 0.5 * rng.uniform(0.0, 1.0, n - 2 * k)
        inside = rng.uniform(0.500, 0.501, k)
        outside = 0.501 + 1e-4 * rng.exponential(1.0, k)
        return np.sort(np.concatenate([bg, inside, outside]))
    if cfg == 5:
        # quarter-circle density sqrt(4 - s^2)/pi on [0, 2], inverse CDF by interpolation
        grid, cdf = _quarter_circle_cdf_grid()
        return np.sort(np.interp(rng.uniform(0.0, 1.0, n), cdf, grid))
    raise ValueError(cfg)


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def _haar_device(rows: int, cols: int, seed: int, device):
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    x = torch.randn(rows, cols, dtype=torch.float64, device=device, generator=g)
    q, r = torch.linalg.qr(x, mode="reduced")
    del x
    return q * torch.sign(torch.diagonal(r))[None, :]


def _haar_host(rows: int, cols: int, rng: np.random.Generator) -> np.ndarray:
    g = rng.standard_normal((rows, cols))
    q, r = np.linalg.qr(g, mode="reduced")
    return q * np.sign(np.diag(r))[None, :]


def make_operator(cfg: int, seed: int = 7, m: Optional[int] = None, n: Optional[int] = None,
                  device: Optional[str] = None, out=None):
    """Returns (A column-major m x n float64 numpy array, sigma sorted ascending).

    device: "cuda" (default when a GPU is present; bit-reproducible across B200 boxes) or "cpu".
    out: optional preallocated (n, m) C-contiguous float64 array (e.g. pinned) that receives A^T,
    i.e. A column-major; the returned A is then a Fortran view of it."""
    w = CONFIGS[cfg]
    m = w.m if m is None else m
    n = w.n if n is None else n
    rng = np.random.default_rng(seed)
    sigma = spectrum(cfg, n, rng)
    if device is None:
        device = "cuda" if gpu_available() else "cpu"
    if device == "cpu":
        u = _haar_host(m, n, rng)
        v = _haar_host(n, n, rng)
        a = np.asfortranarray((u * sigma[None, :]) @ v.T)
        if out is not None:
            out[...] = a.T
            a = out.T
        return a, np.sort(sigma)
    import torch
    dev = torch.device(device)
    with torch.no_grad():
        u = _haar_device(m, n, seed, dev)
        u *= torch.from_numpy(sigma).to(dev)[None, :]
        v = _haar_device(n, n, seed + 1, dev)
        at = torch.matmul(v, u.T)   # A^T (n x m) row-major == A column-major
        del u, v
        if out is None:
            out = np.empty((n, m), dtype=np.float64)
        torch.from_numpy(out).copy_(at)
        del at
        torch.cuda.empty_cache()
    return out.T, np.sort(sigma)


def sha256(a: np.ndarray) -> str:
    """SHA-256 of A's column-major bytes."""
    at = a.T if a.flags.f_contiguous else np.asfortranarray(a).T
    return hashlib.sha256(np.ascontiguousarray(at).view(np.uint8)).hexdigest()


def phase_flops(n: int, L: int, h: int) -> float:
    """Shifted-solve phase flops h (8n^3/3 + 8n^2 L)."""
    return h * (8.0 * n ** 3 / 3.0 + 8.0 * n * n * L)
