"""Synthetic inputs for the five BASELINE.json configurations (and small variants).

BASELINE.json names no dataset: each config is A = U diag(sigma) V^T with Haar U, V (QR of a
seeded standard-Gaussian matrix, columns sign-fixed by diag(R)) and a stated spectrum. The
generator is seeded (numpy PCG64, seed 7 = the reference's model seed, problems.hpp:27); the
bench and the tests hash A (SHA-256) so the CPU and GPU legs provably read the same bits.
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


def spectrum(cfg: int, n: int, rng: np.random.Generator) -> np.ndarray:
    if cfg == 1:
        return np.arange(1, n + 1, dtype=np.float64) / n
    if cfg == 2:
        return np.sort(rng.uniform(0.0, 1.0, n))
    if cfg == 3:
        i = np.arange(n, dtype=np.float64)
        return 10.0 ** (-3.0 * i / (n - 1))
    if cfg == 4:
        k = 200
        bg = 1.0 + 0.5 * rng.uniform(0.0, 1.0, n - 2 * k)
        inside = rng.uniform(0.500, 0.501, k)
        outside = 0.501 + 1e-4 * rng.exponential(1.0, k)
        return np.sort(np.concatenate([bg, inside, outside]))
    if cfg == 5:
        # quarter-circle density sqrt(4 - s^2)/pi on [0, 2], inverse CDF by interpolation
        grid = np.linspace(0.0, 2.0, 200001)
        cdf = (grid * np.sqrt(4.0 - grid ** 2) / 2.0 + 2.0 * np.arcsin(grid / 2.0)) / math.pi
        return np.sort(np.interp(rng.uniform(0.0, 1.0, n), cdf, grid))
    raise ValueError(cfg)


def haar(rows: int, cols: int, rng: np.random.Generator, use_torch: bool = False) -> np.ndarray:
    g = rng.standard_normal((rows, cols))
    if use_torch:
        import torch
        t = torch.from_numpy(g).cuda()
        q, r = torch.linalg.qr(t, mode="reduced")
        q = q * torch.sign(torch.diagonal(r))[None, :]
        return q.cpu().numpy()
    q, r = np.linalg.qr(g, mode="reduced")
    return q * np.sign(np.diag(r))[None, :]


def make_operator(cfg: int, seed: int = 7, m: Optional[int] = None, n: Optional[int] = None,
                  use_torch: Optional[bool] = None):
    """Returns (A column-major m x n float64, sigma sorted ascending)."""
    w = CONFIGS[cfg]
    m = w.m if m is None else m
    n = w.n if n is None else n
    rng = np.random.default_rng(seed)
    if use_torch is None:
        use_torch = n > 4096
    u = haar(m, n, rng, use_torch)
    v = haar(n, n, rng, use_torch)
    sigma = spectrum(cfg, n, rng)
    if use_torch:
        import torch
        ut = torch.from_numpy(u).cuda()
        vt = torch.from_numpy(v).cuda()
        st = torch.from_numpy(sigma).cuda()
        a = ((ut * st[None, :]) @ vt.T).cpu().numpy()
    else:
        a = (u * sigma[None, :]) @ v.T
    return np.asfortranarray(a), np.sort(sigma)


def sha256(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8)).hexdigest()


def phase_flops(n: int, L: int, h: int) -> float:
    """Shifted-solve phase flops h (8n^3/3 + 8n^2 L)."""
    return h * (8.0 * n ** 3 / 3.0 + 8.0 * n * n * L)
