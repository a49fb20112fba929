"""Seeded input generators (nodes and spectra) for BASELINE.json configs 1-5.

Recipe:
  * generator: numpy default_rng(SEED_BASE + cfg_id [+ variant offset]) (PCG64);
  * uniform nodes: rng.random(shape) - 0.5, which lies in [-1/2, 1/2) exactly;
  * complex normal spectra: real part = standard_normal, then imag = standard_normal;
  * cfg3: half uniform, half 0.05*N(0,1)^2 clustered at the origin (rows outside
    [-1/2,1/2)^2 re-drawn), concatenated and permuted;
  * cfg4: complex normal scaled by exp(-|k|^2 / (2 (M/4)^2)), k centred;
  * cfg5: 4096 radial lines (directions uniform on the sphere) x 4096 equispaced radii
    r_i = -1/2 + i/4096, line-major; 64 independent spectra.

Nothing here computes any step of Algorithm 2.  Parameters such as L are passed in
by the caller where a generator needs them (feasible box, grid points).
"""
from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Optional, Tuple

import numpy as np

SEED_BASE = 2502071550


@dataclass(frozen=True)
class Config:
    cfg_id: int
    d: int
    M: int
    sigma: float
    m: int
    N: int
    batch: int
    precs: Tuple[str, ...]      # "c128" / "c64"
    windows: Tuple[str, ...]    # "sinh" / "gauss" / "ckb"
    nodes: str                  # "uniform" | "mixed" | "radial"
    spectrum: str               # "normal" | "gauss_decay"

    def scaled(self, **kw) -> "Config":
        return replace(self, **kw)


# BASELINE.json "configs" 0..4 -> cfg ids 1..5
CONFIGS = {
    1: Config(1, 1, 64, 2.0, 5, 1000, 1, ("c128",), ("sinh",), "uniform", "normal"),
    2: Config(2, 1, 1 << 20, 2.0, 8, 1 << 24, 1, ("c128", "c64"), ("sinh", "gauss"),
              "uniform", "normal"),
    3: Config(3, 2, 1024, 2.0, 6, 1 << 22, 1, ("c64",), ("sinh",), "mixed", "normal"),
    4: Config(4, 3, 256, 2.0, 4, 1 << 26, 1, ("c64",), ("sinh",), "uniform", "gauss_decay"),
    5: Config(5, 3, 128, 2.0, 4, 1 << 24, 64, ("c64",), ("sinh",), "radial", "normal"),
}


def _rng(cfg_id: int, variant: int = 0) -> np.random.Generator:
    return np.random.default_rng(SEED_BASE + cfg_id + 1000 * variant)


def make_nodes(cfg: Config, N: Optional[int] = None, variant: int = 0,
               rng: Optional[np.random.Generator] = None) -> np.ndarray:
    """Nodes x_j in [-1/2, 1/2)^d, float64, shape (N, d), row-major, user order."""
    N = cfg.N if N is None else N
    rng = _rng(cfg.cfg_id, variant) if rng is None else rng
    d = cfg.d
    if cfg.nodes == "uniform":
        return rng.random((N, d)) - 0.5
    if cfg.nodes == "mixed":
        n_u = N // 2
        n_c = N - n_u
        uni = rng.random((n_u, d)) - 0.5
        clu = 0.05 * rng.standard_normal((n_c, d))
        bad = np.any((clu < -0.5) | (clu >= 0.5), axis=1)
        while bad.any():
            clu[bad] = 0.05 * rng.standard_normal((int(bad.sum()), d))
            bad = np.any((clu < -0.5) | (clu >= 0.5), axis=1)
        x = np.concatenate([uni, clu], axis=0)
        return x[rng.permutation(N)]
    if cfg.nodes == "radial":
        # N = n_lines * n_radii with n_lines = n_radii when N is a square, else
        # n_radii = 4096 capped by N.
        n_rad = int(round(np.sqrt(N)))
        if n_rad * n_rad != N:
            n_rad = min(4096, N)
        n_lines = -(-N // n_rad)
        g = rng.standard_normal((n_lines, d))
        u = g / np.linalg.norm(g, axis=1, keepdims=True)
        r = -0.5 + np.arange(n_rad) / n_rad
        x = (u[:, None, :] * r[None, :, None]).reshape(-1, d)[:N]
        # |r u_t| <= 1/2 with equality only if |u_t| == 1 and r == -1/2; fold that
        # measure-zero case back into the half-open box.
        x[x >= 0.5] = np.nextafter(0.5, 0.0)
        return np.ascontiguousarray(x)
    raise ValueError(cfg.nodes)


def make_spectrum(cfg: Config, M: Optional[int] = None, batch: Optional[int] = None,
                  variant: int = 0, rng: Optional[np.random.Generator] = None,
                  prec: str = "c128") -> np.ndarray:
    """f^(k), k in I_M, centred row-major (index k_t + M/2, last dim fastest).

    Shape (batch, M, ..., M) complex128; for prec == "c64" the same draw rounded to
    complex64 (the oracle then consumes the rounded values).
    """
    M = cfg.M if M is None else M
    B = cfg.batch if batch is None else batch
    rng = _rng(cfg.cfg_id, variant + 7) if rng is None else rng
    shape = (B,) + (M,) * cfg.d
    re = rng.standard_normal(shape)
    im = rng.standard_normal(shape)
    f = re + 1j * im
    if cfg.spectrum == "gauss_decay":
        k = np.arange(M) - M // 2
        k2 = np.zeros((M,) * cfg.d)
        for t in range(cfg.d):
            sh = [1] * cfg.d
            sh[t] = M
            k2 = k2 + (k.reshape(sh) ** 2)
        f = f * np.exp(-k2 / (2.0 * (M / 4.0) ** 2))[None]
    if prec == "c64":
        f = f.astype(np.complex64)
    return f


def feasible_box_nodes(N: int, d: int, L: int, m: int, seed: int = 0) -> np.ndarray:
    """Uniform nodes inside the feasible box [-1/2+m/L, 1/2-m/L)^d."""
    rng = np.random.default_rng(SEED_BASE + 500 + seed)
    lo, hi = -0.5 + m / L, 0.5 - m / L
    return lo + (hi - lo) * rng.random((N, d))


def grid_point_nodes(N: int, d: int, L: int, seed: int = 0) -> np.ndarray:
    """Nodes exactly on the grid (1/L) Z^d inside [-1/2,1/2)^d (interpolation pin P:328-333)."""
    rng = np.random.default_rng(SEED_BASE + 600 + seed)
    k = rng.integers(-L // 2, L // 2, size=(N, d))
    return k.astype(np.float64) / L


def ones_spectrum(M: int, d: int = 1) -> np.ndarray:
    """f^ == 1 on I_M (BASELINE.json configs[0] closed-form check)."""
    return np.ones((1,) + (M,) * d, dtype=np.complex128)


def triangle_spectrum(M: int) -> np.ndarray:
    """Example 5.3: f^(v) = (2/M)(1 - |2v/M|) for |v| <= M/2, sampled on I_M."""
    k = np.arange(M) - M // 2
    return ((2.0 / M) * np.clip(1.0 - np.abs(2.0 * k / M), 0.0, None)).astype(np.complex128)[None]


def chebyshev_nodes(N: int, L: int, m: int) -> np.ndarray:
    """Scaled Chebyshev nodes, eq. points_cheb_scaled."""
    j = np.arange(1, N + 1)
    return (np.cos((j - 1) * np.pi / N) * (0.5 - m / L))[:, None]
