"""Oracle: Algorithm 1 (the classical NFFT, §2) and the paper's §5 comparison.

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.  float64 numpy, shares no code with the GPU path.

Algorithm 1, for nodes on the torus x_j in T^d = [-1/2, 1/2)^d:
  0(a) phi^(k), k in I_M: Fourier coefficients of the 1-periodic window.  Our windows are
       supported on [-m/L, m/L], so the truncated window equals the window and
       phi^(k) = 2 int_0^{m/L} phi(t) cos(2 pi k t) dt (same quadrature as psi^, without the sinc).
  1    g^_k = f^_k / phi^(k) on I_M, 0 on I_{M_sigma} \\ I_M
  2    g_l = |I_{M_sigma}|^{-1} sum_{k in I_M} g^_k e^{2 pi i k l / M_sigma}
  3    f~_j = sum_{l in I_{M_sigma,m}(x_j)} g_l phi~_m(x_j - l/M_sigma), periodic index set
       I_{M_sigma,m}(x) (eq. indexset_x), phi~_m the 1-periodisation of phi_m.
Matrix form A ~ B F D: D = diag(1/(|I_Msigma| phi^(k))), F as in Alg. 2, B sparse.

Pins (tests/test_oracle_nfft.py): fast == dense B F D; the NFFT approximates the trig sum
eq. nfft on the whole torus to its window error; periodic shift invariance of the index set
(S:95); phi^ vs QUADPACK; the exponential identities eq. approx_exp_nfft / approx_exp_nfft_like
 reduce to Algorithm 1/2 with f^ = delta_k at integer k.
"""
from __future__ import annotations

import math
from typing import Dict, Optional

import numpy as np

from .bandlimited import (grid_length, phi_grid, psi_grid, psihat_multi,
                          step1_deconvolve_pad, step2_inverse_fft)

__all__ = ["default_shape_nfft", "phihat_1d", "phihat_table", "algorithm1", "dense_apply_nfft", "periodic_index_set",
           "exp_error_nfft", "exp_error_alg2"]


def default_shape_nfft(window: str, m: int, M: int, L: int) -> float:
    """Window parameter for Algorithm 1 when none is given.  The paper says only "certain beta > 0"
    and points to the NFFT literature for these windows ([PoTa21a]); reading A17 takes that
    literature's choices: sinh / cKB beta = 2 pi m (1 - 1/(2 sigma)), Gaussian exp(-(L x)^2 / b) with
    b = 2 sigma m / ((2 sigma - 1) pi), i.e. s = sqrt(b/2) / L in our x-unit parametrisation."""
    sigma = L / M
    if window in ("sinh", "ckb"):
        return 2.0 * math.pi * m * (1.0 - 1.0 / (2.0 * sigma))
    if window == "gauss":
        b = 2.0 * sigma * m / ((2.0 * sigma - 1.0) * math.pi)
        return math.sqrt(b / 2.0) / L
    raise ValueError(window)


def phihat_1d(window: str, v, m: int, L: int, shape: float, n: int = 64):
    """phi^(v) = 2 int_0^{m/L} phi(t) cos(2 pi v t) dt (even window, support [-m/L, m/L]); the same
    t = (m/L) sin(theta) substitution and n-point Gauss-Legendre as psihat_1d (reading A4)."""
    v = np.asarray(v, dtype=np.float64)
    xg, wg = np.polynomial.legendre.leggauss(n)
    theta = (xg + 1.0) * (np.pi / 4.0)
    wq = wg * (np.pi / 4.0)
    tau = m * np.sin(theta)
    g = phi_grid(window, tau, m, L, shape) * (m / L) * np.cos(theta)
    return 2.0 * np.cos(2.0 * np.pi * np.multiply.outer(v, tau / L)) @ (wq * g)


def phihat_table(window: str, M: int, m: int, L: int, shape: float, n: int = 64) -> np.ndarray:
    k = np.arange(M, dtype=np.float64) - M // 2
    return phihat_1d(window, k, m, L, shape, n)


def periodic_index_set(x_t: float, L: int, m: int):
    """I_{M_sigma,m}(x) per coordinate (eq. indexset_x): l in I_L with some z in Z such
    that -m <= L (x + z) - l <= m, listed as (l, tau = L(x+z) - l) pairs, by brute force over z."""
    out = []
    for z in (-1, 0, 1):
        Lx = L * (x_t + z) if z else L * x_t
        for l in range(math.ceil(Lx - m), math.floor(Lx + m) + 1):
            if -L // 2 <= l < L // 2:
                out.append((l, Lx - l))
    return sorted(out)


def step3_periodic(g: np.ndarray, x: np.ndarray, window: str, m: int, shape: float) -> np.ndarray:
    """f~_j = sum over l in I_{L,m}(x_j) of g_l phi~_m(x_j - l/L).  For l reached through
    the unwrapped integer l' = l + zL (|L x_j - l'| <= m), phi~_m(x_j - l/L) = phi(tau/L) with
    tau = L x_j - l' formed exactly; since m/L < 1/2 only one periodic image contributes.
    Lexicographic accumulation over the unwrapped l'.  g: (B, L, ..., L) centred."""
    B = g.shape[0]
    d = g.ndim - 1
    L = g.shape[1]
    N = x.shape[0]
    Lx = L * x
    lo = np.ceil(Lx - m).astype(np.int64)
    hi = np.floor(Lx + m).astype(np.int64)
    ncand = 2 * m + 1
    ell = lo[:, :, None] + np.arange(ncand)[None, None, :]
    valid = ell <= hi[:, :, None]
    tau = Lx[:, :, None] - ell
    w = np.where(valid, phi_grid(window, tau, m, L, shape), 0.0)
    wrapped = np.mod(ell + L // 2, L)            # periodic index of l' in centred storage
    flat_g = g.reshape(B, -1)
    f = np.zeros((B, N), dtype=np.complex128)
    for combo in np.ndindex(*([ncand] * d)):
        wt = np.ones(N)
        ok = np.ones(N, dtype=bool)
        flat = np.zeros(N, dtype=np.int64)
        for t in range(d):
            o = combo[t]
            wt = wt * w[:, t, o]
            ok &= valid[:, t, o]
            flat = flat * L + wrapped[:, t, o]
        if ok.any():
            f += np.where(ok[None, :], flat_g[:, flat] * wt[None, :], 0.0)
    return f


def algorithm1(x: np.ndarray, fhat: np.ndarray, M: int, sigma: float, m: int, window: str = "sinh",
               shape: Optional[float] = None, quad_n: int = 64) -> Dict[str, np.ndarray]:
    """Algorithm 1, steps 0(a), 1, 2, 3; nodes on the torus [-1/2, 1/2)^d."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[:, None]
    if fhat.ndim == x.shape[1]:
        fhat = fhat[None]
    d = x.shape[1]
    L = grid_length(M, sigma)
    if 2 * m >= L:
        raise ValueError("2m < M_sigma required")
    if shape is None or shape <= 0:
        shape = default_shape_nfft(window, m, M, L)
    table = phihat_table(window, M, m, L, shape, quad_n)               # step 0(a)
    g_hat = step1_deconvolve_pad(fhat, psihat_multi(table, d), L)       # step 1
    g = step2_inverse_fft(g_hat)                                        # step 2 (1/|I_Msigma|)
    f = step3_periodic(g, x, window, m, shape)                          # step 3
    return {"f": f, "g": g, "phihat": table, "L": L, "shape": shape}


def dense_apply_nfft(x: np.ndarray, fhat: np.ndarray, M: int, sigma: float, m: int,
                     window: str = "sinh", shape: Optional[float] = None) -> np.ndarray:
    """A f^ ~ B F D f^ with dense matrices, D = diag(1/(|I_Msigma| phi^(k))) (eq. matrix_D),
    F (eq. matrix_F), B_{j,l} = phi~_m(x_j - l/M_sigma) (eq. matrix_B) by explicit periodisation
    sum over r in {-1, 0, 1} (m/L < 1/2).  L^d <= 4096."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[:, None]
    if fhat.ndim == x.shape[1]:
        fhat = fhat[None]
    d = x.shape[1]
    L = grid_length(M, sigma)
    if L ** d > 4096:
        raise ValueError("dense guard")
    if shape is None or shape <= 0:
        shape = default_shape_nfft(window, m, M, L)
    kM = np.arange(M) - M // 2
    kL = np.arange(L) - L // 2
    KM = np.stack([gg.ravel() for gg in np.meshgrid(*([kM] * d), indexing="ij")], axis=1)
    KL = np.stack([gg.ravel() for gg in np.meshgrid(*([kL] * d), indexing="ij")], axis=1)
    ph = np.prod(phihat_table(window, M, m, L, shape)[KM + M // 2], axis=1)
    D = np.diag(1.0 / (float(L) ** d * ph))
    F = np.exp(2j * np.pi * (KL @ KM.T) / L)
    Bm = np.ones((x.shape[0], KL.shape[0]))
    for t in range(d):
        per = np.zeros((x.shape[0], KL.shape[0]))
        for r in (-1, 0, 1):
            tau = L * (x[:, None, t] + r) - KL[None, :, t]
            per += phi_grid(window, tau, m, L, shape)
        Bm *= per
    return (Bm @ (F @ (D @ fhat.reshape(fhat.shape[0], -1).T))).T


# ----------------------------------------------------------------------------- §5 exp approximations
def exp_error_nfft(v: np.ndarray, xp: np.ndarray, M: int, m: int, L: int, window: str, shape: float):
    """e(v) = max_p |e^{2 pi i v x_p} - h(x_p)| with h the right-hand side of eq. approx_exp_nfft
    (P:570-578): h(x) = (|I_L| phi^(v))^{-1} sum_{l in I_L} e^{2 pi i v l/L} phi~_m(x - l/L)."""
    v = np.atleast_1d(v)
    ph = phihat_1d(window, v, m, L, shape)
    out = np.empty(len(v))
    Lx = L * xp
    lo = np.ceil(Lx - m).astype(np.int64)
    for i, vv in enumerate(v):
        h = np.zeros(len(xp), dtype=np.complex128)
        for o in range(2 * m + 1):
            ell = lo + o
            tau = Lx - ell
            ok = np.abs(tau) <= m
            wl = np.mod(ell + L // 2, L) - L // 2          # periodic index l in I_L
            h += np.where(ok, np.exp(2j * np.pi * vv * wl / L) * phi_grid(window, tau, m, L, shape), 0)
        h /= L * ph[i]
        out[i] = np.max(np.abs(np.exp(2j * np.pi * vv * xp) - h))
    return out


def exp_error_alg2(v: np.ndarray, xp: np.ndarray, M: int, m: int, L: int, window: str, shape: float,
                   with_psihat: bool = True):
    """e(v) for Algorithm 2's kernel.  with_psihat: h(x) = (|I_L| psi^(v))^{-1} sum_{l in I_L}
    e^{2 pi i v l/L} psi(x - l/L) (the approximation Psi F D_psihat of P:599-610 with D_psihat kept);
    otherwise eq. approx_exp_nfft_like with |I_L| psi^ ~ 1 dropped (reading A16)."""
    from .bandlimited import psihat_1d
    v = np.atleast_1d(v)
    ph = psihat_1d(window, v, m, L, shape) if with_psihat else np.full(len(v), 1.0 / L)
    out = np.empty(len(v))
    Lx = L * xp
    lo = np.ceil(Lx - m).astype(np.int64)
    for i, vv in enumerate(v):
        h = np.zeros(len(xp), dtype=np.complex128)
        for o in range(2 * m + 1):
            ell = lo + o
            tau = Lx - ell
            ok = (np.abs(tau) <= m) & (ell >= -L // 2) & (ell < L // 2)   # l in I_L, no wrap
            h += np.where(ok, np.exp(2j * np.pi * vv * ell / L) * psi_grid(window, tau, m, L, shape), 0)
        h /= L * ph[i]
        out[i] = np.max(np.abs(np.exp(2j * np.pi * vv * xp) - h))
    return out
