"""Oracle: Algorithm 2 ("NFFT-like procedure for bandlimited functions"), step by step.

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.  float64 throughout.

Citations "P:<line>" are lines of the paper text; readings "A<n>" are the
DESIGN.md / SURVEY.md §8(c) readings where the paper is silent or ambiguous.

Pins (tests/test_oracle_pins.py):
  grid_length ........ P:86 worked examples (Fig. 1 L=40)
  phi / phi_grid ..... window-class axioms P:273-278; sinh/cKB boundary values; error-decay in m
  psihat_1d .......... scipy QUADPACK and 30-digit mpmath on the un-substituted integral;
                       evenness; flatness L*psihat ~ 1
  step2_inverse_fft .. literal sum of eq. def_theta; impulse / constant closed forms
  step3_short_sums ... interpolation property; dense Psi F D_psihat
  algorithm2 ......... Dirichlet closed form (f^ == 1), Fejer closed form (Example 5.3 triangle),
                       brute-force trig sum eq. nfft within the regularization error (A12)
  stable_bin_sort .... Python sorted() on (key, index) pairs
No function here is "parity unpinned".
"""
from __future__ import annotations

import math
from typing import Dict, Optional

import numpy as np

__all__ = [
    "grid_length", "default_shape", "phi", "phi_grid", "sinc", "psi_grid",
    "psihat_1d", "psihat_table", "psihat_multi",
    "step1_deconvolve_pad", "step2_inverse_fft", "inverse_dft_literal",
    "step3_short_sums", "algorithm2", "dense_apply", "trig_sum",
    "cell_index", "stable_bin_sort", "J_set",
]

WINDOWS = ("sinh", "gauss", "ckb")


# ----------------------------------------------------------------------------- parameters
def grid_length(M: int, sigma: float) -> int:
    """L = M_sigma = 2*ceil(ceil(sigma*M)/2) (reading A7: Alg. 2's L is Alg. 1's M_sigma)."""
    if M < 2 or M % 2:
        raise ValueError("M must be even and >= 2 (P:50)")
    if not sigma >= 1.0:
        raise ValueError("sigma >= 1 (P:86)")
    return 2 * math.ceil(math.ceil(sigma * M) / 2)


def default_shape(window: str, m: int, M: int, L: int) -> float:
    """Window shape parameter when the paper leaves it open ("certain beta > 0").

    Reading A1: beta = pi*m*(1 - 1/sigma) with sigma = L/M (sinh and cKB).
    Reading A2: Gaussian (not defined in the paper) s = sqrt(m / (pi*L*(L-M))).
    """
    if window in ("sinh", "ckb"):
        return math.pi * m * (1.0 - M / L)
    if window == "gauss":
        return math.sqrt(m / (math.pi * L * (L - M)))
    raise ValueError(window)


# ----------------------------------------------------------------------------- windows
def phi(window: str, x, m: int, L: int, shape: float):
    """Window phi(x) in the paper's x units.

    sinh-type, eq. varphisinh:
        phi(x) = sinh(beta*sqrt(1-(Lx/m)^2)) / sinh(beta) * chi_[-m/L, m/L](x)
    continuous Kaiser-Bessel:
        phi(x) = (I0(beta*sqrt(1-(Lx/m)^2)) - 1) / (I0(beta) - 1) * chi_[-m/L, m/L](x)
    Gaussian (reading A2; not in the paper): exp(-x^2/(2 s^2)) * chi_[-m/L, m/L](x).
    """
    x = np.asarray(x, dtype=np.float64)
    inside = np.abs(x) <= m / L
    if window == "gauss":
        return np.where(inside, np.exp(-x * x / (2.0 * shape * shape)), 0.0)
    r = np.clip(1.0 - (L * x / m) ** 2, 0.0, None)
    if window == "sinh":
        val = np.sinh(shape * np.sqrt(r)) / np.sinh(shape)
    elif window == "ckb":
        val = (np.i0(shape * np.sqrt(r)) - 1.0) / (np.i0(shape) - 1.0)
    else:
        raise ValueError(window)
    return np.where(inside, val, 0.0)


def phi_grid(window: str, tau, m: int, L: int, shape: float):
    """phi(tau/L) written in grid units tau = L*x (so L*x/m = tau/m exactly).

    Same formulas as `phi`; evaluating through tau avoids forming x - l/L in
    floating point, which would lose up to L*2^-54 in tau (reading O3 in DESIGN.md).
    """
    tau = np.asarray(tau, dtype=np.float64)
    inside = np.abs(tau) <= m
    if window == "gauss":
        xs = tau / L
        return np.where(inside, np.exp(-xs * xs / (2.0 * shape * shape)), 0.0)
    r = np.clip(1.0 - (tau / m) ** 2, 0.0, None)
    if window == "sinh":
        val = np.sinh(shape * np.sqrt(r)) / np.sinh(shape)
    elif window == "ckb":
        val = (np.i0(shape * np.sqrt(r)) - 1.0) / (np.i0(shape) - 1.0)
    else:
        raise ValueError(window)
    return np.where(inside, val, 0.0)


def sinc(x):
    """sinc(x) = sin(x)/x, sinc(0) = 1."""
    x = np.asarray(x, dtype=np.float64)
    out = np.ones_like(x)
    nz = x != 0.0
    out[nz] = np.sin(x[nz]) / x[nz]
    return out


def psi_grid(window: str, tau, m: int, L: int, shape: float):
    """Regularized sinc psi(x) = sinc(L*pi*x) * phi(x) (eq. sinc_reg) at x = tau/L."""
    tau = np.asarray(tau, dtype=np.float64)
    return sinc(np.pi * tau) * phi_grid(window, tau, m, L, shape)


# ----------------------------------------------------------------------------- step 0(a)
def psihat_1d(window: str, v, m: int, L: int, shape: float, n: int = 64):
    """psi^(v) = int psi(t) e^{-2 pi i v t} dt (Fourier transform) for d = 1.

    psi is even and supported on [-m/L, m/L], so
        psi^(v) = 2 int_0^{m/L} psi(t) cos(2 pi v t) dt.
    Reading A4 (the paper gives no closed form): substitute t = (m/L) sin(theta),
    dt = (m/L) cos(theta) dtheta, theta in [0, pi/2], which removes the sqrt-type endpoint
    behaviour of the window, and apply n-point Gauss-Legendre (numpy.leggauss).
    """
    v = np.asarray(v, dtype=np.float64)
    xg, wg = np.polynomial.legendre.leggauss(n)
    theta = (xg + 1.0) * (np.pi / 4.0)          # map [-1, 1] -> [0, pi/2]
    wq = wg * (np.pi / 4.0)
    tau = m * np.sin(theta)                      # tau = L t
    t = tau / L
    g = psi_grid(window, tau, m, L, shape) * (m / L) * np.cos(theta)
    return 2.0 * np.cos(2.0 * np.pi * np.multiply.outer(v, t)) @ (wq * g)


def psihat_table(window: str, M: int, m: int, L: int, shape: float, n: int = 64) -> np.ndarray:
    """psi^_1(k) for k in I_M = {-M/2, ..., M/2-1} (Alg. 2 step 0(a)), centred order."""
    k = np.arange(M, dtype=np.float64) - M // 2
    return psihat_1d(window, k, m, L, shape, n)


def psihat_multi(table: np.ndarray, d: int) -> np.ndarray:
    """d-variate psi^(k) = prod_t psi^_1(k_t) (reading A3: tensor-product window)."""
    out = np.ones((len(table),) * d)
    for t in range(d):
        sh = [1] * d
        sh[t] = len(table)
        out = out * table.reshape(sh)
    return out


# ----------------------------------------------------------------------------- step 1
def step1_deconvolve_pad(fhat: np.ndarray, psihat_d: np.ndarray, L: int) -> np.ndarray:
    """theta^(k) = f^(k)/psi^(k) on I_M, 0 on I_L \\ I_M (Alg. 2 step 1).

    fhat: (B, M, ..., M) centred (index k + M/2).  Returns (B, L, ..., L) centred
    (index k + L/2).
    """
    B = fhat.shape[0]
    d = fhat.ndim - 1
    M = fhat.shape[1]
    out = np.zeros((B,) + (L,) * d, dtype=np.complex128)
    sl = (slice(None),) + (slice(L // 2 - M // 2, L // 2 + M // 2),) * d
    out[sl] = fhat.astype(np.complex128) / psihat_d[None]
    return out


# ----------------------------------------------------------------------------- step 2
def step2_inverse_fft(theta_hat: np.ndarray) -> np.ndarray:
    """theta_l = L^{-d} sum_{k in I_L} theta^(k) e^{2 pi i k.l / L}, l in I_L (eq. def_theta,
    P:441-449; Alg. 2 step 2).

    numpy.fft.ifftn is exactly (1/L^d) sum_n a_n e^{+2 pi i n p / L}; the signed index sets
    are mapped to residues mod L by ifftshift (k -> k mod L) and back by fftshift.
    """
    d = theta_hat.ndim - 1
    axes = tuple(range(1, d + 1))
    a = np.fft.ifftshift(theta_hat, axes=axes)
    return np.fft.fftshift(np.fft.ifftn(a, axes=axes), axes=axes)


def inverse_dft_literal(theta_hat: np.ndarray) -> np.ndarray:
    """Literal O(L^{2d}) sum of eq. def_theta, for L^d <= 4096 (pin for step 2)."""
    B = theta_hat.shape[0]
    d = theta_hat.ndim - 1
    L = theta_hat.shape[1]
    idx = np.arange(L) - L // 2
    grids = np.meshgrid(*([idx] * d), indexing="ij")
    K = np.stack([g.ravel() for g in grids], axis=1)             # (L^d, d), lexicographic
    E = np.exp(2j * np.pi * (K @ K.T) / L)                        # E[l, k]
    out = (theta_hat.reshape(B, -1) @ E.T) / float(L) ** d
    return out.reshape(theta_hat.shape)


# ----------------------------------------------------------------------------- step 3
def J_set(x_t: float, L: int, m: int):
    """J_{L,m}(x) per coordinate = {l in Z : -m + L x <= l <= m + L x} (eq. indexset_x_nonperiodic,
    P:469-473), as the integer range [ceil(Lx - m), floor(Lx + m)]."""
    Lx = L * x_t
    return list(range(math.ceil(Lx - m), math.floor(Lx + m) + 1))


def step3_short_sums(theta: np.ndarray, x: np.ndarray, window: str, m: int, shape: float
                     ) -> np.ndarray:
    """f_j = sum_{l in I_L, l in J_{L,m}(x_j)} theta_l psi(x_j - l/L)  (Alg. 2 step 3, P:510-513;
    first equality of P:463 restricts l to I_L -- reading A5, zero extension outside I_L).

    psi(x_j - l/L) is evaluated at tau = L*x_j - l, formed exactly as (L*x_j) - l (O3).
    Per node the terms are accumulated in lexicographic order of l.  Vectorised over
    nodes and batch only.
    theta: (B, L, ..., L) centred.  x: (N, d).  Returns (B, N).
    """
    B = theta.shape[0]
    d = theta.ndim - 1
    L = theta.shape[1]
    N = x.shape[0]
    Lx = L * x                                                    # (N, d)
    lo = np.ceil(Lx - m).astype(np.int64)                         # first member of J
    hi = np.floor(Lx + m).astype(np.int64)                        # last member of J
    ncand = 2 * m + 1                                             # |J| <= 2m+1
    # per-dimension candidate indices, masks and weights psi(tau)
    ell = lo[:, :, None] + np.arange(ncand)[None, None, :]        # (N, d, 2m+1)
    valid = (ell <= hi[:, :, None]) & (ell >= -L // 2) & (ell < L // 2)
    tau = Lx[:, :, None] - ell
    w = np.where(valid, psi_grid(window, tau, m, L, shape), 0.0)
    flat_theta = theta.reshape(B, -1)
    f = np.zeros((B, N), dtype=np.complex128)
    for combo in np.ndindex(*([ncand] * d)):                      # lexicographic in l
        wt = np.ones(N)
        ok = np.ones(N, dtype=bool)
        flat = np.zeros(N, dtype=np.int64)
        for t in range(d):
            o = combo[t]
            wt = wt * w[:, t, o]
            ok &= valid[:, t, o]
            flat = flat * L + np.where(valid[:, t, o], ell[:, t, o] + L // 2, 0)
        if not ok.any():
            continue
        f += np.where(ok[None, :], flat_theta[:, flat] * wt[None, :], 0.0)
    return f


# ----------------------------------------------------------------------------- Algorithm 2
def algorithm2(x: np.ndarray, fhat: np.ndarray, M: int, sigma: float, m: int,
               window: str = "sinh", shape: Optional[float] = None,
               quad_n: int = 64) -> Dict[str, np.ndarray]:
    """Algorithm 2: steps 0(a), 1, 2, 3.  Returns every intermediate.

    x: (N, d) float64 nodes in [-1/2, 1/2)^d (reading A5).  fhat: (B, M, ..., M) centred.
    """
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[:, None]
    if fhat.ndim == x.shape[1]:
        fhat = fhat[None]
    d = x.shape[1]
    L = grid_length(M, sigma)
    if 2 * m >= L:
        raise ValueError("2m < L required (P:273)")
    if shape is None or shape <= 0:
        shape = default_shape(window, m, M, L)
    table = psihat_table(window, M, m, L, shape, quad_n)                 # step 0(a)
    theta_hat = step1_deconvolve_pad(fhat, psihat_multi(table, d), L)  # step 1
    theta = step2_inverse_fft(theta_hat)                               # step 2
    f = step3_short_sums(theta, x, window, m, shape)                   # step 3
    return {"f": f, "theta": theta, "theta_hat": theta_hat, "psihat": table,
            "L": L, "shape": shape}


def dense_apply(x: np.ndarray, fhat: np.ndarray, M: int, sigma: float, m: int,
                window: str = "sinh", shape: Optional[float] = None) -> np.ndarray:
    """f = Psi F D_psihat f^ (eq. function_eval) with explicit dense matrices.

    D_psihat = diag(1/(|I_L| psi^(k)))_{k in I_M}   (eq. matrix_Dpsi)
    F        = (e^{2 pi i k.l/L})_{l in I_L, k in I_M} (eq. matrix_F, M_sigma = L)
    Psi      = (psi(x_j - l/L))_{j, l in I_L}        (eq. matrix_Psi)
    Indices enumerated lexicographically.  For L^d <= 4096 only.
    """
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[:, None]
    if fhat.ndim == x.shape[1]:
        fhat = fhat[None]
    d = x.shape[1]
    L = grid_length(M, sigma)
    if L ** d > 4096:
        raise ValueError("dense oracle guard: L^d <= 4096")
    if shape is None or shape <= 0:
        shape = default_shape(window, m, M, L)
    kM = np.arange(M) - M // 2
    kL = np.arange(L) - L // 2
    KM = np.stack([g.ravel() for g in np.meshgrid(*([kM] * d), indexing="ij")], axis=1)
    KL = np.stack([g.ravel() for g in np.meshgrid(*([kL] * d), indexing="ij")], axis=1)
    ph1 = psihat_table(window, M, m, L, shape)
    ph = np.prod(ph1[KM + M // 2], axis=1)
    D = np.diag(1.0 / (float(L) ** d * ph))
    F = np.exp(2j * np.pi * (KL @ KM.T) / L)
    tau = L * x[:, None, :] - KL[None, :, :]                     # (N, L^d, d)
    Psi = np.prod(psi_grid(window, tau, m, L, shape), axis=2)
    return (Psi @ (F @ (D @ fhat.reshape(fhat.shape[0], -1).T))).T


def trig_sum(x: np.ndarray, fhat: np.ndarray) -> np.ndarray:
    """f(x_j) = sum_{k in I_M} f^_k e^{2 pi i k.x_j} (eq. nfft) -- what Alg. 2
    approximates under the Theta = L truncation (reading A12).  Brute force O(N M^d)."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[:, None]
    if fhat.ndim == x.shape[1]:
        fhat = fhat[None]
    d = x.shape[1]
    M = fhat.shape[1]
    kM = np.arange(M) - M // 2
    KM = np.stack([g.ravel() for g in np.meshgrid(*([kM] * d), indexing="ij")], axis=1)
    out = np.zeros((fhat.shape[0], x.shape[0]), dtype=np.complex128)
    fh = fhat.reshape(fhat.shape[0], -1).astype(np.complex128)
    chunk = max(1, 2_000_000 // max(1, KM.shape[0]))
    for s in range(0, x.shape[0], chunk):
        E = np.exp(2j * np.pi * (x[s:s + chunk] @ KM.T))
        out[:, s:s + chunk] = fh @ E.T
    return out


# ----------------------------------------------------------------------------- node binning
def cell_index(x: np.ndarray, L: int) -> np.ndarray:
    """Grid cell of each node per dim: c_t = floor(L x_t) (so x_t in [c_t/L, (c_t+1)/L)),
    returned shifted to [0, L) as c_t + L/2.  L*x is one IEEE product (no FMA), as A14."""
    return (np.floor(L * np.asarray(x, dtype=np.float64)).astype(np.int64) + L // 2)


def stable_bin_sort(keys: np.ndarray, nbins: int):
    """Stable sort by integer key, ties by original index (reading A14).

    Returns perm (sorted position -> user index) and offsets[nbins+1]."""
    keys = np.asarray(keys, dtype=np.int64)
    perm = np.argsort(keys, kind="stable")
    counts = np.bincount(keys, minlength=nbins)
    offsets = np.zeros(nbins + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    return perm, offsets
