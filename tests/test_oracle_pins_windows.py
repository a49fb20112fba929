"""Pins of the oracle's continuous Kaiser-Bessel and Gaussian windows (no GPU).

VERDICT round 1 "What's weak #1": cKB was pinned only by the window axioms and a decay-slope fit,
and the 30-digit pin covered sinh only, so a slip such as a dropped square root inside I_0 could
pass.  Here both windows and their psi^ tables are compared with formulas typed independently in
30-digit mpmath (its own besseli / exp / sin / quadrature), and each pin is shown to reject the
plausible mutations of the formula it pins.

  cKB:       phi(x) = (I_0(beta sqrt(1 - (L x / m)^2)) - 1) / (I_0(beta) - 1) on |x| <= m/L
  Gaussian (reading A2): phi(x) = exp(-x^2 / (2 s^2)),  s = sqrt(m / (pi L (L - M)))
  psi^(v) = 2 int_0^{m/L} sinc(L pi t) phi(t) cos(2 pi v t) dt   (psi even, supported on
                                                                  [-m/L, m/L])
"""
import numpy as np
import pytest

import oracle as O

mp = pytest.importorskip("mpmath")
mp.mp.dps = 30


def ckb_mp(x, m, L, beta):
    r = 1 - (L * x / m) ** 2
    if r < 0:
        return mp.mpf(0)
    return (mp.besseli(0, beta * mp.sqrt(r)) - 1) / (mp.besseli(0, beta) - 1)


def gauss_mp(x, m, M, L):
    s2 = mp.mpf(m) / (mp.pi * L * (L - M))
    if abs(L * x) > m:
        return mp.mpf(0)
    return mp.exp(-x * x / (2 * s2))


def test_bessel_i0_reference_value():
    """I_0(1) = 1.2660658777520083356... (SPEC's sanity value); the oracle's np.i0 as well."""
    assert abs(mp.besseli(0, 1) - mp.mpf("1.26606587775200833559824462521")) < mp.mpf("1e-28")
    assert abs(float(np.i0(1.0)) - 1.2660658777520083) < 4e-16


@pytest.mark.parametrize("m,M", [(4, 64), (5, 64), (8, 256)])
def test_ckb_window_vs_mpmath(m, M):
    L = O.grid_length(M, 2.0)
    beta = O.default_shape("ckb", m, M, L)
    xs = np.array([0.0, 0.1, 0.37, 0.5, 0.8, 0.95, 0.999, 1.0]) * m / L
    got = O.phi("ckb", xs, m, L, beta)
    ref = np.array([float(ckb_mp(mp.mpf(float(x)), m, L, mp.mpf(beta))) for x in xs])
    assert np.max(np.abs(got - ref)) <= 1e-15
    # the pin rejects plausible slips: sqrt dropped inside I_0, "- 1" dropped
    r = 1 - (L * xs / m) ** 2
    no_sqrt = (np.i0(beta * r) - 1) / (np.i0(beta) - 1)
    no_minus = np.i0(beta * np.sqrt(r)) / np.i0(beta)
    for bad in (no_sqrt, no_minus):
        assert np.max(np.abs(bad - ref)) > 1e-9      # far outside the 1e-15 pin


@pytest.mark.parametrize("m,M", [(4, 64), (8, 256), (8, 1 << 20)])
def test_gauss_window_vs_mpmath(m, M):
    L = O.grid_length(M, 2.0)
    s = O.default_shape("gauss", m, M, L)
    assert abs(s - float(mp.sqrt(mp.mpf(m) / (mp.pi * L * (L - M))))) <= 1e-16 * s
    xs = np.array([0.0, 0.2, 0.5, 0.77, 1.0]) * m / L
    got = O.phi("gauss", xs, m, L, s)
    ref = np.array([float(gauss_mp(mp.mpf(float(x)), m, M, L)) for x in xs])
    assert np.max(np.abs(got - ref)) <= 2e-16
    bad = np.exp(-xs * xs / (s * s))           # missing factor 2 in the exponent
    assert np.max(np.abs(bad - ref)) > 1e-3


def psihat_mp(phi_mp, v, m, L):
    def psi(t):
        tau = L * t
        sinc = mp.mpf(1) if tau == 0 else mp.sin(mp.pi * tau) / (mp.pi * tau)
        return sinc * phi_mp(t)
    return 2 * mp.quad(lambda t: psi(t) * mp.cos(2 * mp.pi * v * t), [0, mp.mpf(m) / L / 2, mp.mpf(m) / L])


@pytest.mark.parametrize("window,m,M,ks", [("ckb", 5, 64, (0, 9, 31, -32)), ("ckb", 8, 256, (0, 77, -128)),
                                           ("gauss", 5, 64, (0, 9, 31, -32)), ("gauss", 8, 256, (0, 77, -128))])
def test_psihat_ckb_gauss_vs_mpmath(window, m, M, ks):
    """Step 0(a) for the cKB and Gaussian windows against 30-digit quadrature of an independently
    typed integrand (the QUADPACK pin of test_oracle_pins integrates the oracle's own psi)."""
    L = O.grid_length(M, 2.0)
    shape = O.default_shape(window, m, M, L)
    if window == "ckb":
        beta = mp.mpf(shape)

        def phi_mp(t):
            return ckb_mp(t, m, L, beta)
    else:
        def phi_mp(t):
            return gauss_mp(t, m, M, L)
    for k in ks:
        ref = float(psihat_mp(phi_mp, k, m, L))
        got = float(O.psihat_1d(window, np.array([float(k)]), m, L, shape)[0])
        # the Gaussian is cut at |x| = m/L (a jump, A2): its integrand has a kink-free but
        # non-analytic end, so the sin-substituted 64-point rule is checked to 1e-12 there
        tol = 4e-14 if window == "ckb" else 1e-12
        assert abs(got - ref) <= tol * abs(ref) + 1e-18, (window, k, got, ref)
