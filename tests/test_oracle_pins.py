"""Pins of the CPU oracle against what the paper and the mathematics fix (no GPU).

Each test names the passage it pins.  None of these re-types an oracle formula: they
compare against closed forms, independent quadrature libraries, literal sums, brute
force, invariants, or values printed in the paper (tests/golden/paper_params.json).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle as O
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_params.json")))


def rel_l2(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))


# ----------------------------------------------------------------------------- parameters
def test_grid_length_paper_examples():
    for M, sigma, L in GOLD["M_sigma"]["cases"]:
        assert O.grid_length(M, sigma) == L
    f1 = GOLD["fig1"]
    assert O.grid_length(f1["M"], 1 + f1["lambda"]) == f1["L"]


def test_grid_length_rejects_bad_bandwidth():
    with pytest.raises(ValueError):
        O.grid_length(7, 2.0)
    with pytest.raises(ValueError):
        O.grid_length(8, 0.9)


def test_J_set_examples():
    for x, L, m, members in GOLD["J_set"]["cases"]:
        assert O.J_set(x, L, m) == members
    # |J| is 2m for L x not an integer, 2m+1 otherwise ("at most (2m+1)^d")
    rng = np.random.default_rng(1)
    for x in rng.random(200) - 0.5:
        assert len(O.J_set(x, 64, 3)) in (6, 7)


# ----------------------------------------------------------------------------- windows
@pytest.mark.parametrize("window", ["sinh", "gauss", "ckb"])
def test_window_class_axioms(window):
    """Phi_{m,L}: even, supported on [-m/L, m/L], values in [0,1],
    non-increasing on [0, inf), phi(0) = 1."""
    m, M, L = 5, 20, 40
    s = O.default_shape(window, m, M, L)
    x = np.linspace(-1.5 * m / L, 1.5 * m / L, 4001)
    p = O.phi(window, x, m, L, s)
    assert np.array_equal(p, O.phi(window, -x, m, L, s))
    assert np.all(p[np.abs(x) > m / L] == 0.0)
    assert np.all((p >= 0) & (p <= 1))
    pos = p[x >= 0]
    assert np.all(np.diff(pos) <= 0)
    assert O.phi(window, np.array([0.0]), m, L, s)[0] == 1.0
    if window in ("sinh", "ckb"):            # C0: vanishes at the support edge
        assert O.phi(window, np.array([m / L]), m, L, s)[0] == 0.0
    # grid-unit evaluation agrees with x-unit evaluation (tau = L x)
    tau = np.linspace(-m, m, 257)
    assert np.allclose(O.phi_grid(window, tau, m, L, s), O.phi(window, tau / L, m, L, s),
                       rtol=1e-14, atol=1e-16)


def test_sinc_special_values():
    assert O.sinc(np.array([0.0]))[0] == 1.0
    assert abs(O.sinc(np.array([np.pi]))[0]) < 1e-16
    assert abs(O.sinc(np.array([np.pi / 2]))[0] - 2 / np.pi) < 1e-16


def test_psi_kronecker():
    """psi(l/L) = delta_{l,0} up to rounding of sin(pi l)."""
    for w in ("sinh", "gauss", "ckb"):
        s = O.default_shape(w, 4, 32, 64)
        v = O.psi_grid(w, np.arange(-4, 5, dtype=float), 4, 64, s)
        assert v[4] == 1.0
        assert np.all(np.abs(np.delete(v, 4)) < 1e-16)


# ----------------------------------------------------------------------------- step 0(a)
@pytest.mark.parametrize("window,m,M", [("sinh", 5, 64), ("sinh", 8, 256), ("gauss", 8, 256),
                                        ("ckb", 5, 64), ("sinh", 4, 128)])
def test_psihat_vs_quadpack(window, m, M):
    """psi^(v) = 2 int_0^{m/L} psi(t) cos(2 pi v t) dt, computed by scipy QUADPACK on the
    un-substituted integral (independent rule, adaptive)."""
    from scipy.integrate import quad
    L = O.grid_length(M, 2.0)
    s = O.default_shape(window, m, M, L)
    for v in (0.0, 1.0, M / 4 - 1, -M / 2, M / 2 - 1, 0.37 * M):
        def g(t):
            return float(O.psi_grid(window, np.array([L * t]), m, L, s)[0]) * math.cos(2 * math.pi * v * t)
        ref, err = quad(g, 0.0, m / L, epsabs=1e-17, epsrel=1e-14, limit=400)
        ref *= 2
        got = float(O.psihat_1d(window, np.array([v]), m, L, s)[0])
        assert abs(got - ref) <= 2e-13 * abs(ref) + 1e-17, (v, got, ref)


def test_psihat_vs_mpmath_30_digits():
    """Same integral in 30-digit arithmetic with mpmath's own sinh/sin/cos (tanh-sinh);
    agreement to a few ulp of psi^(k).  Covers cfg1 (m=5) and cfg2-like (m=8) parameters."""
    mp = pytest.importorskip("mpmath")
    mp.mp.dps = 30
    for m, M, ks in ((5, 64, (0, 7, 31, -32)), (8, 256, (0, 50, -128))):
        L = O.grid_length(M, 2.0)
        beta = mp.pi * m * (1 - mp.mpf(M) / L)

        def psi_mp(t):
            tau = L * t
            sinc = mp.mpf(1) if tau == 0 else mp.sin(mp.pi * tau) / (mp.pi * tau)
            r = 1 - (tau / m) ** 2
            return sinc * mp.sinh(beta * mp.sqrt(r)) / mp.sinh(beta) if r > 0 else mp.mpf(0)

        for k in ks:
            ref = 2 * mp.quad(lambda t: psi_mp(t) * mp.cos(2 * mp.pi * k * t),
                              [0, mp.mpf(m) / L / 2, mp.mpf(m) / L])
            got = O.psihat_1d("sinh", np.array([float(k)]), m, L, float(beta))[0]
            assert abs(got - float(ref)) <= 4e-14 * abs(float(ref)), (m, k, got, ref)


def test_psihat_even_and_flat():
    """psi^ is real and even (psi even); L psi^(k) ~ 1 on I_M (P:602 'numerical experiments')."""
    for w, bound in (("sinh", 1e-3), ("ckb", 1e-3), ("gauss", 5e-3)):
        M, m = 64, 5
        L = O.grid_length(M, 2.0)
        s = O.default_shape(w, m, M, L)
        k = np.arange(1, M // 2)
        a = O.psihat_1d(w, k.astype(float), m, L, s)
        b = O.psihat_1d(w, -k.astype(float), m, L, s)
        assert np.array_equal(a, b)
        tab = O.psihat_table(w, M, m, L, s)
        assert np.max(np.abs(L * tab - 1)) < bound


def test_psihat_quadrature_converged():
    """After the sin substitution (A4) the n = 48 and n = 64 Gauss-Legendre sums agree to
    rounding level (the rule has converged; leggauss itself limits larger n to ~1e-13)."""
    for w in ("sinh", "gauss", "ckb"):
        M, m = 256, 8
        L = O.grid_length(M, 2.0)
        s = O.default_shape(w, m, M, L)
        a = O.psihat_table(w, M, m, L, s, n=48)
        b = O.psihat_table(w, M, m, L, s, n=64)
        assert np.max(np.abs(a - b) / np.abs(b)) <= 1.5e-13


# ----------------------------------------------------------------------------- step 1
def test_step1_placement():
    """M=2, L=4, d=1: inner (a at k=-1, b at k=0) -> (0, a, b, 0) in I_4 order."""
    f = np.array([[2.0 + 1j, 3.0 - 1j]])
    out = O.step1_deconvolve_pad(f, np.array([1.0, 1.0]), 4)
    assert np.array_equal(out[0], np.array([0, 2 + 1j, 3 - 1j, 0]))
    out = O.step1_deconvolve_pad(f, np.array([2.0, 4.0]), 4)
    assert np.array_equal(out[0], np.array([0, (2 + 1j) / 2, (3 - 1j) / 4, 0]))


# ----------------------------------------------------------------------------- step 2
@pytest.mark.parametrize("L,d", [(4, 1), (8, 1), (12, 1), (16, 1), (20, 1), (40, 1),
                                 (4, 2), (8, 2), (12, 2), (16, 2)])
def test_step2_matches_literal_sum(L, d):
    rng = np.random.default_rng(L * 10 + d)
    th = rng.standard_normal((2,) + (L,) * d) + 1j * rng.standard_normal((2,) + (L,) * d)
    assert rel_l2(O.step2_inverse_fft(th), O.inverse_dft_literal(th)) < 1e-13


def test_step2_closed_forms():
    L, d = 16, 2
    ones = np.ones((1, L, L), dtype=complex)
    out = O.step2_inverse_fft(ones)       # sum_k e^{2 pi i k l/L} / L^d = delta_{l,0}
    ref = np.zeros_like(ones)
    ref[0, L // 2, L // 2] = 1.0
    assert np.max(np.abs(out - ref)) < 1e-15
    imp = np.zeros((1, L, L), dtype=complex)
    imp[0, L // 2, L // 2] = L ** d             # delta at k = 0 (centred index L/2)
    assert np.max(np.abs(O.step2_inverse_fft(imp) - 1.0)) < 1e-15
    # Parseval for the 1/L^d-normalised inverse
    rng = np.random.default_rng(3)
    th = rng.standard_normal((1, L, L)) + 1j * rng.standard_normal((1, L, L))
    s = O.step2_inverse_fft(th)
    assert abs(np.sum(np.abs(s) ** 2) * L ** d - np.sum(np.abs(th) ** 2)) < 1e-12 * np.sum(np.abs(th) ** 2)


# ----------------------------------------------------------------------------- step 3
@pytest.mark.parametrize("d", [1, 2, 3])
def test_interpolation_property(d):
    """(R f)(k/L) = f(k/L): at grid nodes the short sum returns theta_k."""
    M, m = 16, 3
    L = O.grid_length(M, 2.0)
    rng = np.random.default_rng(d)
    th = rng.standard_normal((2,) + (L,) * d) + 1j * rng.standard_normal((2,) + (L,) * d)
    x = synth.grid_point_nodes(50, d, L, seed=d)
    for w in ("sinh", "gauss"):
        f = O.step3_short_sums(th, x, w, m, O.default_shape(w, m, M, L))
        idx = tuple((np.round(x * L).astype(int) + L // 2).T)
        ref = th[(slice(None),) + idx]
        assert np.max(np.abs(f - ref)) < 1e-14 * np.max(np.abs(th)) * (2 * m + 1) ** d


@pytest.mark.parametrize("d,M,sigma,shape", [(1, 4, 2.0, None), (1, 8, 2.0, None), (1, 8, 1.0, 6.0),
                                             (2, 4, 2.0, None), (2, 8, 2.0, None), (2, 8, 1.0, 6.0),
                                             (1, 8, 1.5, None)])
def test_fast_equals_dense(d, M, sigma, shape):
    """Fast steps 1-3 == dense Psi F D_psihat f^ (eq. function_eval), m=2, N=7."""
    m = 2
    L = O.grid_length(M, sigma)
    x = synth.feasible_box_nodes(7, d, L, m, seed=M + d)
    rng = np.random.default_rng(11)
    fh = rng.standard_normal((20,) + (M,) * d) + 1j * rng.standard_normal((20,) + (M,) * d)
    for w in ("sinh", "ckb", "gauss"):
        sh = shape if (shape is not None and w != "gauss") else None
        if sigma == 1.0 and w == "gauss":
            continue                          # A2's s is undefined at L = M
        a = O.algorithm2(x, fh, M, sigma, m, window=w, shape=sh)["f"]
        b = O.dense_apply(x, fh, M, sigma, m, window=w, shape=sh)
        assert rel_l2(a, b) < 1e-12


def test_dense_row_sparsity():
    """Each row of Psi has at most (2m+1)^d nonzeros."""
    M, m, d = 8, 2, 2
    L = O.grid_length(M, 2.0)
    x = synth.feasible_box_nodes(9, d, L, m, seed=3)
    KL = np.stack([g.ravel() for g in np.meshgrid(*([np.arange(L) - L // 2] * d), indexing="ij")], 1)
    tau = L * x[:, None, :] - KL[None]
    Psi = np.prod(O.psi_grid("sinh", tau, m, L, O.default_shape("sinh", m, M, L)), axis=2)
    assert np.all(np.count_nonzero(Psi, axis=1) <= (2 * m + 1) ** d)


# ----------------------------------------------------------------------------- end to end
def test_end_to_end_vs_trig_sum_cfg1():
    """Alg. 2 approximates sum_k f^(k) e^{2 pi i k x} (eq. nfft; reading A12) on the
    feasible box to the regularization error (cfg1 shapes: d=1, M=64, sigma=2, m=5, sinh)."""
    cfg = synth.CONFIGS[1]
    L = O.grid_length(cfg.M, cfg.sigma)
    x = synth.feasible_box_nodes(cfg.N, 1, L, cfg.m)
    fh = synth.make_spectrum(cfg)
    f = O.algorithm2(x, fh, cfg.M, cfg.sigma, cfg.m)["f"]
    err = rel_l2(f, O.trig_sum(x, fh))
    assert 1e-6 < err < 2e-4


def test_end_to_end_vs_trig_sum_d2_d3():
    for d, M, m, bound in ((2, 16, 5, 3e-4), (3, 8, 4, 2e-3)):
        L = O.grid_length(M, 2.0)
        x = synth.feasible_box_nodes(300, d, L, m, seed=d)
        rng = np.random.default_rng(d)
        fh = rng.standard_normal((1,) + (M,) * d) + 1j * rng.standard_normal((1,) + (M,) * d)
        f = O.algorithm2(x, fh, M, 2.0, m)["f"]
        assert rel_l2(f, O.trig_sum(x, fh)) < bound


def test_dirichlet_closed_form():
    """f^ == 1 on I_M: the target sum_{k=-M/2}^{M/2-1} e^{2 pi i k x} = sin(pi M x) e^{-i pi x}/sin(pi x)
    (geometric series; value M at x = 0).  BASELINE.json configs[0] closed-form check."""
    M, m = 64, 5
    L = O.grid_length(M, 2.0)
    x = synth.feasible_box_nodes(1000, 1, L, m)
    f = O.algorithm2(x, synth.ones_spectrum(M), M, 2.0, m)["f"][0]
    xx = x[:, 0]
    ref = np.sin(np.pi * M * xx) * np.exp(-1j * np.pi * xx) / np.sin(np.pi * xx)
    assert rel_l2(f, ref) < 2e-4
    # at x = 0 the value is M (up to the regularization error)
    f0 = O.algorithm2(np.zeros((1, 1)), synth.ones_spectrum(M), M, 2.0, m)["f"][0, 0]
    assert abs(f0 - M) < 1e-2
    # d = 2: product of the 1-D forms
    M2 = 16
    L2 = O.grid_length(M2, 2.0)
    x2 = synth.feasible_box_nodes(200, 2, L2, m, seed=2)
    f2 = O.algorithm2(x2, synth.ones_spectrum(M2, 2), M2, 2.0, m)["f"][0]
    ref2 = np.prod(np.sin(np.pi * M2 * x2) * np.exp(-1j * np.pi * x2) / np.sin(np.pi * x2), axis=1)
    assert rel_l2(f2, ref2) < 5e-4


def test_fejer_closed_form_example53():
    """Example 5.3 triangle f^(v) = (2/M)(1-|2v/M|).  Its I_M trig sum is the Fejer
    kernel (sin(pi M x/2) / ((M/2) sin(pi x)))^2; the paper's sinc^2(M pi x/2) differs from it
    only by aliasing (reading A12).  Chebyshev nodes, N = M/2, m = 5, lambda = 1."""
    ex = GOLD["example53"]
    tri = synth.triangle_spectrum(20)[0]
    k = np.arange(20) - 10
    for kk, val in zip(ex["triangle_at_M20"]["k"], ex["triangle_at_M20"]["fhat"]):
        assert abs(tri[k == kk][0] - val) < 1e-15
    for M in (20, 64, 200):
        L = O.grid_length(M, 1 + ex["lambda"])
        x = synth.chebyshev_nodes(M // 2, L, ex["m"])
        f = O.algorithm2(x, synth.triangle_spectrum(M), M, 2.0, ex["m"])["f"][0]
        xx = x[:, 0]
        with np.errstate(invalid="ignore", divide="ignore"):
            fej = np.where(xx == 0, 1.0, (np.sin(np.pi * M * xx / 2) / ((M / 2) * np.sin(np.pi * xx))) ** 2)
        assert np.max(np.abs(f - fej)) < 1e-4
        sinc2 = np.sinc(M * xx / 2) ** 2           # numpy sinc(y) = sin(pi y)/(pi y)
        assert np.max(np.abs(f - sinc2)) < 5e-3     # aliasing ~ 1/M^2 (P:697-699 qualitative)
    c = GOLD["example53"]["cheb_M20_first_last"]
    xc = synth.chebyshev_nodes(c["N"], c["L"], 5)[:, 0]
    assert xc[0] == c["x1"] and abs(xc[5]) < 1e-16


def test_error_decay_in_m():
    """BASELINE north_star check (iii): error decays in m for each window.  The paper states
    no rate (P:334 cites KiPoTa22/23); measured log-ratio per unit m must be near
    -pi(1-1/sigma) (sinh, cKB) and -pi(1-1/sigma)/2 (Gaussian, reading A2), within 25%."""
    M, sigma = 64, 2.0
    L = O.grid_length(M, sigma)
    x = synth.feasible_box_nodes(600, 1, L, 12)
    fh = synth.make_spectrum(synth.CONFIGS[1])
    ts = O.trig_sum(x, fh)
    for w, rate in (("sinh", math.pi * 0.5), ("ckb", math.pi * 0.5), ("gauss", math.pi * 0.25)):
        ms = list(range(2, 12))
        e = [rel_l2(O.algorithm2(x, fh, M, sigma, m, window=w)["f"], ts) for m in ms]
        assert all(e[i + 1] < e[i] for i in range(len(e) - 1)), e
        slope = np.polyfit(ms, np.log(e), 1)[0]
        assert abs(-slope - rate) < 0.25 * rate, (w, slope)


def test_linearity_and_real_symmetry():
    M, m, d = 16, 4, 2
    L = O.grid_length(M, 2.0)
    x = synth.feasible_box_nodes(100, d, L, m, seed=9)
    rng = np.random.default_rng(4)
    a = rng.standard_normal((1, M, M)) + 1j * rng.standard_normal((1, M, M))
    b = rng.standard_normal((1, M, M)) + 1j * rng.standard_normal((1, M, M))
    fa = O.algorithm2(x, a, M, 2.0, m)["f"]
    fb = O.algorithm2(x, b, M, 2.0, m)["f"]
    fab = O.algorithm2(x, 2.5 * a - 1j * b, M, 2.0, m)["f"]
    assert rel_l2(fab, 2.5 * fa - 1j * fb) < 1e-13
    # Hermitian spectrum supported on the symmetric subset (f^(-M/2) = 0): real output
    h = a.copy()
    h[:, 0, :] = 0
    h[:, :, 0] = 0
    hs = h[:, 1:, 1:]
    hs = 0.5 * (hs + np.conj(hs[:, ::-1, ::-1]))
    h[:, 1:, 1:] = hs
    f = O.algorithm2(x, h, M, 2.0, m)["f"]
    assert np.max(np.abs(f.imag)) < 1e-12 * np.max(np.abs(f))


# ----------------------------------------------------------------------------- node binning
def test_stable_bin_sort_bruteforce():
    rng = np.random.default_rng(5)
    keys = rng.integers(0, 37, size=3000)
    keys[100:400] = 5                       # long run of ties
    perm, off = O.stable_bin_sort(keys, 37)
    ref = [i for _, i in sorted((int(k), i) for i, k in enumerate(keys))]
    assert perm.tolist() == ref
    assert off[0] == 0 and off[-1] == len(keys)
    for b in range(37):
        assert np.all(keys[perm[off[b]:off[b + 1]]] == b)


def test_cell_index():
    L = 40
    x = np.array([-0.5, -0.5 + 1 / L, 0.0, 0.3, 0.5 - 1e-12])
    assert O.cell_index(x, L).tolist() == [0, 1, 20, 32, 39]
