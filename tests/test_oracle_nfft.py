"""Pins of the Algorithm 1 (classical NFFT) oracle, oracle/nfft.py (no GPU)."""
import math

import numpy as np
import pytest

import oracle as O
import synth
from oracle import nfft as N


def rel_l2(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))


@pytest.mark.parametrize("d,M,sigma", [(1, 8, 2.0), (1, 8, 1.5), (2, 8, 2.0), (2, 4, 2.0)])
def test_fast_equals_dense_BFD(d, M, sigma):
    """Algorithm 1 steps 1-3 == dense B F D f^, including wrap-around nodes."""
    m = 2
    L = O.grid_length(M, sigma)
    rng = np.random.default_rng(d * 7 + M)
    x = rng.random((9, d)) - 0.5
    x[0] = -0.5
    x[1] = 0.5 - 1e-3
    fh = rng.standard_normal((5,) + (M,) * d) + 1j * rng.standard_normal((5,) + (M,) * d)
    for w in ("sinh", "ckb"):
        a = N.algorithm1(x, fh, M, sigma, m, window=w)["f"]
        b = N.dense_apply_nfft(x, fh, M, sigma, m, window=w)
        assert rel_l2(a, b) < 1e-12


def test_nfft_approximates_trig_sum_on_torus():
    """The NFFT approximates eq. nfft on the whole torus; error falls with m (window error
    ~ e^{-2 pi m (1 - 1/(2 sigma))} for the sinh window of reading A17)."""
    cfg = synth.CONFIGS[1]
    x = synth.make_nodes(cfg, N=600)
    fh = synth.make_spectrum(cfg)
    ts = O.trig_sum(x, fh)
    errs = [rel_l2(N.algorithm1(x, fh, cfg.M, 2.0, m)["f"], ts) for m in range(2, 8)]
    assert all(errs[i + 1] < errs[i] for i in range(len(errs) - 1))
    assert errs[3] < 1e-8                          # m = 5
    slope = np.polyfit(range(2, 8), np.log(errs), 1)[0]
    rate = 2 * math.pi * (1 - 1 / 4)
    assert abs(-slope - rate) < 0.3 * rate


def test_periodic_index_set():
    """eq. indexset_x: |I| = 2m+1 at grid nodes, 2m otherwise; invariant under x -> x + 1."""
    # L x = 19.6: l in [17.6, 21.6] -> {18, 19, 20, 21}, wrapped to I_40 -> {-20, -19, 18, 19}
    assert [l for l, _ in N.periodic_index_set(0.49, 40, 2)] == [-20, -19, 18, 19]
    assert len(N.periodic_index_set(0.3, 40, 1)) == 3
    for x in (0.123, -0.4999, 0.37):
        a = [l for l, _ in N.periodic_index_set(x, 40, 3)]
        b = [l for l, _ in N.periodic_index_set(x + 1.0 - 1.0, 40, 3)]
        assert a == b and len(a) == 6


def test_phihat_vs_quadpack():
    from scipy.integrate import quad
    M, m = 64, 5
    L = O.grid_length(M, 2.0)
    s = N.default_shape_nfft("sinh", m, M, L)
    for v in (0.0, 3.0, -32.0, 17.5):
        ref = 2 * quad(lambda t: float(O.phi("sinh", np.array([t]), m, L, s)[0]) * math.cos(2 * math.pi * v * t),
                       0, m / L, epsabs=1e-17, epsrel=1e-14, limit=400)[0]
        got = N.phihat_1d("sinh", np.array([v]), m, L, s)[0]
        assert abs(got - ref) <= 2e-13 * abs(ref)


def test_exp_identities_reduce_to_algorithms():
    """At integer v = k, eq. approx_exp_nfft is Algorithm 1 applied to f^ = delta_k and
    the D_psihat-kept form of eq. approx_exp_nfft_like is Algorithm 2 applied to it."""
    M, m, L = 20, 5, 40
    xp = synth.feasible_box_nodes(400, 1, L, m)[:, 0]
    for k in (-10, -3, 0, 7):
        fh = np.zeros((1, M), dtype=complex)
        fh[0, k + M // 2] = 1.0
        e_exact = np.exp(2j * np.pi * k * xp)
        a1 = N.algorithm1(xp[:, None], fh, M, 2.0, m)["f"][0]
        a2 = O.algorithm2(xp[:, None], fh, M, 2.0, m)["f"][0]
        assert abs(np.max(np.abs(e_exact - a1)) - N.exp_error_nfft(
            np.array([float(k)]), xp, M, m, L, "sinh", N.default_shape_nfft("sinh", m, M, L))[0]) < 1e-13
        assert abs(np.max(np.abs(e_exact - a2)) - N.exp_error_alg2(
            np.array([float(k)]), xp, M, m, L, "sinh", O.default_shape("sinh", m, M, L))[0]) < 1e-13
