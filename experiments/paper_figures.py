"""The paper's §5 experiments on the GPU path, through the C ABI only.

Figure 1: e(v) = max_p |e^{2 pi i v x_p} - h(x_p)| (eq. maxerr_comparison_nfft) for
v_s = -M/2 - m + s/S, s = 0..S(M+2m) (eq. ..._evaluation_points), M = 20, lambda = 1 (L = 40), m = 5,
sinh window, P equispaced points on [-1/2, 1/2) (full) and on [-1/2+m/L, 1/2-m/L) (truncated).
  NFFT   h: eq. approx_exp_nfft  = (L phi^(v))^{-1} sum_l e^{2 pi i v l/L} phi~_m(x - l/L)
  Alg. 2 h: P:599-610 with D_psihat kept      = (L psi^(v))^{-1} sum_l e^{2 pi i v l/L} psi(x - l/L)
  Alg. 2 h without psi^ (eq. approx_exp_nfft_like, reading A16): sum_l e^{2 pi i v l/L} psi(x - l/L)
Figure 2 / Example 5.3: f(x) = sinc^2(M pi x/2), f^ the triangle, scaled Chebyshev nodes
(eq. points_cheb_scaled), N = M/2, m = 5, lambda = 1, M = 20, 40, ..., 1000: max_j |f_j - f(x_j)| for
Algorithm 2 and Algorithm 1 (f^(k) as the NFFT's Fourier coefficients).
The figures' values are not in the paper text; the paper's claims are qualitative.

usage: python experiments/paper_figures.py [--P 100000] [--S 32] [--out profiles/r01_paper_figures.json]
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def beta_a1(M, L, m):
    """Reading A1 (Algorithm 2's default sinh beta), also used for the NFFT in the 'same-beta' runs."""
    return math.pi * m * (1.0 - M / L)


def fig1(bn, torch, P=100_000, S=32, M=20, m=5, sigma=2.0, window="sinh"):
    L = 2 * math.ceil(math.ceil(sigma * M) / 2)
    xp = -0.5 + np.arange(P) / P
    res = {"M": M, "L": L, "m": m, "P": P, "S": S, "window": window}
    v = -M / 2 - m + np.arange(S * (M + 2 * m) + 1) / S
    res["v"] = v.tolist()
    ell = (np.arange(L) - L // 2).astype(np.float64)
    for dom in ("full", "truncated"):
        x = xp if dom == "full" else xp[(xp >= -0.5 + m / L) & (xp < 0.5 - m / L)]
        xd = torch.from_numpy(np.ascontiguousarray(x[:, None])).cuda()
        e = np.exp(2j * np.pi * np.multiply.outer(v, x))            # (nv, P)
        for name, alg1, use_hat, shape in (("nfft", True, True, 0.0), ("nfft_samebeta", True, True, beta_a1(M, L, m)),
                                           ("alg2", False, True, 0.0), ("alg2_nohat", False, False, 0.0)):
            plan = bn.Plan(1, M, sigma, m, window, "c128", alg1=alg1, shape=shape)
            plan.set_nodes(xd)
            hat = plan.kernel_hat(v) if use_hat else np.full(len(v), 1.0 / L)
            errs = np.empty(len(v))
            for i, vv in enumerate(v):
                s = np.exp(2j * np.pi * vv * ell / L) / (L * hat[i])
                h = plan.interpolate(torch.from_numpy(s[None]).cuda())[0].cpu().numpy()
                errs[i] = np.max(np.abs(e[i] - h))
            res[f"{name}_{dom}"] = errs.tolist()
            plan.close()
    return res


def fig2(bn, torch, Ms=tuple(range(20, 1001, 20)), m=5, sigma=2.0, window="sinh"):
    out = {"M": list(Ms), "m": m, "window": window, "alg2": [], "nfft": [], "nfft_samebeta": []}
    for M in Ms:
        L = 2 * math.ceil(math.ceil(sigma * M) / 2)
        N = M // 2
        j = np.arange(1, N + 1)
        x = np.cos((j - 1) * np.pi / N) * (0.5 - m / L)
        k = np.arange(M) - M // 2
        fh = ((2.0 / M) * np.clip(1.0 - np.abs(2.0 * k / M), 0.0, None)).astype(np.complex128)[None]
        exact = np.sinc(M * x / 2) ** 2                      # numpy sinc(y) = sin(pi y)/(pi y)
        xd = torch.from_numpy(np.ascontiguousarray(x[:, None])).cuda()
        for name, alg1, shape in (("alg2", False, 0.0), ("nfft", True, 0.0), ("nfft_samebeta", True, beta_a1(M, L, m))):
            plan = bn.Plan(1, M, sigma, m, window, "c128", alg1=alg1, shape=shape)
            plan.set_nodes(xd)
            f = plan.execute(torch.from_numpy(fh).cuda())[0].cpu().numpy()
            out[name].append(float(np.max(np.abs(f - exact))))
            plan.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--P", type=int, default=100_000)
    ap.add_argument("--S", type=int, default=32)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_paper_figures.json"))
    a = ap.parse_args()
    import torch
    from paper_2502_07155_b200 import bnfft as bn
    t0 = time.time()
    r1 = fig1(bn, torch, P=a.P, S=a.S)
    r2 = fig2(bn, torch)
    v = np.array(r1["v"])
    inner = np.abs(v) <= r1["M"] / 2 - r1["m"] / r1["L"]
    summary = {
        "fig1_max_err_truncated_inband": {k: float(np.max(np.array(r1[f"{k}_truncated"])[inner]))
                                          for k in ("nfft", "nfft_samebeta", "alg2", "alg2_nohat")},
        "fig1_max_err_full_inband": {k: float(np.max(np.array(r1[f"{k}_full"])[inner]))
                                     for k in ("nfft", "nfft_samebeta", "alg2", "alg2_nohat")},
        "fig2_M>80_alg2_better_fraction": float(np.mean([a2 < nf for M, a2, nf in zip(r2["M"], r2["alg2"], r2["nfft"]) if M > 80])),
        "fig2_M>80_alg2_better_fraction_samebeta": float(np.mean([a2 < nf for M, a2, nf in zip(r2["M"], r2["alg2"], r2["nfft_samebeta"]) if M > 80])),
        "seconds": time.time() - t0,
    }
    json.dump({"fig1": r1, "fig2": r2, "summary": summary}, open(a.out, "w"))
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
