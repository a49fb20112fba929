"""GPU parity of Algorithm 1 (classical NFFT, BNFFT_ALG1) against the oracle (oracle/nfft.py)."""
import numpy as np
import pytest

import oracle as O
import synth
from oracle import nfft as NF

pytestmark = pytest.mark.gpu
TOL = {"c128": 1e-12, "c64": 1e-5}


def rel_l2(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))


@pytest.mark.parametrize("prec", ["c128", "c64"])
@pytest.mark.parametrize("window", ["sinh", "ckb"])
@pytest.mark.parametrize("M,m,N", [(64, 5, 1000), (1 << 12, 8, 40_001), (1 << 14, 6, 2_000)])
def test_alg1_parity(prec, window, M, m, N):
    import torch
    from paper_2502_07155_b200 import bnfft
    cfg = synth.CONFIGS[2].scaled(M=M, m=m, N=N)
    x = synth.make_nodes(cfg, variant=11)
    x[:3, 0] = [-0.5, 0.5 - 1e-12, 0.0]                  # wrap-around and grid nodes
    fh = synth.make_spectrum(cfg, variant=11, prec=prec)
    plan = bnfft.Plan(1, M, 2.0, m, window, prec, alg1=True)
    plan.set_nodes(torch.from_numpy(x).cuda())
    f = plan.execute(torch.from_numpy(fh).cuda()).cpu().numpy()
    ref = NF.algorithm1(x, fh.astype(np.complex128), M, 2.0, m, window)
    assert abs(plan.info().shape - ref["shape"]) < 1e-12 * ref["shape"]
    assert np.max(np.abs(plan.psihat() - ref["phihat"]) / np.abs(ref["phihat"])) < 2e-13
    assert rel_l2(f, ref["f"]) <= TOL[prec]
    plan.close()


def test_alg1_unsupported_combinations():
    from paper_2502_07155_b200 import bnfft
    for kw in (dict(d=2), dict(window="gauss"), dict(batch=2)):
        args = dict(d=1, window="sinh", batch=1)
        args.update(kw)
        with pytest.raises(bnfft.BnfftError) as ei:
            bnfft.Plan(args["d"], 64, 2.0, 4, args["window"], "c64", batch=args["batch"], alg1=True)
        assert ei.value.code == bnfft.BNFFT_E_UNSUPPORTED


def test_interpolate_and_kernel_hat_match_oracle_exp_errors():
    """The Figure 1 path (bnfft_interpolate + bnfft_kernel_hat) reproduces the oracle's e(v)
    (eq. maxerr_comparison_nfft) for the NFFT and Algorithm 2 approximations."""
    import math
    import torch
    from paper_2502_07155_b200 import bnfft
    M, m, L = 20, 5, 40
    xp = -0.5 + np.arange(4000) / 4000
    xt = xp[(xp >= -0.5 + m / L) & (xp < 0.5 - m / L)]
    ell = (np.arange(L) - L // 2).astype(np.float64)
    v = np.array([-12.25, -7.0, -3.5 + 1 / 32, 0.0, 9.96875])
    for alg1 in (True, False):
        plan = bnfft.Plan(1, M, 2.0, m, "sinh", "c128", alg1=alg1)
        plan.set_nodes(torch.from_numpy(xt[:, None].copy()).cuda())
        hat = plan.kernel_hat(v)
        sh = plan.info().shape
        ref_hat = (NF.phihat_1d if alg1 else O.psihat_1d)("sinh", v, m, L, sh)
        assert np.max(np.abs(hat - ref_hat) / np.abs(ref_hat)) < 1e-13
        errs = []
        for i, vv in enumerate(v):
            s = np.exp(2j * np.pi * vv * ell / L) / (L * hat[i])
            h = plan.interpolate(torch.from_numpy(s[None]).cuda())[0].cpu().numpy()
            errs.append(np.max(np.abs(np.exp(2j * np.pi * vv * xt) - h)))
        ref = (NF.exp_error_nfft if alg1 else NF.exp_error_alg2)(v, xt, M, m, L, "sinh", sh)
        assert np.allclose(errs, ref, rtol=1e-9, atol=1e-13), (alg1, errs, ref)
        plan.close()
