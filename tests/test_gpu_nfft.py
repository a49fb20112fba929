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
