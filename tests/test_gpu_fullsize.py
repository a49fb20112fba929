"""Parity at the full BASELINE.json sizes, in the launch configuration bench.py times.

The oracle cannot evaluate 2^24-2^26 nodes, so it computes steps 0(a)-2 at full size (the theta grid)
and step 3 on a seeded sample of nodes; the GPU output at those nodes must match within the
north_star tolerances (relative l2 1e-12 complex128, 1e-5 complex64).  The bin sort is checked at full
size through properties that hold at any size: perm is a permutation, keys are non-decreasing along
it, and equal keys keep increasing user indices (stability)."""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

TOL = {"c128": 1e-12, "c64": 1e-5}
SAMPLE = 3000


def rel_l2(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))


def check_sort_properties(torch, plan, x_dev):
    info = plan.info()
    perm = plan.perm().long()
    n = x_dev.shape[0]
    assert perm.numel() == n
    assert torch.equal(torch.sort(perm).values, torch.arange(n, device=perm.device))
    L = float(info.L)
    key = torch.zeros(n, dtype=torch.int64, device=x_dev.device)
    for t in range(info.d):
        c = torch.floor(x_dev[:, t] * L).long() + info.L // 2
        c = torch.clamp(c, max=info.L - 1)
        key = key * info.bins_per_dim[t] + (c >> info.bin_log2[t])
    key = (torch.arange(n, device=x_dev.device) >> info.user_block_log2) * info.nbins + key
    cb = int(info.key_col_bits)   # minor sort digit: the y column inside the bin (bnfft_info)
    if info.d >= 2 and cb:
        c1 = torch.clamp(torch.floor(x_dev[:, 1] * L).long() + info.L // 2, max=info.L - 1)
        key = key * (1 << cb) + (c1 & ((1 << cb) - 1))
    ks = key[perm]
    assert bool(torch.all(ks[1:] >= ks[:-1]))
    same = ks[1:] == ks[:-1]
    assert bool(torch.all(perm[1:][same] > perm[:-1][same]))


def run_case(torch, cid, prec, window, spectra=(0,)):
    from paper_2502_07155_b200 import bnfft
    cfg = synth.CONFIGS[cid]
    x = synth.make_nodes(cfg)
    fh = synth.make_spectrum(cfg, prec=prec)
    x_dev = torch.from_numpy(x).cuda()
    plan = bnfft.Plan(cfg.d, cfg.M, cfg.sigma, cfg.m, window, prec, batch=cfg.batch)
    plan.set_nodes(x_dev)
    f = plan.execute(torch.from_numpy(fh).cuda())
    check_sort_properties(torch, plan, x_dev)
    rng = np.random.default_rng(17 + cid)
    idx = np.sort(rng.choice(cfg.N, size=SAMPLE, replace=False))
    idx = np.concatenate([idx, [0, cfg.N - 1]])
    L = O.grid_length(cfg.M, cfg.sigma)
    shape = O.default_shape(window, cfg.m, cfg.M, L)
    tab = O.psihat_table(window, cfg.M, cfg.m, L, shape)
    ph = O.psihat_multi(tab, cfg.d)
    for b in spectra:
        theta = O.step2_inverse_fft(O.step1_deconvolve_pad(fh[b:b + 1].astype(np.complex128), ph, L))
        ref = O.step3_short_sums(theta, x[idx], window, cfg.m, shape)[0]
        got = f[b, torch.from_numpy(idx).cuda()].cpu().numpy()
        err = rel_l2(got, ref)
        assert err <= TOL[prec], (cid, prec, window, b, err)
    plan.close()


@pytest.fixture(scope="module")
def torch():
    import torch as _t
    return _t


@pytest.mark.parametrize("prec,window", [("c64", "sinh"), ("c128", "sinh"), ("c64", "gauss"),
                                         ("c128", "gauss")])
def test_cfg2_full(torch, prec, window):
    run_case(torch, 2, prec, window)


def test_cfg3_full(torch):
    run_case(torch, 3, "c64", "sinh")


def test_cfg4_full(torch):
    run_case(torch, 4, "c64", "sinh")


def test_cfg5_full(torch):
    run_case(torch, 5, "c64", "sinh", spectra=(0, 63))
