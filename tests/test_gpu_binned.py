"""GPU parity of the d = 1 large-grid path (plan.d1_binned: 2^(ceil log2 L - 9)-cell bins, one 9-bit
radix pass that also writes the sorted node copy, per-bin gather1b) against the oracle, on sampled
nodes (the oracle computes steps 0(a)-2 on the full grid and step 3 at the sampled nodes)."""
import numpy as np
import pytest

import oracle as O
import synth
from oracle import nfft as NF

pytestmark = pytest.mark.gpu
TOL = {"c128": 1e-12, "c64": 1e-5}
SAMPLE = 2500


def rel_l2(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))


@pytest.fixture(scope="module")
def torch():
    import torch as _t
    return _t


def sampled_ref(x, fh, M, sigma, m, window, idx, alg1=False):
    L = O.grid_length(M, sigma)
    if alg1:
        ref = NF.algorithm1(x[idx], fh.astype(np.complex128), M, sigma, m, window)
        return ref["f"]
    shape = O.default_shape(window, m, M, L)
    ph = O.psihat_multi(O.psihat_table(window, M, m, L, shape), 1)
    theta = O.step2_inverse_fft(O.step1_deconvolve_pad(fh.astype(np.complex128), ph, L))
    return O.step3_short_sums(theta, x[idx], window, m, shape)


CASES = [  # id, M, sigma, m, window, prec, N, exact, alg1
    ("sinh-c64", 1 << 17, 2.0, 8, "sinh", "c64", 1 << 20, False, False),
    ("gauss-c64", 1 << 17, 2.0, 6, "gauss", "c64", 700_001, False, False),
    ("sinh-c128", 1 << 17, 2.0, 8, "sinh", "c128", 300_007, False, False),
    ("gauss-c128-alg1-free", 1 << 16, 2.0, 7, "gauss", "c128", 200_003, False, False),
    ("ckb-exact-c64", 1 << 17, 2.0, 5, "ckb", "c64", 300_007, True, False),
    ("nonpow2-L", 150_000, 2.0, 7, "sinh", "c64", 500_003, False, False),
    ("sigma1.5", 1 << 17, 1.5, 4, "sinh", "c64", 400_009, False, False),
    ("alg1-sinh-c64", 1 << 17, 2.0, 6, "sinh", "c64", 300_001, False, True),
    ("sparse", 1 << 18, 2.0, 8, "sinh", "c64", 20_011, False, False),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_binned_parity(torch, case):
    from paper_2502_07155_b200 import bnfft as bn
    _, M, sigma, m, window, prec, N, exact, alg1 = case
    cfg = synth.CONFIGS[2].scaled(M=M, m=m, N=N)
    x = synth.make_nodes(cfg, variant=21)
    x[:4, 0] = [-0.5, 0.5 - 1e-12, 0.0, 0.25]            # grid ends (wrap for Algorithm 1), grid nodes
    fh = synth.make_spectrum(cfg, variant=21, prec=prec)
    plan = bn.Plan(1, M, sigma, m, window, prec, exact_taps=exact, alg1=alg1)
    info = plan.info()
    assert info.gather_kernel == 1 and info.sort_passes == 1, (info.gather_kernel, info.sort_passes)
    assert info.nbins <= 512
    x_dev = torch.from_numpy(x).cuda()
    plan.set_nodes(x_dev)
    f = plan.execute(torch.from_numpy(fh).cuda()).cpu().numpy()[0]
    rng = np.random.default_rng(5)
    idx = np.sort(np.concatenate([[0, 1, 2, 3, N - 1], rng.choice(N, size=SAMPLE, replace=False)]))
    idx = np.unique(idx)
    ref = sampled_ref(x, fh, M, sigma, m, window, idx, alg1)
    ref = np.ravel(ref)
    assert rel_l2(f[idx], ref) <= TOL[prec], rel_l2(f[idx], ref)
    # permutation: a stable bin sort (keys recomputed on the host)
    info = plan.info()
    L = info.L
    W = 1 << info.bin_log2[0]
    c = np.minimum(np.floor(x[:, 0] * L).astype(np.int64) + L // 2, L - 1)
    key = (np.arange(N) >> info.user_block_log2) * info.nbins + (c // W)
    perm = plan.perm().cpu().numpy().astype(np.int64)
    assert np.array_equal(perm, np.argsort(key, kind="stable"))
    off = plan.bin_offsets().cpu().numpy().astype(np.int64)
    assert np.array_equal(off, np.searchsorted(key[perm], np.arange(info.nkeys + 1), side="left"))
    plan.close()


def test_binned_interpolation_and_shards(torch):
    """Grid nodes return theta exactly and node shards reproduce the full plan bitwise
    on the per-bin path."""
    from paper_2502_07155_b200 import bnfft as bn
    from paper_2502_07155_b200 import shard
    M, m = 1 << 17, 8
    L = 2 * M
    cfg = synth.CONFIGS[2].scaled(M=M, m=m, N=400_000)
    rng = np.random.default_rng(9)
    ell = rng.integers(-L // 2, L // 2, size=20_000)
    x = np.concatenate([synth.make_nodes(cfg, variant=22), (ell / L)[:, None]])
    fh = synth.make_spectrum(cfg, variant=22, prec="c64")
    full = bn.Plan(1, M, 2.0, m, "sinh", "c64")
    assert full.info().gather_kernel == 1
    xd = torch.from_numpy(x).cuda()
    full.set_nodes(xd)
    ft = torch.from_numpy(fh).cuda()
    f = full.execute(ft).clone()
    theta = full.grid().cpu().numpy().reshape(-1)
    got = f.cpu().numpy()[0, -ell.size:]
    assert np.array_equal(got, theta[ell + L // 2])
    parts = []
    for r in range(3):
        a, b = shard.node_shard(x.shape[0], r, 3)
        p = bn.Plan(1, M, 2.0, m, "sinh", "c64")
        p.set_nodes(xd[a:b].contiguous())
        parts.append(p.execute(ft).clone())
        p.close()
    assert torch.equal(torch.cat(parts, dim=1), f)
    full.close()
