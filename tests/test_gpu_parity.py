"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on identical seeded
inputs.  Tolerances (BASELINE.json north_star): relative l2 <= 1e-12 (complex128), <= 1e-5
(complex64); the node bin-sort bit-exact.  Sizes span several sort tiles / gather chunks and a
ragged tail; full BASELINE sizes are checked on sampled outputs in test_gpu_fullsize.py."""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu

TOL = {"c128": 1e-12, "c64": 1e-5}


def rel_l2(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))


@pytest.fixture(scope="module")
def torch():
    import torch as _t
    return _t


@pytest.fixture(scope="module")
def bn():
    from paper_2502_07155_b200 import bnfft
    return bnfft


def run_gpu(bn, torch, x, fh, d, M, sigma, m, window, prec, batch=1, **kw):
    dev = torch.device("cuda:0")
    plan = bn.Plan(d, M, sigma, m, window, prec, batch=batch, **kw)
    plan.set_nodes(torch.from_numpy(np.ascontiguousarray(x)).to(dev))
    ft = torch.from_numpy(np.ascontiguousarray(fh.astype(np.complex128 if prec == "c128" else np.complex64))).to(dev)
    f = plan.execute(ft).cpu().numpy()
    return f, plan


def oracle_f(x, fh, M, sigma, m, window):
    return O.algorithm2(x, fh.astype(np.complex128), M, sigma, m, window)


# ----------------------------------------------------------------------------- cfg1 (exact size)
def test_cfg1_full(bn, torch):
    cfg = synth.CONFIGS[1]
    x = synth.make_nodes(cfg)
    fh = synth.make_spectrum(cfg)
    f, plan = run_gpu(bn, torch, x, fh, 1, cfg.M, cfg.sigma, cfg.m, "sinh", "c128")
    ref = oracle_f(x, fh, cfg.M, cfg.sigma, cfg.m, "sinh")
    assert rel_l2(f, ref["f"]) <= TOL["c128"]
    # stage parity: psi^ table and the theta grid
    assert np.max(np.abs(plan.psihat() - ref["psihat"]) / np.abs(ref["psihat"])) < 2e-13
    assert rel_l2(plan.grid().cpu().numpy(), ref["theta"]) < 1e-13
    plan.close()


def test_cfg1_closed_forms(bn, torch):
    """f^ == 1 (Dirichlet form) and the Example 5.3 triangle (Fejer form) on the feasible box."""
    M, m = 64, 5
    L = O.grid_length(M, 2.0)
    x = synth.feasible_box_nodes(1000, 1, L, m)
    f, _ = run_gpu(bn, torch, x, synth.ones_spectrum(M), 1, M, 2.0, m, "sinh", "c128")
    xx = x[:, 0]
    ref = np.sin(np.pi * M * xx) * np.exp(-1j * np.pi * xx) / np.sin(np.pi * xx)
    assert rel_l2(f[0], ref) < 2e-4
    f, _ = run_gpu(bn, torch, x, synth.triangle_spectrum(M), 1, M, 2.0, m, "sinh", "c128")
    fej = (np.sin(np.pi * M * xx / 2) / ((M / 2) * np.sin(np.pi * xx))) ** 2
    assert np.max(np.abs(f[0] - fej)) < 1e-4


# ----------------------------------------------------------------------------- reduced configs
CASES = [
    # (name, cfg_id, d, M, m, N, batch, window, prec)
    ("cfg2-sinh-c128", 2, 1, 1 << 12, 8, 50_003, 1, "sinh", "c128"),
    ("cfg2-sinh-c64", 2, 1, 1 << 12, 8, 50_003, 1, "sinh", "c64"),
    ("cfg2-gauss-c128", 2, 1, 1 << 12, 8, 50_003, 1, "gauss", "c128"),
    ("cfg2-gauss-c64", 2, 1, 1 << 12, 8, 50_003, 1, "gauss", "c64"),
    ("cfg3-c64", 3, 2, 128, 6, 30_011, 1, "sinh", "c64"),
    ("cfg3-c128", 3, 2, 128, 6, 30_011, 1, "sinh", "c128"),
    ("cfg4-c64", 4, 3, 32, 4, 20_001, 1, "sinh", "c64"),
    ("cfg4-c128", 4, 3, 32, 4, 20_001, 1, "sinh", "c128"),
    ("cfg5-c64", 5, 3, 16, 4, 4096, 8, "sinh", "c64"),
    ("ckb-d1-c128", 1, 1, 256, 6, 9_999, 1, "ckb", "c128"),
    ("ckb-d2-c64", 3, 2, 64, 5, 9_999, 1, "ckb", "c64"),
    ("d2-gauss-c128", 3, 2, 64, 7, 7_777, 2, "gauss", "c128"),
    ("d1-m1-c128", 1, 1, 64, 1, 3_001, 1, "sinh", "c128"),
    ("d1-m16-c64", 2, 1, 512, 16, 12_345, 1, "sinh", "c64"),
    ("d1-batch3-c128", 2, 1, 1 << 10, 8, 20_000, 3, "sinh", "c128"),
    ("d1-batch4-c64", 2, 1, 1 << 10, 6, 20_000, 4, "gauss", "c64"),
    ("d1-sparse-c64", 2, 1, 1 << 16, 8, 3_000, 1, "sinh", "c64"),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_reduced_configs(bn, torch, case):
    name, cid, d, M, m, N, batch, window, prec = case
    cfg = synth.CONFIGS[cid].scaled(d=d, M=M, m=m, N=N, batch=batch)
    x = synth.make_nodes(cfg, variant=1)
    fh = synth.make_spectrum(cfg, variant=1, prec=prec)
    f, plan = run_gpu(bn, torch, x, fh, d, M, 2.0, m, window, prec, batch=batch)
    ref = oracle_f(x, fh, M, 2.0, m, window)
    err = rel_l2(f, ref["f"])
    assert err <= TOL[prec], err
    g = plan.grid().cpu().numpy()
    assert rel_l2(g, ref["theta"]) <= (1e-13 if prec == "c128" else 2e-6)
    plan.close()


# ----------------------------------------------------------------------------- bin sort
@pytest.mark.parametrize("cid,d,M,N", [(2, 1, 1 << 16, 100_000), (2, 1, 1 << 16, 3_000_017),
                                       (3, 2, 256, 70_000), (3, 2, 1024, 2_500_000),
                                       (4, 3, 64, 50_000), (5, 3, 64, 40_000)])
def test_bin_sort_bit_exact(bn, torch, cid, d, M, N):
    cfg = synth.CONFIGS[cid].scaled(d=d, M=M, N=N, batch=1)
    x = synth.make_nodes(cfg, variant=2)
    if cid == 5:
        x[:500] = 0.0                    # a long run of identical keys (ties)
    plan = bn.Plan(d, M, 2.0, 4, "sinh", "c64")
    plan.set_nodes(torch.from_numpy(x).cuda())
    info = plan.info()
    cells = O.cell_index(x, info.L)
    cells = np.minimum(cells, info.L - 1)
    key = np.zeros(N, dtype=np.int64)
    for t in range(d):
        key = key * info.bins_per_dim[t] + (cells[:, t] >> info.bin_log2[t])
    # sort key ((user block, bin), y column) as documented in include/bnfft.h (bnfft_info); offsets
    # per (user block, bin)
    key = (np.arange(N, dtype=np.int64) >> info.user_block_log2) * info.nbins + key
    assert info.nkeys == (((N - 1) >> info.user_block_log2) + 1) * info.nbins
    cb = int(info.key_col_bits)
    if d >= 2 and cb:
        key = key * (1 << cb) + (cells[:, 1] & ((1 << cb) - 1))
    perm_ref, _ = O.stable_bin_sort(key, int(info.nkeys) << cb)
    _, off_ref = O.stable_bin_sort(key >> cb, int(info.nkeys))
    perm = plan.perm().cpu().numpy().astype(np.int64)
    off = plan.bin_offsets().cpu().numpy().astype(np.int64)
    assert np.array_equal(perm, perm_ref)
    assert np.array_equal(off, off_ref)
    plan.close()


@pytest.mark.parametrize("prec", ["c128", "c64"])
@pytest.mark.parametrize("window", ["sinh", "gauss", "ckb"])
def test_exact_taps_path(bn, torch, prec, window):
    """BNFFT_EXACT_TAPS (direct sinc * phi) and the default tap polynomials both meet parity."""
    cfg = synth.CONFIGS[2].scaled(M=1 << 10, m=6, N=20_011)
    x = synth.make_nodes(cfg, variant=6)
    fh = synth.make_spectrum(cfg, variant=6, prec=prec)
    ref = oracle_f(x, fh, cfg.M, 2.0, 6, window)["f"]
    for exact in (False, True):
        f, plan = run_gpu(bn, torch, x, fh, 1, cfg.M, 2.0, 6, window, prec, exact_taps=exact)
        assert plan.info().tap_poly == (0 if exact else 1)
        assert rel_l2(f, ref) <= TOL[prec]
        plan.close()


def test_tap_fit_check_consistent_for_sharp_shapes(bn, torch):
    """Very sharp sinh windows: whatever the plan-time fit check decides (tap polynomials or the
    exact fallback), the decision matches the reported fit error and parity holds."""
    M, m = 256, 6
    x = synth.make_nodes(synth.CONFIGS[1], N=5000)
    rng = np.random.default_rng(3)
    fh = rng.standard_normal((1, M)) + 1j * rng.standard_normal((1, M))
    for prec, beta in (("c128", 150.0), ("c128", 60.0), ("c64", 60.0)):
        f, plan = run_gpu(bn, torch, x, fh, 1, M, 2.0, m, "sinh", prec, shape=beta)
        info = plan.info()
        tol = 1e-13 if prec == "c128" else 2e-6
        assert info.tap_poly == (1 if info.tap_fit_err <= tol else 0)
        ref = O.algorithm2(x, fh, M, 2.0, m, "sinh", shape=beta)["f"]
        assert rel_l2(f, ref) <= TOL[prec]
        plan.close()


# ----------------------------------------------------------------------------- exactness / determinism
@pytest.mark.parametrize("prec", ["c128", "c64"])
@pytest.mark.parametrize("d", [1, 2, 3])
def test_interpolation_bitwise(bn, torch, d, prec):
    """Grid nodes x = k/L: f_j == theta_k bitwise (u == 0 Kronecker branch)."""
    M, m = 32, 4
    L = O.grid_length(M, 2.0)
    x = synth.grid_point_nodes(3000, d, L, seed=d)
    rng = np.random.default_rng(d)
    fh = rng.standard_normal((1,) + (M,) * d) + 1j * rng.standard_normal((1,) + (M,) * d)
    f, plan = run_gpu(bn, torch, x, fh, d, M, 2.0, m, "sinh", prec)
    g = plan.grid().cpu().numpy()
    idx = tuple((np.round(x * L).astype(int) + L // 2).T)
    assert np.array_equal(f[0], g[(0,) + idx])
    plan.close()


def test_deterministic_and_fft_input_preserved(bn, torch):
    cfg = synth.CONFIGS[4].scaled(M=32, N=30_000)
    x = torch.from_numpy(synth.make_nodes(cfg, variant=3)).cuda()
    a = torch.from_numpy(synth.make_spectrum(cfg, variant=3, prec="c64")).cuda()
    b = torch.from_numpy(synth.make_spectrum(cfg, variant=4, prec="c64")).cuda()
    p1 = bn.Plan(3, 32, 2.0, 4, "sinh", "c64")
    p1.set_nodes(x)
    fa1 = p1.execute(a).clone()
    fb1 = p1.execute(b).clone()
    fa2 = p1.execute(a).clone()
    p2 = bn.Plan(3, 32, 2.0, 4, "sinh", "c64")
    p2.set_nodes(x)
    fb2 = p2.execute(b)
    assert torch.equal(fa1, fa2)
    assert torch.equal(fb1, fb2)
    p1.close()
    p2.close()


def test_transform_host_matches_device(bn, torch):
    cfg = synth.CONFIGS[2].scaled(M=1 << 10, N=20_000)
    x = synth.make_nodes(cfg, variant=5)
    fh = synth.make_spectrum(cfg, variant=5, prec="c64")
    f_dev, plan = run_gpu(bn, torch, x, fh, 1, cfg.M, 2.0, 8, "sinh", "c64")
    xh = torch.from_numpy(x).pin_memory()
    fhh = torch.from_numpy(fh).pin_memory()
    out = torch.empty((1, x.shape[0]), dtype=torch.complex64).pin_memory()
    plan.transform_host(xh, fhh, out)
    assert np.array_equal(out.numpy(), f_dev)
    plan.close()


@pytest.mark.parametrize("d,M,m,prec,N", [(1, 1 << 12, 8, "c64", 50_000), (3, 32, 4, "c64", 60_000),
                                           (2, 64, 5, "c128", 30_000)])
def test_transform_one_call(bn, torch, d, M, m, prec, N):
    """bnfft_transform (grid stage on the side stream, concurrent with the sort): bitwise equal to
    precompute + set_nodes + execute, over repeated calls with changing nodes and spectra; a bad
    node is reported and the plan stays usable."""
    cfg = synth.CONFIGS[{1: 2, 2: 3, 3: 4}[d]].scaled(M=M, N=N)
    dev = torch.device("cuda:0")
    cd = np.complex128 if prec == "c128" else np.complex64
    plan = bn.Plan(d, M, 2.0, m, "sinh", prec)
    ref_plan = bn.Plan(d, M, 2.0, m, "sinh", prec)
    for v in range(3):
        x = synth.make_nodes(cfg, variant=v)[: N - 1000 * v]
        fh = synth.make_spectrum(cfg, variant=v, prec=prec).astype(cd)
        xt = torch.from_numpy(np.ascontiguousarray(x)).to(dev)
        ft = torch.from_numpy(np.ascontiguousarray(fh)).to(dev)
        f1 = plan.transform(xt, ft)
        ref_plan.precompute()
        ref_plan.set_nodes(xt)
        f2 = ref_plan.execute(ft)
        assert torch.equal(f1, f2)
        if v == 0:
            ref = oracle_f(x, fh, M, 2.0, m, "sinh")
            assert rel_l2(f1.cpu().numpy(), ref["f"]) <= TOL[prec]
    xb = x.copy()
    xb[123] = 0.75
    with pytest.raises(bn.BnfftError) as ei:
        plan.transform(torch.from_numpy(xb).to(dev), ft)
    assert ei.value.first_bad == 123
    f1 = plan.transform(xt, ft)
    assert torch.equal(f1, f2)
    plan.close()
    ref_plan.close()


@pytest.mark.parametrize("d", [1, 2, 3])
def test_transform_empty_and_single_node(bn, torch, d):
    """bnfft_transform with n = 0 (nothing written) and n = 1, then a regular node set on the same plan."""
    M, m = (256, 4) if d == 1 else (32, 4)
    cfg = synth.CONFIGS[{1: 2, 2: 3, 3: 4}[d]].scaled(M=M, N=5000, m=m)
    dev = torch.device("cuda:0")
    fh = synth.make_spectrum(cfg, variant=2, prec="c64")
    ft = torch.from_numpy(fh).to(dev)
    x = synth.make_nodes(cfg, variant=2)
    plan = bn.Plan(d, M, 2.0, m, "sinh", "c64")
    f0 = plan.transform(torch.empty((0, d), dtype=torch.float64, device=dev), ft)
    assert f0.shape == (1, 0)
    f1 = plan.transform(torch.from_numpy(x[:1].copy()).to(dev), ft).cpu().numpy()
    fa = plan.transform(torch.from_numpy(x).to(dev), ft).cpu().numpy()
    ref = oracle_f(x, fh, M, 2.0, m, "sinh")["f"]
    assert rel_l2(fa, ref) <= TOL["c64"]
    assert abs(f1[0, 0] - ref[0, 0]) <= 1e-5 * np.abs(ref).max()
    plan.close()


@pytest.mark.parametrize("d,M,m,prec", [(1, 1 << 10, 8, "c64"), (3, 16, 4, "c64"), (2, 32, 5, "c128")])
def test_transform_host_many_pipelined(bn, torch, d, M, m, prec):
    """bnfft_transform_host_many: five steps with different node sets and spectra, each equal bitwise
    to the device path (set_nodes + execute) on the same inputs; a bad node in one step is reported
    with its step-local index."""
    cid = {1: 2, 2: 3, 3: 4}[d]
    cfg = synth.CONFIGS[cid].scaled(d=d, M=M, N=3001, batch=1)
    K = 5
    xs = [synth.make_nodes(cfg, variant=20 + k) for k in range(K)]
    fhs = [synth.make_spectrum(cfg, variant=20 + k, prec=prec) for k in range(K)]
    ct = torch.complex128 if prec == "c128" else torch.complex64
    plan = bn.Plan(d, M, 2.0, m, "sinh", prec)
    ref = []
    for k in range(K):
        plan.set_nodes(torch.from_numpy(xs[k]).cuda())
        ref.append(plan.execute(torch.from_numpy(fhs[k]).cuda()).cpu().numpy())
    xh = [torch.from_numpy(x).pin_memory() for x in xs]
    fhh = [torch.from_numpy(f).pin_memory() for f in fhs]
    outs = [torch.empty((1, cfg.N), dtype=ct).pin_memory() for _ in range(K)]
    plan.transform_host_many(xh, fhh, outs)
    for k in range(K):
        assert np.array_equal(outs[k].numpy(), ref[k]), k
    bad = [x.copy() for x in xs[:3]]
    bad[2][77, 0] = 0.5                      # outside [-1/2, 1/2): BNFFT_E_NODE_OUT_OF_RANGE
    with pytest.raises(bn.BnfftError) as ei:
        plan.transform_host_many([torch.from_numpy(x).pin_memory() for x in bad], fhh[:3], outs[:3])
    assert ei.value.code == -8 and ei.value.first_bad == 77
    plan.close()


# ----------------------------------------------------------------------------- edge cases
def test_empty_and_tiny_node_sets(bn, torch):
    plan = bn.Plan(2, 16, 2.0, 3, "sinh", "c128")
    plan.set_nodes(torch.empty((0, 2), dtype=torch.float64, device="cuda"))
    fh = torch.ones((1, 16, 16), dtype=torch.complex128, device="cuda")
    assert plan.execute(fh).shape == (1, 0)
    for n in (1, 2, 255, 256, 257, 4097):
        x = synth.feasible_box_nodes(n, 2, 32, 3, seed=n)
        plan.set_nodes(torch.from_numpy(x).cuda())
        f = plan.execute(fh).cpu().numpy()
        ref = O.algorithm2(x, fh.cpu().numpy(), 16, 2.0, 3)["f"]
        assert rel_l2(f, ref) <= 1e-12
    plan.close()


def test_boundary_and_identical_nodes(bn, torch):
    M, m = 64, 5
    x = np.array([[-0.5], [-0.5], [0.5 - 2 ** -53], [0.0], [0.0], [0.25], [-0.25 + 1e-17]])
    x = np.concatenate([x, np.zeros((3000, 1)), synth.make_nodes(synth.CONFIGS[1], N=2000)])
    fh = synth.make_spectrum(synth.CONFIGS[1])
    f, plan = run_gpu(bn, torch, x, fh, 1, M, 2.0, m, "sinh", "c128")
    ref = O.algorithm2(x, fh, M, 2.0, m)["f"]
    assert np.max(np.abs(f - ref)) <= 1e-12 * np.max(np.abs(ref))
    plan.close()


def test_non_power_of_two_grid(bn, torch):
    """sigma = 1.5 and M = 20: L = 30; fl(L x) may round to L/2 for x < 1/2."""
    M, m = 20, 3
    L = O.grid_length(M, 1.5)
    assert L == 30
    x = np.concatenate([synth.make_nodes(synth.CONFIGS[1], N=3000), [[np.nextafter(0.5, 0)]]])
    rng = np.random.default_rng(8)
    fh = rng.standard_normal((1, M)) + 1j * rng.standard_normal((1, M))
    f, plan = run_gpu(bn, torch, x, fh, 1, M, 1.5, m, "sinh", "c128")
    ref = O.algorithm2(x, fh, M, 1.5, m)["f"]
    assert np.max(np.abs(f - ref)) <= 1e-12 * np.max(np.abs(ref))
    plan.close()


def test_invalid_nodes_report_first_bad(bn, torch):
    plan = bn.Plan(2, 16, 2.0, 3, "sinh", "c64", strict=False)
    x = synth.feasible_box_nodes(5000, 2, 32, 3)
    for idx, val, code in ((4000, np.nan, bn.BNFFT_E_NODE_NOT_FINITE),
                           (17, 0.5, bn.BNFFT_E_NODE_OUT_OF_RANGE),
                           (333, -0.5000001, bn.BNFFT_E_NODE_OUT_OF_RANGE),
                           (2, np.inf, bn.BNFFT_E_NODE_NOT_FINITE)):
        xb = x.copy()
        xb[idx, 1] = val
        xb[idx + 100, 0] = val
        with pytest.raises(bn.BnfftError) as ei:
            plan.set_nodes(torch.from_numpy(xb).cuda())
        assert ei.value.code == code and ei.value.first_bad == idx
    with pytest.raises(bn.BnfftError) as ei:
        plan.execute(torch.zeros((1, 16, 16), dtype=torch.complex64, device="cuda"))
    assert ei.value.code == bn.BNFFT_E_NODES_NOT_SET
    plan.close()
    strict = bn.Plan(1, 16, 2.0, 3, "sinh", "c64", strict=True)
    xs = np.array([[0.0], [0.5 - 3 / 32], [0.41], [-0.45]])
    with pytest.raises(bn.BnfftError) as ei:
        strict.set_nodes(torch.from_numpy(xs).cuda())
    assert ei.value.code == bn.BNFFT_E_NODE_OUTSIDE_FEASIBLE_BOX and ei.value.first_bad == 2
    strict.set_nodes(torch.from_numpy(xs[:2]).cuda())        # closed box accepted
    strict.close()


def test_reset_nodes_grow_and_shrink(bn, torch):
    cfg = synth.CONFIGS[3].scaled(M=64, N=1)
    plan = bn.Plan(2, 64, 2.0, 6, "sinh", "c64")
    fh = synth.make_spectrum(cfg, prec="c64")
    ft = torch.from_numpy(fh).cuda()
    for n in (10_000, 50_000, 3_000):
        x = synth.make_nodes(cfg, N=n, variant=n)
        plan.set_nodes(torch.from_numpy(x).cuda())
        f = plan.execute(ft).cpu().numpy()
        assert rel_l2(f, O.algorithm2(x, fh.astype(np.complex128), 64, 2.0, 6)["f"]) <= 1e-5
    plan.close()


@pytest.mark.parametrize("cid,d,M,N,prec", [(2, 1, 1 << 12, 100_001, "c64"), (3, 2, 128, 40_000, "c128"),
                                           (4, 3, 32, 30_000, "c64")])
def test_shards_bitwise(bn, torch, cid, d, M, N, prec):
    """Node sharding (the multi-GPU layout): plans over disjoint node shards with the
    same spectrum reproduce the single-plan result bitwise (per-node work is independent)."""
    from paper_2502_07155_b200 import shard
    cfg = synth.CONFIGS[cid].scaled(d=d, M=M, N=N)
    x = torch.from_numpy(synth.make_nodes(cfg, variant=9)).cuda()
    fh = torch.from_numpy(synth.make_spectrum(cfg, variant=9, prec=prec)).cuda()
    full = bn.Plan(d, M, 2.0, cfg.m, "sinh", prec)
    full.set_nodes(x)
    ref = full.execute(fh).clone()
    parts = []
    for r in range(3):
        a, b = shard.node_shard(N, r, 3)
        p = bn.Plan(d, M, 2.0, cfg.m, "sinh", prec)
        p.set_nodes(x[a:b].contiguous())
        parts.append(p.execute(fh).clone())
        p.close()
    assert torch.equal(torch.cat(parts, dim=1), ref)
    full.close()


# ----------------------------------------------------------------------------- step 0(b): PRECOMPUTE_PSI
@pytest.mark.parametrize("prec,m,window,exact", [("c64", 4, "sinh", False), ("c128", 5, "sinh", False),
                                                 ("c64", 3, "gauss", False), ("c64", 7, "ckb", True),
                                                 ("c128", 2, "sinh", False)])
def test_precompute_psi(bn, torch, prec, m, window, exact):
    """BNFFT_PRECOMPUTE_PSI (Algorithm 2 step 0(b)): the stored per-node weights are the same
    numbers the gather evaluates on the fly, so the result equals the default path bitwise and meets
    parity with the oracle; odd m exercises the 16-byte row padding."""
    cfg = synth.CONFIGS[2].scaled(M=1 << 11, m=m, N=70_001)
    x = synth.make_nodes(cfg, variant=11)
    fh = synth.make_spectrum(cfg, variant=11, prec=prec)
    ref = oracle_f(x, fh, cfg.M, 2.0, m, window)["f"]
    f0, p0 = run_gpu(bn, torch, x, fh, 1, cfg.M, 2.0, m, window, prec, exact_taps=exact)
    f1, p1 = run_gpu(bn, torch, x, fh, 1, cfg.M, 2.0, m, window, prec, exact_taps=exact, precompute_psi=True)
    assert np.array_equal(f0, f1)
    assert rel_l2(f1, ref) <= TOL[prec]
    # new nodes (fewer, then more) recompute the table
    for n, v in ((5_003, 12), (90_001, 13)):
        xn = synth.make_nodes(cfg, N=n, variant=v)
        p1.set_nodes(torch.from_numpy(xn).cuda())
        ft = torch.from_numpy(fh.astype(np.complex128 if prec == "c128" else np.complex64)).cuda()
        fn = p1.execute(ft).cpu().numpy()
        assert rel_l2(fn, oracle_f(xn, fh, cfg.M, 2.0, m, window)["f"]) <= TOL[prec]
    p0.close()
    p1.close()


def test_precompute_psi_unsupported(bn):
    for d, batch in ((2, 1), (3, 1), (1, 4)):
        with pytest.raises(bn.BnfftError) as ei:
            bn.Plan(d, 64, 2.0, 4, "sinh", "c64", batch=batch, precompute_psi=True)
        assert ei.value.code == bn.BNFFT_E_UNSUPPORTED


def test_precompute_side_stream_join(bn, torch):
    """Step 0(a) runs on the plan's side stream: a precompute issued right before execute (and a
    psihat read right after it) must see the finished quadrature (fork/join ordering)."""
    cfg = synth.CONFIGS[2].scaled(M=1 << 16, m=8, N=200_003)
    x = torch.from_numpy(synth.make_nodes(cfg, variant=31)).cuda()
    fh = torch.from_numpy(synth.make_spectrum(cfg, variant=31, prec="c64")).cuda()
    plan = bn.Plan(1, cfg.M, 2.0, 8, "sinh", "c64")
    plan.set_nodes(x)
    ref = plan.execute(fh).clone()
    ph0 = plan.psihat().copy()
    for _ in range(3):
        plan.precompute()
        assert torch.equal(plan.execute(fh), ref)
        plan.precompute()
        assert np.array_equal(plan.psihat(), ph0)
    plan.close()
