"""GPU parity for the round-2 paths, through the C ABI against the CPU oracle:

* the d = 3, m = 4, complex64 gathers (y-sweep gather3y, the default; z-sweep gather3s): clustered
  node sets that overflow a bin's stash or an x-line's chunk, many nodes in one cell, grid nodes
  (Kronecker case), the global grid ends, sparse node sets, several grid sizes, and the half-warp
  kernel gather3c (BNFFT_GATHER3C) and the half-height y-sweep gather3q (BNFFT_GATHER3Q) as further
  witnesses;
* the d = 2 complex64 quarter-warp kernel gather2c (m <= 7) and gatherN (BNFFT_GATHER2N, m = 8): cfg3's
  mixed node recipe, grid nodes, the grid ends, one cell;
* the NCCL transport's self-test on a one-rank communicator;
* BNFFT_SORTED_OUTPUT: f_sorted[i] == f_user[perm[i]] bitwise;
* repeated executes on d = 2 and d = 3 plans are bitwise equal (the FFT input's zero padding is
  written once at plan creation);
* multi-rank execution with the in-process transport (one thread per rank on this GPU):
  BNFFT_DIST_REPLICATE is bitwise equal to one rank; BNFFT_DIST_SLAB (distributed slab FFT,
  halo exchange, node redistribution, output return) matches the oracle at the complex64 /
  complex128 tolerances, with equal and node-balanced cut points.
Tolerances: BASELINE.json north_star (rel. l2 1e-5 complex64, 1e-12 complex128)."""
import os
import threading

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


def cdt(prec):
    return np.complex128 if prec == "c128" else np.complex64


def gpu_run(bn, torch, x, fh, M, m, prec, window="sinh", **kw):
    dev = torch.device("cuda:0")
    d = x.shape[1]
    plan = bn.Plan(d, M, 2.0, m, window, prec, batch=fh.shape[0], **kw)
    plan.set_nodes(torch.from_numpy(np.ascontiguousarray(x)).to(dev))
    f = plan.execute(torch.from_numpy(np.ascontiguousarray(fh.astype(cdt(prec)))).to(dev)).cpu().numpy()
    return f, plan


def oracle_f(x, fh, M, m, window="sinh"):
    return O.algorithm2(x, fh.astype(np.complex128), M, 2.0, m, window)["f"]


# ----------------------------------------------------------------------------- d = 3, m = 4 gathers
# Three kernels serve d = 3, m = 4, complex64, batch 1 (chosen at plan creation): the y-sweep kernel
# gather3y (default: x-line bins of 1 x 16 x 8 cells, rows in registers), the half-warp kernel gather3c
# (BNFFT_GATHER3C) and the z-sweep kernel gather3s (BNFFT_GATHER3S), both on 8 x 8 x 16-cell bins.
def _sweep_inputs(kind, M, N, seed):
    rng = np.random.default_rng(seed)
    L = 2 * M
    if kind == "uniform":
        x = rng.random((N, 3)) - 0.5
    elif kind == "one_bin":            # every node in one 8x8x16-cell bin: chunked bins / x-lines
        x = (rng.random((N, 3)) * np.array([8, 8, 16]) + np.array([3, -20, 5])) / L
    elif kind == "one_xline":          # every node in one 1x16x8-cell x-line: > CAP nodes, chunks
        x = (rng.random((N, 3)) * np.array([1, 16, 8]) + np.array([5, -16, 8])) / L
    elif kind == "one_cell":           # all nodes in one cell: one column, one z step
        x = (rng.random((N, 3)) + np.array([-7, 2, 11])) / L
    elif kind == "grid_nodes":         # Kronecker case u == 0 in every dimension
        x = rng.integers(-L // 2, L // 2, size=(N, 3)).astype(np.float64) / L
    elif kind == "edges":              # near the global grid ends (zero extension, reading A5)
        x = rng.random((N, 3)) - 0.5
        x[: N // 2, 0] = -0.5 + rng.random(N // 2) * 3 / L
        x[N // 2:, 2] = 0.5 - rng.random(N - N // 2) * 3 / L
    elif kind == "sparse":             # a few nodes: most items and x-lines empty
        x = rng.random((N, 3)) - 0.5
    else:
        raise ValueError(kind)
    return np.clip(x, -0.5, np.nextafter(0.5, 0))


KERNEL3 = {"y": ("gather3y_kernel", None), "c": ("gather3c_kernel", "BNFFT_GATHER3C"),
           "s": ("gather3s_kernel", "BNFFT_GATHER3S"), "q": ("gather3q_kernel", "BNFFT_GATHER3Q")}


def _use_kernel3(monkeypatch, which):
    monkeypatch.delenv("BNFFT_GATHER3C", raising=False)
    monkeypatch.delenv("BNFFT_GATHER3S", raising=False)
    monkeypatch.delenv("BNFFT_GATHER3Q", raising=False)
    env = KERNEL3[which][1]
    if env:
        monkeypatch.setenv(env, "1")


@pytest.mark.parametrize("which", ["y", "s", "q"])
@pytest.mark.parametrize("kind", ["uniform", "one_bin", "one_xline", "one_cell", "grid_nodes", "edges", "sparse"])
def test_sweep3_parity(bn, torch, kind, which, monkeypatch):
    M, m = 32, 4
    N = {"uniform": 40_003, "one_xline": 700, "sparse": 17}.get(kind, 3000)
    x = _sweep_inputs(kind, M, N, 11)
    cfg = synth.CONFIGS[4].scaled(M=M, N=N)
    fh = synth.make_spectrum(cfg, variant=3, prec="c64")
    _use_kernel3(monkeypatch, which)
    f, plan = gpu_run(bn, torch, x, fh, M, m, "c64")
    assert bn.GATHER_KERNELS[plan.info().gather_kernel].endswith(KERNEL3[which][0])
    ref = oracle_f(x, fh, M, m)
    assert rel_l2(f, ref) <= TOL["c64"]
    if kind == "grid_nodes":   # interpolation property: f_j == theta at the node's cell
        g = plan.grid().cpu().numpy()[0]
        L = 2 * M
        c = np.floor(L * x).astype(np.int64) + L // 2
        assert np.array_equal(f[0], g[c[:, 0], c[:, 1], c[:, 2]])
    plan.close()


@pytest.mark.parametrize("which", ["y", "q"])
@pytest.mark.parametrize("M", [8, 24, 32])
def test_ysweep3_grid_sizes(bn, torch, M, which, monkeypatch):
    """L = 16 (one item), L = 48 (partial y bins and a partial 8-x-line item), L = 64."""
    m, N = 4, 5000
    x = _sweep_inputs("uniform", M, N, 13)
    cfg = synth.CONFIGS[4].scaled(M=M, N=N)
    fh = synth.make_spectrum(cfg, variant=5, prec="c64")
    _use_kernel3(monkeypatch, which)
    f, plan = gpu_run(bn, torch, x, fh, M, m, "c64")
    assert bn.GATHER_KERNELS[plan.info().gather_kernel].endswith(KERNEL3[which][0])
    assert rel_l2(f, oracle_f(x, fh, M, m)) <= TOL["c64"]
    plan.close()


def test_sweep3_kernels_agree(bn, torch, monkeypatch):
    """The three d = 3, m = 4 kernels on the same inputs: each within tolerance of the oracle and
    within 1e-6 of each other."""
    M, m, N = 32, 4, 20_001
    cfg = synth.CONFIGS[4].scaled(M=M, N=N)
    x = synth.make_nodes(cfg, variant=2)
    fh = synth.make_spectrum(cfg, variant=2, prec="c64")
    ref = oracle_f(x, fh, M, m)
    res = {}
    for which in ("y", "c", "s"):
        _use_kernel3(monkeypatch, which)
        f, p = gpu_run(bn, torch, x, fh, M, m, "c64")
        assert bn.GATHER_KERNELS[p.info().gather_kernel].endswith(KERNEL3[which][0])
        assert rel_l2(f, ref) <= TOL["c64"], which
        res[which] = f
        p.close()
    assert rel_l2(res["y"], res["c"]) <= 1e-6 and rel_l2(res["s"], res["c"]) <= 1e-6


@pytest.mark.parametrize("which", ["y", "s"])
def test_sweep3_repeat_bitwise(bn, torch, which, monkeypatch):
    M, m, N = 32, 4, 30_000
    cfg = synth.CONFIGS[4].scaled(M=M, N=N)
    x = synth.make_nodes(cfg, variant=4)
    fh = synth.make_spectrum(cfg, variant=4, prec="c64")
    _use_kernel3(monkeypatch, which)
    f1, plan = gpu_run(bn, torch, x, fh, M, m, "c64")
    ft = torch.from_numpy(fh).to("cuda:0")
    for _ in range(3):
        assert np.array_equal(plan.execute(ft).cpu().numpy(), f1)
    # a permuted copy of the node set gives the same value per node, bitwise (in-bin order free)
    perm = np.random.default_rng(5).permutation(N)
    plan.set_nodes(torch.from_numpy(np.ascontiguousarray(x[perm])).to("cuda:0"))
    assert np.array_equal(plan.execute(ft).cpu().numpy()[0], f1[0][perm])
    plan.close()
# ----------------------------------------------------------------------------- sorted output
@pytest.mark.parametrize("d,M,m,prec", [(1, 1 << 12, 8, "c64"), (1, 1 << 16, 8, "c128"), (2, 64, 6, "c64"),
                                        (3, 32, 4, "c64"), (3, 16, 3, "c128")])
def test_sorted_output(bn, torch, d, M, m, prec):
    N = 20_011
    cfg = synth.CONFIGS[{1: 2, 2: 3, 3: 4}[d]].scaled(d=d, M=M, m=m, N=N)
    x = synth.make_nodes(cfg, variant=5)
    fh = synth.make_spectrum(cfg, variant=5, prec=prec)
    fu, pu = gpu_run(bn, torch, x, fh, M, m, prec)
    fs, ps = gpu_run(bn, torch, x, fh, M, m, prec, sorted_output=True)
    perm = ps.perm().cpu().numpy().astype(np.int64)
    assert np.array_equal(np.sort(perm), np.arange(N))
    assert np.array_equal(fs[0], fu[0][perm])
    pu.close()
    ps.close()


# ----------------------------------------------------------------------------- repeated executes
@pytest.mark.parametrize("d,M,m,prec", [(2, 128, 6, "c64"), (2, 64, 5, "c128"), (3, 32, 4, "c64"),
                                        (3, 16, 4, "c128")])
def test_repeat_execute_bitwise(bn, torch, d, M, m, prec):
    N = 10_007
    cfg = synth.CONFIGS[{2: 3, 3: 4}[d]].scaled(d=d, M=M, m=m, N=N)
    x = synth.make_nodes(cfg, variant=6)
    fh = synth.make_spectrum(cfg, variant=6, prec=prec)
    fh2 = synth.make_spectrum(cfg, variant=7, prec=prec)
    f1, plan = gpu_run(bn, torch, x, fh, M, m, prec)
    dev = torch.device("cuda:0")
    a, b = torch.from_numpy(fh).to(dev), torch.from_numpy(fh2).to(dev)
    f2 = plan.execute(b).cpu().numpy()          # another spectrum in between
    assert np.array_equal(plan.execute(a).cpu().numpy(), f1)
    assert np.array_equal(plan.execute(b).cpu().numpy(), f2)
    assert rel_l2(f1, oracle_f(x, fh, M, m)) <= TOL[prec]
    plan.close()


# ----------------------------------------------------------------------------- multi-rank
def run_ranks(bn, torch, P, x_parts, fh, M, m, prec, dist, **kw):
    """P ranks of one in-process group, each in its own thread with its own stream."""
    grp = bn.Group(P)
    out, errs = [None] * P, []
    info = [None] * P

    def worker(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                plan = bn.Plan(3, M, 2.0, m, "sinh", prec, device=0, stream=st.cuda_stream, rank=r, nranks=P,
                               local_group=grp.handle, dist=dist, **kw)
                xd = torch.from_numpy(np.ascontiguousarray(x_parts[r])).to("cuda:0")
                plan.set_nodes(xd)
                fd = torch.from_numpy(np.ascontiguousarray(fh.astype(cdt(prec)))).to("cuda:0")
                o = torch.empty((1, len(x_parts[r])), dtype=plan.cdtype, device="cuda:0")
                plan.execute(fd, o)
                plan.execute(fd, o)    # twice: buffers reused across executes
                st.synchronize()
                out[r] = o.cpu().numpy()
                info[r] = plan.info()
                plan.close()
        except Exception as e:   # pragma: no cover - reported below
            errs.append((r, repr(e)))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    grp.close()
    assert not errs, errs
    return out, info


@pytest.mark.parametrize("P,prec,balanced,kind", [(2, "c64", False, "uniform"), (4, "c64", False, "uniform"),
                                                  (4, "c64", True, "mixed"), (2, "c128", False, "uniform"),
                                                  (3, "c64", True, "mixed")])
def test_slab_ranks(bn, torch, P, prec, balanced, kind):
    M, m, N = 32, 4, 24_011
    L = 2 * M
    rng = np.random.default_rng(17 + P)
    if kind == "uniform":
        x = rng.random((N, 3)) - 0.5
    else:   # half uniform, half clustered in the second coordinate (unbalanced slabs)
        x = rng.random((N, 3)) - 0.5
        x[N // 2:, 1] = np.clip(0.05 * rng.standard_normal(N - N // 2), -0.5, 0.49)
    cfg = synth.CONFIGS[4].scaled(M=M, N=N)
    fh = synth.make_spectrum(cfg, variant=8, prec=prec)
    cuts = np.linspace(0, N, P + 1).astype(int)
    parts = [x[cuts[r]:cuts[r + 1]] for r in range(P)]
    out, info = run_ranks(bn, torch, P, parts, fh, M, m, prec, "slab", balanced_slabs=balanced)
    f = np.concatenate([o[0] for o in out])
    ref = oracle_f(x, fh, M, m)
    assert rel_l2(f, ref) <= TOL[prec]
    lo = [i.slab_lo for i in info]
    hi = [i.slab_hi for i in info]
    assert lo[0] == 0 and hi[-1] == L and all(hi[r] == lo[r + 1] for r in range(P - 1))
    owned = sum(i.n_owned for i in info)
    assert owned == N
    # every rank received m-1 planes from below and m from above, except at the global ends
    cs = 16 if prec == "c128" else 8
    for r, i in enumerate(info):
        exp = ((m - 1) if r > 0 else 0) + (m if r < P - 1 else 0)
        assert i.halo_bytes == exp * L * L * cs
    # cut points: the library's host rule (bnfft_slab_cuts) on the whole node set's plane histogram
    # must equal what the ranks agreed on from their device histograms (all-gathered)
    c = np.minimum(np.floor(L * x[:, 1]).astype(np.int64) + L // 2, L - 1)
    hist = np.bincount(c, minlength=L)
    align = 1 << info[0].bin_log2[1]      # cut points are whole bins of the sort (row a1)
    exp = bn.slab_cuts(L, P, align, hist if balanced else None)
    assert lo + [hi[-1]] == list(exp)
    assert [i.n_owned for i in info] == [int(hist[exp[r]:exp[r + 1]].sum()) for r in range(P)]


def test_replicate_ranks_bitwise(bn, torch):
    M, m, N, P = 32, 4, 20_000, 3
    cfg = synth.CONFIGS[4].scaled(M=M, N=N)
    x = synth.make_nodes(cfg, variant=9)
    fh = synth.make_spectrum(cfg, variant=9, prec="c64")
    f1, p1 = gpu_run(bn, torch, x, fh, M, m, "c64")
    p1.close()
    cuts = np.linspace(0, N, P + 1).astype(int)
    out, _ = run_ranks(bn, torch, P, [x[cuts[r]:cuts[r + 1]] for r in range(P)], fh, M, m, "c64", "replicate")
    assert np.array_equal(np.concatenate([o[0] for o in out]), f1[0])


def test_slab_rejects_bad_node_on_all_ranks(bn, torch):
    M, m, P = 16, 4, 2
    x = np.random.default_rng(3).random((1000, 3)) - 0.5
    x[700, 2] = 0.75
    grp = bn.Group(P)
    codes = [None] * P

    def worker(r):
        torch.cuda.set_device(0)
        st = torch.cuda.Stream()
        plan = bn.Plan(3, M, 2.0, m, "sinh", "c64", device=0, stream=st.cuda_stream, rank=r, nranks=P,
                       local_group=grp.handle, dist="slab")
        try:
            plan.set_nodes(torch.from_numpy(np.ascontiguousarray(x[500 * r:500 * (r + 1)])).to("cuda:0"))
            codes[r] = 0
        except bn.BnfftError as e:
            codes[r] = (e.code, getattr(e, "first_bad", None))
        plan.close()

    th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
    [t.start() for t in th]
    [t.join(timeout=120) for t in th]
    grp.close()
    assert codes[1] == (bn.BNFFT_E_NODE_OUT_OF_RANGE, 200)
    assert codes[0][0] == bn.BNFFT_E_NODE_OUT_OF_RANGE and codes[0][1] == -1


# ----------------------------------------------------------------------------- NCCL transport
def test_nccl_transport_selftest(bn, torch):
    """The library's NCCL transport (run-time libnccl, communicator init, grouped ncclSend/ncclRecv
    exchange, host all-gather) on a one-rank communicator: every call the slab path makes over NCCL,
    with this rank as its own peer (NCCL refuses two ranks on one GPU, so more ranks need more GPUs;
    the slab logic itself runs over the in-process transport above)."""
    torch.cuda.set_device(0)
    torch.zeros(1, device="cuda:0")
    comm = bn.nccl_comm_init(bn.nccl_unique_id(), 1, 0, 0)
    try:
        for nbytes in (1, 4096, (1 << 22) + 3):
            bn.nccl_selftest(comm, nbytes, torch.cuda.current_stream().cuda_stream)
    finally:
        bn.nccl_comm_destroy(comm)


# ----------------------------------------------------------------------------- d = 2 cooperative gather
@pytest.mark.parametrize("m", [1, 2, 4, 6, 7, 8])
@pytest.mark.parametrize("kind", ["mixed", "grid_nodes", "edges", "one_cell"])
def test_gather2c_parity(bn, torch, m, kind, monkeypatch):
    """d = 2 complex64: the quarter-warp kernel gather2c (m <= 7; gatherN beyond) against the oracle and,
    bitwise for Kronecker nodes, against theta; BNFFT_GATHER2N selects gatherN."""
    M, N = 64, 20_011
    L = 2 * M
    rng = np.random.default_rng(100 + m)
    if kind == "mixed":          # cfg3's recipe: half uniform, half clustered around the origin
        x = rng.random((N, 2)) - 0.5
        x[N // 2:] = np.clip(0.05 * rng.standard_normal((N - N // 2, 2)), -0.5, 0.49)
    elif kind == "grid_nodes":
        x = rng.integers(-L // 2, L // 2, size=(N, 2)).astype(np.float64) / L
    elif kind == "edges":        # windows reaching past the grid ends (zero extension, reading A5)
        x = rng.random((N, 2)) - 0.5
        x[: N // 2, 0] = -0.5 + rng.random(N // 2) * 3 / L
        x[N // 2:, 1] = 0.5 - rng.random(N - N // 2) * 3 / L
    else:                        # one cell: every batch reads the same window
        x = (rng.random((3000, 2)) + np.array([-7, 21])) / L
    x = np.clip(x, -0.5, np.nextafter(0.5, 0))
    cfg = synth.CONFIGS[3].scaled(M=M, N=len(x), m=m)
    fh = synth.make_spectrum(cfg, variant=4, prec="c64")
    dev = torch.device("cuda:0")
    xt, ft = torch.from_numpy(x).to(dev), torch.from_numpy(fh).to(dev)
    plan = bn.Plan(2, M, 2.0, m, "sinh", "c64")
    want = "gather2c_kernel" if m <= 7 else "gatherN_kernel"
    assert bn.GATHER_KERNELS[plan.info().gather_kernel].endswith(want)
    plan.set_nodes(xt)
    f = plan.execute(ft).cpu().numpy()
    ref = O.algorithm2(x, fh.astype(np.complex128), M, 2.0, m, "sinh")["f"]
    assert rel_l2(f, ref) <= TOL["c64"]
    if kind == "grid_nodes":     # interpolation property
        g = plan.grid().cpu().numpy()[0]
        c = np.floor(L * x).astype(np.int64) + L // 2
        assert np.array_equal(f[0], g[c[:, 0], c[:, 1]])
    plan.close()
    monkeypatch.setenv("BNFFT_GATHER2N", "1")
    plan = bn.Plan(2, M, 2.0, m, "sinh", "c64")
    assert bn.GATHER_KERNELS[plan.info().gather_kernel].endswith("gatherN_kernel")
    plan.set_nodes(xt)
    assert rel_l2(plan.execute(ft).cpu().numpy(), ref) <= TOL["c64"]
    plan.close()


def test_gather3q_sort_bit_exact(bn, torch, monkeypatch):
    """The gather3q plan's sort key (bin, (z half, y column)) as documented in include/bnfft.h: the
    permutation and the key offsets equal the oracle's stable sort bit for bit."""
    M, N = 64, 50_000
    cfg = synth.CONFIGS[4].scaled(M=M, N=N)
    x = synth.make_nodes(cfg, variant=2)
    x[:300] = 0.0   # a run of identical keys (ties by user index)
    _use_kernel3(monkeypatch, "q")
    plan = bn.Plan(3, M, 2.0, 4, "sinh", "c64")
    plan.set_nodes(torch.from_numpy(x).cuda())
    info = plan.info()
    assert int(info.key_col_bits) == 5
    cells = np.minimum(O.cell_index(x, info.L), info.L - 1)
    key = np.zeros(N, dtype=np.int64)
    for t in range(3):
        key = key * info.bins_per_dim[t] + (cells[:, t] >> info.bin_log2[t])
    minor = (((cells[:, 2] >> 2) & 1) << 4) | (cells[:, 1] & 15)
    perm_ref, _ = O.stable_bin_sort(key * 32 + minor, int(info.nkeys) << 5)
    _, off_ref = O.stable_bin_sort(key, int(info.nkeys))
    assert np.array_equal(plan.perm().cpu().numpy().astype(np.int64), perm_ref)
    assert np.array_equal(plan.bin_offsets().cpu().numpy().astype(np.int64), off_ref)
    plan.close()


@pytest.mark.parametrize("M,m", [(4, 2), (14, 4), (8, 7), (24, 6)])
def test_gather2c_small_grids(bn, torch, M, m):
    """d = 2 grids smaller than or not a multiple of the 16-cell bins (L = 8, 28, 16, 48): partial bins,
    windows mostly outside the grid (zero extension, reading A5)."""
    N = 4001
    rng = np.random.default_rng(7 * M + m)
    x = np.clip(rng.random((N, 2)) - 0.5, -0.5, np.nextafter(0.5, 0))
    cfg = synth.CONFIGS[3].scaled(M=M, N=N, m=m)
    fh = synth.make_spectrum(cfg, variant=6, prec="c64")
    dev = torch.device("cuda:0")
    plan = bn.Plan(2, M, 2.0, m, "sinh", "c64")
    assert bn.GATHER_KERNELS[plan.info().gather_kernel].endswith("gather2c_kernel")
    f = plan.transform(torch.from_numpy(x).to(dev), torch.from_numpy(fh).to(dev)).cpu().numpy()
    ref = O.algorithm2(x, fh.astype(np.complex128), M, 2.0, m, "sinh")["f"]
    assert rel_l2(f, ref) <= TOL["c64"]
    plan.close()
