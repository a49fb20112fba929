"""Multi-rank host logic on CPU: world_size-2 gloo process group (no GPU).

The product path shards nodes across ranks with a replicated grid.  These tests cover
the shard split, the max-over-ranks timing reduction and the aggregate rate, and check with the CPU
oracle that Algorithm 2's step 3 is per-node independent: evaluating two shards separately and
concatenating reproduces the unsharded result bitwise."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2502_07155_b200 import shard


def test_node_shard_partition():
    for n in (0, 1, 7, 1000, 2 ** 20 + 3):
        for world in (1, 2, 3, 8):
            spans = [shard.node_shard(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard.node_shard(10, 2, 2)


def test_aggregate_rate():
    assert shard.aggregate_rate(1000, 4, 2.0) == pytest.approx(2e6)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    import oracle as O
    import synth
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        # timing reduction
        t = shard.max_over_ranks(1.5 + rank)
        # node-parallel evaluation of one shard with the (replicated) grid
        cfg = synth.CONFIGS[3].scaled(M=32, N=2001)
        x = synth.make_nodes(cfg)
        fh = synth.make_spectrum(cfg)
        L = O.grid_length(cfg.M, cfg.sigma)
        shape = O.default_shape("sinh", cfg.m, cfg.M, L)
        theta = O.step2_inverse_fft(O.step1_deconvolve_pad(
            fh, O.psihat_multi(O.psihat_table("sinh", cfg.M, cfg.m, L, shape), cfg.d), L))
        a, b = shard.node_shard(len(x), rank, world)
        f = O.step3_short_sums(theta, x[a:b], "sinh", cfg.m, shape)
        parts = [None] * world
        dist.all_gather_object(parts, (a, b, f))
        if rank == 0:
            full = O.step3_short_sums(theta, x, "sinh", cfg.m, shape)
            cat = np.concatenate([p[2] for p in sorted(parts, key=lambda z: z[0])], axis=1)
            q.put((t, bool(np.array_equal(cat, full))))
        else:
            q.put((t, True))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharding():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(t == 2.5 for t, _ in res)          # max over ranks of 1.5 + rank
    assert all(ok for _, ok in res)


def test_reference_arm_nonzero_rank_is_silent(capsys, monkeypatch):
    """Under torchrun only rank 0 runs the CPU reference arm; other ranks exit 0 without output."""
    import bench
    monkeypatch.setenv("RANK", "1")
    args = type("A", (), dict(gpus=2, steps=1, warmup=0, impl="reference", cfg=1, prec=None,
                              window=None, N=None))()
    assert bench.run_reference(args) == 0
    assert capsys.readouterr().out == ""


# ----------------------------------------------------------------------------- library partition logic
def test_slab_cuts_equal_and_balanced():
    from paper_2502_07155_b200 import bnfft as bn
    for L, P, align in ((512, 8, 8), (64, 3, 8), (512, 5, 16), (100, 4, 8)):
        cuts = bn.slab_cuts(L, P, align)
        assert cuts[0] == 0 and cuts[-1] == L
        assert all(c % align == 0 for c in cuts[:-1])
        w = np.diff(cuts)
        assert (w > 0).all() and w.max() - w.min() <= align
    # balanced: every rank's node count within one align-block of the ideal share
    rng = np.random.default_rng(1)
    L, P, align = 512, 8, 8
    pc = rng.poisson(5, L)
    pc[200:260] += 400                              # a dense band
    cuts = bn.slab_cuts(L, P, align, pc)
    share = np.array([pc[cuts[r]:cuts[r + 1]].sum() for r in range(P)])
    blk = pc.reshape(-1, align).sum(1).max()
    assert np.abs(share - pc.sum() / P).max() <= blk
    assert np.array_equal(bn.slab_cuts(L, P, align, np.ones(L, np.int64)), bn.slab_cuts(L, P, align))
    # owners and halo ranges
    for c in range(L):
        r = bn.slab_owner(cuts, c)
        assert cuts[r] <= c < cuts[r + 1]
    for r in range(P):
        lo, hi = bn.halo_ranges(cuts, r, 4, L)
        assert lo == max(0, cuts[r] - 3) and hi == min(L, cuts[r + 1] + 4)
    with pytest.raises(bn.BnfftError):
        bn.slab_cuts(64, 16, 8)                      # fewer bin rows than ranks


def _slab_worker(rank, world, port, q):
    """Each rank: its own nodes -> plane histogram -> all-reduce (gloo) -> the library's cut points
    (bnfft_slab_cuts) -> owners (bnfft_slab_owner) -> node exchange (gloo) -> halo ranges."""
    import torch
    import torch.distributed as dist
    from paper_2502_07155_b200 import bnfft as bn
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        L, m, align = 128, 4, 8
        rng = np.random.default_rng(100 + rank)
        x = rng.random((5000, 3)) - 0.5
        if rank == 1:                                    # this rank's nodes cluster in y
            x[:, 1] = np.clip(0.03 * rng.standard_normal(5000), -0.5, 0.49)
        c = np.minimum(np.floor(L * x[:, 1]).astype(np.int64) + L // 2, L - 1)
        h = torch.from_numpy(np.bincount(c, minlength=L).astype(np.int64))
        dist.all_reduce(h)
        cuts = bn.slab_cuts(L, world, align, h.numpy())
        allcuts = [None] * world
        dist.all_gather_object(allcuts, cuts.tolist())
        owner = np.array([bn.slab_owner(cuts, int(ci)) for ci in c])
        send = [x[owner == r] for r in range(world)]
        recv = [None] * world
        dist.all_gather_object(recv, send)
        mine = np.concatenate([recv[s][rank] for s in range(world)])
        cm = np.minimum(np.floor(L * mine[:, 1]).astype(np.int64) + L // 2, L - 1)
        lo, hi = bn.halo_ranges(cuts, rank, m, L)
        q.put((rank, allcuts[0] == allcuts[1], bool(((cm >= cuts[rank]) & (cm < cuts[rank + 1])).all()),
               len(mine), int(h.sum()), lo, hi, cuts.tolist()))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_slab_partition():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, same0, in0, n0, tot, lo0, hi0, cuts), (r1, same1, in1, n1, _, lo1, hi1, _) = res
    assert same0 and same1 and in0 and in1
    assert n0 + n1 == tot == 10000
    assert abs(n0 - n1) <= 0.25 * tot                    # balanced by the all-reduced histogram
    assert (lo0, hi0) == (0, cuts[1] + 4) and (lo1, hi1) == (cuts[1] - 3, 128)
