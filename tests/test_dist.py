"""Multi-rank host logic on CPU (gloo, world_size 2 and 3).

The device path shards particles over ranks with dist.ShardPlan and
all-gathers the likelihood shards (one packed block per rank,
dist.allgather_packed) before the
replicated update (smc.DeviceSmcRun.update); the exhaustive search shards
node ranges and reduces (value, index) pairs with the lowest-index
tie-break.  Here the same host functions run under torch.distributed/gloo
with the C oracle standing in for the per-rank measurement (test only), and
the results must be bit-identical to the single-process run.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as td
import torch.multiprocessing as mp

from paper_2504_19930_b200 import dist

from .conftest import golden


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_shard_plan_partitions_exactly():
    for n in (1, 2, 5, 500, 2000, 262144):
        for w in (1, 2, 3, 4, 8):
            plans = [dist.ShardPlan(n, w, r) for r in range(w)]
            owned = np.concatenate([np.arange(p.lo, p.hi) for p in plans])
            assert np.array_equal(owned, np.arange(n))
            assert all(p.count <= p.shard for p in plans)
            assert all(p.lo == min(n, r * p.shard) for r, p in enumerate(plans))


def _c1():
    g = golden("smc.npz")
    dims = tuple(int(x) for x in g["c1_dims"])
    n = int(np.prod(dims))
    t = np.unpackbits(g["c1_target_bits"])[:n].reshape(dims).astype(np.float64)
    s = np.unpackbits(g["c1_source_bits"])[:n].reshape(dims).astype(np.float64)
    return t, s, dims


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import kernels as ok
        from oracle import smc as osmc

        t, s, dims = _c1()
        geom = (dims, (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
        cfg = osmc.Cfg(mode="mask", n_particles=90, n_iterations=4, seed=5)
        plan = dist.plan(cfg.n_particles)
        assert (plan.world, plan.rank) == (world, rank)

        def sharded_measure(a, b, overlap):
            z_local = torch.zeros(plan.shard, dtype=torch.float64)
            d_local = torch.zeros(plan.shard, dtype=torch.uint8)
            if plan.count:
                z, d = ok.ncc_measure_batch(t, s, a[plan.lo:plan.hi], b[plan.lo:plan.hi],
                                            overlap, workers=1)
                z_local[: plan.count] = torch.from_numpy(z)
                d_local[: plan.count] = torch.from_numpy(d.astype(np.uint8))
            z_all = dist.allgather_shards(
                z_local, plan, torch.zeros(plan.shard * world, dtype=torch.float64))
            d_all = dist.allgather_shards(
                d_local, plan, torch.zeros(plan.shard * world, dtype=torch.uint8))
            return z_all.numpy().copy(), d_all.numpy().astype(bool)

        est, tr = osmc.register(t, s, geom, geom, cfg, measure=sharded_measure)

        # exhaustive-style node-range sharding + (value, index) reduction
        scores = np.random.default_rng(0).random(1000)
        scores[[17, 640]] = 2.0   # a tie across ranks: lowest index must win
        per = -(-scores.size // world)
        lo, hi = min(scores.size, rank * per), min(scores.size, (rank + 1) * per)
        best = torch.tensor([-1.0, -1.0], dtype=torch.float64)
        if hi > lo:
            i = int(np.argmax(scores[lo:hi]))
            best = torch.tensor([scores[lo + i], float(lo + i)], dtype=torch.float64)
        allb = torch.zeros(2 * world, dtype=torch.float64)
        td.all_gather_into_tensor(allb, best)
        bv, bi = -1.0, -1
        for v, i in allb.view(world, 2).numpy():
            if v > bv:
                bv, bi = float(v), int(i)
        out_q.put((rank, est, np.stack(tr.z), tr.resampled, bi))
    finally:
        td.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_smc_and_grid_bit_identical(world):
    from oracle import kernels as ok
    from oracle import smc as osmc

    ok.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    t, s, dims = _c1()
    geom = (dims, (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    cfg = osmc.Cfg(mode="mask", n_particles=90, n_iterations=4, seed=5)
    est1, tr1 = osmc.register(t, s, geom, geom, cfg)
    for rank, est, z, resampled, bi in results:
        assert np.array_equal(est, est1), rank        # replicated update: identical
        assert np.array_equal(z, np.stack(tr1.z)), rank
        assert resampled == tr1.resampled
        assert bi == 17                                # lowest index wins the tie


def _frames_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2504_19930_b200 import errors, pipeline

        seen = []

        def scorer(tgt, src, tm, sm, matrix):  # stands in for the device warp + scores
            seen.append(tgt)
            if tgt == 6 and matrix is None:
                raise errors.DegenerateInput("constant")
            has = tm is not None and sm is not None
            return [tgt + 0.5, -tgt, float(has), tgt * 0.01 if has else 0.0, 0.3, 0.0]

        frames = list(range(7))
        masks = [1, None, 1, 1, None, 1, 1]
        res = pipeline.score_frames(frames, frames, masks, masks, np.eye(4), scorer=scorer)
        try:
            pipeline.score_frames(frames, frames, masks, masks, None, scorer=scorer)
            raised = None
        except errors.DegenerateInput as e:
            raised = str(e)
        out_q.put((rank, res, seen, raised))
    finally:
        td.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_score_frames_sharded_over_ranks(world):
    """The 4D scoring shards frames (contiguous ranges) and all-gathers the
    per-frame rows: every rank returns the full lists, in frame order, with
    None DSC for mask-less frames; a degenerate frame on one rank raises on
    all of them instead of leaving the others in the collective."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_frames_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect_b = [f + 0.5 for f in range(7)]
    expect_dsc = [None if f in (1, 4) else f * 0.01 for f in range(7)]
    owned = []
    for rank, (nb, na, db, da), seen, raised in results:
        assert nb == expect_b and na == [-float(f) for f in range(7)]
        assert db == expect_dsc
        assert da == [None if f in (1, 4) else 0.3 for f in range(7)]
        plan = dist.ShardPlan(7, world, rank)
        assert seen[: plan.count] == list(range(plan.lo, plan.hi))
        owned += seen[: plan.count]
        assert raised is not None and "frame 6" in raised
    assert sorted(owned) == list(range(7))


def _packed_worker(rank, world, port, n, out_q):
    """One SMC iteration's exchange as DeviceSmcRun does it, on CPU tensors:
    each rank writes its shard of z and degenerate flags into ONE packed
    block, ONE all_gather, then every rank reads particle i back the way
    er_smc_update_gathered's ZPacked accessor does."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = dist.plan(n)
        S = plan.shard
        block = dist.packed_block_bytes(S)
        local = torch.zeros(block, dtype=torch.uint8)
        z_local = local[: 8 * S].view(torch.float64)
        dg_local = local[8 * S: 9 * S]
        g = np.random.default_rng(123)
        z_all = g.random(n)
        dg_all = (g.random(n) < 0.2).astype(np.uint8)
        z_local[: plan.count] = torch.from_numpy(z_all[plan.lo: plan.hi])
        dg_local[: plan.count] = torch.from_numpy(dg_all[plan.lo: plan.hi])
        out = torch.zeros(block * world, dtype=torch.uint8)
        calls = []
        orig = td.all_gather_into_tensor

        def counting(*a, **k):
            calls.append(1)
            return orig(*a, **k)

        td.all_gather_into_tensor = counting
        try:
            dist.allgather_packed(local, out)
        finally:
            td.all_gather_into_tensor = orig
        buf = out.numpy()
        z = np.array([buf[(i // S) * block: (i // S) * block + 8 * S].view(np.float64)[i % S]
                      for i in range(n)])
        dg = np.array([buf[(i // S) * block + 8 * S + i % S] for i in range(n)])
        out_q.put((rank, len(calls), np.array_equal(z, z_all), np.array_equal(dg, dg_all)))
    finally:
        td.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 2000), (3, 101), (2, 7)])
def test_one_packed_allgather_carries_z_and_flags(world, n):
    """The exchange of an SMC iteration is exactly ONE collective, and the
    packed rank blocks decode to every particle's z and degenerate flag
    (the layout er_smc_update_gathered reads; block size % 8 == 0)."""
    assert dist.packed_block_bytes(n) % 8 == 0 and dist.packed_block_bytes(n) >= 9 * n
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_packed_worker, args=(r, world, port, n, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == list(range(world))
    for _, ncalls, z_ok, dg_ok in res:
        assert ncalls == 1 and z_ok and dg_ok
