"""Multi-rank host logic on CPU (gloo, world_size 2 and 3).

The device path shards particles over ranks with dist.ShardPlan and
all-gathers the likelihood shards with dist.allgather_shards before the
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
