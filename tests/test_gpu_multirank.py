"""The product's particle-sharded path executed at world size 2 on the one
leased GPU.

Two processes join a gloo process group (host-staged collectives, so the two
ranks' kernels never wait on each other on the device) and each runs the
device code paths exactly as N GPUs would: register_smc through DeviceSmcRun
(its shard of the particles, the ONE packed all-gather per iteration,
er_smc_update_gathered), register_exhaustive (node-range shards, the
(value, index) all-gather) and score_frames (frame shards, the score-row
all-gather).  Every rank's outputs must be BITWISE equal to the 1-rank run:
the reference's worker-count invariance contract
(/root/reference/pkg/src/echoreg/kernels_numba.py:6-8,
/root/reference/pkg/tests/test_kernels.py:106-116).
"""

import math
import multiprocessing as mp
import os
import socket
import sys

import numpy as np
import pytest

from .conftest import ROOT

pytestmark = pytest.mark.gpu


def _case():
    from paper_2504_19930_b200 import PhantomSpec, RigidParams, make_pair, make_phantom

    spec = PhantomSpec(dims=(28, 26, 30), frames=3, outer_semiaxes=(10.0, 8.5, 11.0),
                       inner_semiaxes=(6.5, 5.0, 7.5), speckle_sigma=0.25, amplitude=0.2,
                       seed=6)
    seq, masks = make_phantom(spec)
    truth = RigidParams(math.radians(4.0), math.radians(-2.0), math.radians(3.0), 1.5, -1.0, 0.8)
    case = make_pair(seq, masks, truth)
    return {
        "spacing": spec.spacing,
        "t": [f.data for f in case.target.frames], "s": [f.data for f in case.source.frames],
        "tm": [m.data for m in case.target_masks], "sm": [m.data for m in case.source_masks],
    }


def _run_all(arrays):
    """Everything the sharded paths touch; returns plain numpy results."""
    from paper_2504_19930_b200 import (GridSpec, RigidParams, SmcConfig, Volume3, binarize,
                                       normalize_zscore, register_exhaustive, register_smc,
                                       to_matrix)
    from paper_2504_19930_b200.pipeline import score_frames

    sp = arrays["spacing"]
    t = [normalize_zscore(Volume3(a, sp)) for a in arrays["t"]]
    s = [normalize_zscore(Volume3(a, sp)) for a in arrays["s"]]
    tm = [binarize(Volume3(a, sp), 0.5) for a in arrays["tm"]]
    sm = [binarize(Volume3(a, sp), 0.5) for a in arrays["sm"]]
    out = {}
    # odd particle count: the last rank's shard is padded
    for name, tv, sv, cfg in (
        ("image", t[0], s[0], SmcConfig(mode="image", n_particles=101, n_iterations=8, seed=3,
                                        t_limit=4.0, r_limit=6.0)),
        ("mask", tm[0], sm[0], SmcConfig(mode="mask", n_particles=96, n_iterations=6, seed=1,
                                         t_limit=4.0, r_limit=6.0)),
        ("overlap", t[0], s[0], SmcConfig(mode="image", n_particles=64, n_iterations=5, seed=2,
                                          t_limit=4.0, r_limit=6.0, ncc_region="overlap")),
    ):
        est, tr = register_smc(tv, sv, cfg)
        out[f"{name}_estimate"] = est.to_array()
        out[f"{name}_ess"] = np.array(tr.ess)
        out[f"{name}_resampled"] = np.array(tr.resampled)
        out[f"{name}_mean"] = np.array(tr.mean_measurement)
        out[f"{name}_best"] = (tr.best_particle.to_array() if tr.best_particle is not None
                               else np.zeros(6))
    g = GridSpec(half_counts=(1, 1, 1, 1, 2, 1), step_t=1.0, step_r=2.0)
    best, value = register_exhaustive(t[0], s[0], g)
    out["grid_best"] = best.to_array()
    out["grid_value"] = np.array(float(value))
    m = to_matrix(RigidParams.from_array(out["image_estimate"]), t[0].physical_center())
    nb, na, db, da = score_frames(t, s, tm, sm, m)
    out["score"] = np.array([nb, na, db, da], dtype=np.float64)
    return out


def _worker(rank, world, port, arrays, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    try:
        import torch
        import torch.distributed as td

        torch.cuda.set_device(0)
        td.init_process_group("gloo", rank=rank, world_size=world)
        try:
            from paper_2504_19930_b200 import dist

            assert dist.world()[:2] == (world, rank)
            q.put((rank, _run_all(arrays), None))
        finally:
            td.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback

        q.put((rank, None, traceback.format_exc() + repr(e)))


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def test_world2_sharded_paths_are_bitwise_equal_to_one_rank():
    arrays = _case()
    single = _run_all(arrays)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, arrays, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = {}
    try:
        for _ in procs:
            rank, res, err = q.get(timeout=600)
            assert err is None, f"rank {rank} failed:\n{err}"
            results[rank] = res
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    assert sorted(results) == [0, 1]
    for rank, res in results.items():
        assert res.keys() == single.keys()
        for k, v in single.items():
            assert np.array_equal(res[k], v, equal_nan=True), (rank, k, res[k], v)
