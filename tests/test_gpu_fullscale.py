"""Echo-scale (176x176x208) checks against the reference's algorithms, sized
to run in seconds: exhaustive search on the C2 pair over a 3^6 grid (winner
and every node's likelihood vs the C oracle), and the 4D pipeline's per-frame
scores on a 3-frame cycle (tools/parity_c3_scores.py restatements).  The
full-size runs are tools/parity_c4_grid.py and tools/parity_c3_scores.py."""

import os
import sys

import numpy as np
import pytest

from .conftest import ROOT

pytestmark = pytest.mark.gpu


def test_exhaustive_grid_on_the_echo_pair_matches_the_oracle():
    sys.path.insert(0, ROOT)
    import bench
    from oracle import kernels as ok
    from paper_2504_19930_b200 import Executor, GridSpec, RigidParams, register_exhaustive
    from paper_2504_19930_b200.exhaustive import _node_states
    from paper_2504_19930_b200.geometry import index_affine_batch, to_matrix

    t, s, _ = bench.make_workload()
    g = GridSpec(half_counts=(1, 1, 1, 1, 1, 1))
    states = _node_states(g)
    mats = np.stack([to_matrix(RigidParams(*st), t.physical_center()) for st in states])
    a, b = index_affine_batch(mats, s.spacing, s.origin, t.spacing, t.origin)
    z_ref, _ = ok.ncc_measure_batch(t.data, s.data, a, b, False, ok.max_threads())
    best_ref = int(np.argmax(z_ref))
    for prec, rtol in (("f32", 1e-6), ("f64", 1e-9)):
        ex = Executor(precision=prec)
        best, _ = register_exhaustive(t, s, g, ex)
        assert np.array_equal(np.asarray(best.to_array()), states[best_ref]), prec
        z = ex.measure_ncc(t, s, mats)[0]
        assert np.all(np.abs(z - z_ref) <= rtol * np.abs(z_ref)), prec


def test_pipeline_scores_on_an_echo_cycle_match_the_reference_algorithms():
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import parity_c3_scores as pc
    from oracle import kernels as ok
    from paper_2504_19930_b200 import (Executor, SmcConfig, binarize, register_sequence,
                                       register_smc, to_matrix)
    from paper_2504_19930_b200.geometry import index_affine
    from paper_2504_19930_b200.phantom_device import echo_case_device

    case = echo_case_device(frames=3, seed=0)
    cfg = SmcConfig(mode="mask", n_particles=256, n_iterations=6, seed=0)
    rep = register_sequence(case.target, case.source, case.target_masks, case.source_masks,
                            cfg, Executor())
    reg_t = binarize(case.target_masks[0], 0.5)
    reg_s = binarize(case.source_masks[0], 0.5)
    est, _ = register_smc(reg_t, reg_s, cfg, Executor(), trace_masks=(reg_t, reg_s))
    m = to_matrix(est, reg_t.physical_center())
    for f in range(3):
        tf, sf = case.target.frames[f], case.source.frames[f]
        tz, sz = pc.zscore(tf.codec.raw), pc.zscore(sf.codec.raw)
        assert rep.ncc_before[f] == pytest.approx(pc.ncc_ref(tz, sz), rel=1e-12)
        a, b = index_affine(m, sf, tf)
        moved = ok.resample_trilinear(sz, a, b, tf.dims, ok.max_threads())
        assert rep.ncc_after[f] == pytest.approx(pc.ncc_ref(tz, moved), rel=1e-12)
        tm = case.target_masks[f].codec.raw.astype(np.float64)
        sm = case.source_masks[f].codec.raw.astype(np.float64)
        am, bm = index_affine(m, case.source_masks[f], case.target_masks[f])
        mm = (ok.resample_trilinear(sm, am, bm, tf.dims, ok.max_threads()) > 0.5)
        assert rep.dsc_before[f] == pc.dice_ref(tm, sm)
        assert rep.dsc_after[f] == pc.dice_ref(mm.astype(np.float64), tm)


def test_c5_scale_measurement_matches_the_oracle_and_is_batch_invariant():
    """BASELINE configs[4] at full size: the 256^3 z-scored echo pair (its oct
    layout, 136 MB, exceeds L2, so the kernel runs the 8-lanes-per-row
    variant), 16,384 particles of SMC iteration 0 measured in one launch.
    Per-particle parity on a spread of 48 of them against the bit-exact C
    oracle (f32 bar 1e-4, counts exact) and two size-independent properties
    of the full batch: every particle's result is bitwise the same when it is
    measured alone in a small batch (fixed tiling: batch/shard invariance),
    and z is in [0, 1]."""
    sys.path.insert(0, ROOT)
    import torch

    from oracle import kernels as ok
    from paper_2504_19930_b200 import Executor, SmcConfig, normalize_zscore, ops
    from paper_2504_19930_b200 import smc as dsmc
    from paper_2504_19930_b200.phantom_device import echo_case_device

    case = echo_case_device(dims=(256, 256, 256), spacing=(0.8, 0.8, 0.8), frames=1, seed=0)
    t = normalize_zscore(case.target.frames[0])
    s = normalize_zscore(case.source.frames[0])
    P = 16384
    run = dsmc.DeviceSmcRun(t, s, SmcConfig(mode="image", n_particles=P, n_iterations=1, seed=0),
                            Executor())
    run.predict(0)
    run.measure()
    z = run.z_local[:P].cpu().numpy().copy()
    n = run.n_local[:P].cpu().numpy().copy()
    dg = run.dg_local[:P].cpu().numpy().astype(bool)
    assert np.all((z >= 0) & (z <= 1))
    idx = np.linspace(0, P - 1, 48).astype(np.int64)
    A = run.A[:P][torch.as_tensor(idx, device=run.A.device)].contiguous()
    B = run.B[:P][torch.as_tensor(idx, device=run.B.device)].contiguous()
    zs, ds, ns = (x.cpu().numpy() for x in ops.measure(run.tdv, run.sdv, A, B, False, "f32"))
    assert np.array_equal(zs, z[idx]) and np.array_equal(ns, n[idx])
    assert np.array_equal(ds.astype(bool), dg[idx])
    a = A.cpu().numpy().reshape(-1, 3, 3)
    b = B.cpu().numpy()
    zo, do, no = ok.ncc_measure_batch(t.data, s.data, a, b, False, ok.max_threads(),
                                      return_counts=True)
    assert np.array_equal(ns, no) and np.array_equal(ds.astype(bool), do)
    assert np.all(np.abs(zs - zo) <= 1e-4 * np.abs(zo) + 1e-12)
