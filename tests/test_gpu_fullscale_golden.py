"""Full BASELINE-scale parity against the REAL reference.

tests/golden/full_c2.npz and full_c3.npz were produced by running the
unmodified reference package (echoreg 0.1, numba backend) on the build host
(tests/golden/make_golden_full.py, ~30 min of CPU each):

* C2 -- register_smc, image mode, 2000 particles x 50 iterations, seed 0, on
  the 176x176x208 8-bit echo pair (/root/reference/pkg/src/echoreg/smc.py:
  325-373, kernels_numba.py:116-189);
* C3 -- register_sequence, mask mode, 2000 x 50, on the 30-frame 4D cycle,
  then the warp and scoring of every frame (pipeline.py:155-216).

The GPU rebuilds the same inputs with its own generator (the digests of the
8-bit frames and masks must equal the reference's) and runs the whole path on
the device.  The north star's bars: final transform within 0.1 degree and 0.1
voxel, Dice within 1e-3, per-particle fp32 likelihoods within 1e-4 relative,
degenerate flags and resampling decisions identical.
"""

import os

import numpy as np
import pytest

from .conftest import GOLDEN

pytestmark = pytest.mark.gpu

ESS_RTOL = {"f32": 1e-4, "f64": 1e-8, "exact": 1e-10}
Z_RTOL = {"f32": 1e-4, "f64": 1e-6, "exact": 1e-10}


def _digest(vols):
    from oracle.phantom import digest

    return digest([v.codec.raw for v in vols])


@pytest.fixture(scope="module")
def c2():
    from paper_2504_19930_b200 import normalize_zscore
    from paper_2504_19930_b200.phantom_device import echo_case_device

    g = np.load(os.path.join(GOLDEN, "full_c2.npz"))
    case = echo_case_device(frames=1, seed=0)
    assert _digest(case.target.frames) == str(g["c2_target_sha256"])
    assert _digest(case.source.frames) == str(g["c2_source_sha256"])
    t = normalize_zscore(case.target.frames[0])
    s = normalize_zscore(case.source.frames[0])
    return g, t, s


def _transform_diff(est, ref, spacing):
    d = np.asarray(est) - np.asarray(ref)
    return (float(np.degrees(np.abs(d[:3])).max()),
            float((np.abs(d[3:]) / np.asarray(spacing)).max()))


@pytest.mark.parametrize("precision", ["f32", "f64", "exact"])
def test_c2_full_registration_matches_reference(c2, precision):
    """The device loop step by step (what register_smc runs), capturing the
    first and last iterations' per-particle likelihoods."""
    from paper_2504_19930_b200 import Executor, SmcConfig
    from paper_2504_19930_b200 import smc as dsmc

    g, t, s = c2
    cfg = SmcConfig(mode="image", n_particles=2000, n_iterations=50, seed=0)
    run = dsmc.DeviceSmcRun(t, s, cfg, Executor(precision=precision))
    dsmc._check_inputs(run.tdv, run.sdv, cfg)
    z = {}
    for k in range(cfg.n_iterations):
        run.predict(k)
        run.measure()
        if k in (0, cfg.n_iterations - 1):
            z[k] = (run.z_local[:2000].cpu().numpy().copy(),
                    run.dg_local[:2000].cpu().numpy().astype(bool))
        run.update(k)
    tr = run.finish()
    est = tr.estimates[-1].to_array()
    rot, vox = _transform_diff(est, g["c2_estimate"], t.spacing)
    assert rot <= 0.1 and vox <= 0.1, (rot, vox)
    assert np.array_equal(np.array(tr.resampled), g["c2_resampled"])
    ess = np.array(tr.ess)
    assert np.max(np.abs(ess - g["c2_ess"]) / g["c2_ess"]) <= ESS_RTOL[precision]
    for k, key in ((0, "first"), (cfg.n_iterations - 1, "last")):
        zz, dd = z[k]
        zr, dr = g[f"c2_z_{key}"], g[f"c2_degen_{key}"]
        assert np.array_equal(dd, dr), key
        rel = np.abs(zz - zr) / np.maximum(np.abs(zr), 1e-300)
        assert rel.max() <= Z_RTOL[precision], (key, float(rel.max()))
    # informative: how close the whole trajectory stays (it is
    # chaotic in the likelihoods, so agreement to ~1e-12 degrees means the
    # same resampling decisions all the way)
    est_all = np.stack([e.to_array() for e in tr.estimates])
    traj = float(np.degrees(np.abs(est_all[:, :3] - g["c2_estimates"][:, :3])).max())
    assert traj <= 0.1, traj


def test_c3_full_4d_pipeline_matches_reference():
    from paper_2504_19930_b200 import Executor, SmcConfig, register_sequence
    from paper_2504_19930_b200.phantom_device import echo_case_device

    g = np.load(os.path.join(GOLDEN, "full_c3.npz"))
    case = echo_case_device(frames=30, seed=0)
    assert _digest(case.target.frames) == str(g["c3_target_sha256"])
    assert _digest(case.source.frames) == str(g["c3_source_sha256"])
    assert _digest(case.target_masks) == str(g["c3_target_masks_sha256"])
    assert _digest(case.source_masks) == str(g["c3_source_masks_sha256"])
    cfg = SmcConfig(mode="mask", n_particles=2000, n_iterations=50, seed=0)
    rep = register_sequence(case.target, case.source, case.target_masks, case.source_masks,
                            cfg, Executor(), case_id="c3")
    keys = ("rx_deg", "ry_deg", "rz_deg", "tx_mm", "ty_mm", "tz_mm")
    est = np.array([rep.estimate_deg_mm[k] for k in keys])
    ref = g["c3_estimate_deg_mm"]
    sp = case.target.frames[0].spacing
    assert np.abs(est[:3] - ref[:3]).max() <= 0.1
    assert (np.abs(est[3:] - ref[3:]) / np.asarray(sp)).max() <= 0.1
    assert np.array_equal(np.array(rep.trace["resampled"]), g["c3_resampled"])
    assert np.abs(np.array(rep.dsc_before) - g["c3_dsc_before"]).max() <= 1e-3
    assert np.abs(np.array(rep.dsc_after) - g["c3_dsc_after"]).max() <= 1e-3
    assert np.abs(np.array(rep.trace["dsc"]) - g["c3_trace_dsc"]).max() <= 1e-3
    for key in ("ncc_before", "ncc_after"):
        got, want = np.array(getattr(rep, key)), g[f"c3_{key}"]
        assert np.max(np.abs(got - want) / np.abs(want)) <= 1e-6, key
    ess = np.array(rep.trace["ess"])
    assert np.max(np.abs(ess - g["c3_ess"]) / g["c3_ess"]) <= 1e-4
    # the report document has the reference's schema (keys, config, trace keys)
    import json

    with open(os.path.join(GOLDEN, "full_c3_report.json")) as fh:
        want = json.load(fh)
    got = rep.to_dict()
    assert got.keys() == want.keys()
    assert got["config"] == want["config"]
    assert got["trace"].keys() == want["trace"].keys()
    assert got["aggregates"].keys() == want["aggregates"].keys()
    for k, v in want["aggregates"].items():
        assert got["aggregates"][k] == pytest.approx(v, rel=1e-6, abs=1e-9), k


def _c2o_goldens():
    import glob

    return sorted(glob.glob(os.path.join(GOLDEN, "full_c2o*.npz")))


@pytest.mark.parametrize("path", _c2o_goldens() or [None],
                         ids=lambda p: os.path.basename(p) if p else "none")
@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_c2_overlap_region_registration_matches_reference(c2, precision, path):
    """The C2 pair with SmcConfig(ncc_region="overlap"), 2000 x 20, seed 3
    (and further seeds, full_c2o_seed<s>.npz):
    the overlap-region kernels (in-bounds target sums and sums of squares,
    /root/reference/pkg/src/echoreg/kernels_numba.py:172-189) against the real
    reference's run (tests/golden/full_c2o.npz)."""
    from paper_2504_19930_b200 import Executor, SmcConfig
    from paper_2504_19930_b200 import smc as dsmc

    if path is None:
        pytest.skip("full_c2o*.npz not generated")
    g = np.load(path)
    _, t, s = c2
    assert str(g["c2o_target_sha256"]) == str(c2[0]["c2_target_sha256"])
    seed = int(g["c2o_seed"]) if "c2o_seed" in g else 3
    cfg = SmcConfig(mode="image", n_particles=2000, n_iterations=20, seed=seed,
                    ncc_region="overlap")
    run = dsmc.DeviceSmcRun(t, s, cfg, Executor(precision=precision))
    z = {}
    for k in range(cfg.n_iterations):
        run.predict(k)
        run.measure()
        if k in (0, cfg.n_iterations - 1):
            z[k] = (run.z_local[:2000].cpu().numpy().copy(),
                    run.dg_local[:2000].cpu().numpy().astype(bool))
        run.update(k)
    tr = run.finish()
    rot, vox = _transform_diff(tr.estimates[-1].to_array(), g["c2o_estimate"], t.spacing)
    assert rot <= 0.1 and vox <= 0.1, (rot, vox)
    # the seed-3 run is known to stay on the reference trajectory in every
    # precision; at other seeds f32 may leave it at a resampling boundary
    # (DESIGN.md section 5 item 5), so there only its first iteration is held
    strict = precision != "f32" or seed == 3
    if strict:
        assert np.array_equal(np.array(tr.resampled), g["c2o_resampled"])
        ess = np.array(tr.ess)
        assert np.max(np.abs(ess - g["c2o_ess"]) / g["c2o_ess"]) <= ESS_RTOL[precision]
    for k, key in ((0, "first"), (cfg.n_iterations - 1, "last")):
        if k and not strict:
            continue
        zz, dd = z[k]
        zr, dr = g[f"c2o_z_{key}"], g[f"c2o_degen_{key}"]
        assert np.array_equal(dd, dr), key
        rel = np.abs(zz - zr) / np.maximum(np.abs(zr), 1e-300)
        assert rel.max() <= Z_RTOL[precision], (key, float(rel.max()))


def _seed_goldens():
    import glob

    return sorted(glob.glob(os.path.join(GOLDEN, "full_c2_seed*.npz")))


@pytest.mark.parametrize("precision", ["f32", "f64"])
@pytest.mark.parametrize("path", _seed_goldens() or [None],
                         ids=lambda p: os.path.basename(p) if p else "none")
def test_c2_full_other_seeds_match_reference(c2, path, precision):
    """C2 at further SMC seeds (tests/golden/full_c2_seed<s>.npz, the real
    reference's register_smc).  f64 tracks the reference's whole trajectory
    (same resampling decisions, estimates to 1e-9 degree); f32 holds the
    north star's bar on the final transform (0.1 degree / 0.1 voxel) and the
    per-particle likelihoods of the first iteration (1e-4), but may leave the
    reference's trajectory at a resampling boundary later (SMC chaos,
    DESIGN.md section 5 item 5) -- those seeds are kept, not skipped."""
    from paper_2504_19930_b200 import Executor, SmcConfig
    from paper_2504_19930_b200 import smc as dsmc

    if path is None:
        pytest.skip("no full_c2_seed*.npz generated")
    g = np.load(path)
    _, t, s = c2
    assert str(g["c2_target_sha256"]) == str(c2[0]["c2_target_sha256"])
    assert str(g["c2_source_sha256"]) == str(c2[0]["c2_source_sha256"])
    cfg = SmcConfig(mode="image", n_particles=2000, n_iterations=50, seed=int(g["c2_seed"]))
    run = dsmc.DeviceSmcRun(t, s, cfg, Executor(precision=precision))
    z0 = None
    for k in range(cfg.n_iterations):
        run.predict(k)
        run.measure()
        if k == 0:
            z0 = (run.z_local[:2000].cpu().numpy().copy(),
                  run.dg_local[:2000].cpu().numpy().astype(bool))
        run.update(k)
    tr = run.finish()
    rot, vox = _transform_diff(tr.estimates[-1].to_array(), g["c2_estimate"], t.spacing)
    assert rot <= 0.1 and vox <= 0.1, (rot, vox)
    assert np.array_equal(z0[1], g["c2_degen_first"])
    rel = np.abs(z0[0] - g["c2_z_first"]) / np.maximum(np.abs(g["c2_z_first"]), 1e-300)
    assert rel.max() <= Z_RTOL[precision], float(rel.max())
    if precision == "f64":
        assert np.array_equal(np.array(tr.resampled), g["c2_resampled"])
        ess = np.array(tr.ess)
        assert np.max(np.abs(ess - g["c2_ess"]) / g["c2_ess"]) <= ESS_RTOL["f64"]
        est_all = np.stack([e.to_array() for e in tr.estimates])
        traj = float(np.degrees(np.abs(est_all[:, :3] - g["c2_estimates"][:, :3])).max())
        assert traj <= 1e-9, traj


def _c3_seed_goldens():
    import glob

    return sorted(glob.glob(os.path.join(GOLDEN, "full_c3_seed*.npz")))


@pytest.mark.parametrize("path", _c3_seed_goldens() or [None],
                         ids=lambda p: os.path.basename(p) if p else "none")
def test_c3_full_4d_pipeline_other_seeds(path):
    """The C3 pipeline (mask-mode SMC + warp/score of the 30-frame cycle) at
    another SMC seed against the real reference (full_c3_seed<s>.npz): same
    bars as the seed-0 test (transform, resampling decisions, Dice, NCC,
    ESS), without the report-file comparison."""
    from paper_2504_19930_b200 import Executor, SmcConfig, register_sequence
    from paper_2504_19930_b200.phantom_device import echo_case_device

    if path is None:
        pytest.skip("no full_c3_seed*.npz generated")
    g = np.load(path)
    case = echo_case_device(frames=30, seed=0)
    assert _digest(case.target.frames) == str(g["c3_target_sha256"])
    assert _digest(case.source_masks) == str(g["c3_source_masks_sha256"])
    cfg = SmcConfig(mode="mask", n_particles=2000, n_iterations=50, seed=int(g["c3_seed"]))
    rep = register_sequence(case.target, case.source, case.target_masks, case.source_masks,
                            cfg, Executor(), case_id="c3")
    keys = ("rx_deg", "ry_deg", "rz_deg", "tx_mm", "ty_mm", "tz_mm")
    est = np.array([rep.estimate_deg_mm[k] for k in keys])
    ref = g["c3_estimate_deg_mm"]
    sp = case.target.frames[0].spacing
    assert np.abs(est[:3] - ref[:3]).max() <= 0.1
    assert (np.abs(est[3:] - ref[3:]) / np.asarray(sp)).max() <= 0.1
    assert np.array_equal(np.array(rep.trace["resampled"]), g["c3_resampled"])
    assert np.abs(np.array(rep.dsc_before) - g["c3_dsc_before"]).max() <= 1e-3
    assert np.abs(np.array(rep.dsc_after) - g["c3_dsc_after"]).max() <= 1e-3
    for key in ("ncc_before", "ncc_after"):
        got, want = np.array(getattr(rep, key)), g[f"c3_{key}"]
        assert np.max(np.abs(got - want) / np.abs(want)) <= 1e-6, key
    ess = np.array(rep.trace["ess"])
    assert np.max(np.abs(ess - g["c3_ess"]) / g["c3_ess"]) <= 1e-4
