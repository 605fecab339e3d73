"""Behavioural properties the reference's own test suite asserts
(T/test_metrics.py, T/test_smc.py, T/test_exhaustive.py), checked on this
package's device path: the invariants a user of the reference relies on,
beyond the golden-vector parity of the other test modules."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _vol(a, spacing=(1.0, 1.0, 1.0)):
    from paper_2504_19930_b200 import Volume3

    return Volume3(np.asarray(a, dtype=np.float64), spacing)


# ---- metrics (E/metrics.py:49-93) -----------------------------------------

def test_ncc_self_similarity_symmetry_and_affine_invariance():
    from paper_2504_19930_b200 import ncc

    g = np.random.default_rng(1)
    a, b = g.standard_normal((12, 10, 14)), g.standard_normal((12, 10, 14))
    assert abs(float(ncc(_vol(a), _vol(a))) - 1.0) < 1e-12
    assert abs(float(ncc(_vol(a), _vol(2.5 * a - 7.0))) - 1.0) < 1e-12
    assert abs(float(ncc(_vol(a), _vol(b))) - float(ncc(_vol(b), _vol(a)))) < 1e-15
    for _ in range(5):
        v = float(ncc(_vol(g.standard_normal((6, 7, 8))), _vol(g.standard_normal((6, 7, 8)))))
        assert 0.0 <= v <= 1.0


def test_ncc_errors():
    from paper_2504_19930_b200 import ncc
    from paper_2504_19930_b200.errors import DegenerateInput, DimMismatch

    g = np.random.default_rng(2)
    with pytest.raises(DimMismatch):
        ncc(_vol(g.random((4, 4, 4))), _vol(g.random((4, 4, 5))))
    with pytest.raises(DegenerateInput):
        ncc(_vol(np.full((4, 4, 4), 3.0)), _vol(g.random((4, 4, 4))))


def test_dice_conventions():
    from paper_2504_19930_b200 import dice

    z = np.zeros((5, 6, 7))
    a = z.copy()
    a[1:3, 2:5, 1:6] = 1.0
    b = z.copy()
    b[3:5, :, :] = 1.0
    assert float(dice(_vol(z), _vol(z))) == 1.0          # both empty
    assert float(dice(_vol(a), _vol(z))) == 0.0          # one empty
    assert float(dice(_vol(a), _vol(a))) == 1.0
    assert float(dice(_vol(a), _vol(b))) == 0.0          # disjoint
    with pytest.raises(ValueError):
        dice(_vol(a * 0.5), _vol(a))                     # not binary


def test_dice_under_transform_identity_and_integer_shift():
    from paper_2504_19930_b200 import RigidParams, dice, dice_under_transform, to_matrix

    m = np.zeros((20, 20, 20))
    m[6:12, 7:13, 5:11] = 1.0
    ma = _vol(m)
    assert float(dice_under_transform(ma, ma, np.eye(4))) == float(dice(ma, ma)) == 1.0
    shifted = np.zeros_like(m)
    shifted[8:14, 6:12, 5:11] = 1.0
    # the target is the mask moved by (+2, -1, 0) voxels: pull it back exactly
    # (dice_under_transform pulls the first mask back through m: moved(x) = a(m x))
    mat = to_matrix(RigidParams(tx=-2.0, ty=1.0, tz=0.0))
    assert float(dice_under_transform(ma, _vol(shifted), mat)) == 1.0


# ---- particle machinery (E/smc.py:145-259) ---------------------------------

def test_zero_noise_predict_keeps_states_and_clamps_to_double_limits():
    from paper_2504_19930_b200 import SmcConfig
    from paper_2504_19930_b200.smc import init_particles, predict

    cfg = SmcConfig(n_particles=64, sigma0_t=0.0, sigma0_r=0.0, seed=3)
    ps = init_particles(cfg)
    assert np.array_equal(predict(ps, cfg).states, ps.states)
    wild = SmcConfig(n_particles=256, sigma0_t=500.0, sigma0_r=500.0, seed=3)
    out = predict(init_particles(wild), wild).states
    lim = 2.0 * wild.state_limits()
    assert np.all(np.abs(out) <= lim) and np.any(np.abs(out) == lim)


def test_per_particle_streams_do_not_depend_on_population():
    from paper_2504_19930_b200 import SmcConfig
    from paper_2504_19930_b200.smc import ParticleSet, predict

    rows = np.random.default_rng(4).uniform(-0.1, 0.1, (40, 6))
    outs = []
    for n in (10, 40):
        cfg = SmcConfig(n_particles=n, seed=9)
        ps = ParticleSet(states=rows[:n].copy(), weights=np.full(n, 1.0 / n),
                         measurements=np.zeros(n), iteration=2, rng_seed=9)
        outs.append(predict(ps, cfg).states)
    assert np.array_equal(outs[0], outs[1][:10])


def test_init_is_deterministic_and_inside_the_box():
    from paper_2504_19930_b200 import SmcConfig
    from paper_2504_19930_b200.smc import init_particles

    cfg = SmcConfig(n_particles=500, seed=11)
    a, b = init_particles(cfg).states, init_particles(cfg).states
    assert np.array_equal(a, b)
    assert np.all(np.abs(a) <= cfg.state_limits())


# ---- registration (E/smc.py:325-373, E/exhaustive.py:78-113) --------------

def _small_case():
    """The reference suite's small phantom case (T/test_smc.py:242-256)."""
    from paper_2504_19930_b200 import PhantomSpec, RigidParams, make_pair, make_phantom

    spec = PhantomSpec(dims=(24, 24, 24), frames=1, outer_semiaxes=(9.0, 7.5, 10.0),
                       inner_semiaxes=(6.0, 4.5, 7.0), speckle_sigma=0.2, amplitude=0.0,
                       seed=2)
    seq, masks = make_phantom(spec)
    truth = RigidParams(math.radians(4.0), 0.0, math.radians(-3.0), 2.5, -1.5, 1.0)
    return make_pair(seq, masks, truth), truth


def _phantom_pair(truth):
    from paper_2504_19930_b200 import PhantomSpec, make_pair, make_phantom

    seq, masks = make_phantom(PhantomSpec(dims=(48, 48, 48), frames=1, seed=2,
                                          outer_semiaxes=(16.0, 13.0, 19.0),
                                          inner_semiaxes=(10.0, 8.0, 12.0)))
    return make_pair(seq, masks, truth)


def test_already_aligned_source_stays_near_identity():
    # image mode on the z-scored speckled frame, as T/test_smc.py's
    # already-aligned case (a smooth cavity mask carries little rotation signal)
    from paper_2504_19930_b200 import Executor, SmcConfig, normalize_zscore, register_smc

    case, _ = _small_case()
    v = normalize_zscore(case.target.frames[0])
    cfg = SmcConfig(n_particles=128, n_iterations=30, t_limit=6.0, r_limit=8.0, seed=0)
    est, trace = register_smc(v, v, cfg, Executor(workers=2))
    a = est.to_array()
    assert np.all(np.abs(np.degrees(a[:3])) <= 0.5) and np.all(np.abs(a[3:]) <= 0.5)
    assert len(trace) == 30
    assert all(1.0 - 1e-9 <= e <= 128.0 + 1e-9 for e in trace.ess)
    assert all(mn <= mx + 1e-12 for mn, mx in zip(trace.mean_measurement,
                                                  trace.max_measurement))


def test_truth_beats_random_states_and_worker_count_is_irrelevant():
    from paper_2504_19930_b200 import Executor, RigidParams, SmcConfig, register_smc, to_matrix

    truth = RigidParams(math.radians(4), math.radians(-3), math.radians(2), 3.0, -2.0, 1.5)
    case = _phantom_pair(truth)
    tm, sm = case.target_masks[0], case.source_masks[0]
    center = tm.physical_center()
    g = np.random.default_rng(5)
    rand = [RigidParams(*g.uniform(-0.2, 0.2, 3), *g.uniform(-8, 8, 3)) for _ in range(32)]
    mats = np.stack([to_matrix(p, center) for p in [truth] + rand])
    z, _ = Executor().measure_ncc(tm, sm, mats)
    assert z[0] >= z[1:].max()
    cfg = SmcConfig(mode="mask", n_particles=300, n_iterations=15, seed=4)
    e1, _ = register_smc(tm, sm, cfg, Executor(workers=1))
    e8, _ = register_smc(tm, sm, cfg, Executor(workers=8))
    assert np.array_equal(e1.to_array(), e8.to_array())


def test_exhaustive_finds_a_truth_on_the_grid():
    from paper_2504_19930_b200 import GridSpec, RigidParams, register_exhaustive

    truth = RigidParams(math.radians(2.0), 0.0, math.radians(-2.0), 2.5, 0.0, -2.5)
    case = _phantom_pair(truth)
    g = GridSpec(half_counts=(1, 1, 1, 1, 1, 1), step_r=2.0, step_t=2.5)
    best, value = register_exhaustive(case.target_masks[0], case.source_masks[0], g)
    assert np.allclose(best.to_array(), truth.to_array(), atol=1e-12)
    assert 0.0 < float(value) <= 1.0


def test_recovers_the_reference_small_case():
    """T/test_smc.py:312-330 with the reference's own bounds."""
    from paper_2504_19930_b200 import (Executor, SmcConfig, dice_under_transform,
                                       register_smc, to_matrix)

    case, truth = _small_case()
    tm, sm = case.target_masks[0], case.source_masks[0]
    cfg = SmcConfig(mode="mask", n_particles=128, n_iterations=25, t_limit=6.0, r_limit=8.0,
                    seed=1)
    est, trace = register_smc(tm, sm, cfg, Executor(workers=2))
    err = np.abs(est.to_array() - truth.to_array())
    assert np.all(np.degrees(err[:3]) <= 6.0) and np.all(err[3:] <= 0.5)
    assert float(dice_under_transform(sm, tm, to_matrix(est, tm.physical_center()))) >= 0.94
    assert trace.ess[0] >= 1.0


# ---- resampling and the fused measurement (E/geometry.py:188-200,
#      E/kernels_numba.py:116-189; T/test_geometry.py, T/test_kernels.py) ----

def test_resample_identity_integer_shift_and_trilinear_fields():
    from paper_2504_19930_b200 import RigidParams, resample, to_matrix

    g = np.random.default_rng(6)
    src = g.standard_normal((9, 8, 10))
    v = _vol(src)
    assert np.array_equal(resample(v, v, np.eye(4)).data, src)
    # integer translation == array shift with fill 0 (pull-back: out(x) = src(x + d))
    moved = resample(v, v, to_matrix(RigidParams(tx=2.0, ty=-1.0, tz=0.0))).data
    want = np.zeros_like(src)
    want[:-2, 1:, :] = src[2:, :-1, :]
    assert np.array_equal(moved, want)
    # a trilinear polynomial field is reproduced exactly (up to rounding) anywhere
    i, j, k = np.meshgrid(np.arange(9.0), np.arange(8.0), np.arange(10.0), indexing="ij")
    c = g.uniform(-1, 1, 8)
    f = lambda x, y, z: (c[0] + c[1] * x + c[2] * y + c[3] * z + c[4] * x * y + c[5] * x * z
                         + c[6] * y * z + c[7] * x * y * z)
    m = to_matrix(RigidParams(0.03, -0.02, 0.05, 0.3, -0.4, 0.2), v.physical_center())
    out = resample(_vol(f(i, j, k)), v, m).data
    pts = np.einsum("ab,bijk->aijk", m[:3, :3], np.stack([i, j, k])) + m[:3, 3][:, None, None, None]
    inside = np.all((pts >= 0) & (pts <= np.array([8, 7, 9])[:, None, None, None]), axis=0)
    assert inside.sum() > 300
    assert np.allclose(out[inside], f(*pts)[inside], rtol=0, atol=1e-12)
    assert np.all(out[~inside] == 0.0)


@pytest.mark.parametrize("precision,tol", [("exact", 1e-9), ("f64", 1e-9), ("f32", 1e-4)])
def test_fused_measurement_equals_composed_warp_then_ncc(precision, tol):
    from paper_2504_19930_b200 import Executor, RigidParams, ncc, resample, to_matrix

    g = np.random.default_rng(7)
    t = _vol(g.integers(0, 256, (14, 12, 16)).astype(np.float64))
    s = _vol(np.roll(t.data, 1, axis=0) + g.integers(0, 40, (14, 12, 16)))
    mats = [to_matrix(RigidParams(*g.uniform(-0.1, 0.1, 3), *g.uniform(-2, 2, 3)),
                      t.physical_center()) for _ in range(6)]
    z, _ = Executor(precision=precision).measure_ncc(t, s, np.stack(mats))
    for p, m in enumerate(mats):
        want = float(ncc(t, resample(s, t, m)))
        assert abs(z[p] - want) <= tol * max(want, 1e-12), (p, z[p], want)


# ---- 4D pipeline, exhaustive search, phantom (T/test_pipeline.py,
#      T/test_exhaustive.py, T/test_phantom.py) -------------------------------

def _cycle(frames=3, amplitude=0.25, seed=3):
    from paper_2504_19930_b200 import PhantomSpec, RigidParams, make_pair
    from paper_2504_19930_b200.phantom_device import make_phantom_device

    spec = PhantomSpec(dims=(24, 24, 24), frames=frames, outer_semiaxes=(9.0, 7.5, 10.0),
                       inner_semiaxes=(6.0, 4.5, 7.0), amplitude=amplitude, seed=seed)
    seq, masks = make_phantom_device(spec)
    truth = RigidParams(math.radians(3.0), 0.0, math.radians(-2.0), 1.5, -1.0, 0.5)
    return make_pair(seq, masks, truth)


def test_pipeline_reports_errors_and_aggregates():
    from paper_2504_19930_b200 import (Executor, Sequence4, SmcConfig, Volume3,
                                       register_sequence)
    from paper_2504_19930_b200.errors import GeometryMismatch, MissingMasks

    case = _cycle()
    cfg = SmcConfig(mode="mask", n_particles=64, n_iterations=4, seed=1)
    rep = register_sequence(case.target, case.source, case.target_masks, case.source_masks,
                            cfg, Executor(workers=2))
    agg = rep.aggregates
    assert abs(agg["ncc_after_mean"] - float(np.mean(rep.ncc_after))) <= 1e-12
    assert abs(agg["dsc_before_std"] - float(np.std(rep.dsc_before))) <= 1e-12
    assert len(rep.dsc_after) == len(rep.ncc_before) == 3
    img = register_sequence(case.target, case.source, None, None,
                            SmcConfig(n_particles=32, n_iterations=3, seed=1))
    assert all(d is None for d in img.dsc_before + img.dsc_after)
    with pytest.raises(MissingMasks):
        register_sequence(case.target, case.source, None, None, cfg)
    other = Sequence4([Volume3(f.data, (1.0, 1.0, 1.1)) for f in case.source.frames])
    with pytest.raises(GeometryMismatch):
        register_sequence(case.target, other, case.target_masks, case.source_masks, cfg)


def test_exhaustive_identity_wins_when_aligned_and_beats_identity_score():
    from paper_2504_19930_b200 import Executor, GridSpec, RigidParams, register_exhaustive

    case = _cycle(frames=1)
    tm, sm = case.target_masks[0], case.source_masks[0]
    g = GridSpec(half_counts=(1, 0, 1, 1, 1, 0), step_r=3.0, step_t=1.5)
    best, _ = register_exhaustive(tm, tm, g)
    assert np.array_equal(best.to_array(), RigidParams().to_array())
    best, value = register_exhaustive(tm, sm, g)
    ident, _ = Executor().measure_ncc(tm, sm, np.eye(4))
    assert float(value) >= float(ident[0])


def test_device_phantom_cycle_properties():
    from paper_2504_19930_b200 import PhantomSpec
    from paper_2504_19930_b200.phantom_device import make_phantom_device

    spec = PhantomSpec(dims=(24, 24, 24), frames=4, outer_semiaxes=(9.0, 7.5, 10.0),
                       inner_semiaxes=(6.0, 4.5, 7.0), amplitude=0.3, seed=1)
    seq, masks = make_phantom_device(spec)
    assert seq.ed_index == 0
    raw = [m.codec.raw for m in masks]
    assert all(set(np.unique(r)) <= {0, 1} for r in raw)
    assert np.all(raw[0] >= raw[2]) and raw[0].sum() > raw[2].sum()   # ED contains mid-cycle
    frozen, _ = make_phantom_device(PhantomSpec(dims=(16, 16, 16), frames=3, amplitude=0.0,
                                                outer_semiaxes=(6.0, 5.0, 7.0),
                                                inner_semiaxes=(4.0, 3.0, 5.0), seed=4))
    assert all(np.array_equal(f.data, frozen.frames[0].data) for f in frozen.frames)
