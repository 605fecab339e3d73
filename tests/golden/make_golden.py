"""Generate golden fixtures from the REAL reference package (run in the build
container only; /root/reference does not exist on the GPU box).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Every array written here comes out of the reference's own code path
(echoreg.kernels_numba through echoreg.backend.Executor, echoreg.smc,
echoreg.exhaustive, echoreg.geometry, numpy's Philox streams as used by
echoreg.smc._stream).  The fixtures pin the C oracle (tests/test_oracle.py)
and the sm_100a kernels (tests/test_gpu_*.py).
"""

from __future__ import annotations

import hashlib
import math
import os
import sys

os.environ.setdefault("NUMBA_NUM_THREADS", "8")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import echoreg  # noqa: E402
from echoreg import geometry, kernels_numba, kernels_numpy, smc  # noqa: E402
from echoreg.backend import Executor  # noqa: E402
from echoreg.exhaustive import GridSpec, _node_states, register_exhaustive  # noqa: E402
from echoreg.geometry import RigidParams, index_affine, to_matrix  # noqa: E402
from echoreg.phantom import PhantomSpec, make_pair, make_phantom  # noqa: E402
from echoreg.volume import Volume3, normalize_zscore  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def random_volume(rng, dims, spacing=None, origin=None):
    """Same construction as the reference's tests/conftest.py:30-41."""
    data = rng.random(dims, dtype=np.float32).astype(np.float64)
    spacing = spacing or tuple(np.float32(s) for s in rng.uniform(0.5, 2.0, 3))
    origin = origin if origin is not None else tuple(
        np.float32(o) for o in rng.uniform(-10.0, 10.0, 3)
    )
    return Volume3(data, spacing, origin)


def random_mats(rng, center, count, rmax=0.4, tmax=6.0):
    mats = []
    for _ in range(count):
        p = RigidParams(*rng.uniform(-rmax, rmax, 3), *rng.uniform(-tmax, tmax, 3))
        mats.append(to_matrix(p, center))
    return np.stack(mats)


def affines(mats, source, target):
    a = np.empty((len(mats), 3, 3))
    b = np.empty((len(mats), 3))
    for i, m in enumerate(mats):
        a[i], b[i] = index_affine(m, source, target)
    return a, b


def overlap_counts(tgt, src, a, b):
    """In-bounds counts from the reference's numpy backend mask
    (kernels_numpy.sample_with_mask, kernels_numpy.py:40-62)."""
    return np.array(
        [int(kernels_numpy.sample_with_mask(src, a[p], b[p], tgt.shape)[1].sum())
         for p in range(a.shape[0])],
        dtype=np.int64,
    )


def kernels_cases():
    rng = np.random.default_rng(12345)
    cases = {}
    specs = [
        ("cube10", (10, 9, 8), (10, 9, 8), 24, 0.4, 6.0, True),
        ("ragged", (7, 11, 5), (9, 6, 13), 24, 0.6, 4.0, False),
        ("flat", (5, 1, 7), (6, 3, 7), 12, 0.3, 2.0, False),
        ("wide", (12, 11, 10), (12, 11, 10), 32, 1.2, 9.0, True),
        ("tiny_src", (4, 4, 4), (1, 1, 1), 6, 0.2, 0.5, False),
    ]
    for name, tdims, sdims, count, rmax, tmax, same_grid in specs:
        tgt = random_volume(rng, tdims)
        if same_grid:
            src = random_volume(rng, sdims, spacing=tgt.spacing, origin=tgt.origin)
        else:
            src = random_volume(rng, sdims)
        mats = random_mats(rng, tgt.physical_center(), count, rmax, tmax)
        # extra rows: identity, far out of frame, exact quarter turn
        extra = [np.eye(4), to_matrix(RigidParams(tx=1e5)),
                 to_matrix(RigidParams(rz=math.pi / 2), tgt.physical_center())]
        mats = np.concatenate([mats, np.stack(extra)])
        a, b = affines(mats, src, tgt)
        full, dfull = Executor(backend="numba").measure_ncc(tgt, src, mats, False)
        over, dover = Executor(backend="numba").measure_ncc(tgt, src, mats, True)
        counts = overlap_counts(tgt.data, src.data, a, b)
        res = np.stack([
            kernels_numba.resample_trilinear(src.data, a[p], b[p], tgt.dims)
            for p in range(min(4, len(mats)))
        ])
        cases[name] = dict(
            tgt=tgt.data, src=src.data,
            tgt_spacing=np.array(tgt.spacing), tgt_origin=np.array(tgt.origin),
            src_spacing=np.array(src.spacing), src_origin=np.array(src.origin),
            mats=mats, a=a, b=b, ncc_full=full, degen_full=dfull,
            ncc_overlap=over, degen_overlap=dover, n_in=counts, resampled=res,
        )
    # binary-mask case with rotations (reference tests/test_kernels.py:126-138)
    arr = np.zeros((12, 12, 12))
    arr[3:9, 4:8, 2:10] = 1.0
    tgt = Volume3(arr)
    mats = np.stack([
        to_matrix(RigidParams(rx=math.radians(d), tz=1.5, ry=math.radians(-d / 2)),
                  tgt.physical_center())
        for d in (-20, -10, -3, 0, 3, 10, 20)
    ])
    a, b = affines(mats, tgt, tgt)
    full, dfull = Executor(backend="numba").measure_ncc(tgt, tgt, mats, False)
    over, dover = Executor(backend="numba").measure_ncc(tgt, tgt, mats, True)
    cases["mask12"] = dict(
        tgt=tgt.data, src=tgt.data,
        tgt_spacing=np.ones(3), tgt_origin=np.zeros(3),
        src_spacing=np.ones(3), src_origin=np.zeros(3),
        mats=mats, a=a, b=b, ncc_full=full, degen_full=dfull,
        ncc_overlap=over, degen_overlap=dover,
        n_in=overlap_counts(tgt.data, tgt.data, a, b),
        resampled=np.stack([kernels_numba.resample_trilinear(tgt.data, a[p], b[p], tgt.dims)
                            for p in range(4)]),
    )
    flat = {}
    for name, d in cases.items():
        for k, v in d.items():
            flat[f"{name}__{k}"] = np.asarray(v)
    flat["case_names"] = np.array(list(cases.keys()))
    np.savez_compressed(os.path.join(OUT, "kernels.npz"), **flat)
    print("kernels.npz", len(cases), "cases")


def rng_cases():
    out = {}
    for seed, n in ((0, 500), (99, 7), (3, 2000)):
        cfg = smc.SmcConfig(n_particles=n, seed=seed)
        out[f"init_{seed}_{n}"] = smc.init_particles(cfg).states
    idx = np.arange(1000)
    for seed, k in ((0, 0), (0, 3), (7, 19), (2**31 + 5, 1)):
        out[f"normals_{seed}_{k}"] = np.stack(
            [smc._stream(seed, 1, k, int(i)).standard_normal(6) for i in idx])
    for seed in (0, 9):
        out[f"resample_u0_{seed}"] = np.array(
            [smc._stream(seed, 2, k, 0).uniform(0.0, 1.0 / 500) for k in range(50)])
    # a long single stream exercises the ziggurat wedge and tail branches
    out["long_normals"] = smc._stream(5, 1, 2, 3).standard_normal(300_000)
    # predict() end to end on a known population
    cfg = smc.SmcConfig(n_particles=300, seed=4, sigma0_r=3.0, sigma0_t=4.0)
    ps = smc.init_particles(cfg)
    ps.iteration = 6
    out["predict_in"] = ps.states
    out["predict_out"] = smc.predict(ps, cfg).states
    # hard clamp exercise
    cfg2 = smc.SmcConfig(n_particles=64, sigma0_t=500.0, sigma0_r=500.0, seed=1)
    ps2 = smc.init_particles(cfg2)
    out["clamp_in"] = ps2.states
    out["clamp_out"] = smc.predict(ps2, cfg2).states
    np.savez_compressed(os.path.join(OUT, "rng.npz"), **out)
    print("rng.npz")


def geometry_cases():
    rng = np.random.default_rng(777)
    params = np.concatenate([
        rng.uniform(-0.6, 0.6, (300, 3)), rng.uniform(-25.0, 25.0, (300, 3))], axis=1)
    centers = rng.uniform(-40, 80, (300, 3))
    mats = np.stack([to_matrix(RigidParams.from_array(p), c)
                     for p, c in zip(params, centers)])
    tgt = random_volume(rng, (5, 6, 7))
    src = random_volume(rng, (6, 5, 4))
    a, b = affines(mats, src, tgt)
    np.savez_compressed(
        os.path.join(OUT, "geometry.npz"), params=params, centers=centers, mats=mats,
        tgt_spacing=np.array(tgt.spacing), tgt_origin=np.array(tgt.origin),
        src_spacing=np.array(src.spacing), src_origin=np.array(src.origin),
        a=a, b=b)
    print("geometry.npz")


class RecordingExecutor(Executor):
    """Records every batch the SMC loop measures (reference seam,
    backend.py:78-108) without changing behaviour."""

    def __init__(self, *args, **kw):
        super().__init__(*args, **kw)
        object.__setattr__(self, "log", [])

    def measure_ncc(self, target, source, mats, overlap_only=False):
        out = super().measure_ncc(target, source, mats, overlap_only)
        self.log.append((np.array(mats), out[0].copy(), out[1].copy()))
        return out


def trace_arrays(prefix, est, trace, rec):
    d = {
        f"{prefix}estimate": est.to_array(),
        f"{prefix}estimates": np.stack([e.to_array() for e in trace.estimates]),
        f"{prefix}mean_measurement": np.array(trace.mean_measurement),
        f"{prefix}max_measurement": np.array(trace.max_measurement),
        f"{prefix}best_measurement": np.array(trace.best_measurement),
        f"{prefix}ess": np.array(trace.ess),
        f"{prefix}resampled": np.array(trace.resampled),
        f"{prefix}best_particle": (trace.best_particle.to_array()
                                   if trace.best_particle else np.zeros(0)),
        f"{prefix}z": np.stack([z for _, z, _ in rec.log]),
        f"{prefix}degen": np.stack([dg for _, _, dg in rec.log]),
    }
    dsc = [x if x is not None else np.nan for x in trace.dsc]
    d[f"{prefix}dsc"] = np.array(dsc, dtype=np.float64)
    return d


def smc_cases():
    out = {}
    # C1: SPEC acceptance case, mask mode 64^3, 500 x 20
    seq, masks = make_phantom(PhantomSpec(dims=(64, 64, 64), frames=1, seed=0))
    truth = RigidParams(math.radians(5), math.radians(-8), math.radians(4), 6.0, -4.0, 3.0)
    case = make_pair(seq, masks, truth)
    tm, sm = case.target_masks[0], case.source_masks[0]
    cfg = smc.SmcConfig(mode="mask", n_particles=500, n_iterations=20, seed=0)
    rec = RecordingExecutor(workers=8)
    est, trace = smc.register_smc(tm, sm, cfg, rec)
    out.update(trace_arrays("c1_", est, trace, rec))
    out["c1_target_bits"] = np.packbits(tm.data.astype(np.uint8).ravel())
    out["c1_source_bits"] = np.packbits(sm.data.astype(np.uint8).ravel())
    out["c1_dims"] = np.array(tm.dims)
    out["c1_truth"] = truth.to_array()
    # iteration-0 and iteration-1 particle matrices (lock-step inputs)
    out["c1_mats_it0"] = rec.log[0][0]
    out["c1_mats_it1"] = rec.log[1][0]
    a, b = affines(rec.log[0][0], sm, tm)
    out["c1_a_it0"], out["c1_b_it0"] = a, b
    # the same run in overlap mode (short) for n_in-sensitive parity
    cfg_o = smc.SmcConfig(mode="mask", n_particles=200, n_iterations=6, seed=3,
                          ncc_region="overlap")
    rec_o = RecordingExecutor(workers=8)
    est_o, trace_o = smc.register_smc(tm, sm, cfg_o, rec_o)
    out.update(trace_arrays("c1o_", est_o, trace_o, rec_o))

    # image mode on a 32^3 normalized phantom (float64 speckle, not quantized)
    seq, masks = make_phantom(PhantomSpec(
        dims=(32, 32, 32), frames=1, seed=4, outer_semiaxes=(11.0, 9.0, 13.0),
        inner_semiaxes=(7.0, 5.5, 8.5), speckle_sigma=0.3))
    truth = RigidParams(math.radians(3), math.radians(-4), math.radians(2), 2.0, -1.5, 1.0)
    case = make_pair(seq, masks, truth)
    ti = normalize_zscore(case.target.frames[0])
    si = normalize_zscore(case.source.frames[0])
    cfg_i = smc.SmcConfig(mode="image", n_particles=96, n_iterations=10, seed=2,
                          t_limit=6.0, r_limit=8.0)
    rec_i = RecordingExecutor(workers=8)
    est_i, trace_i = smc.register_smc(ti, si, cfg_i, rec_i,
                                      trace_masks=(case.target_masks[0], case.source_masks[0]))
    out.update(trace_arrays("img_", est_i, trace_i, rec_i))
    out["img_target"] = ti.data
    out["img_source"] = si.data
    out["img_target_mask"] = case.target_masks[0].data.astype(np.uint8)
    out["img_source_mask"] = case.source_masks[0].data.astype(np.uint8)
    out["img_truth"] = truth.to_array()
    np.savez_compressed(os.path.join(OUT, "smc.npz"), **out)
    print("smc.npz c1 est", np.degrees(est.to_array()[:3]), est.to_array()[3:])


def c1seeds_cases():
    """C1 (SPEC acceptance case, mask mode 64^3, 500 x 20) at SMC seeds 1..8:
    the reference's trajectory per seed (c1_seeds.npz)."""
    seq, masks = make_phantom(PhantomSpec(dims=(64, 64, 64), frames=1, seed=0))
    truth = RigidParams(math.radians(5), math.radians(-8), math.radians(4), 6.0, -4.0, 3.0)
    case = make_pair(seq, masks, truth)
    tm, sm = case.target_masks[0], case.source_masks[0]
    out = {"seeds": np.arange(1, 9)}
    est_all, ess_all, res_all = [], [], []
    for seed in range(1, 9):
        cfg = smc.SmcConfig(mode="mask", n_particles=500, n_iterations=20, seed=seed)
        est, trace = smc.register_smc(tm, sm, cfg, Executor(workers=8))
        est_all.append(np.stack([e.to_array() for e in trace.estimates]))
        ess_all.append(np.array(trace.ess))
        res_all.append(np.array(trace.resampled))
    out["estimates"] = np.stack(est_all)
    out["ess"] = np.stack(ess_all)
    out["resampled"] = np.stack(res_all)
    out["target_bits"] = np.packbits(tm.data.astype(np.uint8).ravel())
    out["source_bits"] = np.packbits(sm.data.astype(np.uint8).ravel())
    np.savez_compressed(os.path.join(OUT, "c1_seeds.npz"), **out)
    print("c1_seeds.npz final estimates (deg)", np.degrees(out["estimates"][:, -1, :3]))


def exhaustive_cases():
    spec = PhantomSpec(dims=(16, 16, 16), frames=1, outer_semiaxes=(6.0, 5.0, 7.0),
                       inner_semiaxes=(4.0, 3.0, 5.0), speckle_sigma=0.25,
                       amplitude=0.0, seed=5)
    seq, masks = make_phantom(spec)
    truth = RigidParams(tx=1.0, ty=-1.0)
    case = make_pair(seq, masks, truth)
    t = normalize_zscore(case.target.frames[0])
    s = normalize_zscore(case.source.frames[0])
    out = {"target": t.data, "source": s.data}
    for name, g in (("g1", GridSpec(half_counts=(1, 1, 1, 1, 1, 1), step_t=1.0, step_r=2.0)),
                    ("g2", GridSpec(half_counts=(0, 1, 0, 2, 2, 0), step_t=0.5, step_r=3.0))):
        best, value = register_exhaustive(t, s, g, Executor(workers=8))
        states = _node_states(g)
        mats = np.stack([to_matrix(RigidParams.from_array(r), t.physical_center())
                         for r in states])
        scores, _ = Executor(workers=8).measure_ncc(t, s, mats)
        out[f"{name}_half_counts"] = np.array(g.half_counts)
        out[f"{name}_steps"] = np.array([g.step_t, g.step_r])
        out[f"{name}_best"] = best.to_array()
        out[f"{name}_value"] = np.array(float(value))
        out[f"{name}_scores"] = scores
        out[f"{name}_states"] = states
    np.savez_compressed(os.path.join(OUT, "exhaustive.npz"), **out)
    print("exhaustive.npz")


def phantom_cases():
    """Digests of the reference generator so our port can be pinned."""
    out = {}
    spec = PhantomSpec(dims=(20, 18, 22), spacing=(1.1, 0.9, 1.3), frames=3, seed=11,
                       outer_semiaxes=(8.0, 7.0, 9.0), inner_semiaxes=(5.0, 4.0, 6.0))
    seq, masks = make_phantom(spec)
    truth = RigidParams(math.radians(6), math.radians(-3), math.radians(2), 1.5, -2.0, 0.5)
    case = make_pair(seq, masks, truth, overlap_crop=0.2)
    out["frames"] = np.stack([f.data for f in seq.frames])
    out["masks"] = np.stack([m.data for m in masks]).astype(np.uint8)
    out["src_frames"] = np.stack([f.data for f in case.source.frames])
    out["src_masks"] = np.stack([m.data for m in case.source_masks]).astype(np.uint8)
    out["initial_dsc"] = np.array(case.initial_dsc)
    np.savez_compressed(os.path.join(OUT, "phantom.npz"), **out)
    print("phantom.npz")


def pipeline_cases():
    from echoreg.pipeline import register_sequence

    spec = PhantomSpec(dims=(24, 24, 24), frames=4, outer_semiaxes=(9.0, 7.5, 10.0),
                       inner_semiaxes=(6.0, 4.5, 7.0), speckle_sigma=0.2, seed=2)
    seq, masks = make_phantom(spec)
    truth = RigidParams(math.radians(4.0), 0.0, math.radians(-3.0), 2.5, -1.5, 1.0)
    case = make_pair(seq, masks, truth)
    cfg = smc.SmcConfig(mode="mask", n_particles=64, n_iterations=8, seed=1,
                        t_limit=6.0, r_limit=8.0)
    rep = register_sequence(case.target, case.source, case.target_masks,
                            case.source_masks, cfg, Executor(workers=8))
    out = {
        "target": np.stack([f.data for f in case.target.frames]),
        "source": np.stack([f.data for f in case.source.frames]),
        "target_masks": np.stack([m.data for m in case.target_masks]).astype(np.uint8),
        "source_masks": np.stack([m.data for m in case.source_masks]).astype(np.uint8),
        "ncc_before": np.array(rep.ncc_before), "ncc_after": np.array(rep.ncc_after),
        "dsc_before": np.array(rep.dsc_before), "dsc_after": np.array(rep.dsc_after),
        "estimate": np.array([rep.estimate_deg_mm[k] for k in
                              ("rx_deg", "ry_deg", "rz_deg", "tx_mm", "ty_mm", "tz_mm")]),
        "trace_dsc": np.array(rep.trace["dsc"], dtype=np.float64),
    }
    np.savez_compressed(os.path.join(OUT, "pipeline.npz"), **out)
    print("pipeline.npz")


def zscore_cases():
    """normalize_zscore on 8-bit data (volume.py:119-130): the reference's mean,
    population std and normalised values for byte volumes of several shapes
    and level distributions."""
    rng = np.random.default_rng(2024)
    out = {}
    shapes = [(5, 6, 7), (17, 9, 23), (40, 36, 44), (64, 64, 64), (88, 88, 104)]
    for i, dims in enumerate(shapes):
        for j, kind in enumerate(("uniform", "skewed", "sparse")):
            if kind == "uniform":
                raw = rng.integers(0, 256, dims)
            elif kind == "skewed":
                raw = np.clip(np.round(rng.lognormal(3.0, 0.8, dims)), 0, 255)
            else:
                raw = np.where(rng.random(dims) < 0.1, rng.integers(1, 256, dims), 0)
            raw = raw.astype(np.uint8)
            v = Volume3(raw.astype(np.float64))
            z = normalize_zscore(v)
            key = f"v{i}_{kind}"
            out[f"{key}__raw"] = raw
            out[f"{key}__mean"] = np.array(float(v.data.mean()))
            out[f"{key}__std"] = np.array(float(v.data.std()))
            if raw.size <= 64 ** 3:
                out[f"{key}__z"] = z.data
    np.savez_compressed(os.path.join(OUT, "zscore.npz"), **out)
    print("zscore.npz", len(out))


def report_cases():
    """RegistrationReport JSON (pipeline.py:32-76), percentile_summary and its
    CSV (pipeline.py:273-308), written by the reference itself."""
    import json

    from echoreg.pipeline import (RegistrationReport, percentile_summary,
                                  write_summary_csv)

    rng = np.random.default_rng(77)
    reports = []
    for c in range(9):
        nf = int(rng.integers(2, 6))
        before = [float(x) for x in rng.uniform(0.5, 0.9, nf)]
        after = [float(min(1.0, b + d)) for b, d in zip(before, rng.uniform(-0.05, 0.3, nf))]
        if c == 3:
            before[1] = after[1] = None          # a frame without masks
        if c == 5:
            before = [None] * nf                 # no DSC at all: excluded from the summary
            after = [None] * nf
        ncc_b = [float(x) for x in rng.uniform(0.1, 0.6, nf)]
        ncc_a = [float(x) for x in rng.uniform(0.4, 0.95, nf)]
        from echoreg.pipeline import _aggregates

        rep = RegistrationReport(
            mode="mask", method="smc", config={"n_particles": 64, "seed": c},
            estimate_deg_mm={"rx_deg": 1.0 * c, "ry_deg": -0.5, "rz_deg": 0.25,
                             "tx_mm": 2.0, "ty_mm": -1.0, "tz_mm": 0.5},
            best_estimate_deg_mm=None, ncc_before=ncc_b, ncc_after=ncc_a,
            dsc_before=before, dsc_after=after,
            aggregates=_aggregates(ncc_b, ncc_a, before, after), trace=None,
            wall_time_s=0.125 * c, case_id=f"case{c:02d}")
        reports.append(rep)
    rows = percentile_summary(reports)
    path_csv = os.path.join(OUT, "report_summary.csv")
    write_summary_csv(rows, path_csv)
    paths = []
    for rep in reports:
        p = os.path.join("/tmp", f"er_report_{rep.case_id}.json")
        rep.save(p)
        paths.append(open(p).read())
    with open(os.path.join(OUT, "report_cases.json"), "w") as fh:
        json.dump({"reports": [r.to_dict() for r in reports], "saved": paths,
                   "summary": rows}, fh, indent=1)
    print("report_cases.json", len(reports))


def exhaustive_sequence_cases():
    """exhaustive_sequence (pipeline.py:219-266) on a small 4D case, image and
    mask mode, through the reference's numba backend."""
    import json

    from echoreg.pipeline import exhaustive_sequence

    spec = PhantomSpec(dims=(20, 18, 22), frames=3, outer_semiaxes=(7.5, 6.5, 8.5),
                       inner_semiaxes=(5.0, 4.0, 5.5), speckle_sigma=0.2, seed=9)
    seq, masks = make_phantom(spec)
    truth = RigidParams(0.0, math.radians(2.0), 0.0, 1.0, -1.0, 0.5)
    case = make_pair(seq, masks, truth)
    grid = GridSpec(half_counts=(0, 1, 0, 1, 1, 1), step_t=0.5, step_r=2.0)
    out = {"target": np.stack([f.data for f in case.target.frames]),
           "source": np.stack([f.data for f in case.source.frames]),
           "target_masks": np.stack([m.data for m in case.target_masks]).astype(np.uint8),
           "source_masks": np.stack([m.data for m in case.source_masks]).astype(np.uint8),
           "spacing": np.array(spec.spacing)}
    reps = {}
    for mode in ("image", "mask"):
        rep = exhaustive_sequence(case.target, case.source, case.target_masks,
                                  case.source_masks, grid, mode=mode,
                                  executor=Executor(workers=8), case_id=f"ex_{mode}")
        d = rep.to_dict()
        d.pop("wall_time_s")
        reps[mode] = d
    np.savez_compressed(os.path.join(OUT, "exhaustive_sequence.npz"), **out)
    with open(os.path.join(OUT, "exhaustive_sequence.json"), "w") as fh:
        json.dump({"grid": {"half_counts": list(grid.half_counts), "step_t": grid.step_t,
                            "step_r": grid.step_r}, "reports": reps}, fh, indent=1)
    print("exhaustive_sequence", {m: r["estimate_deg_mm"] for m, r in reps.items()})


if __name__ == "__main__":
    print("reference echoreg", echoreg.__version__, "numpy", np.__version__)
    which = sys.argv[1:] or ["kernels", "rng", "geometry", "smc", "exhaustive",
                             "phantom", "pipeline", "zscore", "report", "exhaustive_sequence"]
    for w in which:
        globals()[f"{w}_cases"]()
    with open(os.path.join(OUT, "SHA256SUMS"), "w") as fh:
        for f in sorted(os.listdir(OUT)):
            if f.endswith(".npz"):
                h = hashlib.sha256(open(os.path.join(OUT, f), "rb").read()).hexdigest()
                fh.write(f"{h}  {f}\n")
