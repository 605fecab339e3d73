"""Randomised differential test of the measurement against the C oracle
(bit-exact restatement of the reference kernel): random target/source dims
(1..40 per axis, independent), spacings, origins, storage (u8 / binary /
f32-exact / f64), affines (near identity, large rotations, far out of frame)
and region mode, every precision.  Counts and degenerate flags must be
bit-exact; likelihoods within the mode's tolerance (relative, with the absolute
floors below; f32 strictly, since the device re-measures its ill-conditioned
particles in fp64) -- or, in the fp64 modes, for ill-conditioned particles within 2 eps kappa (eps the
mode's unit roundoff, kappa the particle's condition number, conditioning()),
which is the accuracy any evaluation at that precision or in another summation
order allows; a degenerate flag may differ only where 2 eps kappa >= 1 (the
sampled variance is below the precision's resolution).

    python tools/fuzz_measure.py [n_cases] [seed]      (prints a JSON summary)
    python tools/fuzz_measure.py [n_cases] [seed] warp
    python tools/fuzz_measure.py [n_cases] [seed] c1,c2,...  (replay those cases)

Failures carry the particle's condition number kappa (see conditioning()) and
the error in units of eps * kappa, eps the mode's unit roundoff.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

RTOL = {"f32": 1e-4, "f64": 1e-6, "exact": 1e-10}
# absolute floors: fp32 sampling resolves z (in [0, 1]) to ~1e-7 once the
# sts^2 cancellation of a decorrelated particle dominates (e.g. 4 in-bounds
# voxels, z = 3.9e-4: |dz| = 4e-8); the fp64 modes keep 1e-12
ATOL = {"f32": 1e-12, "f64": 1e-12, "exact": 1e-12}


def random_case(g):
    from paper_2504_19930_b200 import Volume3

    tdims = tuple(int(x) for x in g.integers(1, 41, 3))
    sdims = tuple(int(x) for x in g.integers(1, 41, 3)) if g.random() < 0.5 else tdims
    kind = g.choice(["u8", "binary", "f32", "f64"])

    def data(d):
        if kind == "u8":
            return g.integers(0, 256, d).astype(np.float64)
        if kind == "binary":
            return (g.random(d) < g.uniform(0.2, 0.8)).astype(np.float64)
        if kind == "f32":
            return g.standard_normal(d).astype(np.float32).astype(np.float64)
        return g.standard_normal(d)

    sp_t = tuple(g.uniform(0.5, 1.5, 3))
    sp_s = sp_t if g.random() < 0.5 else tuple(g.uniform(0.5, 1.5, 3))
    org = (0.0, 0.0, 0.0) if g.random() < 0.5 else tuple(g.uniform(-3, 3, 3))
    t = Volume3(data(tdims), sp_t)
    s = Volume3(data(sdims), sp_s, org)
    n = int(g.integers(1, 24))
    rot = g.choice([0.05, 0.5, 3.0])
    shift = g.choice([1.0, 5.0, 60.0])
    mats = []
    from paper_2504_19930_b200 import RigidParams, to_matrix

    for _ in range(n):
        p = RigidParams(*g.uniform(-rot, rot, 3), *g.uniform(-shift, shift, 3))
        mats.append(to_matrix(p, t.physical_center()))
    return t, s, np.stack(mats), bool(g.random() < 0.5), kind


EPS = {"f32": 2.0 ** -24, "f64": 2.0 ** -53, "exact": 2.0 ** -53}


def conditioning(t, s, a, b, overlap):
    """Per particle, the condition number of z = sts^2 / (sst sss) under
    perturbations of the samples and of the summation order:
    kappa = kappa_s + kappa_t + 2 kappa_ts with kappa_s = sum x^2 / sss,
    kappa_t = sum t^2 / sst, kappa_ts = sqrt(sum x^2 sum t^2) / |sts| over the
    region (in-bounds voxels in overlap mode, else all; x = 0 outside).  A
    relative error of order eps * kappa is the accuracy any summation order
    or sample rounding of that size allows.  Built on the oracle's
    resampler (the reference's _resample_kernel)."""
    from oracle import kernels as ok

    ones = np.ones(s.dims)
    out = []
    for p in range(a.shape[0]):
        x = ok.resample_trilinear(s.data, a[p], b[p], t.dims)
        m = ok.resample_trilinear(ones, a[p], b[p], t.dims) > 0.5
        if overlap:
            xs, ts = x[m], t.data[m]
        else:
            xs, ts = np.where(m, x, 0.0).ravel(), t.data.ravel()
        n = xs.size
        if n == 0:
            out.append(np.inf)
            continue
        sxx, stt = np.float64((xs * xs).sum()), np.float64((ts * ts).sum())
        sss = sxx - np.float64(xs.sum()) ** 2 / n
        sst = stt - np.float64(ts.sum()) ** 2 / n
        sts = np.float64((xs * ts).sum()) - np.float64(xs.sum()) * np.float64(ts.sum()) / n
        with np.errstate(divide="ignore", invalid="ignore"):
            k = sxx / abs(sss) + stt / abs(sst) + 2.0 * np.sqrt(sxx * stt) / abs(sts)
        out.append(float(k) if np.isfinite(k) else np.inf)
    return np.asarray(out)


def run(n_cases=200, seed=0, only=None, strict=("f32",)):
    """``only``: replay just these case indices of the seed's sequence.
    ``strict``: precisions held to their plain bar (no conditioning
    allowance); f32 by default, whose ill-conditioned particles the
    device refines in fp64."""
    from oracle import kernels as ok
    from paper_2504_19930_b200 import ops
    from paper_2504_19930_b200.device import device_volume, require_cuda, torch
    from paper_2504_19930_b200.geometry import index_affine_batch

    t_ = torch()
    dev = require_cuda()
    g = np.random.default_rng(seed)
    worst = {p: 0.0 for p in RTOL}
    conditioned = {p: [] for p in RTOL}
    failures = []
    for c in range(n_cases):
        t, s, mats, overlap, kind = random_case(g)
        if only is not None and c not in only:
            continue
        a, b = index_affine_batch(mats, s.spacing, s.origin, t.spacing, t.origin)
        zo, do, no = ok.ncc_measure_batch(t.data, s.data, a, b, overlap, return_counts=True)
        tdv, sdv = device_volume(t, dev), device_volume(s, dev)
        A = t_.as_tensor(a.reshape(-1, 9), device=dev)
        B = t_.as_tensor(b.reshape(-1, 3), device=dev)
        kap = None
        for prec, rtol in RTOL.items():
            z, d, n = (x.cpu().numpy() for x in ops.measure(tdv, sdv, A, B, overlap, prec))
            scale = np.maximum(np.abs(zo), 1e-300)
            rel = np.abs(z - zo) / scale
            atol = ATOL[prec]
            flags = d.astype(bool) == do
            bad = (np.abs(z - zo) > rtol * scale + atol) | ((zo == 0) != (z == 0)) | ~flags
            worst[prec] = max(worst[prec], float(np.where(np.abs(z - zo) > atol, rel, 0).max()))
            counts_ok = np.array_equal(n, no)
            if not bad.any() and counts_ok:
                continue
            # the mode's bar missed: accept a particle whose error is within
            # what its conditioning allows at this precision (2 eps kappa), and
            # a degenerate flag only where the variance is not resolved at all
            if kap is None:
                kap = conditioning(t, s, a, b, overlap)
            floor = 2.0 * EPS[prec] * kap
            cond_ok = (rel <= floor) & (flags | (floor >= 1.0))
            if prec in strict:
                cond_ok = np.zeros_like(cond_ok)
            still = bad & ~cond_ok
            for q in np.flatnonzero(bad & cond_ok):
                conditioned[prec].append(float(rel[q] / (EPS[prec] * kap[q])))
            if still.any() or not counts_ok:
                q = int(np.argmax(np.where(still, rel, 0.0))) if still.any() else 0
                failures.append({"case": c, "precision": prec, "kind": kind, "overlap": overlap,
                                 "tdims": t.dims, "sdims": s.dims,
                                 "max_rel": float(rel.max()),
                                 "z_ref": float(zo[q]), "z": float(z[q]),
                                 "kappa": float(kap[q]),
                                 "rel_over_eps_kappa": float(rel[q] / (EPS[prec] * kap[q])),
                                 "counts_equal": bool(counts_ok),
                                 "degen_equal": bool(flags.all())})
    return {"cases": n_cases, "seed": seed, "failures": failures,
            "worst_rel_err_above_atol": worst,
            "within_conditioning_only": {p: {"particles": len(v),
                                             "worst_rel_over_eps_kappa": max(v, default=0.0)}
                                         for p, v in conditioned.items()}}


def run_warp(n_cases=200, seed=0):
    """The warp kernels on random cases: er_resample bit-exact with the
    oracle's resampler (the reference's _resample_kernel), the fused
    warp + Dice counts equal to binarising that warp and counting."""
    from oracle import kernels as ok
    from paper_2504_19930_b200 import RigidParams, Volume3, ops, to_matrix
    from paper_2504_19930_b200.geometry import index_affine

    g = np.random.default_rng(seed)
    failures = []
    for c in range(n_cases):
        t, s, mats, _, kind = random_case(g)
        m = mats[0]
        a, b = index_affine(m, s, t)
        want = ok.resample_trilinear(s.data, a, b, t.dims)
        got = ops.resample_device(s, a, b, t.dims).cpu().numpy()
        ok_resample = np.array_equal(got, want)
        sm = Volume3((g.random(s.dims) < 0.5).astype(np.float64), s.spacing, s.origin)
        tm = Volume3((g.random(t.dims) < 0.5).astype(np.float64), t.spacing, t.origin)
        moved = ok.resample_trilinear(sm.data, a, b, t.dims) > 0.5
        want_counts = [int(moved.sum()), int(tm.data.sum()), int((moved & (tm.data == 1)).sum())]
        got_counts = [int(x) for x in ops.dice_counts(sm, tm, a, b).cpu().numpy()]
        if not ok_resample or got_counts != want_counts:
            failures.append({"case": c, "kind": kind, "tdims": t.dims, "sdims": s.dims,
                             "resample_equal": ok_resample, "counts": got_counts,
                             "want_counts": want_counts})
    return {"cases": n_cases, "seed": seed, "failures": failures}


if __name__ == "__main__":
    if len(sys.argv) > 3 and sys.argv[3] == "warp":
        print(json.dumps(run_warp(int(sys.argv[1]), int(sys.argv[2]))))
        sys.exit(0)
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    sd = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    only = {int(c) for c in sys.argv[3].split(",")} if len(sys.argv) > 3 else None
    print(json.dumps(run(n, sd, only)))
