"""Randomised differential test of the measurement against the C oracle
(bit-exact restatement of the reference kernel): random target/source dims
(1..40 per axis, independent), spacings, origins, storage (u8 / binary /
f32-exact / f64), affines (near identity, large rotations, far out of frame)
and region mode, every precision.  Counts and degenerate flags must be
bit-exact; likelihoods within the mode's tolerance (relative, with the absolute
floors below).

    python tools/fuzz_measure.py [n_cases] [seed]      (prints a JSON summary)
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
ATOL = {"f32": 1e-7, "f64": 1e-12, "exact": 1e-12}


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


def run(n_cases=200, seed=0):
    from oracle import kernels as ok
    from paper_2504_19930_b200 import ops
    from paper_2504_19930_b200.device import device_volume, require_cuda, torch
    from paper_2504_19930_b200.geometry import index_affine_batch

    t_ = torch()
    dev = require_cuda()
    g = np.random.default_rng(seed)
    worst = {p: 0.0 for p in RTOL}
    failures = []
    for c in range(n_cases):
        t, s, mats, overlap, kind = random_case(g)
        a, b = index_affine_batch(mats, s.spacing, s.origin, t.spacing, t.origin)
        zo, do, no = ok.ncc_measure_batch(t.data, s.data, a, b, overlap, return_counts=True)
        tdv, sdv = device_volume(t, dev), device_volume(s, dev)
        A = t_.as_tensor(a.reshape(-1, 9), device=dev)
        B = t_.as_tensor(b.reshape(-1, 3), device=dev)
        for prec, rtol in RTOL.items():
            z, d, n = (x.cpu().numpy() for x in ops.measure(tdv, sdv, A, B, overlap, prec))
            scale = np.maximum(np.abs(zo), 1e-300)
            rel = np.abs(z - zo) / scale
            atol = ATOL[prec]
            bad = (np.abs(z - zo) > rtol * scale + atol) | ((zo == 0) != (z == 0))
            worst[prec] = max(worst[prec], float(np.where(np.abs(z - zo) > atol, rel, 0).max()))
            if bad.any() or not np.array_equal(d.astype(bool), do) or not np.array_equal(n, no):
                failures.append({"case": c, "precision": prec, "kind": kind, "overlap": overlap,
                                 "tdims": t.dims, "sdims": s.dims,
                                 "max_rel": float(rel.max()),
                                 "counts_equal": bool(np.array_equal(n, no)),
                                 "degen_equal": bool(np.array_equal(d.astype(bool), do))})
    return {"cases": n_cases, "seed": seed, "failures": failures,
            "worst_rel_err_above_atol": worst}


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
    print(json.dumps(run(n, sd)))
