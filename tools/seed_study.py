"""Trajectory drift of the fast precision modes at full BASELINE scale.

The reference-op-order mode (precision="exact") reproduces the reference
algorithm's final transform to ~1e-14 (tools/parity_full.py, tests), so it
stands in for the reference here: for seeds 0..N-1 run C2 (image, 2000 x 50)
and a C3-style mask registration (2000 x 50 on the 176x176x208 masks) in
f32 / f64 / exact and report the final-transform differences.

    python tools/seed_study.py [n_seeds] [image,mask] [first_seed]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_2504_19930_b200 import Executor, SmcConfig, binarize, register_smc

n_seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 8
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["image", "mask"]
first = int(sys.argv[3]) if len(sys.argv) > 3 else 0
t, s, case = bench.make_workload()
tm, sm = binarize(case.target_masks[0], 0.5), binarize(case.source_masks[0], 0.5)
sp = np.asarray(t.spacing)
for mode, (a, b) in (("image", (t, s)), ("mask", (tm, sm))):
    if mode not in modes:
        continue
    rows = []
    for seed in range(first, first + n_seeds):
        cfg = SmcConfig(mode=mode, n_particles=2000, n_iterations=50, seed=seed)
        res = {}
        for prec in ("exact", "f64", "f32"):
            t0 = time.perf_counter()
            est, tr = register_smc(a, b, cfg, Executor(precision=prec))
            res[prec] = (est.to_array(), time.perf_counter() - t0, tr.resampled)
        row = {"seed": seed}
        for prec in ("f64", "f32"):
            d = res[prec][0] - res["exact"][0]
            row[f"{prec}_deg"] = float(np.degrees(np.abs(d[:3])).max())
            row[f"{prec}_vox"] = float((np.abs(d[3:]) / sp).max())
            row[f"{prec}_same_flags"] = res[prec][2] == res["exact"][2]
            row[f"{prec}_s"] = res[prec][1]
        row["exact_s"] = res["exact"][1]
        rows.append(row)
        print(mode, json.dumps(row), flush=True)
    for prec in ("f64", "f32"):
        print(mode, prec, "worst deg", max(r[f"{prec}_deg"] for r in rows),
              "worst vox", max(r[f"{prec}_vox"] for r in rows), flush=True)
