"""Full-scale C3 check of the 4D pipeline's scores (E/pipeline.py:110-138,
155-216): register_sequence on the 30-frame 176x176x208 echo pair (mask SMC,
2000 x 50) on the GPU, then every frame's NCC before/after and Dice
before/after recomputed on the host with the reference's algorithms under
the same transform -- the z-score of E/volume.py:119-130 in numpy, the
oracle's resampler (bit-exact restatement of _resample_kernel) and numpy
restatements of metrics.ncc / dice / dice_under_transform
(E/metrics.py:49-93).  The SMC estimate itself is checked against the
reference algorithm by tools/parity_full.py.

    python tools/parity_c3_scores.py [frames]      (prints one JSON line)
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from oracle import kernels as ok  # noqa: E402  (checker)
from paper_2504_19930_b200 import (Executor, SmcConfig, binarize, register_sequence,  # noqa: E402
                                   register_smc, to_matrix)
from paper_2504_19930_b200.geometry import index_affine  # noqa: E402
from paper_2504_19930_b200.phantom_device import echo_case_device  # noqa: E402


def zscore(raw):
    d = raw.astype(np.float64)
    return (d - d.mean()) / d.std()


def ncc_ref(t, s):
    """metrics.ncc (E/metrics.py:49-68); None where it raises DegenerateInput."""
    td, sd = t.ravel(), s.ravel()
    n = td.size
    dt, ds = td - td.mean(), sd - sd.mean()
    sst, sss = float(dt @ dt), float(ds @ ds)
    if sst / n < 1e-12 or sss / n < 1e-12:
        return None
    sts = float(dt @ ds)
    return (sts * sts) / (sst * sss)


def dice_ref(a, b):
    """metrics.dice (E/metrics.py:71-85)."""
    sa, sb = float(a.sum()), float(b.sum())
    if sa == 0.0 and sb == 0.0:
        return 1.0
    return 2.0 * float((a * b).sum()) / (sa + sb)


def main():
    frames = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    ok.build()
    threads = ok.max_threads()
    case = echo_case_device(frames=frames, seed=0)
    cfg = SmcConfig(mode="mask", n_particles=2000, n_iterations=50, seed=0)
    t0 = time.perf_counter()
    rep = register_sequence(case.target, case.source, case.target_masks, case.source_masks,
                            cfg, Executor())
    gpu_s = time.perf_counter() - t0
    # the pipeline's transform (register_sequence: to_matrix(est, ED mask centre))
    ed = case.target.ed_index
    reg_t = binarize(case.target_masks[ed], 0.5)
    reg_s = binarize(case.source_masks[ed], 0.5)
    est, _ = register_smc(reg_t, reg_s, cfg, Executor(), trace_masks=(reg_t, reg_s))
    matrix = to_matrix(est, reg_t.physical_center())
    t0 = time.perf_counter()
    ref = {"ncc_before": [], "ncc_after": [], "dsc_before": [], "dsc_after": []}
    for f in range(frames):
        tf, sf = case.target.frames[f], case.source.frames[f]
        tz, sz = zscore(tf.codec.raw), zscore(sf.codec.raw)
        ref["ncc_before"].append(ncc_ref(tz, sz))
        a, b = index_affine(matrix, sf, tf)
        moved = ok.resample_trilinear(sz, a, b, tf.dims, threads)
        after = ncc_ref(tz, moved)
        ref["ncc_after"].append(0.0 if after is None else after)
        tm = case.target_masks[f].codec.raw.astype(np.float64)
        sm = case.source_masks[f].codec.raw.astype(np.float64)
        ref["dsc_before"].append(dice_ref(tm, sm))
        am, bm = index_affine(matrix, case.source_masks[f], case.target_masks[f])
        mm = (ok.resample_trilinear(sm, am, bm, tf.dims, threads) > 0.5).astype(np.float64)
        ref["dsc_after"].append(dice_ref(mm, tm))
    cpu_s = time.perf_counter() - t0

    def rel(a, b):
        return max(abs(x - y) / max(abs(y), 1e-300) for x, y in zip(a, b))

    out = {
        "config": f"C3: {frames}-frame 176x176x208 echo pair, mask SMC 2000 x 50, register_sequence",
        "gpu_register_sequence_s": gpu_s, "host_rescoring_s": cpu_s, "host_threads": threads,
        "ncc_before_max_rel_diff": rel(rep.ncc_before, ref["ncc_before"]),
        "ncc_after_max_rel_diff": rel(rep.ncc_after, ref["ncc_after"]),
        "dsc_before_identical": rep.dsc_before == ref["dsc_before"],
        "dsc_after_identical": rep.dsc_after == ref["dsc_after"],
        "dsc_after_max_abs_diff": max(abs(x - y) for x, y in zip(rep.dsc_after,
                                                                 ref["dsc_after"])),
        "dsc_before_mean": float(np.mean(ref["dsc_before"])),
        "dsc_after_mean": float(np.mean(ref["dsc_after"])),
        "estimate_deg_mm": rep.estimate_deg_mm,
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
