"""Quad fast path vs the generic gather kernel on C2-shaped NON-8-bit volumes
(the reference's fp64 speckle phantom, z-scored; stored f64, and its fp32
rounding stored f32): evals/s of one measurement launch, and the agreement
with the oracle on the same particles.  usage: quad_probe.py [P]   (GPU)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import kernels as ok  # noqa: E402
from paper_2504_19930_b200 import SmcConfig, Volume3, normalize_zscore, ops  # noqa: E402
from paper_2504_19930_b200 import smc as dsmc  # noqa: E402
from paper_2504_19930_b200.backend import Executor  # noqa: E402
from paper_2504_19930_b200.phantom import ECHO_SPACING, echo_spec, make_pair  # noqa: E402
from paper_2504_19930_b200.phantom_device import make_phantom_device  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
seq, masks = make_phantom_device(echo_spec(frames=1))
case = make_pair(seq, masks, __import__("paper_2504_19930_b200").phantom.ECHO_TRUTH)
t64 = normalize_zscore(case.target.frames[0])
s64 = normalize_zscore(case.source.frames[0])
out = {}
for name, conv in (("f64-stored", lambda v: v),
                   ("f32-stored", lambda v: Volume3(v.data.astype(np.float32).astype(np.float64),
                                                    v.spacing, v.origin))):
    t, s = conv(t64), conv(s64)
    run = dsmc.DeviceSmcRun(t, s, SmcConfig(mode="image", n_particles=P, n_iterations=1, seed=0),
                            Executor())
    run.predict(0)
    A, B = run.A[:P], run.B[:P]
    res = {"storage": int(run.sdv.dtype_code)}
    for path in ("quad", "generic"):
        ops.prepare_layouts(run.tdv, run.sdv, "f32")
        if path == "generic":   # drop the layout and keep it from being rebuilt
            run.sdv.desc.quad_dev = None
            run.sdv.ensure_quad = lambda: None
        z, d, n = ops.measure(run.tdv, run.sdv, A, B, False, "f32")
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            z, d, n = ops.measure(run.tdv, run.sdv, A, B, False, "f32")
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        res[path] = {"ms": ms, "evals_per_s": P * t.data.size / (ms * 1e-3),
                     "refined": ops.refined_count(run.tdv, P)}
        res[path + "_z"] = z.cpu().numpy()
    a = A.cpu().numpy().reshape(-1, 3, 3)
    b = B.cpu().numpy()
    sub = np.arange(0, P, max(1, P // 64))
    zo, do = ok.ncc_measure_batch(t.data, s.data, a[sub], b[sub], False)
    for path in ("quad", "generic"):
        zz = res.pop(path + "_z")[sub]
        res[path]["max_rel_vs_oracle_64_particles"] = float(np.max(np.abs(zz - zo) / np.abs(zo)))
    res["speedup"] = res["generic"]["ms"] / res["quad"]["ms"]
    out[name] = res
    print(name, json.dumps(res), flush=True)
