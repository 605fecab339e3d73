"""Dev probe: per-particle likelihood error of the fast modes against the
reference-op-order mode on the C2 workload, on the particles of SMC iteration
K (default 30: concentrated near the optimum, where the resampling decisions
are made).  usage: zerr_probe.py [K] [P]   (GPU)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2504_19930_b200 import SmcConfig, ops  # noqa: E402
from paper_2504_19930_b200 import smc as dsmc  # noqa: E402
from paper_2504_19930_b200.backend import Executor  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 30
P = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
t, s, _ = bench.make_workload()
cfg = SmcConfig(mode="image", n_particles=P, n_iterations=K + 1, seed=0)
run = dsmc.DeviceSmcRun(t, s, cfg, Executor(precision="exact"))
for k in range(K):
    run.predict(k)
    run.measure()
    run.update(k)
run.predict(K)
A, B = run.A[:P], run.B[:P]
z = {}
for prec in ("exact", "f64", "f32"):
    zz, d, n = ops.measure(run.tdv, run.sdv, A, B, False, prec)
    z[prec] = zz.cpu().numpy().astype(np.float64)
ref = z["exact"]
out = {"iteration": K, "particles": P, "z_median": float(np.median(ref))}
for prec in ("f64", "f32"):
    rel = np.abs(z[prec] - ref) / np.abs(ref)
    # the weights are exp(beta z): what matters for resampling is beta * dz
    out[prec] = {"rel_median": float(np.median(rel)), "rel_p99": float(np.quantile(rel, 0.99)),
                 "rel_max": float(rel.max()), "beta_dz_max": float(50 * np.abs(z[prec] - ref).max()),
                 "beta_dz_rms": float(50 * np.sqrt(np.mean((z[prec] - ref) ** 2)))}
print(json.dumps(out))
