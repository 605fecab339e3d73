"""register_smc at large particle counts (C5-style P) on the C2 pair: the
update (whole-GPU kernel chain at these sizes), workspace sizing, trace."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2504_19930_b200 import Executor, SmcConfig, register_smc  # noqa: E402

t, s, case = bench.make_workload()
for P in (65536, 262144):
    cfg = SmcConfig(n_particles=P, n_iterations=4, seed=0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    est, tr = register_smc(t, s, cfg, Executor())
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    a = est.to_array()
    assert np.all(np.isfinite(a)) and len(tr) == 4
    assert all(1.0 <= e <= P + 1e-6 for e in tr.ess)
    print(f"P={P}: {dt:.2f} s, {P * t.data.size * 4 / dt / 1e9:.0f} G evals/s, ess {[round(e) for e in tr.ess]}, "
          f"resampled {tr.resampled}, est deg {np.degrees(a[:3]).round(2).tolist()} mm {a[3:].round(2).tolist()}")
