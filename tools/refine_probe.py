"""How many particles the f32 measurement refines in fp64, per SMC iteration,
on the C2 workload (image mode, 2000 x 50), and what the refinement costs.
usage: refine_probe.py [P] [iterations]   (GPU)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2504_19930_b200 import SmcConfig, ops  # noqa: E402
from paper_2504_19930_b200 import smc as dsmc  # noqa: E402
from paper_2504_19930_b200.backend import Executor  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
IT = int(sys.argv[2]) if len(sys.argv) > 2 else 50
t, s, _ = bench.make_workload()
cfg = SmcConfig(mode="image", n_particles=P, n_iterations=IT, seed=0)
run = dsmc.DeviceSmcRun(t, s, cfg, Executor())
counts = []
for k in range(IT):
    run.predict(k)
    run.measure()
    counts.append(ops.refined_count(run.tdv, run.plan.count, run.ws))
    run.update(k)
torch.cuda.synchronize()
print(json.dumps({"P": P, "iterations": IT, "refined_per_iteration": counts,
                  "refined_total": sum(counts), "refined_frac": sum(counts) / (P * IT)}))
