"""Dev probe: measurement-kernel throughput on the C2 workload (CUDA events
on the launching stream).  usage: measure_probe.py [P] [precisions] [reps]
(ER_PROBE_MODE=mask: the binary masks of the same pair; ER_PROBE_OVERLAP=1:
the overlap region)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_19930_b200 import SmcConfig, ops  # noqa: E402
from paper_2504_19930_b200 import smc as dsmc  # noqa: E402
from paper_2504_19930_b200.backend import Executor  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
precs = sys.argv[2].split(",") if len(sys.argv) > 2 else ["f32", "f64", "exact"]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
t, s, case = bench.make_workload()
mode = os.environ.get("ER_PROBE_MODE", "image")
if mode == "mask":
    # the C3-style binary masks of the same pair (bit-oct path)
    from paper_2504_19930_b200 import binarize  # noqa: E402
    t, s = binarize(case.target_masks[0], 0.5), binarize(case.source_masks[0], 0.5)
cfg = SmcConfig(mode=mode, n_particles=P, n_iterations=1, seed=0)
run = dsmc.DeviceSmcRun(t, s, cfg, Executor())
run.predict(0)
A, B = run.A[:P], run.B[:P]
nvox = t.data.size
ovl = os.environ.get("ER_PROBE_OVERLAP", "0") == "1"
res = {}
for prec in precs:
    for _ in range(2):
        z, d, n = ops.measure(run.tdv, run.sdv, A, B, ovl, prec)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        z, d, n = ops.measure(run.tdv, run.sdv, A, B, ovl, prec)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    nin = int(n.sum().item())
    res[prec] = dict(ms=ms, evals_per_s=P * nvox / (ms * 1e-3),
                     sampled_per_s=nin / (ms * 1e-3), inbounds_frac=nin / (P * nvox),
                     hbm_frac_9B=nin * 9 / (ms * 1e-3) / 6535.4e9)
    print(prec, json.dumps(res[prec]), flush=True)
    if os.environ.get("ER_PROBE_DUMP"):
        # raw outputs, to compare builds bit for bit
        torch.save({"z": z.cpu(), "d": d.cpu(), "n": n.cpu()},
                   f"{os.environ['ER_PROBE_DUMP']}_{prec}.pt")
