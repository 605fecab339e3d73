"""Throughput of the generic measurement path (non-8-bit data): fp64 and
fp32-representable volumes on the C2 grid, each precision mode."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2504_19930_b200 import SmcConfig, Volume3, normalize_zscore, ops
from paper_2504_19930_b200 import smc as dsmc
from paper_2504_19930_b200.backend import Executor
from paper_2504_19930_b200.phantom import ECHO_TRUTH, echo_spec, make_pair, make_phantom

seq, masks = make_phantom(echo_spec(frames=1, seed=0))
case = make_pair(seq, masks, ECHO_TRUTH)
t64 = normalize_zscore(case.target.frames[0]); s64 = normalize_zscore(case.source.frames[0])
t32 = Volume3(t64.data.astype(np.float32).astype(np.float64), t64.spacing)
s32 = Volume3(s64.data.astype(np.float32).astype(np.float64), s64.spacing)
P = 2000
for name, (t, s) in (("f64 storage", (t64, s64)), ("f32 storage", (t32, s32))):
    run = dsmc.DeviceSmcRun(t, s, SmcConfig(n_particles=P, n_iterations=1), Executor())
    run.predict(0)
    A, B = run.A[:P], run.B[:P]
    print(name, "dtype code", run.sdv.dtype_code)
    for prec in ("f32", "f64", "exact"):
        ops.measure(run.tdv, run.sdv, A, B, False, prec)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); z, d, n = ops.measure(run.tdv, run.sdv, A, B, False, prec); e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"  {prec:6s} {ms:8.2f} ms  {P * t.data.size / ms / 1e6:8.1f} G evals/s")
