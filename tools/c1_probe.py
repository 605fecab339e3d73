"""Where C1's time goes: device time per SMC iteration (events), the
measurement launch alone, and host wall time per iteration."""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_19930_b200 import PhantomSpec, RigidParams, SmcConfig, make_pair, make_phantom  # noqa: E402
from paper_2504_19930_b200 import smc as dsmc  # noqa: E402
from paper_2504_19930_b200.backend import Executor  # noqa: E402

seq, masks = make_phantom(PhantomSpec(dims=(64, 64, 64), frames=1, seed=0))
case = make_pair(seq, masks, RigidParams(math.radians(5), math.radians(-8), math.radians(4),
                                         6.0, -4.0, 3.0))
tm, sm = case.target_masks[0], case.source_masks[0]
cfg = SmcConfig(mode="mask", n_particles=500, n_iterations=20, seed=0)
for rep in range(3):
    run = dsmc.DeviceSmcRun(tm, sm, cfg, Executor())
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    mev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * cfg.n_iterations)]
    t0 = time.perf_counter()
    ev[0].record()
    for k in range(cfg.n_iterations):
        run.predict(k)
        mev[2 * k].record()
        run.measure()
        mev[2 * k + 1].record()
        run.update(k)
    ev[1].record()
    host = time.perf_counter() - t0
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    meas = sum(mev[2 * k].elapsed_time(mev[2 * k + 1]) for k in range(cfg.n_iterations))
    print(f"device {ev[0].elapsed_time(ev[1]):.3f} ms, measure {meas:.3f} ms, "
          f"host enqueue {1e3 * host:.3f} ms, wall {1e3 * wall:.3f} ms")
