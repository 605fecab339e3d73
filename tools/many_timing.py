"""Throughput of concurrent small registrations: 8 C1-sized mask
registrations (64^3, 500 x 20) one after another vs register_smc_many."""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_19930_b200 import (PhantomSpec, RigidParams, SmcConfig, make_pair,  # noqa: E402
                                   make_phantom, register_smc, register_smc_many)

truth = RigidParams(math.radians(5), math.radians(-8), math.radians(4), 6.0, -4.0, 3.0)
pairs = []
for seed in range(8):
    case = make_pair(*make_phantom(PhantomSpec(dims=(64, 64, 64), frames=1, seed=seed)), truth)
    pairs.append((case.target_masks[0], case.source_masks[0]))
cfg = SmcConfig(mode="mask", n_particles=500, n_iterations=20, seed=0)
register_smc_many(pairs[:2], cfg)
for name, fn in (("sequential", lambda: [register_smc(t, s, cfg) for t, s in pairs]),
                 ("register_smc_many", lambda: register_smc_many(pairs, cfg))):
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(f"8 x C1 {name:18s} {1e3 * best:8.2f} ms  ({1e3 * best / 8:.2f} ms per registration)")
