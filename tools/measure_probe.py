"""Dev probe: measurement-kernel throughput on the C2-shaped workload for
each interpolation precision (CUDA events on the launching stream)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2504_19930_b200 import Volume3, normalize_zscore, ops
from paper_2504_19930_b200.device import device_volume, require_cuda
from tests.test_gpu_measure import _echo_pair

dev = require_cuda()
raw_t, raw_s = _echo_pair()
sp = (0.87, 1.08, 0.73)
tv = normalize_zscore(Volume3(raw_t, sp)); sv = normalize_zscore(Volume3(raw_s, sp))
tdv, sdv = device_volume(tv, dev), device_volume(sv, dev)
P = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
states = ops.smc_init(P, 0, np.array([np.radians(15)]*3 + [20.0]*3), dev)
A, B = ops.states_to_affine(states, 0, P, tv.physical_center(), (sp, (0,0,0)), (sp, (0,0,0)))
nvox = tv.data.size
res = {}
for prec in ("f32", "f64", "exact"):
    for _ in range(2):
        z, d, n = ops.measure(tdv, sdv, A, B, False, prec)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        z, d, n = ops.measure(tdv, sdv, A, B, False, prec)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    nin = int(n.sum().item())
    res[prec] = dict(ms=ms, evals_per_s=P * nvox / (ms * 1e-3), sampled_per_s=nin / (ms * 1e-3),
                     inbounds_frac=nin / (P * nvox))
    print(prec, json.dumps(res[prec]))
print(json.dumps(res))
