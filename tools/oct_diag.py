"""Oct fast path vs the C oracle on one of tests/test_gpu_oct.py's grid cases
(anisotropic spacings, offset origins): per-precision relative error and
count parity.  usage: oct_diag.py [case]  (GPU)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import kernels as ok
from tests.test_gpu_oct import CASES, _mats
from paper_2504_19930_b200 import Volume3, ops
from paper_2504_19930_b200.device import device_volume, require_cuda
from paper_2504_19930_b200.geometry import index_affine_batch
case = int(sys.argv[1]) if len(sys.argv) > 1 else 0
tdims, sdims, same = CASES[case]
rng = np.random.default_rng(100 + case)
sp_t = tuple(rng.uniform(0.6, 1.4, 3))
sp_s = sp_t if same else tuple(rng.uniform(0.6, 1.4, 3))
org_s = (0.0, 0.0, 0.0) if same else tuple(rng.uniform(-1.0, 1.0, 3))
t = Volume3(rng.integers(0, 256, tdims).astype(np.float64), sp_t)
s = Volume3(rng.integers(0, 256, sdims).astype(np.float64), sp_s, org_s)
mats = _mats(rng, t.physical_center(), 40, 0.5, 3.0)
a, b = index_affine_batch(mats, s.spacing, s.origin, t.spacing, t.origin)
dev = require_cuda()
tdv, sdv = device_volume(t, dev), device_volume(s, dev)
A = torch.as_tensor(a.reshape(-1, 9), device=dev); B = torch.as_tensor(b.reshape(-1, 3), device=dev)
zo, do, no = ok.ncc_measure_batch(t.data, s.data, a, b, False, return_counts=True)
for prec in ("f32", "f64", "exact"):
    z = ops.measure(tdv, sdv, A, B, False, prec)[0].cpu().numpy()
    rel = np.abs(z - zo) / np.maximum(np.abs(zo), 1e-300)
    i = int(np.argmax(rel))
    print(prec, "max rel", rel.max(), "p", i, "z", zo[i], z[i], "n_in", no[i], "top5", np.sort(rel)[-5:])
