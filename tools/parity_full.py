"""Full-size free-running parity at BASELINE C2 (2000 particles x 50
iterations, 176x176x208 u8 echo pair, image mode): the device path against
the reference algorithm (oracle/smc.py driving the bit-exact C kernel, all
host threads).  Prints one JSON line."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from oracle import kernels as ok
from oracle import smc as osmc
from paper_2504_19930_b200 import Executor, SmcConfig, register_smc

P = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
IT = int(sys.argv[2]) if len(sys.argv) > 2 else 50
mode = sys.argv[3] if len(sys.argv) > 3 else "image"
t, s, case = bench.make_workload()
if mode == "mask":
    from paper_2504_19930_b200 import binarize
    t, s = binarize(case.target_masks[0], 0.5), binarize(case.source_masks[0], 0.5)
out = {"config": f"C2 shape, {mode} mode, {P} x {IT}", "seed": 0}
for prec in ("f32", "f64", "exact"):
    t0 = time.perf_counter()
    est, tr = register_smc(t, s, SmcConfig(mode=mode, n_particles=P, n_iterations=IT, seed=0),
                           Executor(precision=prec))
    out[f"gpu_{prec}_s"] = time.perf_counter() - t0
    out[f"gpu_{prec}_estimate"] = est.to_array().tolist()
    out[f"gpu_{prec}_resampled"] = tr.resampled
    out[f"gpu_{prec}_ess"] = tr.ess
ok.build()
geom = (t.dims, t.spacing, t.origin)
t0 = time.perf_counter()
oest, otr = osmc.register(t.data, s.data, geom, geom,
                          osmc.Cfg(mode=mode, n_particles=P, n_iterations=IT, seed=0))
out["cpu_s"] = time.perf_counter() - t0
out["cpu_threads"] = ok.max_threads()
out["cpu_estimate"] = oest.tolist()
for prec in ("f32", "f64", "exact"):
    d = np.asarray(out[f"gpu_{prec}_estimate"]) - oest
    out[f"{prec}_max_rot_diff_deg"] = float(np.degrees(np.abs(d[:3])).max())
    out[f"{prec}_max_trans_diff_vox"] = float((np.abs(d[3:]) / np.asarray(t.spacing)).max())
    out[f"{prec}_resampled_identical"] = out[f"gpu_{prec}_resampled"] == otr.resampled
    out[f"{prec}_ess_max_rel_diff"] = float(np.max(np.abs(np.asarray(out[f"gpu_{prec}_ess"])
                                                         - np.asarray(otr.ess)) / np.asarray(otr.ess)))
    del out[f"gpu_{prec}_resampled"], out[f"gpu_{prec}_ess"]
print(json.dumps(out))
