"""A/B of an L2 persisting access-policy window over the oct source for the
C2 measurement (the north star's "L2-persistent window"), inside the bench's
conditions (256 MiB L2 flush between launches): cudaLimitPersistingL2CacheSize
+ a cudaAccessPolicyWindow (hitRatio 1, persisting) on the launching stream,
via cuda-python.  usage: l2window_probe.py [reps]   (GPU)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from cuda.bindings import runtime as cudart  # noqa: E402

import bench  # noqa: E402
from paper_2504_19930_b200 import SmcConfig, ops  # noqa: E402
from paper_2504_19930_b200 import smc as dsmc  # noqa: E402
from paper_2504_19930_b200.backend import Executor  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
t, s, _ = bench.make_workload()
P = 2000
run = dsmc.DeviceSmcRun(t, s, SmcConfig(mode="image", n_particles=P, n_iterations=1, seed=0),
                        Executor())
run.predict(0)
A, B = run.A[:P], run.B[:P]
ops.prepare_layouts(run.tdv, run.sdv, "f32")
oct_ptr, oct_bytes = run.sdv.desc.oct_dev, run.sdv.oct.numel() if run.sdv.shared is None \
    else run.sdv.shared.oct.numel()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
stream = torch.cuda.current_stream()


def timed(label):
    ms = []
    for i in range(reps + 2):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ops.measure(run.tdv, run.sdv, A, B, False, "f32")
        e1.record(stream)
        torch.cuda.synchronize()
        if i >= 2:
            ms.append(e0.elapsed_time(e1))
    out = {"case": label, "ms_mean": sum(ms) / len(ms), "ms_min": min(ms)}
    print(json.dumps(out), flush=True)
    return out


base = timed("no window")
prop = cudart.cudaGetDeviceProperties(0)[1]
limit = min(int(prop.persistingL2CacheMaxSize), oct_bytes)
cudart.cudaDeviceSetLimit(cudart.cudaLimit.cudaLimitPersistingL2CacheSize, limit)
attr = cudart.cudaStreamAttrValue()
w = attr.accessPolicyWindow
w.base_ptr = oct_ptr
w.num_bytes = min(oct_bytes, int(prop.accessPolicyMaxWindowSize))
w.hitRatio = 1.0
w.hitProp = cudart.cudaAccessProperty.cudaAccessPropertyPersisting
w.missProp = cudart.cudaAccessProperty.cudaAccessPropertyStreaming
attr.accessPolicyWindow = w
err = cudart.cudaStreamSetAttribute(stream.cuda_stream,
                                    cudart.cudaStreamAttrID.cudaLaunchAttributeAccessPolicyWindow,
                                    attr)
print(json.dumps({"persisting_limit_bytes": limit, "window_bytes": int(w.num_bytes),
                  "oct_bytes": oct_bytes, "set_attribute": str(err[0])}), flush=True)
win = timed("persisting window over the oct source")
print(json.dumps({"speedup": base["ms_mean"] / win["ms_mean"]}))
