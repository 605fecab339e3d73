"""Host (numpy, the reference's algorithm) vs device phantom generation for
the echo workloads: C2 (1 frame) and C3 (30 frames) at 176x176x208, C5
(256^3, 1 frame).  Prints one JSON line per case."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_19930_b200.phantom import echo_case  # noqa: E402
from paper_2504_19930_b200.phantom_device import echo_case_device  # noqa: E402

echo_case_device((40, 36, 44), frames=2)  # warm-up (module load, lazy kernels)
torch.cuda.synchronize()
for name, dims, spacing, frames in (("C2", (176, 176, 208), (0.87, 1.08, 0.73), 1),
                                    ("C3", (176, 176, 208), (0.87, 1.08, 0.73), 30),
                                    ("C5", (256, 256, 256), (0.8, 0.8, 0.8), 1)):
    t0 = time.perf_counter()
    d = echo_case_device(dims, spacing, frames=frames)
    torch.cuda.synchronize()
    td = time.perf_counter() - t0
    row = {"case": name, "dims": dims, "frames": frames, "device_s": round(td, 4)}
    if "--host" in sys.argv and frames <= 30:
        t0 = time.perf_counter()
        h = echo_case(dims, spacing, frames=frames)
        th = time.perf_counter() - t0
        same = all((a.codec.raw == b.codec.raw).all() for a, b in
                   zip(h.target.frames + h.source.frames + h.target_masks + h.source_masks,
                       d.target.frames + d.source.frames + d.target_masks + d.source_masks))
        row.update({"host_s": round(th, 3), "speedup": round(th / td, 1), "identical": same})
    print(json.dumps(row), flush=True)
