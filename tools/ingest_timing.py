"""Ingest of an 8-bit 4D NIfTI on the device vs the host (SURVEY.md §8f rank
1): a C3-sized file (30 frames of 176x176x208 u8, 194 MB) is written, then
read + z-scored (a) by the host reader (the reference's algorithm,
E/io.py:124-187 + E/volume.py:119-130 on numpy) and (b) by
read_volume_device (one H2D copy, one er_ingest_u8 launch with the per-frame
histograms).  Prints one JSON line; outputs are checked equal.

    python tools/ingest_timing.py [frames]
"""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_19930_b200 import Sequence4, Volume3, _lib, normalize_zscore  # noqa: E402
from paper_2504_19930_b200.device import ptr, stream_ptr  # noqa: E402
from paper_2504_19930_b200.io import read_volume, read_volume_device, write_u8_nifti  # noqa: E402


def host_zscore(v):
    """The reference's normalize_zscore on the fp64 data (volume.py:119-130)."""
    d = v.data
    return (d - d.mean()) / d.std()


def main():
    nf = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    dims = (176, 176, 208)
    n = dims[0] * dims[1] * dims[2]
    rng = np.random.default_rng(0)
    base = rng.integers(0, 256, dims, dtype=np.uint8)
    seq = Sequence4([Volume3.from_u8(np.roll(base, k, axis=2), (0.87, 1.08, 0.73))
                     for k in range(nf)], frame_rate=30.0)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "c3.nii")
        write_u8_nifti(seq, path)
        size = os.path.getsize(path)
        read_volume_device(path)  # warm-up (library load, allocator, page cache)
        torch.cuda.synchronize()
        dev_t = []
        for _ in range(3):
            t0 = time.perf_counter()
            dv = read_volume_device(path)
            dz = [normalize_zscore(f) for f in dv.frames]
            torch.cuda.synchronize()
            dev_t.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        hv = read_volume(path)
        hz = [host_zscore(f) for f in hv.frames]
        host_s = time.perf_counter() - t0
        ok = all(np.array_equal(a.codec.raw, b.codec.raw) for a, b in zip(dv.frames, hv.frames))
        ok = ok and all(np.array_equal(z.data, h) for z, h in zip(dz[:3], hz[:3]))
        pay = torch.from_numpy(np.fromfile(path, np.uint8)[352:]).cuda()
    out = torch.empty(nf * n, dtype=torch.uint8, device="cuda")
    hist = torch.empty((nf, 256), dtype=torch.int64, device="cuda")
    res = {}
    for label, h in (("with_hist", ptr(hist)), ("reorder_only", None)):
        for _ in range(3):
            _lib.call("er_ingest_u8", ptr(pay), *dims, nf, ptr(out), h, stream_ptr())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            _lib.call("er_ingest_u8", ptr(pay), *dims, nf, ptr(out), h, stream_ptr())
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        res[label] = {"ms": ms, "gbs": 2 * nf * n / (ms * 1e-3) / 1e9}
    print(json.dumps({
        "file_bytes": size, "frames": nf, "dims": dims,
        "device_read_plus_zscore_s": min(dev_t), "host_read_plus_zscore_s": host_s,
        "speedup": host_s / min(dev_t), "identical": bool(ok),
        "ingest_kernel": res,
        "ingest_kernel_note": "2 bytes of HBM traffic per voxel (read on-disk order, write "
                              "grid order); 10 back-to-back launches, payload 194 MB > L2",
        "cpu": os.cpu_count()}))


if __name__ == "__main__":
    main()
