"""Golden files of the reference's volume I/O (E/io.py): each case is written
by the reference's own ``write_volume`` and read back by its ``read_volume``;
the fixture stores the file bytes and the decoded arrays / geometry, so
tests/test_io.py can check our writer byte for byte and our reader value for
value without /root/reference.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_io.py
"""
import os
import sys
import tempfile

sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from echoreg.io import read_volume, write_volume  # noqa: E402
from echoreg.volume import Sequence4, Volume3  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "io.npz")


def vol(rng, dims, spacing, origin):
    # float32-representable values, as the reference's tests/conftest.py:30-41
    return Volume3(rng.random(dims, dtype=np.float32).astype(np.float64), spacing, origin)


def cases(rng):
    yield "f32_3d", vol(rng, (5, 4, 3), (0.9, 1.1, 0.7), (1.5, -2.0, 3.25)), ".nii", "float32"
    frames = [vol(rng, (4, 3, 2), (1.0, 2.0, 0.5), (0.0, 0.0, 0.0)) for _ in range(3)]
    yield "f32_4d", Sequence4(frames, frame_rate=25.0, ed_index=0), ".nii", "float32"
    m = Volume3((rng.random((6, 5, 4)) > 0.5).astype(np.float64), (0.87, 1.08, 0.73))
    yield "mask_u8", m, ".nii", "uint8"
    frames = [vol(rng, (3, 4, 5), (1.0, 1.0, 1.0), (-1.0, 2.0, 0.5)) for _ in range(2)]
    yield "raw_4d", Sequence4(frames, frame_rate=12.5, ed_index=1), ".raw", None


if __name__ == "__main__":
    rng = np.random.default_rng(2504)
    arrays = {}
    with tempfile.TemporaryDirectory() as d:
        for name, v, ext, dtype in cases(rng):
            path = os.path.join(d, name + ext)
            if dtype:
                write_volume(v, path, dtype=dtype)
            else:
                write_volume(v, path)
            arrays[f"{name}.file"] = np.frombuffer(open(path, "rb").read(), np.uint8)
            if ext == ".raw":
                arrays[f"{name}.json"] = np.frombuffer(
                    open(path[:-4] + ".json", "rb").read(), np.uint8)
            back = read_volume(path)
            fr = back.frames if isinstance(back, Sequence4) else [back]
            arrays[f"{name}.data"] = np.stack([f.data for f in fr])
            arrays[f"{name}.geom"] = np.array([*fr[0].spacing, *fr[0].origin])
            arrays[f"{name}.seq"] = np.array(
                [back.frame_rate, back.ed_index] if isinstance(back, Sequence4) else [-1.0, -1])
            # the written volume, to rewrite with our writer
            src = v.frames if isinstance(v, Sequence4) else [v]
            arrays[f"{name}.src"] = np.stack([f.data for f in src])
    np.savez_compressed(OUT, **arrays)
    print(OUT, sorted(arrays))
