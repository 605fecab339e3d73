"""Small end-to-end exercise of every kernel family, for compute-sanitizer
(one tool per run): generic measurement (f32/f64 storage, 3 precisions),
oct (u8) and bit-oct (binary) fast paths in full and overlap mode, odd
shapes, predict/update, exhaustive grid, warps, Dice, NCC, histogram, 8-bit
NIfTI ingest (word and byte paths, partial tiles, several frames)."""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_19930_b200 import (Executor, GridSpec, RigidParams, Sequence4,  # noqa: E402
                                   SmcConfig, Volume3, dice, dice_under_transform, ncc, normalize_zscore,
                                   register_exhaustive, register_smc, resample, to_matrix)

rng = np.random.default_rng(0)
for dims in ((9, 7, 11), (5, 1, 6), (1, 4, 4), (17, 13, 19)):
    raw = rng.integers(0, 256, dims).astype(np.uint8)
    img = normalize_zscore(Volume3.from_u8(raw, (0.9, 1.1, 1.3)))
    f32 = Volume3(rng.random(dims, dtype=np.float32).astype(np.float64))
    f64 = Volume3(rng.random(dims))
    m = Volume3.from_u8((raw > 128).astype(np.uint8))
    for prec in ("f32", "f64", "exact"):
        ex = Executor(precision=prec)
        for tv, sv in ((img, img), (f32, f32), (f64, f64), (m, m)):
            mats = np.stack([to_matrix(RigidParams(*rng.uniform(-0.5, 0.5, 3),
                                                   *rng.uniform(-3, 3, 3)), tv.physical_center())
                             for _ in range(7)] + [np.eye(4), to_matrix(RigidParams(tx=1e4))])
            for overlap in (False, True):
                ex.measure_ncc(tv, sv, mats, overlap)
    resample(img, img, to_matrix(RigidParams(0.1, 0.2, -0.1, 1, 2, 3), img.physical_center()))
    if (raw > 128).any() and (raw <= 128).any():
        dice(m, m)
        dice_under_transform(m, m, to_matrix(RigidParams(0.1, 0, 0, 1, 0, 0), m.physical_center()))
    if img.data.std() > 0:
        ncc(img, img)
    cfg = SmcConfig(mode="image", n_particles=33, n_iterations=3, seed=1, t_limit=3, r_limit=5)
    register_smc(img, img, cfg)
    register_smc(m, m, SmcConfig(mode="mask", n_particles=17, n_iterations=2,
                                 ncc_region="overlap"), trace_masks=(m, m))
    register_exhaustive(img, img, GridSpec(half_counts=(1, 0, 1, 0, 1, 1), step_t=1.0,
                                           step_r=3.0))
from paper_2504_19930_b200.io import read_volume_device, write_u8_nifti  # noqa: E402

with tempfile.TemporaryDirectory() as d:
    for dims, nf in (((9, 7, 11), 3), ((68, 5, 130), 2), ((64, 3, 64), 1), ((1, 1, 1), 1)):
        seq = Sequence4([Volume3.from_u8(rng.integers(0, 256, dims).astype(np.uint8))
                         for _ in range(nf)])
        write_u8_nifti(seq, os.path.join(d, "v.nii"))
        read_volume_device(os.path.join(d, "v.nii"))
torch.cuda.synchronize()
print("sanitize target done")
from paper_2504_19930_b200 import _lib  # noqa: E402

faults = _lib.bounds_faults()
print("bounds faults:", "n/a (checks compiled out)" if faults is None else faults)
if os.environ.get("ER_ASSERT_NO_BOUNDS_FAULTS") and faults != 0:
    sys.exit(f"bounds check failed: {faults}")
