"""numpy restatement of the reference phantom generator -- TEST INFRASTRUCTURE ONLY.

Follows /root/reference/pkg/src/echoreg/phantom.py:61-166 (make_phantom,
make_pair) line by line, with the warps through the C oracle's resampler
(``oracle.kernels.resample_trilinear``, the bit-exact restatement of
kernels_numba._resample_kernel) and the rigid algebra of geometry.py:76-152
from ``oracle.smc``.  Adds the BASELINE C2/C3 echo recipe (the LV phantom on
the 176x176x208 echo grid, quantised to 8 bit), the same recipe as
paper_2504_19930_b200.phantom.echo_case and tests/golden/make_golden_full.py.

Used by bench.py's CPU legs (``--impl reference`` and ``cpu_baseline``) so
that the reference arm builds its inputs without importing the product
package, and pinned by tests/test_oracle_phantom.py to the SHA-256 digests the
REAL reference generator produced (tests/golden/full_c2.npz, full_c3.npz) and
to tests/golden/phantom.npz.
"""

from __future__ import annotations

import hashlib
import math

import numpy as np

from . import kernels
from .smc import index_affine, physical_center, to_matrix

INTENSITY_BACKGROUND = 0.2   # phantom.py:24-26
INTENSITY_TISSUE = 1.0
INTENSITY_BLOOD = 0.1
FILL_VALUE = 0.0             # geometry.py FILL_VALUE

ECHO_DIMS = (176, 176, 208)
ECHO_SPACING = (0.87, 1.08, 0.73)
ECHO_TRUTH = (math.radians(5.0), math.radians(-8.0), math.radians(4.0), 6.0, -4.0, 3.0)


def _ellipsoid_radius(xs, ys, zs, semiaxes, scale):
    """phantom.py:94-96"""
    ax, ay, az = (a * scale for a in semiaxes)
    return (xs / ax) ** 2 + (ys / ay) ** 2 + (zs / az) ** 2


def make_phantom(dims, spacing, outer, inner, speckle_sigma=0.3, amplitude=0.25, frames=5,
                 seed=0, center=None):
    """phantom.py:61-91: (frames, masks) as lists of fp64 arrays."""
    nx, ny, nz = dims
    sx, sy, sz = spacing
    if center is None:
        center = physical_center(dims, spacing, (0.0, 0.0, 0.0))
    xs = (np.arange(nx) * sx - center[0])[:, None, None]
    ys = (np.arange(ny) * sy - center[1])[None, :, None]
    zs = (np.arange(nz) * sz - center[2])[None, None, :]
    gen = np.random.Generator(np.random.Philox(key=seed))
    speckle = np.exp(speckle_sigma * gen.standard_normal(tuple(dims)))
    out_frames, masks = [], []
    for k in range(frames):
        scale = 1.0 - amplitude * math.sin(math.pi * k / frames) ** 2
        r_out = _ellipsoid_radius(xs, ys, zs, outer, scale)
        r_in = _ellipsoid_radius(xs, ys, zs, inner, scale)
        base = np.full(tuple(dims), INTENSITY_BACKGROUND)
        base[r_out <= 1.0] = INTENSITY_TISSUE
        cavity = r_in <= 1.0
        base[cavity] = INTENSITY_BLOOD
        out_frames.append(base * speckle)
        masks.append(cavity.astype(np.float64))
    return out_frames, masks


def inverse(m):
    """geometry.py:105-112 (closed-form rigid inverse)"""
    r_t = m[:3, :3].T
    out = np.eye(4)
    out[:3, :3] = r_t
    out[:3, 3] = -r_t @ m[:3, 3]
    return out


def resample(data, spacing, m, workers=0):
    """geometry.py:188-200 on one grid (source grid = reference grid)."""
    a, b = index_affine(m, spacing, (0.0, 0.0, 0.0), spacing, (0.0, 0.0, 0.0))
    return kernels.resample_trilinear(data, a, b, data.shape, workers)


def make_pair(frames, masks, spacing, truth, overlap_crop=0.0, workers=0):
    """phantom.py:120-166: (source frames, source masks)."""
    dims = frames[0].shape
    m_inv = inverse(to_matrix(np.asarray(truth, dtype=np.float64),
                              physical_center(dims, spacing, (0.0, 0.0, 0.0))))
    nx = dims[0]
    slab_start = nx - int(round(overlap_crop * nx))
    src_frames, src_masks = [], []
    for frame, mask in zip(frames, masks):
        moved = resample(frame, spacing, m_inv, workers)
        moved_mask = (resample(mask, spacing, m_inv, workers) > 0.5).astype(np.float64)
        if slab_start < nx:
            moved = moved.copy()
            moved[slab_start:, :, :] = FILL_VALUE
            moved_mask[slab_start:, :, :] = 0.0
        src_frames.append(moved)
        src_masks.append(moved_mask)
    return src_frames, src_masks


def echo_spec(dims=ECHO_DIMS, spacing=ECHO_SPACING):
    """The reference's LV phantom scaled to the echo grid:
    semi-axes scaled by extent / 64, speckle 0.3, amplitude 0.25."""
    ext = [d * s for d, s in zip(dims, spacing)]
    f = [e / 64.0 for e in ext]
    outer = tuple(a * k for a, k in zip((22.0, 18.0, 26.0), f))
    inner = tuple(a * k for a, k in zip((14.0, 11.0, 17.0), f))
    return outer, inner


def echo_case(frames=1, seed=0, dims=ECHO_DIMS, spacing=ECHO_SPACING, truth=ECHO_TRUTH,
              workers=0):
    """BASELINE C2/C3 inputs: 8-bit target/source frames (uint8 arrays) and
    the target/source cavity masks (fp64 0/1 arrays)."""
    outer, inner = echo_spec(dims, spacing)
    fr, masks = make_phantom(dims, spacing, outer, inner, 0.3, 0.25, frames, seed)
    src, src_masks = make_pair(fr, masks, spacing, truth, workers=workers)
    scale = 255.0 / float(np.percentile(fr[0], 99.9))

    def q(x):
        return np.clip(np.round(x * scale), 0.0, 255.0).astype(np.uint8)

    return [q(f) for f in fr], [q(f) for f in src], masks, src_masks


def normalize_zscore(data):
    """volume.py:119-130 (population std; ConstantVolume below 1e-12)."""
    mean = float(data.mean())
    std = float(data.std())
    if std < 1e-12:
        raise ValueError(f"standard deviation {std:.3e} too small to normalize")
    return (data - mean) / std


def digest(arrays) -> str:
    """SHA-256 of the arrays' bytes as uint8 (the goldens' input digests)."""
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).astype(np.uint8).tobytes())
    return h.hexdigest()
