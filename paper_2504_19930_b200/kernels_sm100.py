"""The kernel module the reference's backend seam can select.

Same interface as /root/reference/pkg/src/echoreg/kernels_numba.py:22,
192-233 (``NAME``, ``ncc_measure_batch``, ``resample_trilinear``,
``warm_up``): host numpy arrays in, host numpy arrays out.

Volumes arrive as plain fp64 arrays.  They are uploaded once and kept on the
device for as long as the host array lives: the reference treats volumes as
immutable (E/volume.py:20) and passes the same
``target.data`` / ``source.data`` objects on every SMC iteration.  Each call
re-validates the cached copy against a 4096-value sampled fingerprint of the
array and re-uploads on any change.  On upload the storage is chosen
losslessly on the device; for the measurement this includes recognising the
reference's z-scored 8-bit echo data as an affine image of bytes
(device.upload_array(lattice=True)), which puts it on the 8-bit oct fast
path.  The warp (resample_trilinear) keeps exact fp64 storage, so its output
stays bit-identical to _resample_kernel.  There is no CPU path: without a
CUDA device every call raises InternalError.
"""

from __future__ import annotations

import weakref

import numpy as np

from . import ops
from .device import device_volume_from_array, require_cuda, torch

NAME = "sm100"

#: interpolation arithmetic used through this seam (precision)
PRECISION = "f32"


_CACHE: dict = {}


def _fingerprint(a: np.ndarray) -> bytes:
    flat = a.reshape(-1)
    idx = np.linspace(0, flat.size - 1, num=min(flat.size, 4096)).astype(np.int64)
    return flat[idx].tobytes()


def _seam_volume(arr, dev, lattice: bool):
    """Device copy of a host array, cached per live array object."""
    a = np.asarray(arr)
    if a.dtype != np.float64 or not a.flags.c_contiguous or a.ndim != 3:
        return device_volume_from_array(np.ascontiguousarray(a, dtype=np.float64), dev,
                                        lattice=lattice)
    key = (id(a), a.ctypes.data, a.shape, dev.index, lattice)
    fp = _fingerprint(a)
    hit = _CACHE.get(key)
    if hit is not None and hit[0]() is a and hit[1] == fp:
        return hit[2]
    dv = device_volume_from_array(a, dev, lattice=lattice)
    _CACHE[key] = (weakref.ref(a, lambda _r, k=key: _CACHE.pop(k, None)), fp, dv)
    return dv


def ncc_measure_batch(tgt, src, a_batch, b_batch, overlap_only, workers=1):
    """Squared NCC of tgt against src pulled through each (A, b); returns
    (ncc f64[P], degenerate bool[P]) like kernels_numba.ncc_measure_batch.
    ``workers`` is accepted for signature compatibility; the device decides."""
    dev = require_cuda()
    t = torch()
    tdv = _seam_volume(tgt, dev, lattice=True)
    sdv = _seam_volume(src, dev, lattice=True)
    a = np.ascontiguousarray(a_batch, dtype=np.float64).reshape(-1, 9)
    b = np.ascontiguousarray(b_batch, dtype=np.float64).reshape(-1, 3)
    A = t.from_numpy(a).to(dev, non_blocking=False)
    B = t.from_numpy(b).to(dev, non_blocking=False)
    ncc, degen, _ = ops.measure(tdv, sdv, A, B, bool(overlap_only), PRECISION)
    return ncc.cpu().numpy(), degen.cpu().numpy().astype(bool)


def resample_trilinear(src, a, b, out_dims):
    """kernels_numba.resample_trilinear: f64 pull-back warp, fill 0."""
    dev = require_cuda()
    sdv = _seam_volume(src, dev, lattice=False)
    out = ops.resample_device(sdv, a, b, out_dims, dev)
    return out.cpu().numpy()


def warm_up():
    """Load the library and touch every kernel family once on a toy problem."""
    src = np.zeros((2, 2, 2))
    src[1, 1, 1] = 1.0
    eye = np.eye(3)
    zero = np.zeros(3)
    resample_trilinear(src, eye, zero, (2, 2, 2))
    ncc_measure_batch(src, src, eye[np.newaxis], zero[np.newaxis], False, 1)
