"""The kernel module the reference's backend seam can select.

Same interface as /root/reference/pkg/src/echoreg/kernels_numba.py:22,
192-233 (``NAME``, ``ncc_measure_batch``, ``resample_trilinear``,
``warm_up``): host numpy arrays in, host numpy arrays out.

Volumes arrive as plain fp64 arrays.  They are uploaded once and kept on the
device for as long as the host array lives: the reference treats volumes as
immutable (E/volume.py:20) and passes the same
``target.data`` / ``source.data`` objects on every SMC iteration -- but
``Volume3.data`` is a writable numpy array (E/volume.py:32-47), so every call
re-validates each cached copy against a digest of the array's FULL content
(xxh3-128, ~14 GB/s on one host core).  The digest is computed while the
measurement already runs on the cached copy (the launch is asynchronous), so
it costs no wall time; on a mismatch the result is discarded and the call is
repeated on a fresh upload.  On upload the storage is chosen
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


def _digest(a: np.ndarray):
    """Digest of the array's full content."""
    try:
        import xxhash

        return xxhash.xxh3_128_intdigest(memoryview(a).cast("B"))
    except ImportError:  # pragma: no cover - xxhash ships with the image
        u = a.reshape(-1).view(np.uint64)
        return (int(np.add.reduce(u)), int(np.bitwise_xor.reduce(u)), a.size)


def _cacheable(a) -> bool:
    return (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous
            and a.ndim == 3)


def _key(a, dev, lattice):
    return (id(a), a.ctypes.data, a.shape, dev.index, lattice)


def _cached(arr, dev, lattice: bool):
    """(device volume, verified) for a host array: the cached copy for a live
    array object, unverified until _still_valid() confirms its digest; else a fresh
    upload (verified)."""
    if not _cacheable(arr):
        a = np.ascontiguousarray(arr, dtype=np.float64)
        return device_volume_from_array(a, dev, lattice=lattice), True
    hit = _CACHE.get(_key(arr, dev, lattice))
    if hit is not None and hit[0]() is arr:
        return hit[2], False
    return _upload(arr, dev, lattice), True


def _upload(a, dev, lattice):
    key = _key(a, dev, lattice)
    dv = device_volume_from_array(a, dev, lattice=lattice)
    _CACHE[key] = (weakref.ref(a, lambda _r, k=key: _CACHE.pop(k, None)), _digest(a), dv)
    return dv


def _still_valid(arr, dev, lattice) -> bool:
    """Does the cached copy still hold the array's current content?"""
    hit = _CACHE.get(_key(arr, dev, lattice))
    return hit is not None and hit[1] == _digest(arr)


def ncc_measure_batch(tgt, src, a_batch, b_batch, overlap_only, workers=1):
    """Squared NCC of tgt against src pulled through each (A, b); returns
    (ncc f64[P], degenerate bool[P]) like kernels_numba.ncc_measure_batch.
    ``workers`` is accepted for signature compatibility; the device decides."""
    dev = require_cuda()
    t = torch()
    a = np.ascontiguousarray(a_batch, dtype=np.float64).reshape(-1, 9)
    b = np.ascontiguousarray(b_batch, dtype=np.float64).reshape(-1, 3)
    A = t.from_numpy(a).to(dev, non_blocking=False)
    B = t.from_numpy(b).to(dev, non_blocking=False)
    for attempt in range(2):
        tdv, t_ok = _cached(tgt, dev, lattice=True)
        sdv, s_ok = _cached(src, dev, lattice=True)
        ncc, degen, _ = ops.measure(tdv, sdv, A, B, bool(overlap_only), PRECISION)
        # validate the cached copies while the measurement runs
        t_ok = t_ok or _still_valid(tgt, dev, True)
        s_ok = s_ok or _still_valid(src, dev, True)
        if t_ok and s_ok:
            return ncc.cpu().numpy(), degen.cpu().numpy().astype(bool)
        # the host array changed since it was cached: drop the stale copies
        for arr, ok in ((tgt, t_ok), (src, s_ok)):
            if not ok:
                _upload(arr, dev, True)
    raise AssertionError("unreachable: fresh uploads are always valid")


def resample_trilinear(src, a, b, out_dims):
    """kernels_numba.resample_trilinear: f64 pull-back warp, fill 0."""
    dev = require_cuda()
    for attempt in range(2):
        sdv, ok = _cached(src, dev, lattice=False)
        out = ops.resample_device(sdv, a, b, out_dims, dev)
        if ok or _still_valid(src, dev, False):
            return out.cpu().numpy()
        _upload(src, dev, False)
    raise AssertionError("unreachable: fresh uploads are always valid")


def warm_up():
    """Load the library and touch every kernel family once on a toy problem."""
    src = np.zeros((2, 2, 2))
    src[1, 1, 1] = 1.0
    eye = np.eye(3)
    zero = np.zeros(3)
    resample_trilinear(src, eye, zero, (2, 2, 2))
    ncc_measure_batch(src, src, eye[np.newaxis], zero[np.newaxis], False, 1)
