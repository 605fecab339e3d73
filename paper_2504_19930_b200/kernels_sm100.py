"""The kernel module the reference's backend seam can select.

Same interface as /root/reference/pkg/src/echoreg/kernels_numba.py:22,
192-233 (``NAME``, ``ncc_measure_batch``, ``resample_trilinear``,
``warm_up``): host numpy arrays in, host numpy arrays out.  Every call
uploads its volumes (fp64 -> device -> lossless storage chosen on device),
runs the sm_100a kernels and copies the results back -- this is the
"reference-facing plugin with host buffers" that bench.py's e2e number is
measured through.  There is no CPU path: without a CUDA device every call
raises InternalError.
"""

from __future__ import annotations

import numpy as np

from . import ops
from .device import device_volume_from_array, require_cuda, torch

NAME = "sm100"

#: interpolation arithmetic used through this seam (precision)
PRECISION = "f32"


def ncc_measure_batch(tgt, src, a_batch, b_batch, overlap_only, workers=1):
    """Squared NCC of tgt against src pulled through each (A, b); returns
    (ncc f64[P], degenerate bool[P]) like kernels_numba.ncc_measure_batch.
    ``workers`` is accepted for signature compatibility; the device decides."""
    dev = require_cuda()
    t = torch()
    tdv = device_volume_from_array(np.asarray(tgt), dev)
    sdv = device_volume_from_array(np.asarray(src), dev)
    a = np.ascontiguousarray(a_batch, dtype=np.float64).reshape(-1, 9)
    b = np.ascontiguousarray(b_batch, dtype=np.float64).reshape(-1, 3)
    A = t.from_numpy(a).to(dev, non_blocking=False)
    B = t.from_numpy(b).to(dev, non_blocking=False)
    ncc, degen, _ = ops.measure(tdv, sdv, A, B, bool(overlap_only), PRECISION)
    return ncc.cpu().numpy(), degen.cpu().numpy().astype(bool)


def resample_trilinear(src, a, b, out_dims):
    """kernels_numba.resample_trilinear: f64 pull-back warp, fill 0."""
    dev = require_cuda()
    sdv = device_volume_from_array(np.asarray(src), dev)
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
