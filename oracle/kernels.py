"""ctypes binding of the C oracle (test infrastructure only, see __init__).

Interface mirrors the reference kernel module
(/root/reference/pkg/src/echoreg/kernels_numba.py:192-223): ``NAME``,
``ncc_measure_batch``, ``resample_trilinear``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

NAME = "oracle-c"

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

_d = ctypes.POINTER(ctypes.c_double)
_i64 = ctypes.c_int64


def build(force: bool = False) -> str:
    """Compile the oracle with its Makefile (gcc, strict fp64)."""
    src = os.path.join(_HERE, "echoreg_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or (
        os.path.getmtime(_LIB_PATH) < os.path.getmtime(src)
    ):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.or_ncc_measure_batch.argtypes = [
            _d, _i64, _i64, _i64, _d, _i64, _i64, _i64, _d, _d, _i64,
            ctypes.c_int, _d, ctypes.POINTER(ctypes.c_uint8),
            ctypes.POINTER(ctypes.c_int64), ctypes.c_int]
        L.or_ncc_measure_batch.restype = None
        L.or_resample_trilinear.argtypes = [
            _d, _i64, _i64, _i64, _d, _d, _d, _i64, _i64, _i64, ctypes.c_int]
        L.or_resample_trilinear.restype = None
        L.or_k_interval.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                    ctypes.POINTER(ctypes.c_int64),
                                    ctypes.POINTER(ctypes.c_int64)]
        L.or_k_interval.restype = None
        L.or_sample_one.argtypes = [_d, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_double, _i64, _i64, _i64]
        L.or_sample_one.restype = ctypes.c_double
        L.or_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a, t=_d):
    return a.ctypes.data_as(t)


def max_threads() -> int:
    return int(lib().or_max_threads())


def ncc_measure_batch(tgt, src, a_batch, b_batch, overlap_only, workers=0,
                      return_counts=False):
    """Reference kernels_numba.ncc_measure_batch (kernels_numba.py:203-223);
    ``workers=0`` uses every host core.  Optionally also returns the
    in-bounds voxel counts."""
    tgt = np.ascontiguousarray(tgt, dtype=np.float64)
    src = np.ascontiguousarray(src, dtype=np.float64)
    a = np.ascontiguousarray(a_batch, dtype=np.float64).reshape(-1, 9)
    b = np.ascontiguousarray(b_batch, dtype=np.float64).reshape(-1, 3)
    p = a.shape[0]
    ncc = np.zeros(p)
    degen = np.zeros(p, dtype=np.uint8)
    counts = np.zeros(p, dtype=np.int64)
    lib().or_ncc_measure_batch(
        _ptr(tgt), *tgt.shape, _ptr(src), *src.shape, _ptr(a), _ptr(b), p,
        int(bool(overlap_only)), _ptr(ncc), _ptr(degen, ctypes.POINTER(ctypes.c_uint8)),
        _ptr(counts, ctypes.POINTER(ctypes.c_int64)), int(workers))
    if return_counts:
        return ncc, degen.astype(bool), counts
    return ncc, degen.astype(bool)


def resample_trilinear(src, a, b, out_dims, workers=0):
    """Reference kernels_numba.resample_trilinear (kernels_numba.py:192-200)."""
    src = np.ascontiguousarray(src, dtype=np.float64)
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(9)
    b = np.ascontiguousarray(b, dtype=np.float64).reshape(3)
    out = np.empty(tuple(int(d) for d in out_dims))
    lib().or_resample_trilinear(_ptr(src), *src.shape, _ptr(a), _ptr(b), _ptr(out),
                                *out.shape, int(workers))
    return out


def k_interval(c0, slope, limit, k_lo, k_hi):
    lo = ctypes.c_int64(k_lo)
    hi = ctypes.c_int64(k_hi)
    lib().or_k_interval(c0, slope, limit, ctypes.byref(lo), ctypes.byref(hi))
    return lo.value, hi.value
