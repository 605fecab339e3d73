"""ctypes binding of the sm_100a C-ABI library (include/echoreg_b200.h).

There is no fallback: if the library is missing or no CUDA device is
present, every entry point raises ``InternalError`` (the reference's exit
code 3 class) instead of silently computing on the CPU.
"""

from __future__ import annotations

import ctypes
import os

from .errors import BadConfig, InternalError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libechoreg_sm100.so")

ER_OK, ER_EINVAL, ER_ECUDA, ER_EWEIGHTS = 0, 1, 2, 3
ER_U8, ER_F32, ER_F64 = 0, 1, 2
ER_LERP_F32, ER_LERP_F64, ER_LERP_EXACT, ER_LERP_NEAREST = 0, 1, 2, 3
ER_MOMENTS_DOUBLES = 1026
ER_NCC_SUMS_DOUBLES = 1782
ER_TRACE_STRIDE = 12

_p = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_f64 = ctypes.c_double
_d3 = ctypes.c_double * 3
_d6 = ctypes.c_double * 6
_d9 = ctypes.c_double * 9
_i6 = ctypes.c_int32 * 6


class ErVolume(ctypes.Structure):
    _fields_ = [
        ("data_dev", _p),
        ("dtype", _i32),
        ("nx", _i32),
        ("ny", _i32),
        ("nz", _i32),
        ("alpha", _f64),
        ("gamma", _f64),
        ("oct_dev", _p),
        ("bitoct_dev", _p),
        ("quad_dev", _p),
    ]


class ErSmcCtl(ctypes.Structure):
    _fields_ = [
        ("best_measurement", _f64),
        ("best_state", _f64 * 6),
        ("has_best", _i32),
        ("error", _i32),
    ]


_VP = ctypes.POINTER(ErVolume)

# name -> (restype, argtypes)
SIGNATURES = {
    "er_abi_version": (ctypes.c_int, []),
    "er_last_error": (ctypes.c_char_p, []),
    "er_debug_bounds_faults": (ctypes.c_int, [ctypes.POINTER(ctypes.c_ulonglong)]),
    "er_volume_moments": (ctypes.c_int, [_VP, _p, _p]),
    "er_oct_bytes": (ctypes.c_size_t, [_VP]),
    "er_histogram_u8": (ctypes.c_int, [_VP, _p, _p]),
    "er_build_oct": (ctypes.c_int, [_VP, _p, _p]),
    "er_bitoct_bytes": (ctypes.c_size_t, [_VP]),
    "er_build_bitoct": (ctypes.c_int, [_VP, _p, _p]),
    "er_classify_f64": (ctypes.c_int, [_p, _i64, _p, _p]),
    "er_convert_f64": (ctypes.c_int, [_p, _i64, _i32, _p, _p]),
    "er_minmax_f64": (ctypes.c_int, [_p, _i64, _p, _p]),
    "er_lattice_u8": (ctypes.c_int, [_p, _i64, _f64, _f64, _f64, _p, _p, _p]),
    "er_ingest_u8": (ctypes.c_int, [_p, _i64, _i64, _i64, _i64, _p, _p, _p]),
    "er_measure_workspace_bytes": (ctypes.c_size_t, [_VP, _i64]),
    "er_measure_ncc": (ctypes.c_int, [_VP, _VP, _p, _p, _p, _i64, _i32, _i32, _p, _p, _p,
                                      _p, ctypes.c_size_t, _p]),
    "er_smc_init": (ctypes.c_int, [_p, _i64, _u64, _d6, _p]),
    "er_smc_predict": (ctypes.c_int, [_p, _p, _i64, _u64, _i64, _d6, _d6, _p]),
    "er_states_to_affine": (ctypes.c_int, [_p, _i64, _i64, _d3, _d3, _d3, _d3, _d3, _p, _p,
                                           _p]),
    "er_smc_predict_affine": (ctypes.c_int, [_p, _p, _i64, _u64, _i64, _d6, _d6, _i64, _i64,
                                             _d3, _d3, _d3, _d3, _d3, _p, _p, _p]),
    "er_grid_to_affine": (ctypes.c_int, [_i64, _i64, _i6, _d6, _d3, _d3, _d3, _d3, _d3, _p,
                                         _p, _p, _p]),
    "er_argmax_update": (ctypes.c_int, [_p, _i64, _i64, _p, _p]),
    "er_smc_update": (ctypes.c_int, [_p, _p, _p, _p, _p, _p, _p, _i64, _f64, _f64, _u64,
                                     _i64, _i32, _p, _p, _p]),
    "er_probe_read": (ctypes.c_int, [_p, _i64, _i32, _p, _p]),
    "er_quad_bytes": (ctypes.c_size_t, [_VP]),
    "er_build_quad": (ctypes.c_int, [_VP, _p, _p]),
    "er_smc_update_gathered": (ctypes.c_int, [_p, _i64, _i64, _p, _p, _p, _p, _p, _i64, _f64,
                                              _f64, _u64, _i64, _i32, _p, _p, _p]),
    "er_resample": (ctypes.c_int, [_VP, _d9, _d3, _i32, _i32, _i32, _p, _p]),
    "er_warp_dice_counts": (ctypes.c_int, [_VP, _d9, _d3, _VP, _p, _p]),
    "er_warp_ncc_sums": (ctypes.c_int, [_VP, _VP, _d9, _d3, _i32, _p, _p]),
    "er_phantom_scratch_bytes": (ctypes.c_size_t, [_i64]),
    "er_phantom_speckle": (ctypes.c_int, [_u64, _i64, _f64, _p, ctypes.c_size_t, _p, _p, _p]),
    "er_phantom_frame": (ctypes.c_int, [_p, _i32, _i32, _i32, _d3, _d3, _d3, _d3, _p, _p, _p]),
    "er_quantize_u8": (ctypes.c_int, [_p, _i64, _f64, _i64, _p, _p]),
    "er_binarize_u8": (ctypes.c_int, [_p, _i64, _f64, _i64, _p, _p]),
}

_lib = None

#: kernels each entry point launches (for the bench's gpu_launches count)
LAUNCHES_PER_CALL = {
    "er_volume_moments": 2, "er_classify_f64": 2, "er_build_oct": 1, "er_build_bitoct": 1, "er_histogram_u8": 2, "er_convert_f64": 1, "er_minmax_f64": 3, "er_lattice_u8": 2, "er_ingest_u8": 2, "er_measure_ncc": 2,
    "er_smc_init": 1, "er_smc_predict": 1, "er_smc_predict_affine": 1, "er_states_to_affine": 1, "er_grid_to_affine": 1,
    "er_argmax_update": 1, "er_smc_update": 1, "er_smc_update_gathered": 1, "er_probe_read": 1, "er_build_quad": 1, "er_resample": 1, "er_warp_dice_counts": 2,
    "er_warp_ncc_sums": 4, "er_phantom_speckle": 5, "er_phantom_frame": 1, "er_quantize_u8": 1,
    "er_binarize_u8": 1,
}
launch_count = 0


def load():
    """Load the shared library (no CUDA call is made here)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise InternalError(
                f"sm_100a library not built: {LIB_PATH} missing "
                "(run __graft_entry__.build()); there is no CPU fallback")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int, what: str = ""):
    if rc == ER_OK:
        return
    msg = load().er_last_error().decode(errors="replace")
    if rc == ER_EINVAL:
        raise BadConfig(f"{what}: {msg}")
    raise InternalError(f"{what}: {msg} (code {rc})")


def call(name: str, *args):
    global launch_count
    rc = getattr(load(), name)(*args)
    check(rc, name)
    launch_count += LAUNCHES_PER_CALL.get(name, 0)
    return rc


def d3(v) -> "ctypes.Array":
    return _d3(*[float(x) for x in v])


def d6(v) -> "ctypes.Array":
    return _d6(*[float(x) for x in v])


def d9(v) -> "ctypes.Array":
    return _d9(*[float(x) for x in v])


def i6(v) -> "ctypes.Array":
    return _i6(*[int(x) for x in v])


def bounds_faults():
    """Out-of-range gather indices counted by a -DER_BOUNDS_CHECK=1 build
    (None on a normal build, where the checks are compiled out)."""
    n = ctypes.c_ulonglong(0)
    rc = load().er_debug_bounds_faults(ctypes.byref(n))
    return int(n.value) if rc == ER_OK else None
