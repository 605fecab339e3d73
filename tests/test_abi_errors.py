"""Error behaviour of the C-ABI boundary, checked on the CPU build box: every
entry point validates its arguments before touching the device and returns
ER_EINVAL with a message naming itself (the Python layer maps that to the
reference's BadConfig).  Fake non-null device pointers are safe here because
validation precedes any CUDA call."""

import ctypes

import pytest

from paper_2504_19930_b200 import _lib
from paper_2504_19930_b200.errors import BadConfig

FAKE = 0x10000  # never dereferenced: argument checks run first


def _vol(dtype=_lib.ER_U8, dims=(8, 8, 8), data=FAKE):
    v = _lib.ErVolume()
    v.data_dev = data
    v.dtype = dtype
    v.nx, v.ny, v.nz = dims
    v.alpha, v.gamma = 1.0, 0.0
    return v


def _einval(name, *args):
    rc = getattr(_lib.load(), name)(*args)
    assert rc == _lib.ER_EINVAL, (name, rc)
    assert name.encode() in _lib.load().er_last_error(), _lib.load().er_last_error()
    with pytest.raises(BadConfig):
        _lib.check(rc, name)


def test_measure_rejects_bad_arguments():
    t, s = _vol(), _vol()
    by = ctypes.byref
    common = (FAKE, FAKE, FAKE)  # moments, A, b
    _einval("er_measure_ncc", by(_vol(data=None)), by(s), *common, 4, 0, 0, FAKE, FAKE, FAKE,
            FAKE, 1 << 20, None)
    _einval("er_measure_ncc", by(t), by(_vol(dims=(0, 8, 8))), *common, 4, 0, 0, FAKE, FAKE,
            FAKE, FAKE, 1 << 20, None)
    _einval("er_measure_ncc", by(t), by(s), *common, -1, 0, 0, FAKE, FAKE, FAKE, FAKE,
            1 << 20, None)
    _einval("er_measure_ncc", by(t), by(s), *common, 4, 0, 9, FAKE, FAKE, FAKE, FAKE,
            1 << 20, None)                                       # unknown lerp mode
    _einval("er_measure_ncc", by(t), by(s), *common, 4, 0, 0, FAKE, FAKE, FAKE, FAKE,
            1, None)                                             # workspace too small
    _einval("er_measure_ncc", by(t), by(s), None, FAKE, FAKE, 4, 0, 0, FAKE, FAKE, FAKE, FAKE,
            1 << 20, None)                                       # null moments
    assert _lib.load().er_measure_ncc(by(t), by(s), *common, 0, 0, 0, FAKE, FAKE, FAKE, FAKE,
                                      0, None) == _lib.ER_OK  # P = 0: nothing to do


def test_volume_utilities_reject_bad_arguments():
    by = ctypes.byref
    _einval("er_volume_moments", None, FAKE, None)
    _einval("er_histogram_u8", by(_vol(_lib.ER_F32)), FAKE, None)
    _einval("er_build_oct", by(_vol(_lib.ER_F64)), FAKE, None)
    _einval("er_build_bitoct", by(_vol()), None, None)
    _einval("er_classify_f64", None, 10, FAKE, None)
    _einval("er_convert_f64", FAKE, 10, _lib.ER_F64, FAKE, None)   # f64 -> f64 is no conversion
    _einval("er_minmax_f64", FAKE, 0, FAKE, None)
    _einval("er_lattice_u8", FAKE, 10, 0.0, -1.0, 1e-12, FAKE, FAKE, None)  # delta <= 0
    assert _lib.load().er_oct_bytes(by(_vol(dims=(3, 4, 5)))) == 4 * 5 * 6 * 8
    assert _lib.load().er_bitoct_bytes(by(_vol(dims=(3, 4, 5)))) == 4 * 5 * 6


def test_smc_and_warp_entry_points_reject_bad_arguments():
    by = ctypes.byref
    six, three, nine = _lib.d6([1] * 6), _lib.d3([0] * 3), _lib.d9([1, 0, 0, 0, 1, 0, 0, 0, 1])
    _einval("er_smc_init", None, 10, ctypes.c_uint64(0), six, None)
    _einval("er_smc_predict", FAKE, None, 10, ctypes.c_uint64(0), 0, six, six, None)
    _einval("er_smc_update", FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, 10, -1.0, 0.5,
            ctypes.c_uint64(0), 0, 0, FAKE, FAKE, None)          # beta < 0
    _einval("er_smc_update", FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, 0, 50.0, 0.5,
            ctypes.c_uint64(0), 0, 0, FAKE, FAKE, None)          # no particles
    _einval("er_states_to_affine", FAKE, 0, -1, three, three, three, three, three, FAKE, FAKE,
            None)
    _einval("er_argmax_update", None, 10, 0, FAKE, None)
    _einval("er_resample", None, nine, three, 4, 4, 4, FAKE, None)
    _einval("er_warp_dice_counts", None, nine, three, by(_vol()), FAKE, None)
    _einval("er_warp_ncc_sums", None, by(_vol()), nine, three, 0, FAKE, None)


def test_phantom_and_debug_entry_points_reject_bad_arguments():
    three = _lib.d3([1, 1, 1])
    assert _lib.load().er_phantom_scratch_bytes(0) == 0
    _einval("er_phantom_speckle", ctypes.c_uint64(0), 0, 0.3, FAKE, 1 << 30, FAKE, None, None)
    _einval("er_phantom_speckle", ctypes.c_uint64(0), 100, 0.3, FAKE, 16, FAKE, None, None)
    _einval("er_phantom_frame", None, 4, 4, 4, three, three, three, three, FAKE, None, None)
    _einval("er_quantize_u8", None, 10, 1.0, 10, FAKE, None)
    _einval("er_binarize_u8", FAKE, -1, 0.5, 0, FAKE, None)
    assert _lib.load().er_debug_bounds_faults(None) == _lib.ER_EINVAL
