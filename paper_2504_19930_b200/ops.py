"""Thin torch-tensor wrappers over the C ABI (device in, device out).

Each function launches on the current torch stream of the tensors' device
and never synchronises, except where a host value is explicitly returned.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .device import (WORKSPACE, DeviceVolume, device_volume, ptr, require_cuda,
                     stream_ptr, torch)
from .errors import BadConfig

LERP_MODES = {"f32": _lib.ER_LERP_F32, "f64": _lib.ER_LERP_F64, "exact": _lib.ER_LERP_EXACT,
              "nearest": _lib.ER_LERP_NEAREST}


def lerp_code(precision: str) -> int:
    try:
        return LERP_MODES[precision]
    except KeyError:
        raise BadConfig(f"precision must be one of {sorted(LERP_MODES)}, got {precision!r}")


def prepare_layouts(tdv: DeviceVolume, sdv: DeviceVolume, precision: str):
    """Build (once) the source layout the measurement uses in this mode."""
    if precision in ("f32", "nearest"):
        sdv.ensure_fast_layout()       # bit-oct for binary sources, else oct
    elif precision == "f64":
        sdv.ensure_oct()


def workspace_bytes(tdv: DeviceVolume, P: int) -> int:
    return int(_lib.load().er_measure_workspace_bytes(tdv.desc_ptr, int(P)))


def measure(tdv: DeviceVolume, sdv: DeviceVolume, A, B, overlap: bool, precision="f64",
            out=None, workspace=None):
    """Squared NCC per particle on device.  A: (P, 9) f64, B: (P, 3) f64 tensors.
    Returns (ncc f64[P], degenerate u8[P], n_in i64[P]) device tensors.
    ``workspace``: a caller-owned uint8 scratch tensor (else the shared
    per-device one, which concurrent streams must not share)."""
    t = torch()
    dev = A.device
    P = int(A.shape[0])
    if out is None:
        out = (t.empty(P, dtype=t.float64, device=dev), t.empty(P, dtype=t.uint8, device=dev),
               t.empty(P, dtype=t.int64, device=dev))
    ncc, degen, n_in = out
    if P == 0:
        return ncc, degen, n_in
    prepare_layouts(tdv, sdv, precision)
    need = workspace_bytes(tdv, P)
    if workspace is not None and workspace.numel() >= need:
        ws = workspace
    else:
        ws = WORKSPACE.get(dev, need)
    _lib.call("er_measure_ncc", tdv.desc_ptr, sdv.desc_ptr, ptr(tdv.moments), ptr(A), ptr(B),
              P, int(bool(overlap)), lerp_code(precision), ptr(ncc), ptr(degen), ptr(n_in),
              ptr(ws), ws.numel(), stream_ptr(dev))
    if refines(sdv, precision):
        _lib.launch_count += 2   # the refinement pass and its list finalize
    return ncc, degen, n_in


def refines(sdv: DeviceVolume, precision: str) -> bool:
    """Whether er_measure_ncc runs its fp64 refinement pass for this source
    (fp32 lerps on a non-binary u8 source, an f32-stored source, or an
    f64-stored source through its quad layout)."""
    return (precision == "f32" and not sdv.desc.bitoct_dev
            and (sdv.dtype_code != _lib.ER_F64 or bool(sdv.desc.quad_dev)))


def _as_dv(v, device=None) -> DeviceVolume:
    return v if isinstance(v, DeviceVolume) else device_volume(v, device)


def resample_device(source, a, b, out_dims, device=None):
    """er_resample: f64 device tensor of shape out_dims."""
    dv = _as_dv(source, device)
    dev = dv.storage.device
    t = torch()
    out = t.empty(tuple(int(d) for d in out_dims), dtype=t.float64, device=dev)
    _lib.call("er_resample", dv.desc_ptr, _lib.d9(np.ravel(a)), _lib.d3(np.ravel(b)),
              *(int(d) for d in out_dims), ptr(out), stream_ptr(dev))
    return out


def dice_counts(src_mask, tgt_mask, a, b, device=None):
    """(|moved > 0.5|, |target|, |both|) as exact integers (one sync)."""
    s = _as_dv(src_mask, device)
    tm = _as_dv(tgt_mask, device)
    t = torch()
    counts = t.empty(3, dtype=t.int64, device=s.storage.device)
    _lib.call("er_warp_dice_counts", s.desc_ptr, _lib.d9(np.ravel(a)), _lib.d3(np.ravel(b)),
              tm.desc_ptr, ptr(counts), stream_ptr(s.storage.device))
    return counts


def ncc_sums(tgt, src, a=None, b=None, identity=False, device=None):
    """Two-pass centred sums {sst, sss, sts, n} of (tgt, warp(src)) on device."""
    tv = _as_dv(tgt, device)
    sv = _as_dv(src, device)
    t = torch()
    out = t.empty(_lib.ER_NCC_SUMS_DOUBLES, dtype=t.float64, device=tv.storage.device)
    A = _lib.d9(np.ravel(a) if a is not None else np.eye(3).ravel())
    B = _lib.d3(np.ravel(b) if b is not None else np.zeros(3))
    _lib.call("er_warp_ncc_sums", tv.desc_ptr, sv.desc_ptr, A, B, int(bool(identity)),
              ptr(out), stream_ptr(tv.storage.device))
    return out[:4]


def states_to_affine(states, first, count, center, tgt_geom, src_geom, A=None, B=None):
    """Device to_matrix + index_affine for states[first:first+count].
    tgt_geom / src_geom: (spacing, origin)."""
    t = torch()
    dev = states.device
    if A is None:
        A = t.empty((count, 9), dtype=t.float64, device=dev)
        B = t.empty((count, 3), dtype=t.float64, device=dev)
    _lib.call("er_states_to_affine", ptr(states), int(first), int(count), _lib.d3(center),
              _lib.d3(tgt_geom[0]), _lib.d3(tgt_geom[1]), _lib.d3(src_geom[0]),
              _lib.d3(src_geom[1]), ptr(A), ptr(B), stream_ptr(dev))
    return A, B


def smc_init(n, seed, lim, device):
    t = torch()
    states = t.empty((n, 6), dtype=t.float64, device=device)
    _lib.call("er_smc_init", ptr(states), int(n), ctypes.c_uint64(int(seed)), _lib.d6(lim),
              stream_ptr(device))
    return states


def smc_predict(states_in, states_out, seed, k, sigma, clip):
    n = int(states_in.shape[0])
    _lib.call("er_smc_predict", ptr(states_in), ptr(states_out), n, ctypes.c_uint64(int(seed)),
              int(k), _lib.d6(sigma), _lib.d6(clip), stream_ptr(states_in.device))
    return states_out


def require(device=None):
    return require_cuda(device)


def refined_count(tdv: DeviceVolume, P: int, workspace=None) -> int:
    """Number of particles the last f32 measurement with this workspace
    re-measured in fp64 (er_measure_ncc refinement; one sync).  Diagnostic."""
    t = torch()
    need = workspace_bytes(tdv, P)
    ws = workspace if workspace is not None else WORKSPACE.get(require_cuda(), need)
    off = need - 16 - 4 * int(P)
    return int(ws[off:off + 4].view(t.int32).item())
