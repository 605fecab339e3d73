"""On-device phantom generator.

The reference builds its synthetic cases on the CPU (E/phantom.py:61-166):
a log-normal speckle field from numpy's Philox + ziggurat, a speckled
ellipsoidal shell per frame, and the source frames pulled through the
inverse ground truth.  Here every step runs on the GPU with the reference's
exact arithmetic (csrc/phantom.cu):

* speckle normals bit-exact with ``Generator(Philox(key=seed))
  .standard_normal`` (the ziggurat's variable word consumption is resolved
  with a parallel chunked chain walk), ``np.exp`` restated bit-exactly
  (numpy's AVX512 SVML exp, csrc/npexp.cuh);
* frames and cavity masks in numpy's fp64 operation order;
* source frames through ``er_resample`` (the reference resampler's op
  order), 8-bit quantisation ``clip(round(x * scale), 0, 255)`` on device.

Generated volumes are handed to the host API as ordinary ``Volume3``
objects whose device copies are the generated tensors (no re-upload).
``make_phantom_device`` mirrors ``make_phantom``; ``echo_case_device``
mirrors ``phantom.echo_case`` (BASELINE C2/C3/C5 workloads).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _lib
from .device import (_make_desc, adopt_f64, adopt_u8, ptr, require_cuda,
                     stream_ptr, torch)
from .geometry import index_affine, inverse, to_matrix
from .metrics import dice
from .phantom import (ECHO_DIMS, ECHO_SPACING, ECHO_TRUTH, PhantomSpec, RegistrationCase,
                      echo_spec, grid_center, phantom_center)
from .volume import Sequence4, Volume3


def speckle(spec: PhantomSpec, device=None, with_normals: bool = False):
    """exp(sigma * standard_normal(dims)) of Philox(key=seed), flat f64 on device
    (E/phantom.py:76-77).  With ``with_normals`` also returns the normals."""
    dev = require_cuda(device)
    t = torch()
    n = int(np.prod(spec.dims))
    lib = _lib.load()
    scratch = t.empty(int(lib.er_phantom_scratch_bytes(n)), dtype=t.uint8, device=dev)
    out = t.empty(n, dtype=t.float64, device=dev)
    normals = t.empty(n, dtype=t.float64, device=dev) if with_normals else None
    _lib.call("er_phantom_speckle", int(spec.seed), n, float(spec.speckle_sigma), ptr(scratch),
              scratch.numel(), ptr(out), ptr(normals) if normals is not None else None,
              stream_ptr(dev))
    return (out, normals) if with_normals else out


def frame_axes(spec: PhantomSpec, k: int):
    """Semi-axes of frame k, computed as _ellipsoid_radius does (E/phantom.py:80-82,94-95)."""
    scale = 1.0 - spec.amplitude * math.sin(math.pi * k / spec.frames) ** 2
    return (tuple(a * scale for a in spec.outer_semiaxes),
            tuple(a * scale for a in spec.inner_semiaxes))


def frame_device(spec: PhantomSpec, k: int, speckle_dev, frame=True, mask=True, device=None,
                 mask_out=None):
    """Frame k (f64) and its cavity mask (u8) as flat device tensors (the mask
    into ``mask_out`` when given)."""
    dev = require_cuda(device)
    t = torch()
    n = int(np.prod(spec.dims))
    f = t.empty(n, dtype=t.float64, device=dev) if frame else None
    m = mask_out if mask_out is not None else (
        t.empty(n, dtype=t.uint8, device=dev) if mask else None)
    outer, inner = frame_axes(spec, k)
    _lib.call("er_phantom_frame", ptr(speckle_dev) if frame else None,
              *(int(d) for d in spec.dims), _lib.d3(spec.spacing),
              _lib.d3(phantom_center(spec)), _lib.d3(outer), _lib.d3(inner),
              ptr(f) if frame else None, ptr(m) if m is not None else None, stream_ptr(dev))
    return f, m


_PINNED = {}


def _to_host(dev_u8) -> np.ndarray:
    """Device bytes -> a fresh host array through a reused pinned staging
    buffer (pageable device-to-host copies run at a fraction of the speed)."""
    t = torch()
    n = dev_u8.numel()
    buf = _PINNED.get("u8")
    if buf is None or buf.numel() < n:
        buf = t.empty(n, dtype=t.uint8, pin_memory=True)
        _PINNED["u8"] = buf
    buf[:n].copy_(dev_u8.reshape(-1), non_blocking=True)
    t.cuda.current_stream(dev_u8.device).synchronize()
    return buf[:n].numpy().copy()


def _host_u8(dev_u8, dims, spacing, origin=(0.0, 0.0, 0.0)) -> Volume3:
    raw = _to_host(dev_u8).reshape(dims)
    vol = Volume3.from_u8(raw, spacing, origin)
    adopt_u8(raw, dev_u8, dev_u8.device)
    return vol


def make_phantom_device(spec: PhantomSpec, device=None):
    """make_phantom (E/phantom.py:61-91) generated on the GPU: identical frames
    and masks; each frame's device copy is the generated tensor."""
    spec.validate()
    dev = require_cuda(device)
    sp = speckle(spec, dev)
    frames, masks = [], []
    for k in range(spec.frames):
        f, m = frame_device(spec, k, sp, device=dev)
        vol = Volume3(f.reshape(spec.dims).cpu().numpy(), spec.spacing)
        adopt_f64(vol, f, dev)
        frames.append(vol)
        masks.append(_host_u8(m, spec.dims, spec.spacing))
    return Sequence4(frames, frame_rate=spec.frame_rate, ed_index=0), masks


def _resample_flat(storage, code, dims, a, b, dev):
    t = torch()
    desc = _make_desc(storage, code, dims, 1.0, 0.0)
    out = t.empty(int(np.prod(dims)), dtype=t.float64, device=dev)
    _lib.call("er_resample", ctypes.byref(desc), _lib.d9(np.ravel(a)), _lib.d3(np.ravel(b)),
              *(int(d) for d in dims), ptr(out), stream_ptr(dev))
    return out


def _percentile_999(frame0_dev, dims) -> float:
    # np.percentile's own interpolation on the host copy of frame 0 (51 MB at C2)
    return float(np.percentile(frame0_dev.reshape(dims).cpu().numpy(), 99.9))


def echo_case_device(dims=ECHO_DIMS, spacing=ECHO_SPACING, frames=1, seed=0, truth=ECHO_TRUTH,
                     device=None) -> RegistrationCase:
    """phantom.echo_case on the GPU: the echo-sized phantom, the pair under
    ``truth`` (make_pair, E/phantom.py:120-166) and the 8-bit quantisation,
    all device-resident; only the 8-bit results are copied to the host."""
    spec = echo_spec(dims, spacing, frames, seed)
    spec.validate()
    dev = require_cuda(device)
    sp = speckle(spec, dev)
    grid = Volume3(np.zeros((1, 1, 1)), spec.spacing)  # spacing/origin for index_affine
    m_inv = inverse(to_matrix(truth, grid_center(spec.dims, spec.spacing, grid.origin)))
    a, b = index_affine(m_inv, grid, grid)
    n = int(np.prod(spec.dims))
    t = torch()
    f0, _ = frame_device(spec, 0, sp, mask=False, device=dev)
    scale = 255.0 / _percentile_999(f0, spec.dims)
    del f0
    tq, sq, tm, sm = [], [], [], []
    # the 8-bit results stay resident (they become the volumes' device
    # copies): one allocation for all of them, sliced per frame
    outs = t.empty((spec.frames, 4, n), dtype=t.uint8, device=dev)
    for k in range(spec.frames):
        u8, su8, m, sm8 = outs[k]
        f, _ = frame_device(spec, k, sp, device=dev, mask_out=m)
        _lib.call("er_quantize_u8", ptr(f), n, scale, n, ptr(u8), stream_ptr(dev))
        tq.append(_host_u8(u8, spec.dims, spec.spacing))
        moved = _resample_flat(f, _lib.ER_F64, spec.dims, a, b, dev)
        _lib.call("er_quantize_u8", ptr(moved), n, scale, n, ptr(su8), stream_ptr(dev))
        sq.append(_host_u8(su8, spec.dims, spec.spacing))
        mm = _resample_flat(m, _lib.ER_U8, spec.dims, a, b, dev)
        _lib.call("er_binarize_u8", ptr(mm), n, 0.5, n, ptr(sm8), stream_ptr(dev))
        tm.append(_host_u8(m, spec.dims, spec.spacing))
        sm.append(_host_u8(sm8, spec.dims, spec.spacing))
        del f, moved, mm
    ed = 0
    target = Sequence4(tq, frame_rate=spec.frame_rate, ed_index=ed)
    source = Sequence4(sq, frame_rate=spec.frame_rate, ed_index=ed)
    return RegistrationCase(target=target, source=source, target_masks=tm, source_masks=sm,
                            truth=truth, overlap_crop=0.0, seed=0,
                            initial_dsc=float(dice(tm[ed], sm[ed])), case_id="phantom")
