"""Device residency: volumes, streams and small buffers on the B200.

PyTorch is used purely as the allocator/stream plumbing: tensors own the
device memory, raw pointers go to the C ABI.  Every volume is uploaded once
and cached on the (immutable) Volume3 object; its storage type is chosen
losslessly:

* codec hint (raw uint8 + z-score affine)   -> u8, alpha = 1/std, gamma = -mean/std
* binary mask (volume.py:138-140)           -> u8, verbatim
* integers in 0..255                        -> u8, verbatim
* exactly fp32-representable                -> f32, verbatim
* anything else                             -> f64, verbatim
The classification runs on the device (er_classify_f64) on the fp64 upload.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import InternalError

_torch = None
_tls = threading.local()


def torch():
    global _torch
    if _torch is None:
        import torch as t

        _torch = t
    return _torch


def require_cuda(device=None):
    t = torch()
    if not t.cuda.is_available():
        raise InternalError(
            "no CUDA device: the sm_100a path has no CPU fallback "
            "(run on a B200 via gpurun)")
    _lib.load()
    if isinstance(device, t.device):
        return device if device.index is not None else t.device("cuda", t.cuda.current_device())
    return t.device("cuda", t.cuda.current_device() if device is None else int(device))


def stream_ptr(device=None) -> ctypes.c_void_p:
    t = torch()
    s = t.cuda.current_stream(device)
    return ctypes.c_void_p(s.cuda_stream)


def ptr(tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(tensor.data_ptr())


_DT = {_lib.ER_U8: "uint8", _lib.ER_F32: "float32", _lib.ER_F64: "float64"}


@dataclass
class DeviceVolume:
    """A volume resident in HBM plus its C-ABI descriptor."""

    storage: object          # torch tensor (flat)
    desc: _lib.ErVolume
    dims: tuple
    spacing: tuple
    origin: tuple
    moments: object          # torch f64 [ER_MOMENTS_DOUBLES], [0]=sum, [1]=sumsq of stored
    dtype_code: int
    shared: object = None    # _SharedU8 for 8-bit storage (oct / histogram cache)

    @property
    def desc_ptr(self):
        return ctypes.byref(self.desc)

    @property
    def nbytes(self) -> int:
        return int(self.storage.numel() * self.storage.element_size())

    def fast_layout_fits(self) -> bool:
        """The fast kernels index padded cells in 32 bits: a padded grid of
        >= 2^31 cells (only thin volumes, given < 2^31 voxels) gets no fast
        layout and takes the generic gather kernel (er_measure_ncc decides
        the same way)."""
        nx, ny, nz = self.dims
        return (nx + 1) * (ny + 1) * (nz + 1) < 2**31

    def ensure_oct(self):
        """Build (once per 8-bit array) the oct re-layout used by the
        measurement fast path: all 8 trilinear corners of a cell in 8 bytes."""
        if self.dtype_code != _lib.ER_U8 or self.desc.oct_dev or not self.fast_layout_fits():
            return
        sh = self.shared
        if sh is None or sh.oct is None:
            t = torch()
            nbytes = int(_lib.load().er_oct_bytes(ctypes.byref(self.desc)))
            oct_ = t.empty(nbytes, dtype=t.uint8, device=self.storage.device)
            _lib.call("er_build_oct", ctypes.byref(self.desc), ptr(oct_),
                      stream_ptr(self.storage.device))
            if sh is None:
                self.oct = oct_
            else:
                sh.oct = oct_
        self.desc.oct_dev = (sh.oct if sh is not None else self.oct).data_ptr()

    def stored_binary(self) -> bool:
        """True when every stored byte is 0 or 1 (exact, from the histogram)."""
        if self.dtype_code != _lib.ER_U8:
            return False
        b = getattr(self, "_binary", None)
        if b is None:
            b = bool(self.histogram()[2:].sum() == 0)
            self._binary = b
        return b

    def ensure_bitoct(self):
        """Build (once per 8-bit array) the bit-oct re-layout of a binary
        source: the 8 corner bits of a cell in one byte (mask fast path)."""
        if self.desc.bitoct_dev or not self.fast_layout_fits():
            return
        sh = self.shared
        lay = getattr(sh, "bitoct", None) if sh is not None else getattr(self, "bitoct", None)
        if lay is None:
            t = torch()
            nbytes = int(_lib.load().er_bitoct_bytes(ctypes.byref(self.desc)))
            lay = t.empty(nbytes, dtype=t.uint8, device=self.storage.device)
            _lib.call("er_build_bitoct", ctypes.byref(self.desc), ptr(lay),
                      stream_ptr(self.storage.device))
            if sh is not None:
                sh.bitoct = lay
            else:
                self.bitoct = lay
        self.desc.bitoct_dev = lay.data_ptr()

    def quad_fits(self) -> bool:
        nx, ny, nz = self.dims
        return (nx + 1) * (ny + 1) * (nz + 2) < 2**31

    def ensure_quad(self):
        """Build (once) the quad re-layout of an f32/f64-stored source (the
        fp32-lerp fast path for non-8-bit data: two adjacent 16-byte loads per
        sample instead of eight scalar gathers)."""
        if self.dtype_code not in (_lib.ER_F32, _lib.ER_F64) or self.desc.quad_dev \
                or not self.quad_fits():
            return
        lay = getattr(self, "quad", None)
        if lay is None:
            t = torch()
            nbytes = int(_lib.load().er_quad_bytes(ctypes.byref(self.desc)))
            lay = t.empty(nbytes, dtype=t.uint8, device=self.storage.device)
            _lib.call("er_build_quad", ctypes.byref(self.desc), ptr(lay),
                      stream_ptr(self.storage.device))
            self.quad = lay
        self.desc.quad_dev = lay.data_ptr()

    def ensure_fast_layout(self):
        """The fp32-lerp fast-path layout for this source: bit-oct for binary
        8-bit data, oct for other 8-bit data, quad for f32/f64 storage."""
        if self.dtype_code != _lib.ER_U8:
            self.ensure_quad()
        elif self.stored_binary():
            self.ensure_bitoct()
        else:
            self.ensure_oct()

    def histogram(self) -> np.ndarray:
        """Exact 256-bin histogram of 8-bit storage (er_histogram_u8), cached."""
        if self.dtype_code != _lib.ER_U8:
            raise ValueError("histogram needs 8-bit storage")
        sh = self.shared
        if sh is not None and sh.hist is not None:
            return sh.hist
        t = torch()
        h = t.empty(256, dtype=t.int64, device=self.storage.device)
        _lib.call("er_histogram_u8", ctypes.byref(self.desc), ptr(h),
                  stream_ptr(self.storage.device))
        hist = h.cpu().numpy()
        if sh is not None:
            sh.hist = hist
        return hist


@dataclass
class _SharedU8:
    """One device upload of one raw 8-bit host array, shared by every volume
    (any affine) built on it: storage, stored-value moments, oct, histogram."""

    raw_ref: object
    storage: object
    moments: object
    oct: object = None
    hist: object = None
    bitoct: object = None


_U8_STORE: dict = {}


def _make_desc(storage, code, dims, alpha, gamma):
    d = _lib.ErVolume()
    d.data_dev = storage.data_ptr()
    d.dtype = code
    d.nx, d.ny, d.nz = (int(x) for x in dims)
    d.alpha = float(alpha)
    d.gamma = float(gamma)
    return d


def _shared_u8(raw: np.ndarray, device, pinned_staging=False) -> _SharedU8:
    import weakref

    key = (id(raw), device.index)
    hit = _U8_STORE.get(key)
    if hit is not None and hit.raw_ref() is raw:
        return hit
    t = torch()
    flat = np.ascontiguousarray(raw, dtype=np.uint8).reshape(-1)
    host = t.from_numpy(flat)
    if pinned_staging and not host.is_pinned():
        host = host.pin_memory()
    storage = host.to(device, non_blocking=host.is_pinned())
    desc = _make_desc(storage, _lib.ER_U8, raw.shape, 1.0, 0.0)
    moments = t.empty(_lib.ER_MOMENTS_DOUBLES, dtype=t.float64, device=device)
    _lib.call("er_volume_moments", ctypes.byref(desc), ptr(moments), stream_ptr(device))
    try:
        ref = weakref.ref(raw, lambda _r, k=key: _U8_STORE.pop(k, None))
    except TypeError:  # pragma: no cover - non-weakrefable array
        ref = (lambda r=raw: r)
    sh = _SharedU8(ref, storage, moments)
    _U8_STORE[key] = sh
    return sh


def _try_lattice(f64, flat_host: np.ndarray, device, stream):
    """8-bit data behind an affine image (x = x0 + k delta, k in 0..255), e.g.
    the reference's z-score of 8-bit echo data arriving as plain fp64: the
    step comes from the distinct values of a host sample, the offset from the
    exact device minimum, and every voxel is verified on the device
    (er_lattice_u8) to reproduce x within a few hundred ulps.  Returns
    (u8 storage, delta, x0) or None."""
    t = torch()
    n = f64.numel()
    sample = np.unique(flat_host[:: max(1, n // 65536)])
    if sample.size < 2 or sample.size > 256:
        return None
    delta0 = float(np.diff(sample).min())
    if not delta0 > 0.0:
        return None
    mm = t.empty(2, dtype=t.float64, device=device)
    _lib.call("er_minmax_f64", ptr(f64), n, ptr(mm), stream)
    x0, x1 = (float(v) for v in mm.tolist())
    kmax = int(round((x1 - x0) / delta0))
    if kmax < 1 or kmax > 255:
        return None
    delta = (x1 - x0) / kmax
    tol = 256.0 * np.finfo(np.float64).eps * max(abs(x0), abs(x1), delta * 255.0)
    u8 = t.empty(n, dtype=t.uint8, device=device)
    flag = t.empty(1, dtype=t.int32, device=device)
    _lib.call("er_lattice_u8", ptr(f64), n, x0, delta, tol, ptr(u8), ptr(flag), stream)
    if int(flag.item()) != 1:
        return None
    return u8, delta, x0


def upload_array(data: np.ndarray, device, *, pinned_staging=False, lattice=False):
    """Upload one fp64 volume and pick a lossless storage type on the device.
    ``lattice``: also recognise affine images of 8-bit data (stored as u8
    with the affine in the descriptor; values reproduced to ~1e-13)."""
    t = torch()
    dims = tuple(int(x) for x in data.shape)
    if len(dims) != 3:
        raise ValueError("volume must be 3D")
    if int(np.prod(dims)) >= 2**31:
        raise ValueError("volume too large for one device descriptor (>= 2^31 voxels)")
    stream = stream_ptr(device)
    flat = np.ascontiguousarray(data, dtype=np.float64).reshape(-1)
    host = t.from_numpy(flat)
    if pinned_staging:
        host = host.pin_memory()
    f64 = host.to(device, non_blocking=pinned_staging)
    flags = t.empty(3, dtype=t.int32, device=device)
    _lib.call("er_classify_f64", ptr(f64), f64.numel(), ptr(flags), stream)
    binary, f32ok, u8ok = (bool(x) for x in flags.tolist())
    if binary or u8ok:
        storage = t.empty(f64.numel(), dtype=t.uint8, device=device)
        _lib.call("er_convert_f64", ptr(f64), f64.numel(), _lib.ER_U8, ptr(storage), stream)
        code = _lib.ER_U8
    elif f32ok:
        storage = t.empty(f64.numel(), dtype=t.float32, device=device)
        _lib.call("er_convert_f64", ptr(f64), f64.numel(), _lib.ER_F32, ptr(storage), stream)
        code = _lib.ER_F32
    else:
        storage, code = f64, _lib.ER_F64
    alpha, gamma = 1.0, 0.0
    if code == _lib.ER_F64 and lattice:
        hit = _try_lattice(f64, flat, device, stream)
        if hit is not None:
            storage, alpha, gamma = hit
            code = _lib.ER_U8
    desc = _make_desc(storage, code, dims, alpha, gamma)
    moments = t.empty(_lib.ER_MOMENTS_DOUBLES, dtype=t.float64, device=device)
    _lib.call("er_volume_moments", ctypes.byref(desc), ptr(moments), stream)
    return storage, desc, moments, code


def device_volume(v, device=None) -> DeviceVolume:
    """Device copy of a Volume3 (cached on the object; volumes are immutable).
    8-bit codec volumes share one upload per raw array; their fp64 ``data``
    is never touched."""
    dev = require_cuda(device)
    cache = getattr(v, "_er_device_cache", None)
    if cache is None:
        cache = {}
        object.__setattr__(v, "_er_device_cache", cache)
    key = dev.index
    hit = cache.get(key)
    if hit is not None:
        return hit
    codec = getattr(v, "codec", None)
    if codec is not None:
        sh = _shared_u8(codec.raw, dev)
        desc = _make_desc(sh.storage, _lib.ER_U8, v.dims, 1.0 / codec.std,
                          -codec.mean / codec.std)
        dv = DeviceVolume(sh.storage, desc, tuple(v.dims), tuple(v.spacing), tuple(v.origin),
                          sh.moments, _lib.ER_U8, sh)
    else:
        storage, desc, moments, code = upload_array(v.data, dev)
        dv = DeviceVolume(storage, desc, tuple(v.dims), tuple(v.spacing), tuple(v.origin),
                          moments, code)
    cache[key] = dv
    return dv


def device_volume_from_array(data: np.ndarray, device=None, spacing=(1.0, 1.0, 1.0),
                             origin=(0.0, 0.0, 0.0), pinned_staging=False,
                             lattice=False) -> DeviceVolume:
    """Uncached upload of a bare array (kernel-module seam: arrays, not Volume3)."""
    dev = require_cuda(device)
    storage, desc, moments, code = upload_array(np.asarray(data), dev,
                                                pinned_staging=pinned_staging,
                                                lattice=lattice)
    return DeviceVolume(storage, desc, tuple(int(x) for x in data.shape), tuple(spacing),
                        tuple(origin), moments, code)


class Workspace:
    """Grow-only per-device scratch for the measurement partials."""

    def __init__(self):
        self._bufs = {}

    def get(self, device, nbytes: int):
        t = torch()
        key = (device.index if hasattr(device, "index") else int(device))
        buf = self._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = t.empty(max(int(nbytes), 1), dtype=t.uint8, device=device)
            self._bufs[key] = buf
        return buf


WORKSPACE = Workspace()


def u8_histogram(raw: np.ndarray, device=None) -> np.ndarray:
    """Exact 256-bin histogram of a raw 8-bit host array, computed on the
    device from the (shared, cached) upload -- the ingest step of the z-score
    on 8-bit echo data (volume.normalize_zscore)."""
    dev = require_cuda(device)
    sh = _shared_u8(raw, dev)
    if sh.hist is None:
        t = torch()
        desc = _make_desc(sh.storage, _lib.ER_U8, raw.shape, 1.0, 0.0)
        h = t.empty(256, dtype=t.int64, device=dev)
        _lib.call("er_histogram_u8", ctypes.byref(desc), ptr(h), stream_ptr(dev))
        sh.hist = h.cpu().numpy()
    return sh.hist


def adopt_u8(raw: np.ndarray, storage, device=None) -> _SharedU8:
    """Register a u8 tensor already resident on the device as the upload of
    the host array ``raw`` (same bytes), so volumes built on ``raw`` never
    re-upload it (device-generated phantoms)."""
    import weakref

    dev = require_cuda(device)
    key = (id(raw), dev.index)
    desc = _make_desc(storage, _lib.ER_U8, raw.shape, 1.0, 0.0)
    t = torch()
    moments = t.empty(_lib.ER_MOMENTS_DOUBLES, dtype=t.float64, device=dev)
    _lib.call("er_volume_moments", ctypes.byref(desc), ptr(moments), stream_ptr(dev))
    ref = weakref.ref(raw, lambda _r, k=key: _U8_STORE.pop(k, None))
    sh = _SharedU8(ref, storage.reshape(-1), moments)
    _U8_STORE[key] = sh
    return sh


def adopt_f64(v, storage, device=None) -> DeviceVolume:
    """Attach a resident fp64 tensor (same values as ``v.data``) as the device
    copy of the fp64 volume ``v``."""
    dev = require_cuda(device)
    t = torch()
    flat = storage.reshape(-1)
    desc = _make_desc(flat, _lib.ER_F64, v.dims, 1.0, 0.0)
    moments = t.empty(_lib.ER_MOMENTS_DOUBLES, dtype=t.float64, device=dev)
    _lib.call("er_volume_moments", ctypes.byref(desc), ptr(moments), stream_ptr(dev))
    dv = DeviceVolume(flat, desc, tuple(v.dims), tuple(v.spacing), tuple(v.origin), moments,
                      _lib.ER_F64)
    cache = getattr(v, "_er_device_cache", None)
    if cache is None:
        cache = {}
        object.__setattr__(v, "_er_device_cache", cache)
    cache[dev.index] = dv
    return dv
