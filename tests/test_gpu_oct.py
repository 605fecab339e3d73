"""The 8-bit fast path (oct re-layout + fixed-point coordinates) against the
bit-exact C oracle on u8-valued volumes, including the edge cases the
reference handles by cell clamping (kernels_numba.py:32-55): degenerate
axes of length 1, coordinates exactly on the upper face, quarter turns
(coordinates landing exactly on grid nodes), and far out-of-frame poses.
Tolerances: 1e-4 relative (fp32 lerps), 1e-6 relative (fp64 lerps); counts
and degenerate flags bit-exact."""

import math

import numpy as np
import pytest

from oracle import kernels as ok

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ATOL = 1e-12  # floor for numerically-zero likelihoods, as in test_gpu_measure


def _mats(rng, center, n, rmax, tmax, extra=True):
    from paper_2504_19930_b200 import RigidParams, to_matrix

    ms = [to_matrix(RigidParams(*rng.uniform(-rmax, rmax, 3), *rng.uniform(-tmax, tmax, 3)),
                    center) for _ in range(n)]
    if extra:
        ms += [np.eye(4), to_matrix(RigidParams(tx=1e4)),
               to_matrix(RigidParams(rz=math.pi / 2), center),
               to_matrix(RigidParams(rx=math.pi / 2, ty=1.0), center),
               to_matrix(RigidParams(tx=0.5, tz=-0.25), center)]
    return np.stack(ms)


CASES = [
    # target dims, source dims, same grid
    ((12, 11, 10), (12, 11, 10), True),
    ((9, 13, 7), (11, 8, 12), False),
    ((5, 1, 7), (6, 3, 7), False),
    ((4, 4, 4), (1, 1, 1), False),
    ((6, 5, 4), (2, 1, 3), False),
    ((1, 9, 8), (1, 9, 8), True),
]


@pytest.mark.parametrize("precision,rtol", [("f32", 1e-4), ("f64", 1e-6)])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_oct_path_vs_oracle(case, precision, rtol):
    from paper_2504_19930_b200 import Volume3, ops
    from paper_2504_19930_b200.device import device_volume, require_cuda
    from paper_2504_19930_b200.geometry import index_affine_batch

    tdims, sdims, same = CASES[case]
    rng = np.random.default_rng(100 + case)
    sp_t = tuple(rng.uniform(0.6, 1.4, 3))
    sp_s = sp_t if same else tuple(rng.uniform(0.6, 1.4, 3))
    org_s = (0.0, 0.0, 0.0) if same else tuple(rng.uniform(-1.0, 1.0, 3))
    t = Volume3(rng.integers(0, 256, tdims).astype(np.float64), sp_t)
    s = Volume3(rng.integers(0, 256, sdims).astype(np.float64), sp_s, org_s)
    mats = _mats(rng, t.physical_center(), 40, 0.5, 3.0)
    a, b = index_affine_batch(mats, s.spacing, s.origin, t.spacing, t.origin)
    dev = require_cuda()
    tdv, sdv = device_volume(t, dev), device_volume(s, dev)
    assert sdv.dtype_code == 0  # u8 storage
    A = torch.as_tensor(a.reshape(-1, 9), device=dev)
    B = torch.as_tensor(b.reshape(-1, 3), device=dev)
    for overlap in (False, True):
        z, d, n = (x.cpu().numpy() for x in ops.measure(tdv, sdv, A, B, overlap, precision))
        assert sdv.desc.oct_dev  # the fast path was used
        zo, do, no = ok.ncc_measure_batch(t.data, s.data, a, b, overlap, return_counts=True)
        assert np.array_equal(n, no)
        assert np.array_equal(d.astype(bool), do)
        scale = np.maximum(np.abs(zo), 1e-300)
        err = np.abs(z - zo) / scale
        ok_ = (np.abs(z - zo) <= rtol * np.abs(zo) + ATOL) & ((zo == 0) == (z == 0))
        assert np.all(ok_), float(err.max())


def test_oct_matches_generic_path_on_masks():
    """Binary masks: oct fast path vs the plain-gather path (fp64 exact)."""
    from paper_2504_19930_b200 import Volume3, ops
    from paper_2504_19930_b200.device import device_volume, require_cuda
    from paper_2504_19930_b200.geometry import index_affine_batch

    rng = np.random.default_rng(5)
    x, y, z = np.meshgrid(*(np.arange(n) - n / 2 for n in (40, 36, 44)), indexing="ij")
    m = ((x / 12.0) ** 2 + (y / 10.0) ** 2 + (z / 15.0) ** 2 <= 1.0).astype(np.float64)
    t = Volume3(m)
    s = Volume3(np.roll(m, (2, -1, 3), axis=(0, 1, 2)))
    mats = _mats(rng, t.physical_center(), 64, 0.3, 4.0)
    a, b = index_affine_batch(mats, s.spacing, s.origin, t.spacing, t.origin)
    dev = require_cuda()
    A = torch.as_tensor(a.reshape(-1, 9), device=dev)
    B = torch.as_tensor(b.reshape(-1, 3), device=dev)
    tdv, sdv = device_volume(t, dev), device_volume(s, dev)
    ze, de, ne = (v.cpu().numpy() for v in ops.measure(tdv, sdv, A, B, False, "exact"))
    for prec, rtol in (("f64", 1e-6), ("f32", 1e-4)):
        zf, df, nf = (v.cpu().numpy() for v in ops.measure(tdv, sdv, A, B, False, prec))
        assert np.array_equal(nf, ne) and np.array_equal(df, de)
        err = np.abs(zf - ze) / np.maximum(np.abs(ze), 1e-300)
        ok_ = (np.abs(zf - ze) <= rtol * np.abs(ze) + ATOL) & ((ze == 0) == (zf == 0))
        assert np.all(ok_), (prec, float(err.max()))


def test_large_volume_vs_oracle():
    """512^3 u8 pair (134M voxels, a 1.08 GB oct layout): the fixed-point
    stepping over long rows and the 32-bit cell/target indices at size, vs
    the C oracle on a few poses (counts bit-exact)."""
    from paper_2504_19930_b200 import Volume3, ops
    from paper_2504_19930_b200.device import device_volume, require_cuda
    from paper_2504_19930_b200.geometry import index_affine_batch

    dims = (512, 512, 512)
    rng = np.random.default_rng(512)
    # smooth-ish content so the NCC is far from 0: a coarse random field, repeated
    coarse = rng.integers(0, 256, (64, 64, 64), dtype=np.uint8)
    raw = np.repeat(np.repeat(np.repeat(coarse, 8, 0), 8, 1), 8, 2)
    t = Volume3.from_u8(raw, (0.5, 0.5, 0.5))
    s = Volume3.from_u8(np.roll(raw, 3, axis=2), (0.5, 0.5, 0.5))
    mats = _mats(rng, t.physical_center(), 2, 0.2, 4.0, extra=False)
    mats = np.concatenate([mats, [np.eye(4)]])
    a, b = index_affine_batch(mats, s.spacing, s.origin, t.spacing, t.origin)
    dev = require_cuda()
    tdv, sdv = device_volume(t, dev), device_volume(s, dev)
    A = torch.as_tensor(a.reshape(-1, 9), device=dev)
    B = torch.as_tensor(b.reshape(-1, 3), device=dev)
    zo, do, no = ok.ncc_measure_batch(t.data, s.data, a, b, False, return_counts=True)
    for precision, rtol in (("f32", 1e-4), ("f64", 1e-6)):
        z, d, n = (x.cpu().numpy() for x in ops.measure(tdv, sdv, A, B, False, precision))
        assert sdv.desc.oct_dev
        assert np.array_equal(n, no) and np.array_equal(d.astype(bool), do)
        assert np.all(np.abs(z - zo) <= rtol * np.abs(zo) + ATOL), (precision, z, zo)
    assert no.min() > 0.5 * raw.size  # the poses overlap most of the grid


def test_thin_source_beyond_32bit_cells_takes_the_generic_kernel():
    """A 1 x 1 x 2^29 source has < 2^31 voxels but 2^31 + 4 padded cells:
    no fast layout is built and er_measure_ncc takes the generic kernel.  The
    target only reaches the first few thousand source voxels, so a cropped
    source (oct path; and the oracle) must give the same values."""
    from paper_2504_19930_b200 import RigidParams, Volume3, ops, to_matrix
    from paper_2504_19930_b200.device import device_volume, require_cuda
    from paper_2504_19930_b200.geometry import index_affine_batch

    rng = np.random.default_rng(29)
    n_src = 2**29
    head = rng.integers(0, 256, 8192, dtype=np.uint8)
    big = np.zeros((1, 1, n_src), dtype=np.uint8)
    big[0, 0, :8192] = head
    t = Volume3.from_u8(rng.integers(0, 256, (1, 1, 4096), dtype=np.uint8))
    s_big = Volume3.from_u8(big)
    s_crop = Volume3.from_u8(head.reshape(1, 1, -1))
    mats = np.stack([to_matrix(RigidParams(tz=float(tz))) for tz in (0.0, 0.25, 3.5, 1000.75)])
    dev = require_cuda()
    tdv = device_volume(t, dev)
    out = {}
    for name, s in (("big", s_big), ("crop", s_crop)):
        a, b = index_affine_batch(mats, s.spacing, s.origin, t.spacing, t.origin)
        sdv = device_volume(s, dev)
        A = torch.as_tensor(a.reshape(-1, 9), device=dev)
        B = torch.as_tensor(b.reshape(-1, 3), device=dev)
        out[name] = [x.cpu().numpy() for x in ops.measure(tdv, sdv, A, B, False, "f64")]
        assert bool(sdv.desc.oct_dev) == (name == "crop")
    zo, do, no = ok.ncc_measure_batch(t.data, s_crop.data, a, b, False, return_counts=True)
    for name in ("big", "crop"):
        z, d, n = out[name]
        assert np.array_equal(n, no) and np.array_equal(d.astype(bool), do)
        assert np.all(np.abs(z - zo) <= 1e-6 * np.abs(zo) + ATOL), (name, z, zo)
