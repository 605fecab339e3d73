"""Device phantom generator (phantom_device.py, csrc/phantom.cu, SURVEY.md
§8f rank 3) against the reference generator (E/phantom.py:61-166): the
reference's own outputs (tests/golden/phantom.npz), numpy's Philox normals
and numpy's exp (tests/golden/npexp.npz)."""

import ctypes
import math
import os
import subprocess

import numpy as np
import pytest

from .conftest import ROOT, golden

CSRC = os.path.join(ROOT, "paper_2504_19930_b200", "csrc")
HOST_SO = os.path.join(ROOT, "tests", "_build", "libnpexp_host.so")


@pytest.fixture(scope="module")
def npexp_host():
    os.makedirs(os.path.dirname(HOST_SO), exist_ok=True)
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-frounding-math", "-fPIC", "-shared",
                    f"-I{CSRC}", os.path.join(ROOT, "tests", "native", "npexp_host.cpp"),
                    "-o", HOST_SO, "-lm"], check=True)
    lib = ctypes.CDLL(HOST_SO)
    d = ctypes.POINTER(ctypes.c_double)
    lib.er_host_npexp.argtypes = [d, d, ctypes.c_int64]
    return lib


def test_npexp_restatement_bit_exact_with_numpy_exp(npexp_host):
    """csrc/npexp.cuh (numpy's AVX512 SVML exp restated) reproduces np.exp on
    every known-answer vector: the phantom range, the whole non-special
    range, tiny arguments, signed zeros."""
    g = golden("npexp.npz")
    x = np.ascontiguousarray(g["x"])
    y = np.empty_like(x)
    d = ctypes.POINTER(ctypes.c_double)
    npexp_host.er_host_npexp(x.ctypes.data_as(d), y.ctypes.data_as(d), x.size)
    bad = np.flatnonzero(y.view(np.uint64) != g["exp"].view(np.uint64))
    assert bad.size == 0, (x[bad[:5]], y[bad[:5]], g["exp"][bad[:5]])


def test_npexp_vectors_are_not_correctly_rounded_exp():
    """Why the restatement exists: numpy's exp differs from the platform's
    scalar exp on a sizeable share of the phantom's arguments."""
    g = golden("npexp.npz")
    x, want = g["x"][:60000], g["exp"][:60000]
    scalar = np.array([math.exp(v) for v in x])
    assert (scalar != want).sum() > 100


gpu = pytest.mark.gpu


def _phantom_golden_spec():
    from paper_2504_19930_b200 import PhantomSpec

    return PhantomSpec(dims=(20, 18, 22), spacing=(1.1, 0.9, 1.3), frames=3, seed=11,
                       outer_semiaxes=(8.0, 7.0, 9.0), inner_semiaxes=(5.0, 4.0, 6.0))


@gpu
@pytest.mark.parametrize("seed,dims", [(0, (64, 64, 64)), (11, (20, 18, 22)),
                                       (2**40 + 3, (37, 1, 29)), (7, (176, 176, 208))])
def test_speckle_normals_bit_exact_with_numpy(seed, dims):
    from paper_2504_19930_b200 import PhantomSpec
    from paper_2504_19930_b200.phantom_device import speckle

    spec = PhantomSpec(dims=dims, seed=seed)
    sp, z = speckle(spec, with_normals=True)
    want = np.random.Generator(np.random.Philox(key=seed)).standard_normal(dims).reshape(-1)
    got = z.cpu().numpy()
    bad = np.flatnonzero(got != want)
    assert bad.size == 0, (bad[:5], got[bad[:5]], want[bad[:5]])
    from numpy._core._multiarray_umath import __cpu_features__

    if __cpu_features__.get("AVX512_SKX"):  # this host's np.exp is the SVML variant
        assert np.array_equal(sp.cpu().numpy(), np.exp(spec.speckle_sigma * want))


@gpu
def test_make_phantom_device_equals_reference_outputs():
    """Frames and masks bit-identical to the reference generator's own output;
    make_pair on the generated (device-resident) frames reproduces the
    reference's source frames, masks and initial DSC (overlap crop 0.2)."""
    from paper_2504_19930_b200 import RigidParams, make_pair
    from paper_2504_19930_b200.phantom_device import make_phantom_device

    g = golden("phantom.npz")
    seq, masks = make_phantom_device(_phantom_golden_spec())
    assert np.array_equal(np.stack([f.data for f in seq.frames]), g["frames"])
    assert np.array_equal(np.stack([m.codec.raw for m in masks]), g["masks"])
    truth = RigidParams(math.radians(6), math.radians(-3), math.radians(2), 1.5, -2.0, 0.5)
    case = make_pair(seq, masks, truth, overlap_crop=0.2)
    assert np.array_equal(np.stack([f.data for f in case.source.frames]), g["src_frames"])
    assert np.array_equal(np.stack([m.codec.raw for m in case.source_masks]), g["src_masks"])
    assert case.initial_dsc == float(g["initial_dsc"])


@gpu
@pytest.mark.parametrize("dims,frames,seed", [((40, 36, 44), 3, 0), ((176, 176, 208), 1, 0)])
def test_echo_case_device_equals_host_echo_case(dims, frames, seed):
    """The 8-bit echo workload (BASELINE C2/C3) generated on the device equals
    the host pipeline (make_phantom -> make_pair -> quantize) byte for byte."""
    from paper_2504_19930_b200.phantom import echo_case
    from paper_2504_19930_b200.phantom_device import echo_case_device

    spacing = (0.87, 1.08, 0.73)
    host = echo_case(dims, spacing, frames=frames, seed=seed)
    dev = echo_case_device(dims, spacing, frames=frames, seed=seed)
    for a, b in ((host.target.frames, dev.target.frames), (host.source.frames, dev.source.frames),
                 (host.target_masks, dev.target_masks), (host.source_masks, dev.source_masks)):
        assert len(a) == len(b) == frames
        for k, (x, y) in enumerate(zip(a, b)):
            assert np.array_equal(x.codec.raw, y.codec.raw), k
            assert x.spacing == y.spacing and x.origin == y.origin
    assert host.initial_dsc == dev.initial_dsc


@gpu
def test_phantom_abi_rejects_bad_arguments():
    from paper_2504_19930_b200 import _lib
    from paper_2504_19930_b200.errors import BadConfig

    lib = _lib.load()
    assert lib.er_phantom_scratch_bytes(0) == 0
    with pytest.raises(BadConfig):
        _lib.call("er_phantom_speckle", 0, 0, 0.3, None, 0, None, None, None)
    with pytest.raises(BadConfig):
        _lib.call("er_phantom_speckle", 0, 100, 0.3, 1, 16, 1, None, None)  # scratch too small
    with pytest.raises(BadConfig):
        _lib.call("er_phantom_frame", None, 0, 4, 4, _lib.d3((1, 1, 1)), _lib.d3((0, 0, 0)),
                  _lib.d3((1, 1, 1)), _lib.d3((1, 1, 1)), None, None, None)


@gpu
def test_random_phantom_specs_match_the_host_generator():
    """make_phantom_device == make_phantom (the reference's algorithm) bit for
    bit over random specs: dims, frames, semi-axes, amplitude, speckle sigma,
    spacing, centre, seed."""
    from numpy._core._multiarray_umath import __cpu_features__

    if not __cpu_features__.get("AVX512_SKX"):
        pytest.skip("host np.exp is not the SVML variant the device restates")
    from paper_2504_19930_b200 import PhantomSpec, make_phantom
    from paper_2504_19930_b200.phantom_device import make_phantom_device

    g = np.random.default_rng(2504)
    for _ in range(12):
        dims = tuple(int(x) for x in g.integers(4, 33, 3))
        outer = tuple(float(x) for x in g.uniform(3.0, 14.0, 3))
        inner = tuple(float(o * f) for o, f in zip(outer, g.uniform(0.3, 0.9, 3)))
        spec = PhantomSpec(dims=dims, spacing=tuple(float(x) for x in g.uniform(0.6, 1.4, 3)),
                           outer_semiaxes=outer, inner_semiaxes=inner,
                           center=None if g.random() < 0.5 else
                           tuple(float(x) for x in g.uniform(-2.0, 20.0, 3)),
                           speckle_sigma=float(g.choice([0.0, 0.2, 0.3, 0.7])),
                           amplitude=float(g.uniform(0.0, 0.5)),
                           frames=int(g.integers(1, 5)), seed=int(g.integers(0, 2**40)))
        hs, hm = make_phantom(spec)
        ds, dm = make_phantom_device(spec)
        for a, b in zip(hs.frames, ds.frames):
            assert np.array_equal(a.data, b.data), spec
        for a, b in zip(hm, dm):
            assert np.array_equal(a.codec.raw, b.codec.raw), spec
