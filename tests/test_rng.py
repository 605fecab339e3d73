"""The device RNG restatement (csrc/rng.cuh) against numpy's own draws --
the reference's randomness (echoreg/smc.py:38-42, 150, 171, 239).  The
header is compiled for the host here (test only) so the check runs on CPU;
tests/test_gpu_smc.py repeats it on the device."""

import ctypes
import os
import subprocess

import numpy as np
import pytest

from .conftest import ROOT, golden

CSRC = os.path.join(ROOT, "paper_2504_19930_b200", "csrc")
OUT = os.path.join(ROOT, "tests", "_build", "librng_host.so")


@pytest.fixture(scope="module")
def lib():
    from paper_2504_19930_b200 import _build

    _build.build()  # generates zig_tables.h
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-fPIC", "-shared", f"-I{CSRC}",
                    os.path.join(ROOT, "tests", "native", "rng_host.cpp"), "-o", OUT, "-lm"],
                   check=True)
    L = ctypes.CDLL(OUT)
    d = ctypes.POINTER(ctypes.c_double)
    u = ctypes.c_uint64
    L.er_host_normals.argtypes = [u, u, u, u, ctypes.c_int64, d]
    L.er_host_uniforms.argtypes = [u, u, u, u, ctypes.c_int64, ctypes.c_double,
                                   ctypes.c_double, d]
    return L


def normals(L, seed, role, step, index, n):
    out = np.empty(n)
    L.er_host_normals(seed, role, step, index, n, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    return out


def test_long_stream_bit_exact(lib):
    want = golden("rng.npz")["long_normals"]
    got = normals(lib, 5, 1, 2, 3, want.size)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("seed,k", [(0, 0), (0, 3), (7, 19), (2**31 + 5, 1)])
def test_predict_streams_bit_exact(lib, seed, k):
    want = golden("rng.npz")[f"normals_{seed}_{k}"]
    for i in range(0, want.shape[0], 37):
        assert np.array_equal(normals(lib, seed, 1, k, i, 6), want[i]), i


def test_tail_and_wedge_paths_are_exercised():
    """The long golden stream contains draws beyond the ziggurat base strip
    (|x| > r = 3.654), i.e. the idx == 0 tail path was hit and matched."""
    want = golden("rng.npz")["long_normals"]
    assert (np.abs(want) > 3.6541528853610087).sum() >= 5


def test_uniform_matches_numpy(lib):
    for seed in (0, 9):
        want = golden("rng.npz")[f"resample_u0_{seed}"]
        for k in range(0, 50, 7):
            out = np.empty(1)
            lib.er_host_uniforms(seed, 2, k, 0, 1, 0.0, 1.0 / 500,
                                 out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
            assert out[0] == want[k]
    # and against numpy directly on fresh streams
    g = np.random.Generator(np.random.Philox(key=123, counter=[0, 4, 5, 6]))
    want = g.uniform(-2.0, 3.0, size=50)
    out = np.empty(50)
    lib.er_host_uniforms(123, 4, 5, 6, 50, -2.0, 5.0,
                         out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    assert np.array_equal(out, want)


def _host_has_fma():
    try:
        flags = open("/proc/cpuinfo").read()
    except OSError:  # pragma: no cover
        return False
    return " fma " in flags and " avx2 " in flags


@pytest.mark.skipif(not _host_has_fma(), reason="glibc picks its FMA log1p only on FMA hosts")
def test_log1p_is_glibcs(lib):
    """er_log1p (the ziggurat tail's log1p, whose value is returned) equals
    the host's glibc log1p -- what numpy's npy_log1p calls -- bit for bit on
    the tail's arguments -u, u in [0, 1), and across the other branches."""
    import math

    lib.er_host_log1p.argtypes = [ctypes.POINTER(ctypes.c_double)] * 2 + [ctypes.c_int64]
    g = np.random.default_rng(5)
    u = (g.integers(0, 2**53, 400_000, dtype=np.int64) * 2.0**-53)
    x = np.concatenate([-u, g.uniform(-1, 4, 100_000), g.uniform(-1e-6, 1e-6, 20_000),
                        10.0 ** g.uniform(-30, 300, 20_000), -(2.0 ** -np.arange(1, 60)),
                        [0.0, -0.0, 1e-300, -1e-300, 5e-324, 1.0, 0.41421, -0.29289, 1e300]])
    y = np.empty_like(x)
    d = ctypes.POINTER(ctypes.c_double)
    lib.er_host_log1p(x.ctypes.data_as(d), y.ctypes.data_as(d), x.size)
    want = np.array([math.log1p(v) for v in x])
    bad = np.flatnonzero(y.view(np.uint64) != want.view(np.uint64))
    assert bad.size == 0, (x[bad[:5]], y[bad[:5]], want[bad[:5]])


@pytest.mark.parametrize("seed,n", [(0, 262144), (11, 8712), (7, 1_000_000)])
def test_phantom_stream_normals_bit_exact(lib, seed, n):
    """Philox(key=seed).standard_normal(n) -- the phantom speckle's stream
    (E/phantom.py:76-77), counter 0 = stream (seed, 0, 0, 0) -- incl. its
    ~0.03% tail draws."""
    want = np.random.Generator(np.random.Philox(key=seed)).standard_normal(n)
    got = normals(lib, seed, 0, 0, 0, n)
    bad = np.flatnonzero(got != want)
    assert bad.size == 0, (bad[:5], got[bad[:5]], want[bad[:5]])
    assert (np.abs(want) > 3.6541528853610087).sum() > 0
