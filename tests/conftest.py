"""Shared test setup.

Markers: ``gpu`` tests need a B200 (run on the GPU box with ``-m gpu``);
everything else runs on the CPU build box.  CPU tests exercise the oracle
against the reference's golden vectors, the host logic, and that the C-ABI
library loads and exports every declared symbol.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    # a fresh checkout: build the sm_100a library (nvcc cross-compiles without
    # a GPU) and the CPU oracle before any test loads them
    from paper_2504_19930_b200 import _build

    if not os.path.exists(_build.LIB):
        _build.build()
    from oracle import kernels as oracle_kernels

    oracle_kernels.build()


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def golden_kernel_cases():
    g = golden("kernels.npz")
    names = [str(n) for n in g["case_names"]]
    out = {}
    for n in names:
        prefix = f"{n}__"
        out[n] = {k[len(prefix):]: g[k] for k in g.files if k.startswith(prefix)}
    return out


@pytest.fixture()
def rng():
    return np.random.default_rng(12345)


def have_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(autouse=True)
def _no_bounds_faults(request):
    """Under tools/bounds_check.sh (a -DER_BOUNDS_CHECK=1 build), fail the GPU
    test during which any kernel saw an out-of-range gather index."""
    yield
    if os.environ.get("ER_ASSERT_NO_BOUNDS_FAULTS") and request.node.get_closest_marker("gpu"):
        from paper_2504_19930_b200 import _lib

        faults = _lib.bounds_faults()
        assert faults is not None, "ER_ASSERT_NO_BOUNDS_FAULTS set on a build without checks"
        assert faults == 0, f"{faults} out-of-range gather indices"
