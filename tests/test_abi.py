"""CPU checks of the drop-in boundary: the sm_100a library loads (no CUDA
call is made) and exports exactly what include/echoreg_b200.h declares;
the Python binding declares a signature for each of them."""

import ctypes
import os
import re

import pytest

from paper_2504_19930_b200 import _lib

from .conftest import ROOT

HEADER = os.path.join(ROOT, "include", "echoreg_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(er_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    names = declared_functions()
    assert "er_measure_ncc" in names
    assert len(names) >= 15


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_header():
    assert sorted(_lib.SIGNATURES) == declared_functions()


def test_struct_layouts_match_header():
    # er_volume: ptr, 4 x int32, 2 x double, 3 x ptr -> 64 bytes on LP64
    assert ctypes.sizeof(_lib.ErVolume) == 64
    # er_smc_ctl: 7 doubles + 2 int32
    assert ctypes.sizeof(_lib.ErSmcCtl) == 64


def test_abi_version_and_error_text_without_gpu():
    lib = _lib.load()
    assert lib.er_abi_version() == 2
    assert isinstance(lib.er_last_error(), bytes)


def test_bounds_checks_compiled_out_of_the_normal_build():
    if "ER_BOUNDS_CHECK" in os.environ.get("ER_NVCC_EXTRA", ""):
        pytest.skip("debug build")
    assert _lib.bounds_faults() is None
    assert b"ER_BOUNDS_CHECK" in _lib.load().er_last_error()


def test_sass_is_sm100a():
    """The library carries sm_100a SASS (cuobjdump), not PTX-only or another arch."""
    import shutil
    import subprocess

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np

    from paper_2504_19930_b200 import Executor, InternalError, Volume3

    v = Volume3(np.zeros((4, 4, 4)))
    with pytest.raises(InternalError):
        Executor().measure_ncc(v, v, np.eye(4))


def test_docs_state_the_entry_point_count():
    """DESIGN.md and INTEGRATION.md quote the number of C-ABI entry points."""
    n = len(declared_functions())
    design = open(os.path.join(ROOT, "DESIGN.md"), encoding="utf-8").read()
    integ = open(os.path.join(ROOT, "INTEGRATION.md"), encoding="utf-8").read()
    assert re.search(r"(\d+) `extern \"C\"` entry points", design).group(1) == str(n)
    assert re.search(r"all (\d+) entry", integ).group(1) == str(n)
