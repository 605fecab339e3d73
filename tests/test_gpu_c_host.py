"""The C ABI used from a plain C program (examples/measure_demo.c): compiled
with gcc against include/ and the in-tree library, run, and its likelihoods
checked -- identity scores 1, a one-voxel shift less, and a transform that
leaves the source entirely scores 0 with zero in-bounds voxels."""

import os
import re
import subprocess

import pytest

from .conftest import ROOT

pytestmark = pytest.mark.gpu


def test_c_program_calls_the_hot_path(tmp_path):
    exe = str(tmp_path / "measure_demo")
    lib = os.path.join(ROOT, "paper_2504_19930_b200", "_lib")
    subprocess.run(["gcc", "-O2", os.path.join(ROOT, "examples", "measure_demo.c"),
                    "-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include",
                    "-L" + lib, "-lechoreg_sm100", "-L/usr/local/cuda/lib64", "-lcudart",
                    "-lm", "-Wl,-rpath," + lib, "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120, check=True).stdout
    z = [float(m) for m in re.findall(r"ncc ([0-9.]+)", out)]
    n = [int(m) for m in re.findall(r"in-bounds (\d+)", out)]
    assert abs(z[0] - 1.0) < 1e-6 and n[0] == 24 * 20 * 28
    assert 0.0 < z[1] < z[0] and n[1] == 24 * 20 * 27
    assert z[2] == 0.0 and n[2] == 0 and "degenerate 1" in out.splitlines()[2]
