"""INTEGRATION.md's C-ABI walkthrough is executable documentation: extract
the Python block of section 3, run it as written on real inputs, and check
its likelihoods against the oracle."""

import os
import re

import numpy as np
import pytest

from oracle import kernels as ok

from .conftest import ROOT

pytestmark = pytest.mark.gpu


def _snippet():
    text = open(os.path.join(ROOT, "INTEGRATION.md"), encoding="utf-8").read()
    section = text[text.index("## 3. C ABI"):]
    return re.search(r"```python\n(.*?)```", section, re.S).group(1)


def test_c_abi_walkthrough_runs_as_documented():
    from paper_2504_19930_b200 import _lib

    g = np.random.default_rng(8)
    target_u8 = g.integers(0, 256, (20, 18, 22)).astype(np.uint8)
    source_u8 = np.roll(target_u8, 1, axis=2)
    mean_t, std_t = float(target_u8.mean()), float(target_u8.std())
    mean_s, std_s = float(source_u8.mean()), float(source_u8.std())
    a_batch = np.eye(3)[None] + g.uniform(-0.04, 0.04, (16, 3, 3))
    b_batch = g.uniform(-1.5, 1.5, (16, 3))
    ns = {"target_u8": target_u8, "source_u8": source_u8, "mean_t": mean_t, "std_t": std_t,
          "mean_s": mean_s, "std_s": std_s, "a_batch": a_batch, "b_batch": b_batch}
    code = _snippet().replace('ctypes.CDLL("paper_2504_19930_b200/_lib/libechoreg_sm100.so")',
                              f"ctypes.CDLL({_lib.LIB_PATH!r})")
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    assert ns["rc"] == 0
    z = ns["ncc"].cpu().numpy()
    zt = (target_u8 - mean_t) / std_t
    zs = (source_u8 - mean_s) / std_s
    want, _ = ok.ncc_measure_batch(zt, zs, a_batch, b_batch, False)
    assert np.allclose(z, want, rtol=1e-4, atol=1e-12)
    assert np.array_equal(ns["n_in"].cpu().numpy(),
                          ok.ncc_measure_batch(zt, zs, a_batch, b_batch, False,
                                               return_counts=True)[2])
