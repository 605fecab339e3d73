"""A short run of the randomised differential test (tools/fuzz_measure.py):
random dims, spacings, origins, storage types, transforms and region modes
against the C oracle, every precision; counts bit-exact."""

import os
import sys

import pytest

from .conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [1, 2])
def test_random_cases_match_the_oracle(seed):
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import fuzz_measure

    res = fuzz_measure.run(n_cases=40, seed=seed)
    assert not res["failures"], res["failures"][:5]


def test_random_warp_cases_match_the_oracle():
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import fuzz_measure

    res = fuzz_measure.run_warp(n_cases=40, seed=3)
    assert not res["failures"], res["failures"][:5]
