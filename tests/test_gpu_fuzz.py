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


def test_ill_conditioned_particles_meet_the_plain_f32_bar():
    """Two cases the round-1 100k-case run found outside the f32 bar (seed 37):
    particles with z ~ 1 on nearly constant overlaps, condition numbers 1.7e4
    and 1e6.  The finalize now lists such particles and re-measures them in
    fp64 (er_measure_ncc refinement), so they meet the plain 1e-4 bar with
    bit-exact degenerate flags -- no conditioning allowance for f32."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import fuzz_measure

    res = fuzz_measure.run(n_cases=2693, seed=37, only={801, 2692}, strict=("f32",))
    assert not res["failures"], res["failures"]
    assert res["within_conditioning_only"]["f32"]["particles"] == 0
