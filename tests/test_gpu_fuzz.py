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


def test_refinement_pass_remeasures_ill_conditioned_particles():
    """A nearly constant 8-bit source (one 2x2x2 block one byte brighter):
    the sampled variance is tiny next to the stored magnitudes (bytes ~77),
    so fp32 samples cannot resolve sss -- the finalize must list these
    particles, re-measure them in fp64 (er_measure_ncc refinement) and then
    meet the plain f32 bar against the oracle, flags included."""
    import numpy as np

    from oracle import kernels as ok
    from paper_2504_19930_b200 import RigidParams, Volume3, normalize_zscore, ops, to_matrix
    from paper_2504_19930_b200.device import device_volume, require_cuda, torch
    from paper_2504_19930_b200.geometry import index_affine_batch

    rng = np.random.default_rng(5)
    dims = (20, 18, 22)
    t = normalize_zscore(Volume3.from_u8(rng.integers(0, 256, dims).astype(np.uint8)))
    raw = np.full(dims, 77, dtype=np.uint8)
    raw[9:11, 8:10, 10:12] = 78
    s = normalize_zscore(Volume3.from_u8(raw))
    mats = np.stack([to_matrix(RigidParams(*rng.uniform(-0.1, 0.1, 3), *rng.uniform(-2, 2, 3)),
                               t.physical_center()) for _ in range(24)])
    a, b = index_affine_batch(mats, s.spacing, s.origin, t.spacing, t.origin)
    dev = require_cuda()
    tdv, sdv = device_volume(t, dev), device_volume(s, dev)
    A = torch().as_tensor(a.reshape(-1, 9), device=dev)
    B = torch().as_tensor(b.reshape(-1, 3), device=dev)
    for overlap in (False, True):
        z, d, _ = ops.measure(tdv, sdv, A, B, overlap, "f32")
        refined = ops.refined_count(tdv, 24)
        zo, do = ok.ncc_measure_batch(t.data, s.data, a, b, overlap)
        z, d = z.cpu().numpy(), d.cpu().numpy().astype(bool)
        assert refined > 0, overlap
        assert np.array_equal(d, do), overlap
        assert np.all(np.abs(z - zo) <= 1e-4 * np.abs(zo) + 1e-12), overlap
