"""Pin the CPU oracle against golden vectors from the real reference.

The C oracle must be BIT-EXACT with the reference numba kernels (same fp64
operation order, no FMA) and its in-bounds counts must equal the reference
numpy backend's mask counts.  The numpy SMC restatement must reproduce the
reference's recorded registration runs.
"""

import math

import numpy as np
import pytest

from oracle import kernels as ok
from oracle import smc as osmc

from .conftest import golden, golden_kernel_cases


@pytest.fixture(scope="module", autouse=True)
def _build():
    ok.build()


CASES = golden_kernel_cases()


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_measure_bit_exact(name):
    c = CASES[name]
    for overlap, key in ((False, "full"), (True, "overlap")):
        z, d, n = ok.ncc_measure_batch(c["tgt"], c["src"], c["a"], c["b"], overlap,
                                       workers=3, return_counts=True)
        assert np.array_equal(z, c[f"ncc_{key}"]), (name, key)
        assert np.array_equal(d, c[f"degen_{key}"]), (name, key)
        assert np.array_equal(n, c["n_in"]), name


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_resample_bit_exact(name):
    c = CASES[name]
    for p in range(c["resampled"].shape[0]):
        out = ok.resample_trilinear(c["src"], c["a"][p], c["b"][p], c["tgt"].shape)
        assert np.array_equal(out, c["resampled"][p]), (name, p)


def test_oracle_thread_count_invariance():
    c = CASES["wide"]
    base = ok.ncc_measure_batch(c["tgt"], c["src"], c["a"], c["b"], False, workers=1)[0]
    for w in (2, 5, 8):
        got = ok.ncc_measure_batch(c["tgt"], c["src"], c["a"], c["b"], False, workers=w)[0]
        assert np.array_equal(got, base)


def test_k_interval_edge_cases():
    # slope 0 inside / outside (kernels_numba.py:95-98)
    assert ok.k_interval(3.0, 0.0, 5.0, 0, 10) == (0, 10)
    assert ok.k_interval(-0.5, 0.0, 5.0, 0, 10) == (0, 0)
    # positive slope crossing both walls: 0 <= 1 + 0.5k <= 4  -> k in [0, 6]
    assert ok.k_interval(1.0, 0.5, 4.0, 0, 10) == (0, 7)
    # negative slope: 0 <= 4 - k <= 4 -> k in [0, 4]
    assert ok.k_interval(4.0, -1.0, 4.0, 0, 10) == (0, 5)
    # entirely beyond
    assert ok.k_interval(-100.0, 1e-3, 4.0, 0, 10) == (0, 0)


def test_oracle_trilinear_fixture():
    # reference tests/test_geometry.py:156-165: 8-term blend of 0..7 corners
    src = np.arange(8, dtype=np.float64).reshape(2, 2, 2)
    val = ok.lib().or_sample_one(src.ctypes.data_as(ok._d), 0.25, 0.5, 0.75, 2, 2, 2)
    w = 0.0
    for i in (0, 1):
        for j in (0, 1):
            for k in (0, 1):
                w += ((0.25 if i else 0.75) * (0.5 if j else 0.5)
                      * (0.75 if k else 0.25)) * src[i, j, k]
    assert val == pytest.approx(w, abs=1e-15)


def test_geometry_restatement_matches_reference():
    g = golden("geometry.npz")
    for i in range(g["params"].shape[0]):
        m = osmc.to_matrix(g["params"][i], g["centers"][i])
        np.testing.assert_allclose(m, g["mats"][i], rtol=0, atol=1e-12)
        a, b = osmc.index_affine(g["mats"][i], g["src_spacing"], g["src_origin"],
                                 g["tgt_spacing"], g["tgt_origin"])
        assert np.array_equal(a, g["a"][i])
        np.testing.assert_allclose(b, g["b"][i], rtol=1e-15, atol=1e-13)


def test_rng_restatement_matches_reference():
    g = golden("rng.npz")
    for seed, n in ((0, 500), (99, 7), (3, 2000)):
        st = osmc.init_states(osmc.Cfg(n_particles=n, seed=seed))
        assert np.array_equal(st, g[f"init_{seed}_{n}"])
    cfg = osmc.Cfg(n_particles=300, seed=4, sigma0_r=3.0, sigma0_t=4.0)
    assert np.array_equal(osmc.predict(g["predict_in"], 6, cfg), g["predict_out"])


def _c1_inputs():
    g = golden("smc.npz")
    dims = tuple(int(d) for d in g["c1_dims"])
    n = int(np.prod(dims))
    t = np.unpackbits(g["c1_target_bits"])[:n].reshape(dims).astype(np.float64)
    s = np.unpackbits(g["c1_source_bits"])[:n].reshape(dims).astype(np.float64)
    return g, t, s, dims


def test_oracle_c1_lockstep_iteration0():
    g, t, s, dims = _c1_inputs()
    z, d = ok.ncc_measure_batch(t, s, g["c1_a_it0"], g["c1_b_it0"], False)
    assert np.array_equal(z, g["c1_z"][0])
    assert np.array_equal(d, g["c1_degen"][0])


@pytest.mark.parametrize("prefix,mode,n,iters,seed,region", [
    ("c1o_", "mask", 200, 6, 3, "overlap"),
])
def test_oracle_smc_free_run_matches_reference(prefix, mode, n, iters, seed, region):
    g, t, s, dims = _c1_inputs()
    geom = (dims, (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    cfg = osmc.Cfg(mode=mode, n_particles=n, n_iterations=iters, seed=seed,
                   ncc_region=region)
    est, tr = osmc.register(t, s, geom, geom, cfg)
    np.testing.assert_allclose(est, g[f"{prefix}estimate"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(np.stack(tr.z), g[f"{prefix}z"], rtol=0, atol=1e-13)
    assert tr.resampled == list(g[f"{prefix}resampled"])


@pytest.mark.slow
def test_oracle_c1_full_run_matches_reference():
    g, t, s, dims = _c1_inputs()
    geom = (dims, (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    cfg = osmc.Cfg(mode="mask", n_particles=500, n_iterations=20, seed=0)
    est, tr = osmc.register(t, s, geom, geom, cfg)
    np.testing.assert_allclose(est, g["c1_estimate"], rtol=0, atol=1e-12)
    assert tr.resampled == list(g["c1_resampled"])
    assert math.isclose(tr.ess[-1], float(g["c1_ess"][-1]), rel_tol=1e-12)
