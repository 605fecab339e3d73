"""Host-side logic that needs no GPU: report schema and percentile rules
(reference pipeline.py:29-308, tests/test_pipeline.py:164-213), SmcConfig /
GridSpec validation (smc.py:64-89, exhaustive.py:37-45), the exact 8-bit
codec of volume.py, and the reference's geometry conventions."""

import math

import numpy as np
import pytest

from paper_2504_19930_b200 import (BadConfig, EmptyInput, GridSpec, RegistrationReport,
                                   RigidParams, SmcConfig, Volume3, compose, inverse,
                                   percentile_summary, to_matrix)
from paper_2504_19930_b200.volume import LazyVolume3, RawU8Codec, binarize

from .conftest import golden


def _report(case_id, before, after):
    return RegistrationReport(
        mode="mask", method="smc", config={}, estimate_deg_mm={}, best_estimate_deg_mm=None,
        ncc_before=[0.1], ncc_after=[0.2], dsc_before=before, dsc_after=after,
        aggregates={}, trace=None, wall_time_s=0.0, case_id=case_id)


def test_percentile_singleton_and_interpolation():
    rows = percentile_summary([_report("a", [0.5], [0.7])])
    assert [r["stat"] for r in rows] == ["min", "q1", "q2", "q3", "max"]
    assert all(r["case_id"] == "a" for r in rows)
    assert rows[2]["dsc_diff"] == pytest.approx(0.2)
    reps = [_report(str(i), [0.0], [d]) for i, d in enumerate([0.1, 0.2, 0.3, 0.4, 0.5])]
    rows = percentile_summary(reps)
    assert rows[1]["dsc_diff"] == pytest.approx(0.2)
    assert rows[2]["case_id"] == "2"


def test_percentile_empty_raises():
    with pytest.raises(EmptyInput):
        percentile_summary([_report("x", [None], [None])])


def test_report_roundtrip(tmp_path):
    r = _report("case7", [0.4, None], [0.9, None])
    p = tmp_path / "r.json"
    r.save(str(p))
    back = RegistrationReport.load(str(p))
    assert back.to_dict() == r.to_dict()
    assert back.dsc_difference() == pytest.approx(0.5)


def test_config_validation_mirrors_reference():
    with pytest.raises(BadConfig):
        SmcConfig(n_particles=0).validate()
    with pytest.raises(BadConfig):
        SmcConfig(ess_fraction=0.0).validate()
    with pytest.raises(BadConfig):
        SmcConfig(mode="hybrid").validate()
    with pytest.raises(BadConfig):
        GridSpec(half_counts=(1, 1, 1)).validate()
    assert GridSpec().n_nodes == 9 ** 6
    g = GridSpec(half_counts=(1, 0, 2, 0, 1, 1), step_t=1.5, step_r=2.0)
    from paper_2504_19930_b200.exhaustive import _node_states

    states = _node_states(g)
    for i in (0, 7, 44, g.n_nodes - 1):
        assert np.array_equal(g.node_state(i), states[i])


def test_geometry_against_reference_goldens():
    gd = golden("geometry.npz")
    for i in range(0, gd["params"].shape[0], 17):
        m = to_matrix(RigidParams.from_array(gd["params"][i]), gd["centers"][i])
        np.testing.assert_allclose(m, gd["mats"][i], rtol=0, atol=1e-12)
        np.testing.assert_allclose(compose(m, inverse(m)), np.eye(4), atol=1e-12)


def test_u8_codec_volume_semantics():
    rng = np.random.default_rng(4)
    raw = rng.integers(0, 256, (5, 6, 7)).astype(np.uint8)
    v = Volume3.from_u8(raw, (1.0, 2.0, 0.5), (1.0, 0.0, -1.0))
    assert isinstance(v, LazyVolume3)
    assert v.dims == (5, 6, 7)
    assert v.physical_center() == (3.0, 5.0, 0.5)
    assert "_data" not in v.__dict__           # nothing materialised yet
    assert np.array_equal(v.data, raw.astype(np.float64))
    b = binarize(v, 127.5)
    assert np.array_equal(b.codec.raw, (raw > 127.5).astype(np.uint8))
    c = RawU8Codec(raw, 12.5, 3.0)
    np.testing.assert_array_equal(c.decode(), (raw.astype(np.float64) - 12.5) / 3.0)


def test_rigid_params_rejects_nonfinite():
    with pytest.raises(ValueError):
        RigidParams(rx=math.nan)


def test_backend_env_from_a_reference_setup_is_served_by_sm100(monkeypatch, caplog):
    """$ECHOREG_BACKEND=numba/numpy (the reference's CPU backends) must not break
    a default Executor(): logged and served by sm100.  An explicit backend=
    argument naming them is still a configuration error."""
    import logging

    from paper_2504_19930_b200 import BadConfig
    from paper_2504_19930_b200 import backend as bk

    for name in ("numba", "numpy", "NUMBA"):
        monkeypatch.setenv("ECHOREG_BACKEND", name)
        with caplog.at_level(logging.WARNING, logger="echoreg_b200"):
            assert bk.get_backend() is bk.kernels_sm100
        assert "sm100" in caplog.text
        with pytest.raises(BadConfig):
            bk.get_backend(name.lower())
    monkeypatch.setenv("ECHOREG_BACKEND", "cuda-something")
    with pytest.raises(BadConfig):
        bk.get_backend()


def test_seed_beyond_64_bits_is_rejected():
    from paper_2504_19930_b200 import BadConfig, SmcConfig

    SmcConfig(seed=2 ** 64 - 1).validate()
    with pytest.raises(BadConfig):
        SmcConfig(seed=2 ** 64).validate()
