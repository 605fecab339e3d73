"""normalize_zscore on 8-bit data and exhaustive_sequence, pinned to the REAL
reference's outputs (tests/golden/make_golden.py zscore_cases,
exhaustive_sequence_cases)."""

import json
import os

import numpy as np
import pytest

from .conftest import GOLDEN

pytestmark = pytest.mark.gpu


def test_zscore_of_bytes_matches_reference():
    """volume.py:119-130 on 8-bit volumes.  Our statistics come from an exact
    on-device histogram: the mean (an exact integer sum / n) is bit-identical
    to numpy's; the population std is accumulated per level instead of in
    numpy's pairwise voxel order, so it may differ in the last bits -- held to
    4 ulp here -- and the normalised values to 8 ulp of their magnitude."""
    from paper_2504_19930_b200 import Volume3, normalize_zscore

    g = np.load(os.path.join(GOLDEN, "zscore.npz"))
    keys = sorted({k.split("__")[0] for k in g.files})
    worst_std_ulp = 0.0
    for key in keys:
        raw = g[f"{key}__raw"]
        z = normalize_zscore(Volume3.from_u8(raw))
        mean, std = float(g[f"{key}__mean"]), float(g[f"{key}__std"])
        assert z.codec.mean == mean, key
        ulp = abs(z.codec.std - std) / np.spacing(std)
        worst_std_ulp = max(worst_std_ulp, ulp)
        assert ulp <= 4, (key, ulp)
        if f"{key}__z" in g.files:
            want = g[f"{key}__z"]
            tol = 8 * np.spacing(np.maximum(np.abs(want), 1.0))
            assert np.all(np.abs(z.data - want) <= tol), key


@pytest.mark.parametrize("mode", ["image", "mask"])
def test_exhaustive_sequence_matches_reference(mode):
    """pipeline.py:219-266: same winning grid node, same per-frame scores."""
    from paper_2504_19930_b200 import GridSpec, Sequence4, Volume3
    from paper_2504_19930_b200.pipeline import exhaustive_sequence

    g = np.load(os.path.join(GOLDEN, "exhaustive_sequence.npz"))
    with open(os.path.join(GOLDEN, "exhaustive_sequence.json")) as fh:
        ref = json.load(fh)
    sp = tuple(g["spacing"])
    tgt = Sequence4([Volume3(f, sp) for f in g["target"]])
    src = Sequence4([Volume3(f, sp) for f in g["source"]])
    tm = [Volume3.from_u8(m, sp) for m in g["target_masks"]]
    sm = [Volume3.from_u8(m, sp) for m in g["source_masks"]]
    gr = ref["grid"]
    grid = GridSpec(half_counts=tuple(gr["half_counts"]), step_t=gr["step_t"],
                    step_r=gr["step_r"])
    rep = exhaustive_sequence(tgt, src, tm, sm, grid, mode=mode, case_id=f"ex_{mode}")
    want = ref["reports"][mode]
    got = rep.to_dict()
    got.pop("wall_time_s")
    assert got.keys() == want.keys()
    assert got["estimate_deg_mm"] == pytest.approx(want["estimate_deg_mm"], abs=1e-12)
    assert got["config"]["half_counts"] == want["config"]["half_counts"]
    assert got["config"]["best_ncc"] == pytest.approx(want["config"]["best_ncc"], rel=1e-4)
    for key in ("ncc_before", "ncc_after"):
        assert np.allclose(got[key], want[key], rtol=1e-9, atol=0), key
    for key in ("dsc_before", "dsc_after"):
        assert np.allclose(got[key], want[key], rtol=0, atol=1e-12), key
    assert got["trace"] is None and got["method"] == "exhaustive" and got["mode"] == mode
