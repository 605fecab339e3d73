"""The oracle-side phantom generator (oracle/phantom.py) that builds the CPU
reference arm's inputs without the product package: pinned to the bytes the
REAL reference generator produced (tests/golden/phantom.npz from
echoreg.phantom, and the SHA-256 digests of the BASELINE C2 / C3 echo pairs in
tests/golden/full_c2.npz / full_c3.npz, tests/golden/make_golden_full.py)."""

import math
import os
import subprocess
import sys

import numpy as np
import pytest

from .conftest import GOLDEN, ROOT


def test_phantom_matches_reference_golden():
    from oracle import phantom as op

    g = np.load(os.path.join(GOLDEN, "phantom.npz"))
    fr, ms = op.make_phantom((20, 18, 22), (1.1, 0.9, 1.3), (8.0, 7.0, 9.0), (5.0, 4.0, 6.0),
                             0.3, 0.25, 3, 11)
    truth = (math.radians(6), math.radians(-3), math.radians(2), 1.5, -2.0, 0.5)
    src, smk = op.make_pair(fr, ms, (1.1, 0.9, 1.3), truth, overlap_crop=0.2)
    assert np.array_equal(np.stack(fr), g["frames"])
    assert np.array_equal(np.stack(ms).astype(np.uint8), g["masks"])
    assert np.array_equal(np.stack(src), g["src_frames"])
    assert np.array_equal(np.stack(smk).astype(np.uint8), g["src_masks"])


def test_c2_echo_pair_is_the_reference_pair():
    from oracle import phantom as op

    g = np.load(os.path.join(GOLDEN, "full_c2.npz"))
    tq, sq, _, _ = op.echo_case(frames=1)
    assert tq[0].shape == (176, 176, 208)
    assert op.digest(tq) == str(g["c2_target_sha256"])
    assert op.digest(sq) == str(g["c2_source_sha256"])


def test_c3_echo_cycle_is_the_reference_cycle():
    path = os.path.join(GOLDEN, "full_c3.npz")
    if not os.path.exists(path):
        pytest.skip("full_c3.npz not generated")
    from oracle import phantom as op

    g = np.load(path)
    tq, sq, tm, sm = op.echo_case(frames=30)
    assert op.digest(tq) == str(g["c3_target_sha256"])
    assert op.digest(sq) == str(g["c3_source_sha256"])
    assert op.digest(tm) == str(g["c3_target_masks_sha256"])
    assert op.digest(sm) == str(g["c3_source_masks_sha256"])


def test_reference_arm_inputs_never_import_the_product():
    """bench.py --impl reference builds its workload from oracle/ only."""
    code = ("import sys, bench; bench.reference_inputs(8); "
            "bad = [m for m in sys.modules if m.startswith('paper_2504_19930_b200')]; "
            "assert not bad, bad; print('clean')")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "clean" in r.stdout


def test_both_bench_arms_quote_the_same_config():
    """bench.py's two arms build `config` from one function on the same
    workload numbers (the driver compares them)."""
    import bench

    a = bench.workload_config(2000, 176 * 176 * 208, (176, 176, 208))
    b = bench.workload_config(2000, 6443008, [176, 176, 208])
    assert a == b and a["workload"] == bench.WORKLOAD and a["particles"] == 2000
