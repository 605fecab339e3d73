"""bench.py's one-line JSON contract (the driver parses it every round), run
small on the GPU: required keys and types, the roofline / cpu_baseline /
e2e / clocks objects, and the reference arm's line."""

import json
import os
import subprocess
import sys

import pytest

from .conftest import ROOT

pytestmark = pytest.mark.gpu


def _run(*args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_bench_line_contract():
    d = _run("--steps", "3", "--warmup", "3", "--particles", "128", "--e2e-steps", "1",
             "--e2e-iters", "3", "--cpu-seconds", "1")
    for key, typ in (("metric", str), ("value", float), ("unit", str), ("n_gpus", int),
                     ("steps", int), ("warmup", int), ("ms_per_step", float),
                     ("higher_is_better", bool), ("scaling", str), ("dtype", str),
                     ("data", str), ("config", dict), ("gpu_launches", int)):
        assert isinstance(d[key], typ), key
    assert d["metric"] == "particle-voxel evals/sec" and d["unit"] == "evals/s"
    assert d["steps"] == 3 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert "workload" in d["config"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert 0 < r["frac"] < 1.5 and r["l2"]["frac"] > 0
    c = d["cpu_baseline"]
    assert c["kind"] == "port" and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["plugin_seam"]["value"] > 0 and e["plugin_seam"]["cold"]["value"] > 0
    k = d["clocks"]
    assert k["sm_mhz"] > 0 and isinstance(k["reasons"], list)
    assert d["gpu_launches"] >= 4 * 3  # predict+affine, measure x2, update per step


def test_reference_arm_line_contract():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "3", "--particles", "8",
             timeout=900)
    assert d["impl"] == "reference"
    assert d["metric"] == "particle-voxel evals/sec" and d["value"] > 0
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
