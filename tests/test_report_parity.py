"""Report / summary parity with files the REAL reference wrote
(tests/golden/make_golden.py report_cases, exhaustive_sequence_cases;
make_golden_full.py c3): the RegistrationReport JSON (pipeline.py:32-76),
the five-number percentile summary and its CSV (pipeline.py:273-308)."""

import json
import os

import pytest

from .conftest import GOLDEN


@pytest.fixture(scope="module")
def cases():
    with open(os.path.join(GOLDEN, "report_cases.json")) as fh:
        return json.load(fh)


def test_report_json_round_trips_byte_identically(cases, tmp_path):
    from paper_2504_19930_b200 import RegistrationReport

    for d, saved in zip(cases["reports"], cases["saved"]):
        rep = RegistrationReport.from_dict(d)
        p = tmp_path / f"{rep.case_id}.json"
        rep.save(str(p))
        assert p.read_text() == saved
        assert RegistrationReport.load(str(p)).to_dict() == d


def test_percentile_summary_and_csv_match_reference(cases, tmp_path):
    from paper_2504_19930_b200 import RegistrationReport, percentile_summary
    from paper_2504_19930_b200.pipeline import write_summary_csv

    reps = [RegistrationReport.from_dict(d) for d in cases["reports"]]
    rows = percentile_summary(reps)
    assert rows == cases["summary"]
    p = tmp_path / "summary.csv"
    write_summary_csv(rows, str(p))
    with open(os.path.join(GOLDEN, "report_summary.csv"), newline="") as fh:
        want = fh.read()
    with open(p, newline="") as fh:
        assert fh.read() == want


def test_aggregates_match_reference(cases):
    from paper_2504_19930_b200.pipeline import _aggregates

    for d in cases["reports"]:
        assert _aggregates(d["ncc_before"], d["ncc_after"], d["dsc_before"],
                           d["dsc_after"]) == d["aggregates"]


def test_reference_c3_report_loads_with_the_same_schema():
    """The reference's own 30-frame C3 report (make_golden_full.py) loads into
    our RegistrationReport and re-saves to the same JSON document."""
    from paper_2504_19930_b200 import RegistrationReport

    path = os.path.join(GOLDEN, "full_c3_report.json")
    rep = RegistrationReport.load(path)
    with open(path) as fh:
        want = json.load(fh)
    assert rep.to_dict() == want
    assert rep.schema == 1 and rep.method == "smc" and rep.mode == "mask"
    assert len(rep.ncc_before) == 30 and len(rep.trace["ess"]) == 50
