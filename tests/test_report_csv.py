"""Decisions CSV in the reference's report format: rows
written by the host library are read back by the REFERENCE's own
read_decisions_csv (oracle/_ref/ref_golden --check-decisions) and carry the same
mode / reason per request as the reference's routing goldens."""
import csv
import os
import subprocess

import pytest

from paper_2605_23057_b200 import controller as ctl
from paper_2605_23057_b200._capi import ExecRow
from paper_2605_23057_b200.engine import write_decisions_csv

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref", "ref_golden")
GOLD = os.path.join(ROOT, "tests", "golden")


def _rows_from_routing(text):
    rows = []
    for r in ctl.route_ndjson(text):
        row = {f: 0 for f, _ in ExecRow._fields_}
        row["mode"], row["reason"], row["overhead_ms"] = r["mode_id"], ctl.REASONS.index(r["reason"]), 0.0123
        rows.append(row)
    return rows


def test_decisions_csv_format(tmp_path):
    text = open(os.path.join(GOLD, "balanced_55_seed7.ndjson")).read()
    path = str(tmp_path / "decisions.csv")
    write_decisions_csv(text, _rows_from_routing(text), path)
    with open(path) as f:
        rd = list(csv.reader(f))
    assert rd[0] == ["request_id", "mode", "reason", "overhead_ms"]
    gold = list(csv.reader(open(os.path.join(GOLD, "balanced_55_seed7.decisions.csv"))))[1:]
    assert [r[:3] for r in rd[1:]] == [g[:3] for g in gold]  # reference RulePolicy decisions
    assert all(r[3] == "0.0123" for r in rd[1:])  # %.17g


@pytest.mark.skipif(not os.path.exists(REF), reason="oracle/_ref not built (needs /root/reference)")
def test_reference_reader_accepts_decisions(tmp_path):
    text = open(os.path.join(GOLD, "balanced_55_seed7.ndjson")).read()
    path = str(tmp_path / "decisions.csv")
    write_decisions_csv(text, _rows_from_routing(text), path)
    out = subprocess.run([REF, "--check-decisions", path], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout
    gold = list(csv.reader(open(os.path.join(GOLD, "balanced_55_seed7.decisions.csv"))))[1:]
    assert out.stdout.splitlines() == [",".join(g[:3]) for g in gold]
