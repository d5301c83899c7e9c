"""Energy per token: the host library's power-trace reader
and energy_from_power_trace against the reference's own implementation
(sim.cpp:10-78), pinned by tests/golden/power_*.csv written by the reference's
write_power_trace and power_golden.csv (its J/token, %.17g, or the DataError it
raised) from oracle/ref_golden. Bit-exact."""
import csv
import os

import pytest

from paper_2605_23057_b200._capi import MswError
from paper_2605_23057_b200.energy import energy_from_trace

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rows():
    with open(os.path.join(GOLD, "power_golden.csv")) as f:
        return list(csv.DictReader(f))


@pytest.mark.parametrize("row", _rows(), ids=lambda r: r["name"])
def test_energy_matches_reference(row):
    path = os.path.join(GOLD, row["name"] + ".csv")
    tokens = int(row["tokens"])
    if row["joules_per_token"] == "DataError":
        with pytest.raises(MswError) as e:
            energy_from_trace(path, tokens)
        assert e.value.code == 3
    else:
        assert energy_from_trace(path, tokens) == float(row["joules_per_token"])


def test_energy_errors_match_reference_contract(tmp_path):
    bad_header = tmp_path / "h.csv"
    bad_header.write_text("t,p\n0,1\n1,2\n")
    one = tmp_path / "one.csv"
    one.write_text("timestamp_ms,power_w\n0,100\n")
    ok = tmp_path / "ok.csv"
    ok.write_text("timestamp_ms,power_w\n0,100\n1000,300\n")
    for p, tok in ((bad_header, 1), (one, 1), (ok, 0)):
        with pytest.raises(MswError) as e:
            energy_from_trace(str(p), tok)
        assert e.value.code == 3
    assert energy_from_trace(str(ok), 2) == 100.0  # 0.5 * (100 + 300) * 1 s / 2 tokens
