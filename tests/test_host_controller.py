"""Host controller parity (CPU): this repo's libmodeswitch.so against golden
fixtures written by the reference's own proj/core library (oracle/ref_golden.cpp,
regenerated with `make -C oracle ref && oracle/_ref/ref_golden tests/golden`).

Bars: routing decisions (mode, reason), workload class and resolved family
BIT-EXACT on every fixture row; generated traces and canonical trace lines
BYTE-EXACT; strict-schema rejections and error codes as the reference's.
"""
import csv
import ctypes as C
import hashlib
import os

import pytest

from paper_2605_23057_b200 import controller as ctl

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
FIXTURES = ["balanced_55_seed7", "canonical_families", "config1_mixed", "deploy_mix_tagged",
            "deploy_mix_untagged", "boundary_fuzz"]


def _golden(name):
    with open(os.path.join(GOLDEN, name + ".ndjson")) as f:
        text = f.read()
    with open(os.path.join(GOLDEN, name + ".decisions.csv")) as f:
        rows = list(csv.DictReader(f))
    return text, rows


def test_balanced_trace_is_the_surveyed_golden():
    text, rows = _golden("balanced_55_seed7")
    assert hashlib.md5(text.encode()).hexdigest() == "09d8641c4ad33e72a774616032085558"
    assert len(rows) == 605


@pytest.mark.parametrize("name", FIXTURES)
def test_routing_matches_reference(name):
    text, rows = _golden(name)
    got = ctl.route_ndjson(text)
    assert len(got) == len(rows)
    for g, r in zip(got, rows):
        assert g["mode"] == r["mode"], (r["request_id"], g, r)
        assert g["reason"] == r["reason"], r["request_id"]
        assert g["class"] == r["class"], r["request_id"]
        assert g["family"] == r["family"], r["request_id"]


def test_rule_histogram_on_balanced_trace():
    text, _ = _golden("balanced_55_seed7")
    hist = {}
    for g in ctl.route_ndjson(text):
        hist[g["mode"]] = hist.get(g["mode"], 0) + 1
    assert hist == {"gptq4": 220, "gptq_prefix_caching": 55, "int8": 191, "speculative_decoding": 139}


def test_generate_trace_byte_exact():
    text, _ = _golden("balanced_55_seed7")
    assert ctl.generate_trace({f: 55 for f in range(11)}, jitter=0.10, seed=7) == text
    text, _ = _golden("config1_mixed")
    assert ctl.generate_trace({f: 5 for f in range(11)}, jitter=0.10, seed=7,
                              batched_fraction=0.2, batch_pressure=4) == text
    text, _ = _golden("canonical_families")
    assert ctl.generate_trace({f: 2 for f in range(11)}, jitter=0.0, seed=0,
                              batched_fraction=0.5, batch_pressure=4) == text


@pytest.mark.parametrize("name", FIXTURES)
def test_trace_lines_round_trip_byte_exact(name):
    text, _ = _golden(name)
    for line in text.splitlines():
        d = ctl.parse_trace_line(line)
        assert ctl.format_trace_line(d) == line


@pytest.mark.parametrize("line", [
    "not json", "[1,2]",
    '{"request_id":"a","prompt_tokens":1,"expected_output_tokens":1,"shared_prefix":false,'
    '"memory_pressure":false,"batch_pressure":1,"workload_tag":null,"extra":1}',
    '{"request_id":"a","prompt_tokens":1,"expected_output_tokens":1,"shared_prefix":false,'
    '"memory_pressure":false,"batch_pressure":1}',
    '{"request_id":"a","prompt_tokens":0,"expected_output_tokens":1,"shared_prefix":false,'
    '"memory_pressure":false,"batch_pressure":1,"workload_tag":null}',
    '{"request_id":"a","prompt_tokens":1.0,"expected_output_tokens":1,"shared_prefix":false,'
    '"memory_pressure":false,"batch_pressure":1,"workload_tag":null}',
    '{"request_id":"a","prompt_tokens":1,"expected_output_tokens":1,"shared_prefix":0,'
    '"memory_pressure":false,"batch_pressure":1,"workload_tag":null}',
    '{"request_id":"","prompt_tokens":1,"expected_output_tokens":1,"shared_prefix":false,'
    '"memory_pressure":false,"batch_pressure":1,"workload_tag":null}',
    '{"request_id":"a","prompt_tokens":1,"expected_output_tokens":1,"shared_prefix":false,'
    '"memory_pressure":false,"batch_pressure":1,"workload_tag":"NotAFamily"}',
])
def test_malformed_lines_are_data_errors(line):
    with pytest.raises(ctl.MswError) as e:
        ctl.parse_trace_line(line)
    assert e.value.code == 3


def test_config_errors():
    with pytest.raises(ctl.MswError) as e:
        ctl.generate_trace({0: 1}, jitter=0.5, seed=0)
    assert e.value.code == 2
    with pytest.raises(ctl.MswError) as e:
        ctl.route(dict(request_id="x", prompt_tokens=1, expected_output_tokens=1),
                  classifier=dict(long_prompt_threshold=0))
    assert e.value.code == 2


def test_untagged_probes_from_survey():
    # untagged probes and their rules.
    probes = [
        (dict(prompt_tokens=128, expected_output_tokens=32), "int8", "rule7_default"),
        (dict(prompt_tokens=128, expected_output_tokens=512), "speculative_decoding", "rule5_decode_heavy"),
        (dict(prompt_tokens=8192, expected_output_tokens=64, memory_pressure=True), "gptq4",
         "rule3_memory_pressure"),
        (dict(prompt_tokens=128, expected_output_tokens=128, batch_pressure=64),
         "int8_continuous_batching", "rule1_batched"),
        (dict(prompt_tokens=1024, expected_output_tokens=128, shared_prefix=True, batch_pressure=64),
         "int8_continuous_batching", "rule1_batched"),
    ]
    for fields, mode, reason in probes:
        d = ctl.route(dict(request_id="p", **fields))
        assert (d["mode"], d["reason"]) == (mode, reason)


def test_route_cost_is_measured():
    text, _ = _golden("balanced_55_seed7")
    stamp, wall = ctl.route_cost(text, passes=5)
    assert 0 < stamp < 0.1 and 0 < wall < 0.1
