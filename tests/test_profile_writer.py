"""Measured-profile writer: a profile built from engine
measurements is accepted by the REFERENCE's own load_profile + validate
(oracle/_ref/ref_golden --check-profile, compiled from /root/reference), so
the reference's route_oracle / compare_policies can consume B200 numbers."""
import json
import os
import subprocess

import pytest

from paper_2605_23057_b200.configs import (MODE_CHUNKED_PREFILL, MODE_CUDA_GRAPHS, MODE_FP16,
                                           MODE_GPTQ4, MODE_INT8, MODE_INT8_CB, MODE_SPEC)
from paper_2605_23057_b200.profile_writer import NOMINAL, build_profile, fit_baseline, write_profile

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                   "ref_golden")


def _fake_measurements():
    meas = {}
    for i, (fam, (p, o)) in enumerate(NOMINAL.items()):
        base = 20.0 + 0.4 * p + 11.5 * o  # the reference's default FP16 cost model (profile.cpp:281-291)
        for mode, sp in ((MODE_FP16, 1.0), (MODE_INT8, 1.3), (MODE_GPTQ4, 1.5), (MODE_SPEC, 1.2),
                         (MODE_INT8_CB, 0.9), (MODE_CHUNKED_PREFILL, 0.98), (MODE_CUDA_GRAPHS, 1.02)):
            meas[(mode, fam)] = {"latency_ms": base / sp, "tokens": o, "prompt": p,
                                 "energy_j_per_token": 3.0 / sp, "mem_bytes": 16e9 / sp}
    return meas


def test_fit_recovers_linear_cost_model():
    runs = [(p, o, 20.0 + 0.4 * p + 11.5 * o) for p, o in NOMINAL.values()]
    fixed, a, b = fit_baseline(runs)
    assert abs(fixed - 20.0) < 1e-6 and abs(a - 0.4) < 1e-9 and abs(b - 11.5) < 1e-9


def test_profile_schema_and_ratios():
    prof = build_profile(_fake_measurements(), 3.0, 16384.0)
    assert set(prof) == {"baseline_costs", "cells"}
    assert len(prof["cells"]) == 7 * len(NOMINAL)
    assert {c["mode"] for c in prof["cells"]} >= {"chunked_prefill", "cuda_graphs"}
    fp16 = [c for c in prof["cells"] if c["mode"] == "fp16"]
    assert all(c["latency_speedup"] == 1.0 and c["energy_ratio"] == 1.0 for c in fp16)
    g4 = next(c for c in prof["cells"] if c["mode"] == "gptq4" and c["family"] == "GSM8K")
    assert abs(g4["latency_speedup"] - 1.5) < 1e-12 and abs(g4["energy_ratio"] - 1 / 1.5) < 1e-12


@pytest.mark.skipif(not os.path.exists(REF), reason="oracle/_ref not built (needs /root/reference)")
def test_reference_load_profile_accepts_written_profile(tmp_path):
    path = str(tmp_path / "b200_profile.json")
    write_profile(path, build_profile(_fake_measurements(), 3.0, 16384.0))
    out = subprocess.run([REF, "--check-profile", path], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.startswith("ok 11 families")
    # and a broken one is rejected by the reference loader (schema really is checked)
    prof = json.load(open(path))
    prof["cells"][0]["bogus_key"] = 1
    json.dump(prof, open(path, "w"))
    assert subprocess.run([REF, "--check-profile", path], capture_output=True).returncode == 3


@pytest.mark.skipif(not os.path.exists(REF), reason="oracle/_ref not built (needs /root/reference)")
def test_reference_load_profile_accepts_committed_b200_profile():
    """The B200-measured profile committed under profiles/ (10 modes incl. the
    four screening modes x 11 families) loads in the reference's own
    load_profile, so route_oracle / compare_policies can run on it."""
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                        "r02_b200_profile.json")
    prof = json.load(open(path))
    assert len({c["mode"] for c in prof["cells"]}) == 10
    out = subprocess.run([REF, "--check-profile", path], capture_output=True, text=True)
    assert out.returncode == 0 and out.stdout.startswith("ok 11 families"), out.stdout + out.stderr
