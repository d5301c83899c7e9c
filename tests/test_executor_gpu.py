"""The executor seam on the B200 (tiny model): the reference's run_policy /
simulate_request / summarize flow (sim.cpp:80-263) with every request routed
by the C++ RulePolicy and EXECUTED through the engine C ABI.

Checks: routing identical to the reference goldens; every routed mode runs
natively (no FP16 fallback); continuous-batching cohorts, speculative
decoding and prefix-cache reuse are exercised; summary fields follow the reference's aggregation formulas.
"""
import csv
import os

import pytest

from paper_2605_23057_b200 import controller as ctl
from paper_2605_23057_b200 import engine_cfg
from paper_2605_23057_b200.engine import Engine, execute_trace

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def eng(cuda_ok):
    e = Engine(engine_cfg(target="tiny", draft="tiny_draft", seed=9, kv_blocks=2048,
                          max_seq_len=2600))
    yield e
    e.close()


def test_config1_mixed_trace_executes_routed_modes(eng):
    text = open(os.path.join(GOLDEN, "config1_mixed.ndjson")).read()
    gold = list(csv.DictReader(open(os.path.join(GOLDEN, "config1_mixed.decisions.csv"))))
    rows, summ = execute_trace(eng, text, max_output_tokens=24, prefix_len=96)
    assert len(rows) == len(gold) == 55
    for r, g in zip(rows, gold):
        assert ctl.MODES[r["mode"]] == g["mode"]
        assert ctl.REASONS[r["reason"]] == g["reason"]
        assert ctl.FAMILIES[r["family"]] == g["family"]
        assert r["fallback_used"] == 0 and r["executed_mode"] == r["mode"]
        assert r["fp16_latency_ms"] > 0 and r["mode_latency_ms"] > 0
        assert abs(r["speedup"] - r["fp16_latency_ms"] / r["mode_latency_ms"]) < 1e-9
    modes = {ctl.MODES[r["mode"]] for r in rows}
    assert {"int8_continuous_batching", "gptq4", "speculative_decoding", "int8",
            "gptq_prefix_caching"} <= modes
    spec = [r for r in rows if ctl.MODES[r["mode"]] == "speculative_decoding"]
    assert all(r["spec_proposed"] > 0 for r in spec)
    pc = [r for r in rows if ctl.MODES[r["mode"]] == "gptq_prefix_caching"]
    assert pc[-1]["prefix_hit_tokens"] == 96  # shared 96-token prefix reused (6 blocks)
    # reference aggregation (sim.cpp:149-207)
    n = len(rows)
    assert summ["request_count"] == n and summ["fallback_count"] == 0
    assert abs(summ["mean_speedup"] - sum(r["speedup"] for r in rows) / n) < 1e-9
    agg = sum(r["fp16_latency_ms"] for r in rows) / sum(r["mode_latency_ms"] for r in rows)
    assert abs(summ["aggregate_latency_speedup"] - agg) < 1e-9
    assert summ["generated_tokens"] == sum(r["output_tokens"] for r in rows)


def test_single_request_cohort(eng):
    # rule 1 (batch_pressure >= 2) routes to INT8 + continuous batching; a
    # cohort of one still runs through the batch path, not the FP16 fallback
    line = ctl.format_trace_line(dict(request_id="solo", prompt_tokens=40, expected_output_tokens=5,
                                      batch_pressure=2, workload_tag=None))
    rows, summ = execute_trace(eng, line + "\n")
    assert ctl.MODES[rows[0]["executed_mode"]] == "int8_continuous_batching"
    assert summ["fallback_count"] == 0


REF_INTEROP = os.path.join(os.path.dirname(GOLDEN), "..", "oracle", "_ref", "ref_exec_interop")
# quality delta charged per mode (pp): random-init weights have no measurable
# quality, so the executor takes these from the caller (here: illustrative
# values in the reference profile's style)
QUALITY = {1: -0.3, 2: -0.9, 4: 0.0, 10: -0.9, 11: -0.3}


def test_sim_request_result_fields_and_reference_consumers(eng, tmp_path):
    """The executor fills the reference's SimRequestResult fields with
    measured values (energy from the driver counter around the mode and FP16
    runs, memory_ratio from HBM footprints, constraint_violated against the
    ConstraintSet), and the reference's own consumers accept its output:
    evaluate_quality_gate on the rebuilt results agrees with the executor's,
    write_decisions_csv reproduces the executor's decisions file byte for
    byte, and write_comparison_csv reproduces its comparison.csv byte for byte
    (oracle/_ref/ref_exec_interop links the reference library)."""
    import json
    import subprocess
    from paper_2605_23057_b200.engine import write_decisions_csv
    text = open(os.path.join(GOLDEN, "config1_mixed.ndjson")).read()
    res_csv, cmp_csv = str(tmp_path / "results.csv"), str(tmp_path / "comparison.csv")
    rows, summ = execute_trace(eng, text, max_output_tokens=16, prefix_len=96, power_device=0,
                               quality_delta_pp=QUALITY, results_csv=res_csv, comparison_csv=cmp_csv)
    for r in rows:
        m = ctl.MODES[r["executed_mode"]]
        assert r["energy_j"] > 0, "energy not measured"
        # tiny-model requests last a few ms: the ratio of two such windows is
        # noisy (the 8B energy tests hold the accuracy bar), only sane here
        assert 0.0 < r["energy_ratio"] < 1e3
        if m in ("gptq4", "gptq_prefix_caching"):
            assert r["memory_ratio"] < 0.6
        elif m in ("int8", "int8_continuous_batching"):
            assert r["memory_ratio"] < 0.8
        elif m == "speculative_decoding":
            assert r["memory_ratio"] > 1.0  # draft weights + KV on top of FP16
        assert r["quality_delta_pp"] == QUALITY.get(r["executed_mode"], 0.0)
        viol = not (r["quality_delta_pp"] >= -1.5 and r["energy_ratio"] <= 1.0 and r["memory_ratio"] <= 1.10)
        assert bool(r["constraint_violated"]) == viol
    n = len(rows)
    assert abs(summ["mean_memory_ratio"] - sum(r["memory_ratio"] for r in rows) / n) < 1e-12
    assert abs(summ["constraint_violation_rate"] - sum(r["constraint_violated"] for r in rows) / n) < 1e-12
    dec_csv = str(tmp_path / "decisions.ours.csv")
    write_decisions_csv(text, rows, dec_csv)
    if not os.path.exists(REF_INTEROP):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    out_dir = tmp_path / "ref"
    out_dir.mkdir()
    p = subprocess.run([REF_INTEROP, res_csv, cmp_csv, str(out_dir)], capture_output=True, text=True,
                       timeout=60)
    assert p.returncode == 0, p.stderr
    ref = json.loads(p.stdout)
    assert ref["requests"] == n and ref["decisions_read_back"] == n
    assert ref["gate_passed"] == summ["quality_gate_passed"]
    assert float(ref["collapsed_benchmark_delta_pp"]) == pytest.approx(summ["collapsed_benchmark_delta_pp"], abs=1e-12)
    assert ref["benchmark_families"] > 0
    assert open(out_dir / "decisions.csv").read() == open(dec_csv).read()
    assert open(out_dir / "comparison.csv").read() == open(cmp_csv).read()
