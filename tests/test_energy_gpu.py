"""NVML power sampling on the B200 around an executed request: the recorded
trace is in the reference's "timestamp_ms,power_w" format, reads back through
the reference-semantics reader, and integrates to a positive J/token."""
import pytest

from paper_2605_23057_b200 import MODE_GPTQ4, engine_cfg
from paper_2605_23057_b200.energy import PowerSampler, energy_from_trace
from paper_2605_23057_b200.engine import Engine

pytestmark = pytest.mark.gpu


def test_power_trace_round_trip(cuda_ok, tmp_path):
    import numpy as np
    eng = Engine(engine_cfg(target="tiny", draft=None, modes=[MODE_GPTQ4], kv_blocks=64, max_seq_len=256))
    path = str(tmp_path / "power.csv")
    import time
    # >= 2 s of work: the driver's energy counter advances in coarse steps, so a
    # short window cannot be compared with the integrated trace
    n = 0
    with PowerSampler(0, period_ms=5.0, csv_path=path) as ps:
        t0 = time.monotonic()
        while time.monotonic() - t0 < 2.0:
            eng.run(MODE_GPTQ4, np.arange(30, dtype=np.int32), 40)
            n += 40
        jpt = ps.finish(n)
    eng.close()
    assert ps.samples >= 2 and jpt > 0.0
    with open(path) as f:
        assert f.readline().strip() == "timestamp_ms,power_w"
    assert energy_from_trace(path, n) == pytest.approx(jpt, rel=1e-12)
    # instantaneous-power trace vs the driver's energy counter over the same window
    if ps.counter_joules_per_token is not None:
        assert ps.counter_joules_per_token == pytest.approx(jpt, rel=0.3)


def test_profile_writer_measures_tiny_engine(cuda_ok, tmp_path):
    import json
    from paper_2605_23057_b200 import ALL_MODES
    from paper_2605_23057_b200.profile_writer import build_profile, measure, write_profile
    eng = Engine(engine_cfg(target="tiny", draft="tiny_draft", modes=ALL_MODES, kv_blocks=1024,
                            max_seq_len=2560))
    meas = measure(eng, out_cap=6)
    eng.close()
    prof = build_profile(meas, 1.0, 1.0)
    assert len(prof["cells"]) == 10 * 11  # every implemented mode (6 routed + 4 screening) x every family
    assert all(c["latency_speedup"] > 0 and c["provenance"] == "measured" for c in prof["cells"])
    path = str(tmp_path / "p.json")
    write_profile(path, prof)
    assert json.load(open(path))["baseline_costs"]["decode_ms_per_token"] >= 0
