"""Measured-profile writer: B200 measurements of every
engine-implemented mode on each workload family's nominal request, written in
the reference's profile JSON schema so its own `load_profile`
(profile.cpp:132-239), `route_oracle` (routing.cpp:102-165) and
`compare_policies` (sim.cpp:237-263) run on B200 numbers instead of the shipped
mostly-synthesized table (profile.cpp:335-446).

Per (mode, family) cell, all measured on the same GPU:
  latency_speedup = FP16 request latency / mode request latency (domain.cpp:118-123)
  energy_ratio    = mode J/token / FP16 J/token (NVML trace, reference trapezoid rule)
  memory_ratio    = (mode-resident weight bytes + KV bytes of the request) / the same for FP16
  quality_delta_pp = 0.0 (not measured: random-init weights have no task accuracy)
  provenance "measured", anchor = (latency_s, output tokens / latency_s, output tokens)
baseline_costs: the FP16 linear cost model (fixed + prefill/token * prompt +
decode/token * output) least-squares fitted to the FP16 runs, FP16 J/token,
FP16 peak MB.

The schema is pinned by tests/test_profile_writer.py, which loads a written
profile with the reference's own load_profile (oracle/_ref/ref_golden
--check-profile)."""
from __future__ import annotations

import json

import numpy as np

from .configs import (MODE_AWQ4, MODE_CHUNKED_PREFILL, MODE_CUDA_GRAPHS, MODE_KV_COMPRESSION, MODE_FP16, MODE_GPTQ4, MODE_GPTQ_PC,
                      MODE_INT8, MODE_INT8_CB, MODE_NAMES, MODE_SPEC)
from .controller import FAMILIES

# family_nominal_shape (workload.cpp:9-23): prompt, output, shared_prefix, memory_pressure
NOMINAL = {
    "SyntheticSS": (128, 32), "SyntheticSL": (128, 128), "SyntheticLS": (1024, 32),
    "SyntheticLL": (1024, 128), "SharedPrefixChat": (1024, 128),
    "MemoryPressureLongContext": (2048, 64), "MMLUPro": (400, 16), "GSM8K": (250, 256),
    "TruthfulQA": (200, 64), "GPQA": (500, 16), "MLU": (300, 16)}
PROFILE_MODES = (MODE_FP16, MODE_INT8, MODE_GPTQ4, MODE_SPEC, MODE_GPTQ_PC, MODE_INT8_CB,
                 MODE_AWQ4, MODE_CHUNKED_PREFILL, MODE_CUDA_GRAPHS, MODE_KV_COMPRESSION)
CB_COHORT = 4  # co-scheduled requests for the continuous-batching cells (batch_pressure 4)
PREFIX_LEN = 768  # shared tokens of SharedPrefixChat requests


def fit_baseline(fp16_runs):
    """Least-squares fixed + a*prompt + b*output over [(prompt, output, latency_ms)]."""
    A = np.array([[1.0, p, o] for p, o, _ in fp16_runs])
    y = np.array([lat for _, _, lat in fp16_runs])
    (fixed, a, b), *_ = np.linalg.lstsq(A, y, rcond=None)
    return float(max(fixed, 0.0)), float(max(a, 0.0)), float(max(b, 0.0))


def build_profile(meas: dict, fp16_energy_j: float, fp16_peak_mb: float) -> dict:
    """meas[(mode, family)] = dict(latency_ms, tokens, energy_j_per_token or None,
    mem_bytes, prompt). FP16 entries must exist for every family."""
    fixed, a, b = fit_baseline([(m["prompt"], m["tokens"], m["latency_ms"])
                                for (mode, _), m in meas.items() if mode == MODE_FP16])
    cells = []
    for fam in FAMILIES:
        base = meas[(MODE_FP16, fam)]
        for mode in PROFILE_MODES:
            m = meas.get((mode, fam))
            if m is None:
                continue
            e_ratio = 1.0
            if m.get("energy_j_per_token") and base.get("energy_j_per_token"):
                e_ratio = m["energy_j_per_token"] / base["energy_j_per_token"]
            lat_s = m["latency_ms"] / 1000.0
            cells.append({
                "mode": MODE_NAMES[mode], "family": fam,
                "latency_speedup": base["latency_ms"] / m["latency_ms"],
                "energy_ratio": e_ratio,
                "memory_ratio": m["mem_bytes"] / base["mem_bytes"],
                "quality_delta_pp": 0.0, "feasible": True, "provenance": "measured",
                "anchor_latency_s": lat_s, "anchor_throughput_tps": m["tokens"] / lat_s,
                "anchor_tokens": float(m["tokens"])})
    return {"baseline_costs": {"prefill_ms_per_token": a, "decode_ms_per_token": b,
                               "fixed_overhead_ms": fixed,
                               "fp16_energy_j_per_token": fp16_energy_j,
                               "fp16_peak_memory_mb": fp16_peak_mb},
            "cells": cells}


def synth_prompt(key: int, n: int, vocab: int) -> np.ndarray:
    return ((np.arange(n, dtype=np.int64) * 2654435761 + key * 40503) % vocab).astype(np.int32)


def measure(eng, device: int = 0, families=FAMILIES, out_cap: int = 0, energy: bool = True) -> dict:
    """Runs each family's nominal request in every mode the engine has resident.
    out_cap > 0 bounds generated tokens (quick profiles)."""
    from .energy import PowerSampler
    meas = {}
    kv_per_pos = eng.kv_bytes_per_position()
    for fi, fam in enumerate(families):
        plen, olen = NOMINAL[fam]
        if out_cap:
            olen = min(olen, out_cap)
        p = synth_prompt(1000 + fi, plen, eng.vocab)
        for mode in PROFILE_MODES:
            if not eng.has_mode(mode):
                continue
            sampler = PowerSampler(device) if energy else None
            try:
                if sampler:
                    sampler.__enter__()
                if mode == MODE_INT8_CB:
                    prompts = [synth_prompt(2000 + fi * 8 + j, plen, eng.vocab) for j in range(CB_COHORT)]
                    rs = eng.run_batch(mode, prompts, [olen] * CB_COHORT)
                    lat = float(np.mean([r.total_ms for r in rs]))
                    toks, ctx_pos = olen, CB_COHORT * (plen + olen)
                else:
                    if mode == MODE_GPTQ_PC:
                        eng.reset_prefix_cache()
                        if fam == "SharedPrefixChat":  # an earlier request of the group shares the prefix
                            q = synth_prompt(3000 + fi, plen, eng.vocab)
                            q[:PREFIX_LEN] = p[:PREFIX_LEN]
                            eng.run(mode, q, 1)
                    r = eng.run(mode, p, olen)
                    lat, toks, ctx_pos = r.total_ms, olen, plen + olen
                jpt = sampler.finish(toks * (CB_COHORT if mode == MODE_INT8_CB else 1)) if sampler else None
            finally:
                if sampler:
                    sampler.__exit__(None, None, None)
            meas[(mode, fam)] = {"latency_ms": lat, "tokens": toks, "prompt": plen,
                                 "energy_j_per_token": jpt,
                                 "mem_bytes": eng.weight_bytes(mode) + kv_per_pos * ctx_pos}
    return meas


def write_profile(path: str, profile: dict) -> None:
    with open(path, "w") as f:
        json.dump(profile, f, indent=1)
