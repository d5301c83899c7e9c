"""Python handle over the host controller C ABI (include/msw_host.h).

Mirrors the reference's controller entry points with the same names and
error behaviour: parse_trace_line / format_trace_line (trace_io.cpp:34-92),
generate_trace (workload.cpp:61-91), RulePolicy::route (routing.cpp:186-194).
Errors raise MswError with the reference's codes (2 config, 3 data).
"""
from __future__ import annotations

import ctypes as C

from ._capi import (ClassifierCfg, Descriptor, MswError, RouteOut, check_host, host_lib)

FAMILIES = ["SyntheticSS", "SyntheticSL", "SyntheticLS", "SyntheticLL", "SharedPrefixChat",
            "MemoryPressureLongContext", "MMLUPro", "GSM8K", "TruthfulQA", "GPQA", "MLU"]
MODES = ["fp16", "int8", "gptq4", "awq4", "speculative_decoding", "prefix_caching",
         "chunked_prefill", "continuous_batching", "cuda_graphs", "kv_cache_compression",
         "gptq_prefix_caching", "int8_continuous_batching"]
CLASSES = ["batched", "shared_prefix", "memory_pressure", "prefill_heavy", "decode_heavy",
           "balanced"]
REASONS = ["rule1_batched", "rule2_shared_prefix", "rule3_memory_pressure",
           "rule4_synthetic_shape", "rule5_decode_heavy", "rule6_choice_benchmark",
           "rule7_default", "oracle_feasible_fastest", "oracle_fallback_fp16", "static",
           "learned_vote"]

__all__ = ["MswError", "route", "route_ndjson", "parse_trace_line", "format_trace_line",
           "generate_trace", "route_cost", "FAMILIES", "MODES"]


def _cls_cfg(c: dict | None):
    if c is None:
        return None
    cfg = ClassifierCfg(512, 64, 0.5, 2)
    for k, v in c.items():
        setattr(cfg, k, v)
    return C.byref(cfg)


def _desc(d: dict) -> tuple[Descriptor, bytes]:
    rid = d["request_id"].encode()
    tag = d.get("workload_tag")
    tag_i = -1 if tag is None else (FAMILIES.index(tag) if isinstance(tag, str) else int(tag))
    return Descriptor(rid, int(d["prompt_tokens"]), int(d["expected_output_tokens"]),
                      int(bool(d.get("shared_prefix", False))),
                      int(bool(d.get("memory_pressure", False))),
                      int(d.get("batch_pressure", 1)), tag_i), rid


def _route_out(o: RouteOut) -> dict:
    return dict(mode=MODES[o.mode], mode_id=o.mode, reason=REASONS[o.reason],
                **{"class": CLASSES[o.workload_class]}, family=FAMILIES[o.family],
                overhead_ms=o.overhead_ms)


def route(desc: dict, classifier: dict | None = None) -> dict:
    d, _keep = _desc(desc)
    out = RouteOut()
    check_host(host_lib().msw_route_rule(C.byref(d), _cls_cfg(classifier), C.byref(out)))
    return _route_out(out)


def route_ndjson(text: str, classifier: dict | None = None) -> list[dict]:
    n_max = text.count("\n") + 1
    outs = (RouteOut * n_max)()
    n = C.c_int32()
    check_host(host_lib().msw_route_ndjson(text.encode(), _cls_cfg(classifier), n_max, outs,
                                           C.byref(n)))
    return [_route_out(outs[i]) for i in range(n.value)]


def parse_trace_line(line: str) -> dict:
    d = Descriptor()
    buf = C.create_string_buffer(len(line) + 1)
    check_host(host_lib().msw_trace_parse_line(line.encode(), C.byref(d), buf, len(buf)))
    return dict(request_id=buf.value.decode(), prompt_tokens=d.prompt_tokens,
                expected_output_tokens=d.expected_output_tokens,
                shared_prefix=bool(d.shared_prefix), memory_pressure=bool(d.memory_pressure),
                batch_pressure=d.batch_pressure,
                workload_tag=None if d.workload_tag < 0 else FAMILIES[d.workload_tag])


def format_trace_line(desc: dict) -> str:
    d, _keep = _desc(desc)
    need = C.c_size_t()
    host_lib().msw_trace_format_line(C.byref(d), None, 0, C.byref(need))
    buf = C.create_string_buffer(need.value)
    check_host(host_lib().msw_trace_format_line(C.byref(d), buf, need.value, C.byref(need)))
    return buf.value.decode()


def generate_trace(counts: dict, jitter: float = 0.10, seed: int = 0, batch_pressure: int = 4,
                   batched_fraction: float = 0.0) -> str:
    arr = (C.c_int32 * 11)(*[int(counts.get(i, counts.get(FAMILIES[i], 0))) for i in range(11)])
    need = C.c_size_t()
    host_lib().msw_trace_generate(arr, jitter, seed, batch_pressure, batched_fraction, None, 0,
                                  C.byref(need))
    if need.value == 0:
        check_host(host_lib().msw_trace_generate(arr, jitter, seed, batch_pressure,
                                                 batched_fraction, None, 0, C.byref(need)))
    buf = C.create_string_buffer(need.value)
    check_host(host_lib().msw_trace_generate(arr, jitter, seed, batch_pressure, batched_fraction,
                                             buf, need.value, C.byref(need)))
    return buf.value.decode()


def route_cost(text: str, passes: int = 100) -> tuple[float, float]:
    """(mean RulePolicy overhead stamp, wall ms per decision) over `passes` of the trace."""
    a, b = C.c_double(), C.c_double()
    check_host(host_lib().msw_route_cost(text.encode(), passes, C.byref(a), C.byref(b)))
    return a.value, b.value
