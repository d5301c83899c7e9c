"""ctypes mirror of include/msw_engine.h and include/msw_host.h.

Loads the in-tree shared objects built by build.py. Missing libraries are a
hard error: there is no Python or CPU fallback for any product path.
"""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(_PKG, "lib")

MSW_OK, MSW_ERR_OTHER, MSW_ERR_CONFIG, MSW_ERR_DATA = 0, 1, 2, 3
W_FP16, W_INT8, W_W4 = 0, 1, 2
KV_BLOCK = 16
W4_GROUP = 128


class ModelCfg(C.Structure):
    _fields_ = [
        ("hidden", C.c_int32), ("n_layers", C.c_int32), ("n_heads", C.c_int32),
        ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("ffn", C.c_int32),
        ("vocab", C.c_int32), ("rms_eps", C.c_float), ("rope_theta", C.c_float),
        ("rope_factor", C.c_float), ("rope_low_freq_factor", C.c_float),
        ("rope_high_freq_factor", C.c_float), ("rope_orig_ctx", C.c_int32),
    ]


class EngineCfg(C.Structure):
    _fields_ = [
        ("target", ModelCfg), ("draft", ModelCfg), ("has_draft", C.c_int32),
        ("modes_mask", C.c_uint32), ("weight_seed", C.c_uint64),
        ("draft_agree_permille", C.c_int32), ("kv_blocks", C.c_int32),
        ("max_batch", C.c_int32), ("max_seq_len", C.c_int32), ("spec_k", C.c_int32),
        ("use_graphs", C.c_int32),
    ]


class Request(C.Structure):
    _fields_ = [
        ("mode", C.c_int32), ("prompt_ids", C.POINTER(C.c_int32)), ("prompt_len", C.c_int32),
        ("max_new_tokens", C.c_int32), ("prefix_group", C.c_int32), ("prefix_len", C.c_int32),
        ("seq", C.c_uint64),
    ]


class Result(C.Structure):
    _fields_ = [
        ("out_ids", C.POINTER(C.c_int32)), ("n_out", C.c_int32), ("logits", C.POINTER(C.c_float)),
        ("prefill_ms", C.c_double), ("decode_ms", C.c_double), ("total_ms", C.c_double),
        ("spec_rounds", C.c_int32), ("spec_proposed", C.c_int32), ("spec_accepted", C.c_int32),
        ("prefix_hit_tokens", C.c_int32), ("kernel_launches", C.c_int32),
    ]


class Descriptor(C.Structure):
    _fields_ = [
        ("request_id", C.c_char_p), ("prompt_tokens", C.c_int32),
        ("expected_output_tokens", C.c_int32), ("shared_prefix", C.c_int32),
        ("memory_pressure", C.c_int32), ("batch_pressure", C.c_int32),
        ("workload_tag", C.c_int32),
    ]


class ClassifierCfg(C.Structure):
    _fields_ = [
        ("long_prompt_threshold", C.c_int32), ("long_output_threshold", C.c_int32),
        ("decode_heavy_ratio", C.c_double), ("batch_threshold", C.c_int32),
    ]


class RouteOut(C.Structure):
    _fields_ = [
        ("mode", C.c_int32), ("reason", C.c_int32), ("workload_class", C.c_int32),
        ("family", C.c_int32), ("overhead_ms", C.c_double),
    ]


class ExecOpts(C.Structure):
    _fields_ = [
        ("fallback_enabled", C.c_int32), ("zero_overhead", C.c_int32),
        ("extra_overhead_ms", C.c_double), ("measure_fp16_baseline", C.c_int32),
        ("token_seed", C.c_uint64), ("prefix_len", C.c_int32), ("max_output_tokens", C.c_int32),
        ("max_prompt_tokens", C.c_int32), ("cohort_max", C.c_int32),
        ("quality_floor_pp", C.c_double), ("energy_ratio_max", C.c_double),
        ("memory_ratio_max", C.c_double), ("power_device", C.c_int32),
        ("quality_delta_pp", C.POINTER(C.c_double)), ("results_csv", C.c_char_p),
        ("comparison_csv", C.c_char_p), ("prefix_groups", C.c_int32),
    ]


class ExecRow(C.Structure):
    _fields_ = [
        ("mode", C.c_int32), ("reason", C.c_int32), ("executed_mode", C.c_int32),
        ("family", C.c_int32), ("prompt_tokens", C.c_int32), ("output_tokens", C.c_int32),
        ("fallback_used", C.c_int32), ("spec_proposed", C.c_int32), ("spec_accepted", C.c_int32),
        ("prefix_hit_tokens", C.c_int32), ("fp16_latency_ms", C.c_double),
        ("mode_latency_ms", C.c_double), ("speedup", C.c_double), ("overhead_ms", C.c_double),
        ("prefill_ms", C.c_double), ("decode_ms", C.c_double),
        ("energy_j", C.c_double), ("energy_ratio", C.c_double), ("memory_ratio", C.c_double),
        ("quality_delta_pp", C.c_double), ("constraint_violated", C.c_int32),
    ]


class ExecSummary(C.Structure):
    _fields_ = [
        ("request_count", C.c_int32), ("fallback_count", C.c_int32), ("mean_speedup", C.c_double),
        ("aggregate_latency_speedup", C.c_double), ("collapsed_mean_speedup", C.c_double),
        ("mean_overhead_ms", C.c_double), ("mode_time_ms", C.c_double),
        ("generated_tokens", C.c_int64), ("mean_energy_ratio", C.c_double),
        ("mean_memory_ratio", C.c_double), ("mean_quality_delta_pp", C.c_double),
        ("collapsed_mean_energy_ratio", C.c_double), ("constraint_violation_rate", C.c_double),
        ("quality_gate_passed", C.c_int32), ("collapsed_benchmark_delta_pp", C.c_double),
    ]


def _load(name: str) -> C.CDLL:
    path = os.path.join(LIB_DIR, name)
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no fallback path)")
    return C.CDLL(path, mode=C.RTLD_GLOBAL)


_engine = None
_host = None


def engine_lib() -> C.CDLL:
    global _engine
    if _engine is None:
        # MSW_ENGINE_SO selects a diagnostics build (libmsw_engine_trace.so); scripts only
        lib = _load(os.environ.get("MSW_ENGINE_SO", "libmsw_engine.so"))
        vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        lib.msw_engine_create.argtypes = [C.c_int, C.POINTER(EngineCfg), C.POINTER(vp)]
        lib.msw_engine_run.argtypes = [vp, C.POINTER(Request), C.POINTER(Result)]
        lib.msw_engine_run_batch.argtypes = [vp, C.POINTER(Request), i32, C.POINTER(Result)]
        lib.msw_engine_destroy.argtypes = [vp]
        lib.msw_engine_destroy.restype = None
        lib.msw_last_error.restype = C.c_char_p
        lib.msw_engine_weight_bytes.argtypes = [vp, i32, C.POINTER(i64)]
        lib.msw_engine_memory_bytes.argtypes = [vp, i32, i32, C.POINTER(i64)]
        lib.msw_engine_reset_prefix_cache.argtypes = [vp]
        lib.msw_linear.argtypes = [i32, vp, vp, i32, i32, vp, i32, vp, vp]
        lib.msw_gemv_i8_acc.argtypes = [vp, vp, i32, i32, vp, vp]
        lib.msw_linear_i8_raw.argtypes = [vp, i32, i32, vp, i32, vp, vp]
        lib.msw_linear_decode.argtypes = [i32, vp, vp, i32, i32, vp, i32, vp, vp]
        lib.msw_repack_decode.argtypes = [i32, vp, i32, i32, vp, vp]
        lib.msw_fill_fp16.argtypes = [vp, i64, i64, C.c_uint64, C.c_uint64, i32, vp]
        lib.msw_quant_int8_rows.argtypes = [vp, i32, i32, vp, vp, vp]
        lib.msw_quant_w4_rows.argtypes = [vp, i32, i32, vp, vp, vp]
        lib.msw_linear_awq4.argtypes = [vp, vp, vp, i32, i32, vp, i32, vp, vp]
        lib.msw_fp8_e4m3_roundtrip.argtypes = [vp, C.c_int64, vp, vp, vp]
        lib.msw_quant_awq4_rows.argtypes = [vp, i32, i32, vp, vp, vp, vp]
        lib.msw_device_pci_bus_id.argtypes = [i32, C.c_char_p, i32]
        lib.msw_attention_decode.argtypes = [vp, vp, i32, vp, vp, vp, vp, i32, vp, vp, i32, i32, i32,
                                             i32, vp, vp]
        _engine = lib
    return _engine


def host_lib() -> C.CDLL:
    global _host
    if _host is None:
        engine_lib()
        lib = _load("libmodeswitch.so")
        lib.msw_route_rule.argtypes = [C.POINTER(Descriptor), C.POINTER(ClassifierCfg), C.POINTER(RouteOut)]
        lib.msw_route_ndjson.argtypes = [C.c_char_p, C.POINTER(ClassifierCfg), C.c_int32,
                                         C.POINTER(RouteOut), C.POINTER(C.c_int32)]
        lib.msw_trace_parse_line.argtypes = [C.c_char_p, C.POINTER(Descriptor), C.c_char_p, C.c_size_t]
        lib.msw_trace_format_line.argtypes = [C.POINTER(Descriptor), C.c_char_p, C.c_size_t,
                                              C.POINTER(C.c_size_t)]
        lib.msw_trace_generate.argtypes = [C.POINTER(C.c_int32), C.c_double, C.c_uint64, C.c_int32,
                                           C.c_double, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]
        lib.msw_route_cost.argtypes = [C.c_char_p, C.c_int32, C.POINTER(C.c_double),
                                       C.POINTER(C.c_double)]
        lib.msw_execute_trace.argtypes = [C.c_void_p, C.c_int32, C.c_char_p, C.POINTER(ClassifierCfg),
                                          C.POINTER(ExecOpts), C.c_int32, C.POINTER(ExecRow),
                                          C.POINTER(C.c_int32), C.POINTER(ExecSummary)]
        lib.msw_write_decisions_csv.argtypes = [C.c_char_p, C.POINTER(ExecRow), C.c_int32, C.c_char_p]
        lib.msw_power_start.argtypes = [C.c_int32, C.c_double, C.POINTER(C.c_void_p)]
        lib.msw_power_stop.argtypes = [C.c_void_p, C.c_char_p, C.c_int32, C.POINTER(C.c_double),
                                       C.POINTER(C.c_int32), C.POINTER(C.c_double)]
        lib.msw_energy_from_trace.argtypes = [C.c_char_p, C.c_int32, C.POINTER(C.c_double)]
        lib.msw_host_last_error.restype = C.c_char_p
        _host = lib
    return _host


class MswError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def check_engine(rc: int) -> None:
    if rc != MSW_OK:
        raise MswError(rc, (engine_lib().msw_last_error() or b"").decode())


def check_host(rc: int) -> None:
    if rc != MSW_OK:
        raise MswError(rc, (host_lib().msw_host_last_error() or b"").decode())
