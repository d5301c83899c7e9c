"""Python handle over the C-ABI mode executor (include/msw_engine.h).

Thin: every call goes straight to libmsw_engine.so; buffers are host numpy
arrays (the engine does the host<->device copies). No compute happens here
and there is no fallback if the library or the GPU is missing.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from ._capi import Request, Result, check_engine, engine_lib
from .configs import engine_cfg


@dataclass
class RunResult:
    tokens: np.ndarray
    logits: np.ndarray | None
    prefill_ms: float
    decode_ms: float
    total_ms: float
    spec_rounds: int = 0
    spec_proposed: int = 0
    spec_accepted: int = 0
    prefix_hit_tokens: int = 0
    kernel_launches: int = 0
    extra: dict = field(default_factory=dict)


def _i32p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def _f32p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_float))


class Engine:
    """One per GPU. `cfg` is an EngineCfg (see configs.engine_cfg)."""

    def __init__(self, cfg=None, device: int = 0, **kw):
        self.cfg = cfg if cfg is not None else engine_cfg(**kw)
        self.vocab = self.cfg.target.vocab
        h = C.c_void_p()
        check_engine(engine_lib().msw_engine_create(device, C.byref(self.cfg), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            engine_lib().msw_engine_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _mk(self, mode, prompt, n_new, want_logits, seq=0):
        p = np.ascontiguousarray(prompt, dtype=np.int32)
        out = np.zeros(n_new, dtype=np.int32)
        lg = np.zeros((n_new, self.vocab), dtype=np.float32) if want_logits else None
        req = Request(mode=mode, prompt_ids=_i32p(p), prompt_len=len(p), max_new_tokens=n_new,
                      prefix_group=-1, prefix_len=0, seq=seq)
        res = Result(out_ids=_i32p(out), logits=_f32p(lg) if lg is not None else None)
        return p, out, lg, req, res

    @staticmethod
    def _wrap(out, lg, res) -> RunResult:
        return RunResult(tokens=out, logits=lg, prefill_ms=res.prefill_ms, decode_ms=res.decode_ms,
                         total_ms=res.total_ms, spec_rounds=res.spec_rounds,
                         spec_proposed=res.spec_proposed, spec_accepted=res.spec_accepted,
                         prefix_hit_tokens=res.prefix_hit_tokens,
                         kernel_launches=res.kernel_launches)

    def run(self, mode: int, prompt, n_new: int, want_logits: bool = False, seq: int = 0) -> RunResult:
        p, out, lg, req, res = self._mk(mode, prompt, n_new, want_logits, seq)
        check_engine(engine_lib().msw_engine_run(self.h, C.byref(req), C.byref(res)))
        return self._wrap(out, lg, res)

    def run_batch(self, mode: int, prompts, n_new, want_logits: bool = False) -> list[RunResult]:
        n = len(prompts)
        n_new = list(n_new) if hasattr(n_new, "__len__") else [n_new] * n
        keep, reqs, ress = [], (Request * n)(), (Result * n)()
        outs = []
        for i, (pr, nn) in enumerate(zip(prompts, n_new)):
            p, out, lg, req, res = self._mk(mode, pr, nn, want_logits, i)
            keep.append(p)
            reqs[i] = req
            ress[i] = res
            outs.append((out, lg))
        check_engine(engine_lib().msw_engine_run_batch(self.h, reqs, n, ress))
        return [self._wrap(o, l, ress[i]) for i, (o, l) in enumerate(outs)]

    def has_mode(self, mode: int) -> bool:
        """Mode resident in this engine (modes_mask; speculative decoding also needs a draft)."""
        if mode == 4 and not self.cfg.has_draft:
            return False
        return bool(self.cfg.modes_mask & (1 << mode))

    def kv_bytes_per_position(self) -> int:
        """K + V fp16 bytes one token position occupies in the target's paged cache."""
        t = self.cfg.target
        return 2 * t.n_layers * t.n_kv_heads * t.head_dim * 2

    def weight_bytes(self, mode: int) -> int:
        b = C.c_int64()
        check_engine(engine_lib().msw_engine_weight_bytes(self.h, mode, C.byref(b)))
        return b.value

    def memory_bytes(self, mode: int, tokens: int) -> int:
        """HBM footprint of one `tokens`-position request in `mode` (weights + KV)."""
        b = C.c_int64()
        check_engine(engine_lib().msw_engine_memory_bytes(self.h, mode, tokens, C.byref(b)))
        return b.value

    def reset_prefix_cache(self):
        check_engine(engine_lib().msw_engine_reset_prefix_cache(self.h))


__all__ = ["Engine", "RunResult", "_capi"]


def execute_trace(engine: Engine, ndjson: str, *, token_seed: int = 0, prefix_len: int = 768,
                  max_output_tokens: int = 0, max_prompt_tokens: int = 0, fallback: bool = True,
                  measure_fp16: bool = True, zero_overhead: bool = False, cohort_max: int = 64,
                  constraints: tuple[float, float, float] = (-1.5, 1.0, 1.10),
                  power_device: int = -1, quality_delta_pp: dict[int, float] | None = None,
                  results_csv: str | None = None, comparison_csv: str | None = None,
                  prefix_groups: int = 1):
    """Route (RulePolicy) and execute a trace through the C++ executor
    (libmodeswitch msw_execute_trace). constraints = the reference
    ConstraintSet (quality_floor_pp, energy_ratio_max, memory_ratio_max);
    power_device >= 0 measures energy per request; quality_delta_pp maps
    InferenceMode values to the quality delta charged to that mode (the
    reference profile's cells; random-init weights have no measurable
    quality). Returns (rows as dicts, summary dict)."""
    from ._capi import ExecOpts, ExecRow, ExecSummary, check_host, host_lib
    n_max = ndjson.count("\n") + 1
    rows = (ExecRow * n_max)()
    n = C.c_int32()
    summ = ExecSummary()
    qd = None
    if quality_delta_pp:
        qd = (C.c_double * 12)(*[float(quality_delta_pp.get(m, 0.0)) for m in range(12)])
    opts = ExecOpts(int(fallback), int(zero_overhead), 0.0, int(measure_fp16), token_seed, prefix_len,
                    max_output_tokens, max_prompt_tokens, cohort_max, constraints[0], constraints[1],
                    constraints[2], power_device, qd,
                    results_csv.encode() if results_csv else None,
                    comparison_csv.encode() if comparison_csv else None, prefix_groups)
    check_host(host_lib().msw_execute_trace(engine.h, engine.vocab, ndjson.encode(), None,
                                            C.byref(opts), n_max, rows, C.byref(n), C.byref(summ)))
    out = [{f: getattr(rows[i], f) for f, _ in ExecRow._fields_} for i in range(n.value)]
    return out, {f: getattr(summ, f) for f, _ in ExecSummary._fields_}


def write_decisions_csv(ndjson: str, rows: list[dict], path: str) -> None:
    """The reference's decisions CSV (report.cpp:49-61) for rows returned by
    execute_trace (trace order): request_id,mode,reason,overhead_ms."""
    from ._capi import ExecRow, check_host, host_lib
    arr = (ExecRow * max(1, len(rows)))()
    for i, r in enumerate(rows):
        for f, _ in ExecRow._fields_:
            setattr(arr[i], f, r[f])
    check_host(host_lib().msw_write_decisions_csv(ndjson.encode(), arr, len(rows), path.encode()))
