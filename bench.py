#!/usr/bin/env python
"""Benchmark driver (BASELINE.json config 2 by default).

Workload "decode8b": Llama-3.1-8B-shape, K16 random-init weights, batch-1
greedy decode of one synthetic request (prompt 128 -> 128 new tokens, the
SyntheticSS nominal prompt) in each resident mode FP16, INT8 (W8A8) and
GPTQ4 (W4 g128) on every GPU. One step = that request in all three modes,
issued through the C ABI (msw_engine_run) with HOST prompt/token buffers.

  value  = GPTQ4 decode tokens/s (device time: CUDA events on the engine's
           stream around the graph-replayed decode loop), summed over ranks;
  e2e    = GPTQ4 generated tokens / msw_engine_run wall time (H2D prompt,
           prefill, decode, D2H tokens), summed over ranks;
  per_mode / speedup_vs_fp16: every mode's decode tok/s and its mean
           request-latency speedup over FP16 on the same request
           (reference metric, domain.cpp:118-123);
  roofline: the dominant kernel, the W4 GEMV (gate_up, 28672 x 4096),
           timed with CUDA events on torch's stream over rotating weight
           copies larger than L2, against MEASURED_PEAKS.json hbm_gbs;
  cpu_baseline: the CPU oracle (port) on a bounded 8B W4 sample.

Multi-GPU: one process per GPU (torchrun), each rank its own replica and its
own requests (request sharding, no data-path collective); max over ranks.

--impl reference: the reference has no inference path, so the
reference arm times this repo's C oracle port of the same math on the host
cores (kind "port"), plus the reference's own RulePolicy::route cost from
oracle/_ref when present.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MODES = [(0, "fp16"), (1, "int8"), (2, "gptq4")]
PROMPT, NEW = 128, 128


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi style clock / throttle sampling during the timed region (NVML)."""

    def __init__(self, device: int):
        self.device, self.samples, self._stop = device, [], threading.Event()
        self.max_mhz, self.reasons = None, set()

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.hd = nv.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.hd, nv.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception as ex:  # no NVML: record why
            self.nv = None
            self.reasons.add(f"nvml_unavailable:{type(ex).__name__}")
        return self

    def _run(self):
        nv = self.nv
        names = {
            getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8): "hw_slowdown",
            getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4): "sw_power_cap",
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.hd, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.hd)
                for bit, nm in names.items():
                    if r & bit:
                        self.reasons.add(nm)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join(timeout=1)

    def summary(self):
        busy = [s for s in self.samples if s > 300] or self.samples
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": self.max_mhz,
                "samples": len(self.samples), "reasons": sorted(self.reasons)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def synth_prompt(seed: int, n: int, vocab: int):
    import numpy as np
    return np.random.default_rng(seed).integers(0, vocab, size=n).astype(np.int32)


def time_dominant_kernel(iters: int = 50):
    """W4 GEMV on the 8B gate_up shape (28672 x 4096), rotating over weight
    copies larger than L2, CUDA events on torch's current stream."""
    import numpy as np
    import torch
    from paper_2605_23057_b200._capi import check_engine, engine_lib
    n, k = 2 * 14336, 4096
    copies = 5  # 5 x 60.6 MB > 126 MB L2
    lib = engine_lib()
    ws, ss = [], []
    for i in range(copies):
        w16 = torch.empty((n, k), dtype=torch.int16, device="cuda")
        check_engine(lib.msw_fill_fp16(w16.data_ptr(), n, k, 99, 4000 + i, 6, None))
        q = torch.empty((n, k // 8), dtype=torch.int32, device="cuda")
        s = torch.empty((n, k // 128), dtype=torch.int16, device="cuda")
        check_engine(lib.msw_quant_w4_rows(w16.data_ptr(), n, k, q.data_ptr(), s.data_ptr(), None))
        qm = torch.empty_like(q)
        check_engine(lib.msw_repack_decode(2, q.data_ptr(), n, k, qm.data_ptr(), None))
        ws.append(qm)
        del q
        ss.append(s)
        del w16
    x = torch.randn(k, device="cuda", dtype=torch.float32)
    y = torch.empty(n, device="cuda", dtype=torch.float32)
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    for i in range(5):
        check_engine(lib.msw_linear_decode(2, ws[i % copies].data_ptr(), ss[i % copies].data_ptr(), n,
                                           k, x.data_ptr(), 1, y.data_ptr(), sp))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(iters):
        check_engine(lib.msw_linear_decode(2, ws[i % copies].data_ptr(), ss[i % copies].data_ptr(), n,
                                           k, x.data_ptr(), 1, y.data_ptr(), sp))
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    algo_bytes = n * k // 2 + n * (k // 128) * 2 + k * 4 + n * 4  # weights + scales + x + y
    return {"kernel": "gemv_w4_kernel (cp.async.bulk ring, 4 chunks/warp/stage, mma.sync) gate_up 28672x4096, batch 1",
            "ms": ms, "bytes": algo_bytes,
            "gbs": algo_bytes / (ms * 1e-3) / 1e9}


def profiled_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant
    kernel, from the committed `ncu --set full` capture (profiles/)."""
    path = os.path.join(ROOT, "profiles", "r01_ncu_w4_gemv_gate_up.txt")
    try:
        vals = {}
        for line in open(path):
            parts = line.split()
            if parts and parts[0] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[parts[2]]
                vals[parts[0]] = float(parts[1]) * scale
        return vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
    except Exception:
        return None


def cpu_baseline_8b(new_tokens: int = 27, prompt_len: int = 4):
    """CPU oracle (C port, OpenMP over all host cores), 8B shape, W4 mode."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O  # checker / baseline only
    from paper_2605_23057_b200.configs import model_cfg
    t0 = time.perf_counter()
    m = O.OracleModel(model_cfg("llama8b"), seed=0, modes_mask=1 << 2,
                      max_ctx=prompt_len + new_tokens + 1)
    t_init = time.perf_counter() - t0
    p = synth_prompt(1, prompt_len, 128256)
    t0 = time.perf_counter()
    m.generate(2, p, new_tokens)
    dt = time.perf_counter() - t0
    m.close()
    forwards = prompt_len + new_tokens - 1
    return {"value": forwards / dt, "unit": "tokens/s", "cores": O.lib().orc_threads(),
            "kind": "port",
            "sample": f"8B-shape W4 g128 decode, {prompt_len}-token prompt + {new_tokens} new tokens "
                      f"({forwards} full forwards, {dt:.1f} s; weight init {t_init:.1f} s excluded)"}


def ref_route_cost():
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_route_bench")
    trace = os.path.join(ROOT, "tests", "golden", "balanced_55_seed7.ndjson")
    if not (os.path.exists(exe) and os.path.exists(trace)):
        return None
    try:
        out = subprocess.run([exe, trace, "200"], capture_output=True, text=True, timeout=120)
        return json.loads(out.stdout.strip().splitlines()[-1])
    except Exception:
        return None


def default_config(ws):
    """The default workload's `config` (both arms print the same one)."""
    return {"workload": "llama8b batch-1 decode, prompt 128 -> 128 tokens; value = gptq4 mode",
            "model": "llama3.1-8b-shape", "modes": [n for _, n in MODES],
            "parallelism": f"request-sharded replicas x{ws}",
            "l2": "weights stream 4.65-15 GB per token >> 126 MB L2 (no flush needed)"}


def run_reference(args):
    """Reference arm: the reference has no inference path, so the
    C oracle port of the same W4 decode math runs on all host cores; one step
    = one 8B-shape decode token. Rank 0 only."""
    ws, rank, _ = _dist()
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O  # reference-arm baseline (port) only
    from paper_2605_23057_b200.configs import model_cfg
    n_tok = args.warmup + args.steps
    t0 = time.perf_counter()
    m = O.OracleModel(model_cfg("llama8b"), seed=0, modes_mask=1 << 2, max_ctx=n_tok + 4)
    init_s = time.perf_counter() - t0
    p = synth_prompt(1, 1, 128256)
    # generate() runs one full forward per token; time W warm-up + K timed tokens
    t0 = time.perf_counter()
    m.generate(2, p, args.warmup)
    t_warm = time.perf_counter() - t0
    t0 = time.perf_counter()
    m.generate(2, p, n_tok)
    t_all = time.perf_counter() - t0
    m.close()
    dt = max(1e-9, t_all - t_warm)
    v = args.steps / dt
    line = {"metric": "decode tokens/s per mode and routed mix (1/2/4/8 B200); mean latency vs FP16 mode",
            "impl": "reference", "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / v,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "w4a16",
            "data": "synthetic", "config": default_config(ws),
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": O.lib().orc_threads(),
                             "kind": "port",
                             "sample": f"8B-shape W4 g128 decode (the gptq4 arm of the workload), "
                                       f"{args.steps} timed tokens after {args.warmup} warm-up from a "
                                       f"1-token prompt: a bounded sample (a 128-token prompt is 128 "
                                       f"CPU forwards; the weight stream dominates each token either way; "
                                       f"weight init {init_s:.1f} s excluded)"},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "reference_route_cost": ref_route_cost(),
            "note": "reference has no inference path (SPEC.md:20); arm = C oracle port of the same math"}
    print(json.dumps(line), flush=True)


def run_ours(args):
    import numpy as np
    import torch
    ws, rank, local = _dist()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    from paper_2605_23057_b200 import engine_cfg
    from paper_2605_23057_b200.engine import Engine

    cfg = engine_cfg(target="llama8b", draft=None, modes=[m for m, _ in MODES], seed=0,
                     kv_blocks=256, max_batch=8, max_seq_len=PROMPT + NEW + 32, use_graphs=True)
    t0 = time.perf_counter()
    eng = Engine(cfg, device=local)
    init_s = time.perf_counter() - t0
    wbytes = {name: eng.weight_bytes(m) for m, name in MODES}
    prompts = [synth_prompt(1000 * rank + i, PROMPT, 128256) for i in range(args.warmup + args.steps)]

    from paper_2605_23057_b200.energy import PowerSampler
    energy = {name: [] for _, name in MODES}

    def one_step(p, measure_energy=False):
        out = {}
        for m, name in MODES:
            if measure_energy:
                try:  # whole-GPU energy over this request: the driver's energy counter
                    # (instantaneous-power trapezoid where the counter is missing)
                    with PowerSampler(local, period_ms=5.0) as ps:
                        out[name] = eng.run(m, p, NEW)
                        jpt = ps.finish(NEW)
                        energy[name].append(ps.counter_joules_per_token or jpt)
                    continue
                except Exception:
                    pass
            out[name] = eng.run(m, p, NEW)
        return out

    for i in range(args.warmup):
        one_step(prompts[i])
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    agg = {name: {"dec_ms": 0.0, "tot_ms": 0.0, "pre_ms": 0.0, "tokens": 0, "launches": 0} for _, name in MODES}
    speedups = {name: [] for _, name in MODES}
    ref_tokens = None
    with ClockSampler(local) as clk:
        t_wall = time.perf_counter()
        for i in range(args.steps):
            res = one_step(prompts[args.warmup + i], measure_energy=True)
            for _, name in MODES:
                r = res[name]
                a = agg[name]
                a["dec_ms"] += r.decode_ms
                a["tot_ms"] += r.total_ms
                a["pre_ms"] += r.prefill_ms
                a["tokens"] += len(r.tokens)
                a["launches"] += r.kernel_launches
                speedups[name].append(res["fp16"].total_ms / r.total_ms)
            ref_tokens = res["gptq4"].tokens
        torch.cuda.synchronize()
        wall = time.perf_counter() - t_wall
    # max over ranks of the device decode time / e2e time (gptq4 headline)
    dec = torch.tensor([agg["gptq4"]["dec_ms"], agg["gptq4"]["tot_ms"], wall * 1000.0],
                       dtype=torch.float64, device="cuda")
    if ws > 1:
        torch.distributed.all_reduce(dec, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.barrier()
    dec_ms_max, tot_ms_max, wall_max = dec.tolist()
    if rank != 0:
        eng.close()
        if ws > 1:
            torch.distributed.destroy_process_group()
        return
    # decode tokens: first token comes from prefill; the decode loop makes NEW-1 tokens per request
    dec_tokens = (NEW - 1) * args.steps
    value = ws * dec_tokens / (dec_ms_max / 1000.0)
    e2e = ws * NEW * args.steps / (tot_ms_max / 1000.0)
    per_mode = {}
    # algorithmic bytes per decode token = every linear's weights +
    # lm_head + the KV the token's attention reads (context PROMPT + j at step j)
    from paper_2605_23057_b200.configs import model_cfg
    kv_tok = kv_bytes_per_pos(model_cfg("llama8b")) * sum(PROMPT + j for j in range(1, NEW)) / (NEW - 1)
    for _, name in MODES:
        a = agg[name]
        tps = (NEW - 1) * args.steps / (a["dec_ms"] / 1000.0)
        per_mode[name] = {"decode_tok_s": tps, "ms_per_token": a["dec_ms"] / ((NEW - 1) * args.steps),
                          "prefill_ms": a["pre_ms"] / args.steps, "request_ms": a["tot_ms"] / args.steps,
                          "weight_bytes_per_token": wbytes[name],
                          "kv_bytes_per_token": kv_tok,
                          "hbm_frac_of_measured": (wbytes[name] + kv_tok) * tps / 1e9 / peaks()[0],
                          "latency_speedup_vs_fp16": statistics.mean(speedups[name])}
        if energy[name]:
            per_mode[name]["joules_per_token"] = statistics.mean(energy[name])
    if energy["fp16"]:
        for _, name in MODES:
            if energy[name]:  # reference ratio_vs_baseline(mode, fp16) = mode / fp16 (domain.cpp:118-133)
                per_mode[name]["energy_ratio_vs_fp16"] = statistics.mean(energy[name]) / statistics.mean(energy["fp16"])
    kern = time_dominant_kernel()
    peak, peak_kind = peaks()
    launches = sum(agg[n]["launches"] for _, n in MODES)
    cpu = cpu_baseline_8b() if not args.no_cpu_baseline else None
    line = {
        "metric": "decode tokens/s per mode and routed mix (1/2/4/8 B200); mean latency vs FP16 mode",
        "value": value, "unit": "tokens/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": wall_max / args.steps,  # wall_max is in ms; one step = the request in 3 modes
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "w4a16",
        "data": "synthetic (K16 random-init weights, hashed prompt ids)",
        "config": default_config(ws),
        "e2e": {"value": e2e, "unit": "tokens/s", "h2d_bytes_per_step": PROMPT * 4 * len(MODES),
                "d2h_bytes_per_step": NEW * 4 * len(MODES)},
        "per_mode": per_mode,
        "roofline": {"bound": "hbm", "achieved": kern["gbs"], "peak": peak, "unit": "GB/s",
                     "frac": kern["gbs"] / peak, "traffic": profiled_traffic(),
                     "kernel": kern["kernel"],
                     "kernel_ms": kern["ms"], "bytes_per_launch": kern["bytes"],
                     "peak_source": peak_kind,
                     "decode_step_frac": per_mode["gptq4"]["hbm_frac_of_measured"]},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "engine_init_s": init_s,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    eng.close()
    if ws > 1:
        torch.distributed.destroy_process_group()


def deploy_mix_trace(per_class: int, seed: int = 7) -> str:
    """BASELINE config 5: short interactive (SyntheticSS 128->32), long-gen
    (SyntheticSL 128->128, GSM8K 250->256), shared-prefix chat (1024->128),
    8K long-context (MemoryPressureLongContext, prompt x4 -> ~8192, 64 out),
    tagged, jitter 0.10 via the reference generator (workload.cpp:61-91)."""
    from paper_2605_23057_b200 import controller as ctl
    counts = {"SyntheticSS": per_class, "SyntheticSL": per_class, "GSM8K": per_class,
              "SharedPrefixChat": per_class, "MemoryPressureLongContext": per_class}
    lines = []
    for line in ctl.generate_trace(counts, jitter=0.10, seed=seed).splitlines():
        d = ctl.parse_trace_line(line)
        if d["workload_tag"] == "MemoryPressureLongContext":
            d["prompt_tokens"] *= 4  # 2048 nominal -> 8192 (8K long context)
        lines.append(ctl.format_trace_line(d))
    return "\n".join(lines) + "\n"


def run_mix(args):
    """Routed deployment mix (config 5), request-sharded over ranks: each rank
    executes its share through the C++ executor (RulePolicy -> C ABI)."""
    import torch
    ws, rank, local = _dist()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    from paper_2605_23057_b200 import engine_cfg
    from paper_2605_23057_b200.engine import Engine, execute_trace
    eng = Engine(engine_cfg(target="llama8b", draft="llama1b", seed=0, kv_blocks=1536, max_batch=64,
                            max_seq_len=9400, use_graphs=True), device=local)
    from paper_2605_23057_b200.dispatch import aggregate_rows, shard_trace
    text = deploy_mix_trace(args.mix_per_class)
    lines = text.splitlines()
    # cohorts whole, prefix groups sticky, longest-predicted-first onto the least-loaded GPU
    my_idx = shard_trace(text, ws, prefix_groups=args.prefix_groups)[rank]
    mine = "".join(lines[i] + "\n" for i in my_idx)
    execute_trace(eng, "\n".join(lines[:2]) + "\n", max_output_tokens=4)  # warm-up (graphs, attrs)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rows, summ = execute_trace(eng, mine, prefix_len=768, prefix_groups=args.prefix_groups)
    wall = time.perf_counter() - t0
    vals = torch.tensor([summ["generated_tokens"], summ["mode_time_ms"], wall], dtype=torch.float64,
                        device="cuda")
    mine_rows = {i: r for i, r in zip(my_idx, rows)}
    gathered = [mine_rows]
    if ws > 1:
        toks = vals[0].clone()
        torch.distributed.all_reduce(toks)
        torch.distributed.all_reduce(vals, op=torch.distributed.ReduceOp.MAX)
        vals[0] = toks
        gathered = [None] * ws
        torch.distributed.all_gather_object(gathered, mine_rows)
    all_rows = {}
    for g in gathered:
        all_rows.update(g)
    agg = aggregate_rows(all_rows)  # the reference summarize over every request, trace order
    if rank == 0 and args.decisions_out:  # the reference's decisions CSV (report.cpp:49-61)
        from paper_2605_23057_b200.engine import write_decisions_csv
        write_decisions_csv(text, [all_rows[i] for i in sorted(all_rows)], args.decisions_out)
    if rank == 0:
        from paper_2605_23057_b200.controller import MODES
        per_mode = {}
        for r in rows:
            m = MODES[r["mode"]]
            pm = per_mode.setdefault(m, {"requests": 0, "tokens": 0, "mode_ms": 0.0, "speedups": []})
            pm["requests"] += 1
            pm["tokens"] += r["output_tokens"]
            pm["mode_ms"] += r["mode_latency_ms"]
            pm["speedups"].append(r["speedup"])
        for m, pm in per_mode.items():
            pm["tok_s"] = pm["tokens"] / (pm["mode_ms"] / 1000.0)
            pm["mean_speedup_vs_fp16"] = statistics.mean(pm.pop("speedups"))
        print(json.dumps({
            "metric": "decode tokens/s per mode and routed mix (1/2/4/8 B200); mean latency vs FP16 mode",
            "workload": "deploy_mix", "value": vals[0].item() / (vals[1].item() / 1000.0),
            "unit": "tokens/s (generated tokens / routed-mode request time, max over ranks)",
            "n_gpus": ws, "requests": len(lines), "mean_speedup_vs_fp16": agg["mean_speedup"],
            "aggregate_latency_speedup": agg["aggregate_latency_speedup"],
            "collapsed_mean_speedup": agg["collapsed_mean_speedup"],
            "per_family_mean_speedup": agg["per_family_mean_speedup"], "per_mode_rank0": per_mode,
            "placement": f"CB cohorts whole per GPU, {args.prefix_groups} sticky prefix groups, LPT on the "
                         "B200-measured cost model (dispatch.py)",
            "scaling": "weak", "data": "synthetic", "wall_s": vals[2].item()}), flush=True)
    eng.close()
    if ws > 1:
        torch.distributed.destroy_process_group()


# ---- per-config rooflines -----------------------------------
def linear_params(cfg) -> int:
    """Weights of every linear of one forward (QKV, O, gate/up, down x layers + lm_head)."""
    h, f, d = cfg.hidden, cfg.ffn, cfg.head_dim
    qkv = h * (cfg.n_heads + 2 * cfg.n_kv_heads) * d
    return cfg.n_layers * (qkv + cfg.n_heads * d * h + 2 * h * f + f * h) + cfg.vocab * h


def kv_bytes_per_pos(cfg) -> int:
    return 2 * cfg.n_layers * cfg.n_kv_heads * cfg.head_dim * 2


def prefill_flops(cfg, t: int, ctx0: int = 0) -> float:
    """2 * linear params * t + causal attention (QK and PV) over positions
    ctx0 .. ctx0 + t - 1."""
    att = 0.0
    if t > 0:  # sum over query positions p of (p + 1) keys, QK + PV = 4 * Hq * D per key
        att = 4.0 * cfg.n_layers * cfg.n_heads * cfg.head_dim * (t * ctx0 + t * (t + 1) / 2)
    return 2.0 * linear_params(cfg) * t + att


def tensor_peak(kind: str) -> tuple[float, str]:
    """Dense TFLOP/s for the prefill floor: MEASURED_PEAKS bf16 sustained (a
    long step); int8 = 2x that (the B200's nominal int8:bf16 dense ratio)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        bf = float(p.get("bf16_tflops_sustained") or p["bf16_tflops"])
        src = "measured bf16 sustained"
    except Exception:
        bf, src = 1400.0, "fallback"
    return (2.0 * bf, src + " x2 (int8)") if kind == "int8" else (bf, src)


def cpu_mode_sample(mode: int, cfg_name: str = "llama8b", prompt_len: int = 4, new_tokens: int = 3,
                    draft: str | None = None, k: int = 4):
    """The CPU oracle (C port, OpenMP over all host cores) running one mode's
    arithmetic on a bounded sample of the config (8B shape): tokens/s of full
    forwards, and the host-DRAM bytes/s the oracle's storage implies (fp16 2 B,
    int8 1 B, W4 one nibble per byte: 1 B per weight)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O  # checker / baseline only
    from paper_2605_23057_b200.configs import model_cfg
    cfg = model_cfg(cfg_name)
    fmt = {0: 0, 1: 1, 2: 2, 4: 0, 10: 2, 11: 1}[mode]
    omode = {0: 0, 1: 1, 2: 2, 4: 0, 10: 2, 11: 1}[mode]
    t0 = time.perf_counter()
    m = O.OracleModel(cfg, seed=0, modes_mask=1 << omode, max_ctx=prompt_len + new_tokens + 16)
    d = None
    if draft:
        d = O.OracleModel(model_cfg(draft), seed=0, is_draft=True, modes_mask=1, max_ctx=prompt_len + new_tokens + 16)
    t_init = time.perf_counter() - t0
    p = synth_prompt(5, prompt_len, cfg.vocab)
    t0 = time.perf_counter()
    if d is not None:
        _, _, st = O.spec_generate(m, d, k, p, new_tokens)
    else:
        m.generate(omode, p, new_tokens)
    dt = time.perf_counter() - t0
    m.close()
    if d is not None:
        d.close()
    bpw = {0: 2.0, 1: 1.0, 2: 1.0}[fmt]
    if draft:  # per emitted token: the rounds' draft + target forwards
        from paper_2605_23057_b200.configs import model_cfg as mc
        fw = prompt_len + st["rounds"] * (k + 1)  # target verify tokens (approx. forwards)
        sample = (f"{cfg_name} FP16 target + {draft} draft, k={k}: {prompt_len}-token prompt, "
                  f"{new_tokens} tokens, {st['rounds']} rounds in {dt:.1f} s")
        return {"value": new_tokens / dt, "unit": "tokens/s", "cores": O.lib().orc_threads(),
                "kind": "port", "sample": sample, "init_s": round(t_init, 1)}
    forwards = prompt_len + new_tokens - 1
    host_gbs = forwards * linear_params(cfg) * bpw / dt / 1e9
    return {"value": forwards / dt, "unit": "tokens/s (full forwards)", "cores": O.lib().orc_threads(),
            "kind": "port", "host_dram_gbs": round(host_gbs, 1),
            "sample": f"{cfg_name} mode {mode} arithmetic: {prompt_len}-token prompt + {new_tokens} new "
                      f"tokens ({forwards} forwards, {dt:.1f} s; weight init {t_init:.1f} s excluded)"}


def run_configs(args):
    """BASELINE configs 3a (GPTQ + prefix caching), 3b (INT8 + continuous
    batching, ragged batch 64) and 4 (speculative decoding, 1B draft + 8B
    target, k=4) on one GPU, through the C ABI. One JSON line per config, each
    with its roofline (the algorithmic floor: HBM bytes / measured HBM peak +
    prefill FLOPs / tensor peak, against the measured time) and the CPU
    oracle's rate on a bounded sample of the same arithmetic."""
    import numpy as np
    import torch
    from paper_2605_23057_b200 import MODE_FP16, MODE_GPTQ_PC, MODE_INT8_CB, MODE_SPEC, engine_cfg
    from paper_2605_23057_b200.configs import model_cfg
    from paper_2605_23057_b200.engine import Engine
    torch.cuda.set_device(0)
    eng = Engine(engine_cfg(target="llama8b", draft="llama1b", seed=0, kv_blocks=6144, max_batch=64,
                            max_seq_len=2400, use_graphs=True))
    c8, c1 = model_cfg("llama8b"), model_cfg("llama1b")
    hbm, _ = peaks()
    kvp = kv_bytes_per_pos(c8)
    rng = np.random.default_rng(7)
    cpu = not args.no_cpu_baseline
    base = {"metric": "decode tokens/s per mode and routed mix (1/2/4/8 B200); mean latency vs FP16 mode",
            "unit": "tokens/s", "n_gpus": 1, "data": "synthetic"}
    # 3a: shared-prefix chat, 1024+-10% prompts with a shared 768-token prefix, 128+-10% outputs
    shared = synth_prompt(99, 768, 128256)
    n_req = args.cfg_requests
    eng.reset_prefix_cache()
    wb4 = eng.weight_bytes(2)
    tot_tok, tot_ms, dec_ms, pre_ms, hits, floor_dec, floor_pre = 0, 0.0, 0.0, 0.0, 0, 0.0, 0.0
    tp16, _ = tensor_peak("f16")
    for i in range(n_req):
        plen = int(round(1024 * (0.9 + 0.2 * rng.random())))
        p = np.concatenate([shared, synth_prompt(1000 + i, plen - 768, 128256)])
        out = int(round(128 * (0.9 + 0.2 * rng.random())))
        r = eng.run(MODE_GPTQ_PC, p, out)
        tot_tok += out
        tot_ms += r.total_ms
        dec_ms += r.decode_ms
        pre_ms += r.prefill_ms
        hits += r.prefix_hit_tokens
        sfx = plen - r.prefix_hit_tokens
        floor_pre += prefill_flops(c8, sfx, r.prefix_hit_tokens) / (tp16 * 1e12) * 1e3
        floor_dec += sum(wb4 + (plen + j) * kvp for j in range(out - 1)) / (hbm * 1e9) * 1e3
    line = dict(base, config="3a_gptq_prefix_caching", value=tot_tok / (tot_ms / 1e3),
                requests=n_req, prefix_hit_tokens=hits, mean_request_ms=tot_ms / n_req,
                decode_tok_s=(tot_tok - n_req) / (dec_ms / 1e3),
                roofline={"bound": "hbm (decode) + tensor (suffix prefill)",
                          "decode_frac": floor_dec / dec_ms, "prefill_frac": floor_pre / pre_ms,
                          "request_frac": (floor_dec + floor_pre) / tot_ms,
                          "peaks": {"hbm_gbs": hbm, "tensor_tflops": tp16}})
    if cpu:
        line["cpu_baseline"] = cpu_mode_sample(2, new_tokens=27)
    print(json.dumps(line), flush=True)
    # 3b: 64 co-scheduled requests, prompts 1024+-10%, outputs 128+-10%, INT8 + continuous batching
    prompts, outs = [], []
    for i in range(64):
        plen = int(round(1024 * (0.9 + 0.2 * rng.random())))
        prompts.append(synth_prompt(2000 + i, plen, 128256))
        outs.append(int(round(128 * (0.9 + 0.2 * rng.random()))))
    eng.run_batch(MODE_INT8_CB, prompts[:4], [4] * 4)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = eng.run_batch(MODE_INT8_CB, prompts, outs)
    wall = time.perf_counter() - t0
    wb8 = eng.weight_bytes(1)
    tpi8, i8src = tensor_peak("int8")
    pre_wall = max(r.prefill_ms for r in res)  # one packed admission prefill of all 64
    steps = max(outs) - 1
    dec_bytes = 0.0
    for s_ in range(1, steps + 1):  # step s: every sequence with more than s tokens to emit
        live = [len(pr) + s_ for pr, o in zip(prompts, outs) if o > s_]
        dec_bytes += wb8 + sum(live) * kvp
    floor_pre = sum(prefill_flops(c8, len(pr)) for pr in prompts) / (tpi8 * 1e12) * 1e3
    floor_dec = dec_bytes / (hbm * 1e9) * 1e3
    line = dict(base, config="3b_int8_continuous_batching_b64", value=sum(outs) / wall,
                requests=64, generated_tokens=sum(outs), wall_s=wall, prefill_ms=pre_wall,
                decode_ms=wall * 1e3 - pre_wall,
                mean_request_ms=statistics.mean(r.total_ms for r in res),
                roofline={"bound": "tensor (packed 64 x ~1024 prefill) + hbm (decode steps: INT8 "
                                   "weights + every live sequence's KV)",
                          "prefill_floor_ms": floor_pre, "decode_floor_ms": floor_dec,
                          "prefill_frac": floor_pre / pre_wall,
                          "decode_frac": floor_dec / max(1e-9, wall * 1e3 - pre_wall),
                          "frac": (floor_pre + floor_dec) / (wall * 1e3),
                          "peaks": {"hbm_gbs": hbm, "int8_tops": tpi8, "int8_source": i8src}})
    if cpu:
        line["cpu_baseline"] = cpu_mode_sample(1, new_tokens=57)
    print(json.dumps(line), flush=True)
    # 4: speculative decoding on long generations (SyntheticSL-shape prompt, 1024 new tokens),
    # against FP16 batch-1 on the same requests
    wb16, wbd = eng.weight_bytes(0), 2 * linear_params(c1)
    tot_tok, tot_dec, tot16, prop, acc, rounds = 0, 0.0, 0.0, 0, 0, 0
    for i in range(args.cfg_requests // 4 or 1):
        p = synth_prompt(3000 + i, 128, 128256)
        r = eng.run(MODE_SPEC, p, 1024)
        r16 = eng.run(MODE_FP16, p, 1024)
        assert np.array_equal(r.tokens, r16.tokens), "speculative tokens != FP16 greedy tokens"
        tot_tok += 1023
        tot_dec += r.decode_ms
        tot16 += r16.decode_ms
        prop += r.spec_proposed
        acc += r.spec_accepted
        rounds += r.spec_rounds
    k = 4
    # per round: the draft's k forwards (T=2 catch-up + k-1 steps) and one target verify of k+1 tokens
    floor = rounds * (k * wbd + wb16) / (hbm * 1e9) * 1e3
    line = dict(base, config="4_speculative_k4", value=tot_tok / (tot_dec / 1e3),
                acceptance=acc / max(1, prop), rounds=rounds,
                tokens_per_round=tot_tok / max(1, rounds), fp16_tok_s=tot_tok / (tot16 / 1e3),
                speedup_vs_fp16=tot16 / tot_dec, draft="llama1b-shape", target="llama8b-shape",
                roofline={"bound": "hbm", "bytes_per_round": k * wbd + wb16,
                          "frac": floor / tot_dec, "peak_gbs": hbm,
                          "token_ceiling_tok_s": tot_tok / (floor / 1e3)})
    if cpu:
        line["cpu_baseline"] = cpu_mode_sample(4, prompt_len=4, new_tokens=16, draft="llama1b")
    print(json.dumps(line), flush=True)
    eng.close()


def run_profile(args):
    """Measured B200 profile in the reference's load_profile schema:
    every family's nominal request in every mode, 8B target + 1B draft, written
    to --profile-out. Prints one JSON line summarising it."""
    import torch
    from paper_2605_23057_b200 import ALL_MODES, engine_cfg
    from paper_2605_23057_b200.configs import MODE_FP16
    from paper_2605_23057_b200.engine import Engine
    from paper_2605_23057_b200.profile_writer import build_profile, measure, write_profile
    _, rank, local = _dist()
    if rank != 0:
        return
    torch.cuda.set_device(local)
    eng = Engine(engine_cfg(target="llama8b", draft="llama1b", modes=ALL_MODES, seed=0,
                            kv_blocks=1024, max_batch=8, max_seq_len=2048 + 512), device=local)
    t0 = time.perf_counter()
    meas = measure(eng, device=local, out_cap=args.profile_out_cap)
    fp16 = [m for (mode, _), m in meas.items() if mode == MODE_FP16]
    e16 = [m["energy_j_per_token"] for m in fp16 if m["energy_j_per_token"]]
    prof = build_profile(meas, statistics.mean(e16) if e16 else 0.0,
                         max(m["mem_bytes"] for m in fp16) / 2**20)
    write_profile(args.profile_out, prof)
    eng.close()
    print(json.dumps({"workload": "profile", "out": args.profile_out, "cells": len(prof["cells"]),
                      "baseline_costs": prof["baseline_costs"], "wall_s": time.perf_counter() - t0}),
          flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", choices=["decode8b", "mix", "configs", "profile"], default="decode8b")
    ap.add_argument("--profile-out", default="profiles/b200_profile.json")
    ap.add_argument("--decisions-out", default="", help="mix: write the reference-format decisions CSV")
    ap.add_argument("--profile-out-cap", type=int, default=0, help="cap generated tokens per request")
    ap.add_argument("--cfg-requests", type=int, default=8)
    ap.add_argument("--mix-per-class", type=int, default=4)
    ap.add_argument("--prefix-groups", type=int, default=8, help="mix: shared-prefix groups")
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "mix":
        run_mix(args)
    elif args.workload == "configs":
        run_configs(args)
    elif args.workload == "profile":
        run_profile(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
