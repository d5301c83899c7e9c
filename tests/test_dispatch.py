"""Multi-GPU request dispatch on CPU: placement invariants of
shard_trace, and the N > 1 path with world_size 2 over gloo (127.0.0.1): each
rank executes its shard (a deterministic stand-in for the engine, no GPU), rows
are gathered, and the aggregate equals the single-process summary; the timing
reduction is the max over ranks."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_23057_b200 import controller as ctl
from paper_2605_23057_b200.dispatch import (CB_MODE, PC_MODE, CostModel, aggregate_rows, predicted_load,
                                            prefix_group, rank_trace, shard_trace)

COUNTS = {"SyntheticSS": 6, "SyntheticSL": 4, "GSM8K": 4, "SharedPrefixChat": 5,
          "MemoryPressureLongContext": 3, "TruthfulQA": 4}


def _trace():
    return ctl.generate_trace(COUNTS, jitter=0.1, seed=7, batched_fraction=0.5, batch_pressure=4)


def _fake_row(i, line):
    d = ctl.parse_trace_line(line)
    r = ctl.route(d)
    fam = ctl.FAMILIES.index(r["family"])
    fp16 = 10.0 + 0.01 * d["prompt_tokens"] + 0.5 * d["expected_output_tokens"]
    mode = fp16 / (1.1 + 0.05 * (i % 7))
    return {"family": fam, "speedup": fp16 / mode, "fp16_latency_ms": fp16, "mode_latency_ms": mode,
            "fallback_used": 0, "output_tokens": d["expected_output_tokens"]}


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_placement_invariants(world):
    text = _trace()
    lines = [l for l in text.splitlines() if l.strip()]
    routes = ctl.route_ndjson(text)
    shards = shard_trace(text, world)
    flat = sorted(i for s in shards for i in s)
    assert flat == list(range(len(lines)))  # every request exactly once
    owner = {i: r for r, s in enumerate(shards) for i in s}
    for s in shards:
        assert s == sorted(s)  # trace order within a rank
    # CB cohorts (maximal runs of CB-routed requests) whole on one rank
    i = 0
    n_cohorts = 0
    while i < len(lines):
        if routes[i]["mode"] == CB_MODE:
            j = i
            while j < len(lines) and routes[j]["mode"] == CB_MODE:
                j += 1
            assert len({owner[k] for k in range(i, j)}) == 1
            n_cohorts += 1
            i = j
        else:
            i += 1
    assert n_cohorts > 0
    # the shared-prefix group is sticky
    pc = [i for i in range(len(lines)) if routes[i]["mode"] == PC_MODE]
    assert pc and len({owner[i] for i in pc}) == 1


def _deploy_mix(per_class):
    """BASELINE config 5 (bench.py deploy_mix_trace): short interactive, long
    generation, shared-prefix chat and 8K long-context requests, tagged."""
    counts = {"SyntheticSS": per_class, "SyntheticSL": per_class, "GSM8K": per_class,
              "SharedPrefixChat": per_class, "MemoryPressureLongContext": per_class}
    out = []
    for line in ctl.generate_trace(counts, jitter=0.10, seed=7).splitlines():
        d = ctl.parse_trace_line(line)
        if d["workload_tag"] == "MemoryPressureLongContext":
            d["prompt_tokens"] *= 4
        out.append(ctl.format_trace_line(d))
    return "\n".join(out) + "\n"


@pytest.mark.parametrize("world", [2, 4, 8])
def test_config5_predicted_time_balanced(world):
    """On the config-5 deployment mix (64 per class), the B200-measured cost
    model places work so that every GPU's predicted time is within 10% of the
    mean (8 prefix groups, so shared-prefix traffic is not one indivisible unit)."""
    text = _deploy_mix(64)
    cm = CostModel.load()
    shards = shard_trace(text, world, cm, prefix_groups=8)
    load = predicted_load(text, shards, cm, prefix_groups=8)
    mean = sum(load) / world
    assert max(load) <= 1.10 * mean, (load, mean)


def test_prefix_groups_are_sticky_and_spread():
    text = _deploy_mix(16)
    lines = [l for l in text.splitlines() if l.strip()]
    routes = ctl.route_ndjson(text)
    shards = shard_trace(text, 4, prefix_groups=4)
    owner = {i: r for r, s in enumerate(shards) for i in s}
    groups = {}
    for i, l in enumerate(lines):
        if routes[i]["mode"] == PC_MODE:
            groups.setdefault(prefix_group(ctl.parse_trace_line(l)["request_id"], 4), set()).add(owner[i])
    assert len(groups) == 4 and all(len(v) == 1 for v in groups.values())
    assert len({next(iter(v)) for v in groups.values()}) > 1  # groups land on different GPUs
    assert prefix_group("SharedPrefixChat-0", 1) == 0


def test_cost_model_is_the_reference_formula():
    cm = CostModel.load()
    d = {"prompt_tokens": 1000, "expected_output_tokens": 100}
    assert cm.fp16_ms(d) == pytest.approx(cm.fixed + cm.prefill * 1000 + cm.decode * 100)
    sp = cm.speedup[("gptq4", "SyntheticSS")]
    assert cm.mode_ms(d, "gptq4", "SyntheticSS") == pytest.approx(cm.fp16_ms(d) / sp)
    assert cm.decode > 10 * cm.prefill  # a decode token costs far more than a prefill token on B200


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    text = _trace()
    lines = [l for l in text.splitlines() if l.strip()]
    idx = shard_trace(text, world)[rank]
    mine = rank_trace(text, world, rank)
    assert [l for l in mine.splitlines()] == [lines[i] for i in idx]
    rows = {i: _fake_row(i, lines[i]) for i in idx}
    gathered = [None] * world
    dist.all_gather_object(gathered, rows)
    t = torch.tensor([float(sum(r["mode_latency_ms"] for r in rows.values()))], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        merged = {}
        for g in gathered:
            merged.update(g)
        q.put((aggregate_rows(merged), t.item()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_dispatch_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    agg, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    text = _trace()
    lines = [l for l in text.splitlines() if l.strip()]
    ref = aggregate_rows({i: _fake_row(i, l) for i, l in enumerate(lines)})
    assert agg == ref
    shards = shard_trace(text, 2)
    per_rank = [sum(_fake_row(i, lines[i])["mode_latency_ms"] for i in s) for s in shards]
    assert tmax == pytest.approx(max(per_rank))
