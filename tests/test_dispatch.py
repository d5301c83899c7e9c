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
from paper_2605_23057_b200.dispatch import CB_MODE, PC_MODE, aggregate_rows, rank_trace, shard_trace

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
