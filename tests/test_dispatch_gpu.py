"""Request-sharded multi-process execution with the real engine,
on the one GPU the box has: two ranks (gloo, 127.0.0.1) each create their own
engine replica on cuda:0, execute their shard of a mixed routed trace through
the C++ executor (dispatch.shard_trace: cohorts whole, prefix groups sticky,
LPT on the measured cost model), and gather the rows. Per request the
gathered rows equal a single-process execution of the whole trace in every
deterministic field (routing, executed mode, output length, speculative
rounds, prefix-cache hits); latencies are measured and not compared."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_23057_b200 import controller as ctl

pytestmark = pytest.mark.gpu

FIELDS = ("mode", "reason", "executed_mode", "family", "prompt_tokens", "output_tokens",
          "fallback_used", "spec_proposed", "spec_accepted", "prefix_hit_tokens")
OPTS = dict(max_output_tokens=12, prefix_len=48, prefix_groups=2)


def _trace():
    counts = {"SyntheticSS": 3, "SyntheticSL": 2, "GSM8K": 2, "SharedPrefixChat": 4,
              "MemoryPressureLongContext": 2, "TruthfulQA": 2}
    return ctl.generate_trace(counts, jitter=0.1, seed=11, batched_fraction=0.3, batch_pressure=3)


def _engine():
    from paper_2605_23057_b200 import engine_cfg
    from paper_2605_23057_b200.engine import Engine
    return Engine(engine_cfg(target="tiny", draft="tiny_draft", seed=5, kv_blocks=1024,
                             max_seq_len=2600), device=0)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_23057_b200.dispatch import shard_trace
    from paper_2605_23057_b200.engine import execute_trace
    text = _trace()
    lines = [l for l in text.splitlines() if l.strip()]
    idx = shard_trace(text, world, prefix_groups=OPTS["prefix_groups"])[rank]
    eng = _engine()
    rows = {}
    if idx:
        out, _ = execute_trace(eng, "".join(lines[i] + "\n" for i in idx), **OPTS)
        rows = {i: {f: r[f] for f in FIELDS} for i, r in zip(idx, out)}
    eng.close()
    gathered = [None] * world
    dist.all_gather_object(gathered, rows)
    if rank == 0:
        merged = {}
        for g in gathered:
            merged.update(g)
        q.put(merged)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_engine_shards_match_single_process(cuda_ok):
    from paper_2605_23057_b200.engine import execute_trace
    text = _trace()
    eng = _engine()
    ref, _ = execute_trace(eng, text, **OPTS)
    eng.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert sorted(merged) == list(range(len(ref)))
    for i, r in enumerate(ref):
        assert merged[i] == {f: r[f] for f in FIELDS}, f"request {i}"
    assert any(r["prefix_hit_tokens"] > 0 for r in ref)
    assert any(r["spec_proposed"] > 0 for r in ref)
