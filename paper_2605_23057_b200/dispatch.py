"""Multi-GPU request dispatch: one full engine replica per GPU,
requests sharded across ranks with no data-path collective.

Placement (shard_trace), over the trace as routed by the reference RulePolicy:
  * an INT8 + continuous-batching cohort (a maximal run of consecutive
    int8_continuous_batching-routed requests, the executor's cohort rule) goes
    whole to one GPU;
  * shared-prefix requests (gptq_prefix_caching) are sticky per prefix group, so
    prefix-cache hits stay on the GPU that holds the cached blocks (the
    executor keys every SharedPrefixChat request to one group);
  * everything else goes to the GPU with the fewest outstanding tokens
    (prompt + expected output), ties to the lowest rank.
Each rank keeps its requests in trace order. Results are gathered back and
aggregated exactly like the reference's summarize (sim.cpp:149-207): mean of
per-request speedups, per-family means, the collapsed mean of family means,
sum(fp16) / sum(mode), over ALL requests in trace order (aggregate_rows)."""
from __future__ import annotations

import statistics

from . import controller as ctl

CB_MODE = "int8_continuous_batching"
PC_MODE = "gptq_prefix_caching"


def shard_trace(ndjson: str, world: int) -> list[list[int]]:
    """Indices (into the trace's non-empty lines) each rank executes, in trace order."""
    lines = [l for l in ndjson.splitlines() if l.strip()]
    if world < 1:
        raise ValueError("world must be >= 1")
    routes = ctl.route_ndjson("\n".join(lines) + "\n")
    descs = [ctl.parse_trace_line(l) for l in lines]
    units, i = [], 0
    while i < len(lines):  # cohorts: maximal runs of CB-routed requests
        j = i + 1
        if routes[i]["mode"] == CB_MODE:
            while j < len(lines) and routes[j]["mode"] == CB_MODE:
                j += 1
        units.append(list(range(i, j)))
        i = j
    load = [0] * world
    assign: list[list[int]] = [[] for _ in range(world)]
    group_owner: dict[str, int] = {}
    for idxs in units:
        tokens = sum(descs[k]["prompt_tokens"] + descs[k]["expected_output_tokens"] for k in idxs)
        r = min(range(world), key=lambda q: (load[q], q))
        if routes[idxs[0]]["mode"] == PC_MODE:
            key = "prefix-group-0"  # the executor's single SharedPrefixChat group
            r = group_owner.setdefault(key, r)
        assign[r].extend(idxs)
        load[r] += tokens
    return [sorted(a) for a in assign]


def rank_trace(ndjson: str, world: int, rank: int) -> str:
    lines = [l for l in ndjson.splitlines() if l.strip()]
    idx = shard_trace(ndjson, world)[rank]
    return "".join(lines[i] + "\n" for i in idx)


def aggregate_rows(rows_by_index: dict[int, dict]) -> dict:
    """The reference summarize (sim.cpp:149-207) over every request, trace order."""
    rows = [rows_by_index[i] for i in sorted(rows_by_index)]
    if not rows:
        return {"request_count": 0}
    fam: dict[int, list[float]] = {}
    for r in rows:
        fam.setdefault(r["family"], []).append(r["speedup"])
    fam_means = {f: statistics.fmean(v) for f, v in fam.items()}
    return {
        "request_count": len(rows),
        "mean_speedup": statistics.fmean(r["speedup"] for r in rows),
        "aggregate_latency_speedup": sum(r["fp16_latency_ms"] for r in rows)
        / sum(r["mode_latency_ms"] for r in rows),
        "collapsed_mean_speedup": statistics.fmean(fam_means[f] for f in sorted(fam_means)),
        "per_family_mean_speedup": {ctl.FAMILIES[f]: fam_means[f] for f in sorted(fam_means)},
        "fallback_count": sum(int(r["fallback_used"]) for r in rows),
        "generated_tokens": sum(r["output_tokens"] for r in rows),
        "mode_time_ms": sum(r["mode_latency_ms"] for r in rows),
    }
