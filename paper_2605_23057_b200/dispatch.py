"""Multi-GPU request dispatch: one full engine replica per GPU,
requests sharded across ranks with no data-path collective.

Placement (shard_trace), over the trace as routed by the reference RulePolicy:
  * an INT8 + continuous-batching cohort (a maximal run of consecutive
    int8_continuous_batching-routed requests, the executor's cohort rule) goes
    whole to one GPU;
  * shared-prefix requests (gptq_prefix_caching) of one prefix group go to one
    GPU, so prefix-cache hits stay on the GPU that holds the cached blocks.
    The group of a request is FNV-1a-64(request_id) mod prefix_groups, the
    executor's rule (executor.hpp prefix_group);
  * units (cohorts, prefix groups, single requests) are placed longest
    predicted time first on the GPU with the least predicted work (LPT), ties
    to the lowest rank.
Predicted time is the reference's own cost model (fp16_latency, profile.cpp:
281-291, divided by the (mode, family) cell's latency_speedup, sim.cpp:
132-135) evaluated on a B200-MEASURED profile in the reference schema
(profiles/r02_b200_profile.json: FP16 2.75 ms per decode token and 0.021 ms per
prefill token, against the reference's A100-derived 11.5 / 0.4). A cohort runs
its members concurrently, so its time is its slowest member's.
Each rank keeps its requests in trace order. Results are gathered back and
aggregated exactly like the reference's summarize (sim.cpp:149-207): mean of
per-request speedups, per-family means, the collapsed mean of family means,
sum(fp16) / sum(mode), over ALL requests in trace order (aggregate_rows)."""
from __future__ import annotations

import json
import os
import statistics

from . import controller as ctl

CB_MODE = "int8_continuous_batching"
PC_MODE = "gptq_prefix_caching"
DEFAULT_PROFILE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                               "profiles", "r02_b200_profile.json")


class CostModel:
    """Predicted request time on one B200: fp16_latency(costs, request) /
    latency_speedup(mode, family) from a profile in the reference's
    load_profile schema (baseline_costs + cells)."""

    def __init__(self, profile: dict):
        b = profile["baseline_costs"]
        self.fixed = float(b.get("fixed_overhead_ms", 0.0))
        self.prefill = float(b["prefill_ms_per_token"])
        self.decode = float(b["decode_ms_per_token"])
        self.speedup = {(c["mode"], c["family"]): float(c["latency_speedup"])
                        for c in profile["cells"] if c.get("feasible", True)}

    @classmethod
    def load(cls, path: str | None = None) -> "CostModel":
        with open(path or DEFAULT_PROFILE) as f:
            return cls(json.load(f))

    def fp16_ms(self, d: dict) -> float:
        return self.fixed + self.prefill * d["prompt_tokens"] + self.decode * d["expected_output_tokens"]

    def mode_ms(self, d: dict, mode: str, family: str) -> float:
        return self.fp16_ms(d) / self.speedup.get((mode, family), 1.0)


def prefix_group(request_id: str, groups: int) -> int:
    """FNV-1a-64(request_id) mod groups: the executor's rule."""
    if groups <= 1:
        return 0
    h = 0xCBF29CE484222325
    for c in request_id.encode():
        h = ((h ^ c) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h % groups


def plan_units(ndjson: str, cost: CostModel | None = None, prefix_groups: int = 1):
    """Placement units of a routed trace: (indices, predicted ms, kind)."""
    cost = cost or CostModel.load()
    lines = [l for l in ndjson.splitlines() if l.strip()]
    routes = ctl.route_ndjson("\n".join(lines) + "\n")
    descs = [ctl.parse_trace_line(l) for l in lines]
    ms = [cost.mode_ms(d, r["mode"], r["family"]) for d, r in zip(descs, routes)]
    units, groups = [], {}
    i = 0
    while i < len(lines):
        mode = routes[i]["mode"]
        if mode == CB_MODE:  # cohort: maximal run of CB-routed requests, members concurrent
            j = i + 1
            while j < len(lines) and routes[j]["mode"] == CB_MODE:
                j += 1
            units.append((list(range(i, j)), max(ms[i:j]), "cohort"))
            i = j
            continue
        if mode == PC_MODE:
            g = prefix_group(descs[i]["request_id"], prefix_groups)
            groups.setdefault(g, []).append(i)
        else:
            units.append(([i], ms[i], "single"))
        i += 1
    for g, idxs in sorted(groups.items()):
        units.append((idxs, sum(ms[k] for k in idxs), f"prefix-group-{g}"))
    return units


def shard_trace(ndjson: str, world: int, cost: CostModel | None = None,
                prefix_groups: int = 1) -> list[list[int]]:
    """Indices (into the trace's non-empty lines) each rank executes, in trace order."""
    if world < 1:
        raise ValueError("world must be >= 1")
    units = plan_units(ndjson, cost, prefix_groups)
    load = [0.0] * world
    assign: list[list[int]] = [[] for _ in range(world)]
    # longest predicted time first; stable on trace position for equal costs
    for idxs, t, _ in sorted(units, key=lambda u: (-u[1], u[0][0])):
        r = min(range(world), key=lambda q: (load[q], q))
        assign[r].extend(idxs)
        load[r] += t
    return [sorted(a) for a in assign]


def predicted_load(ndjson: str, shards: list[list[int]], cost: CostModel | None = None,
                   prefix_groups: int = 1) -> list[float]:
    """Predicted ms per rank for a placement (cohorts count once, at their slowest member)."""
    owner = {i: r for r, s in enumerate(shards) for i in s}
    load = [0.0] * len(shards)
    for idxs, t, _ in plan_units(ndjson, cost, prefix_groups):
        load[owner[idxs[0]]] += t
    return load


def rank_trace(ndjson: str, world: int, rank: int, prefix_groups: int = 1) -> str:
    lines = [l for l in ndjson.splitlines() if l.strip()]
    idx = shard_trace(ndjson, world, prefix_groups=prefix_groups)[rank]
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
