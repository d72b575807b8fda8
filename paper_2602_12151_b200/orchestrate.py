"""Workload-adaptive re-scheduling over time windows (BASELINE config 4).

Follows the reference's per-window loop `orch::build_adaptive_timeline`
(orchestrate.cpp:94-154) with the GPU scheduling round in place of the
heuristic `search()`:

    for each window w:
        lambda_w = Holt forecast (orchestrate.cpp:75-92; committed in cfg4.json)
        skip if lambda_w == lambda_{w-1}                          (:113)
        found    = full-space GPU round at lambda_w               (K0 + K1)
                   with topk=K: the exact K best plans (packed keys on the
                   device) and the switching batch current -> each of them
                   (K2 key mode, one CTA per pair) — SURVEY §8d config 4
        keep rule: keep current iff found <= keep_obj*(1+min_gain)  (:126-134)
        x        = assignment of the chosen deployment            (:137, K1 detail)
        if the deployment changed: greedy switch plan + estimate  (:141-145, K2)
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

from . import _abi as A
from . import core
from ._native import GpuContext


@dataclass
class TimelineEntry:
    """sim::TimelineEntry (sim.hpp) fields the round produces."""
    span_index: int
    deployment: core.Deployment
    assignment: List[List[int]]
    objective: int
    switch: Optional[core.SwitchPlan] = None
    switch_seconds: float = 0.0
    round_objective: int = 0        # the round's best objective at this window
    kept: bool = False              # keep rule retained the current deployment
    window: int = 0                 # window index (span) this decision was made at


@dataclass
class WindowStat:
    """Per-window record of the round strategy (every evaluated window)."""
    window: int
    seconds: float                  # wall clock of the window's GPU work (synchronous calls)
    round_objective: int = 0
    candidate_keys: List[int] = field(default_factory=list)              # top-K packed keys, best first
    candidate_switch_seconds: List[float] = field(default_factory=list)  # current -> candidate (K2)


@dataclass
class Timeline:
    entries: List[TimelineEntry] = field(default_factory=list)
    windows: int = 0
    rounds: int = 0
    stats: List[WindowStat] = field(default_factory=list)


def build_adaptive_timeline(ctx: GpuContext, types: Sequence[core.WorkloadType], forecasts: Sequence[Sequence[int]],
                            span_seconds: float = 60.0, min_gain: float = 0.01, mode: int = A.SPACE_ORDERED,
                            sizes: Sequence[int] = (), strategy: str = "round", seed: int = 0,
                            search_max_iters: int = 150, search_stale_limit: int = 20, topk: int = 0) -> Timeline:
    """strategy="round": full-space GPU round per window (SURVEY config 4);
    topk=K > 0 also keeps the exact K best plans of every window and costs the
    switch from the current deployment to each of them (K2 batch).
    strategy="search": the reference's own loop exactly — warm-started
    search::search per window (orchestrate.cpp:116-123) on the GPU path."""
    tl = Timeline(windows=len(forecasts))
    current: Optional[core.Deployment] = None
    prev_lam: Optional[List[int]] = None
    prev_x: Optional[List[List[int]]] = None
    d_keys = None
    prepared = False
    if topk and strategy != "search":
        import torch  # device memory for the key list (plumbing)
        d_keys = torch.empty(int(topk), dtype=torch.int64, device=f"cuda:{ctx.device}")
    for w, lam in enumerate(forecasts):
        lam = [int(v) for v in lam]
        if tl.entries and lam == prev_lam:
            continue  # workload unchanged (orchestrate.cpp:113)
        t0 = time.perf_counter()
        ctx.set_workload(types, lam, span_seconds)
        stat = WindowStat(w, 0.0)
        if strategy == "search":
            found, _ = ctx.search(seed=seed, max_iters=search_max_iters, stale_limit=search_stale_limit,
                                  warm_start=current)
        elif d_keys is not None:
            if not prepared:  # the space does not depend on the workload (exact flags and key bits follow it)
                ctx.prepare_space(mode, list(sizes))
                prepared = True
            ctx.round_topk(int(topk), d_keys.data_ptr())
            keys = [int(k) & ((1 << 64) - 1) for k in d_keys.cpu().tolist()]
            found = ctx.decode_key(keys[0])
            stat.candidate_keys = keys
            if current is not None:
                stat.candidate_switch_seconds = ctx.switch_cost_keys(current, d_keys.data_ptr(), int(topk))[0]
        else:
            found = ctx.round(mode, list(sizes))
        stat.round_objective = found.throughput
        tl.rounds += 1
        chosen, kept = found.deployment, False
        if current is not None:
            keep_obj = ctx.evaluate_deployments([current])[0]
            if float(found.throughput) <= float(keep_obj) * (1.0 + min_gain):
                chosen, kept = current, True
        _, lower = ctx.plan_detail(chosen)
        x = lower.assignment.x
        same = current is not None and _same(chosen, current)
        if not tl.entries:
            tl.entries.append(TimelineEntry(w, chosen, x, lower.assignment.objective, None, 0.0,
                                            found.throughput, kept, w))
        elif not same:
            plan = ctx.switch_plan(current, chosen)
            tl.entries.append(TimelineEntry(w, chosen, x, lower.assignment.objective, plan, plan.est_seconds,
                                            found.throughput, kept, w))
        elif x != prev_x:
            tl.entries.append(TimelineEntry(w, chosen, x, lower.assignment.objective, None, 0.0,
                                            found.throughput, kept, w))
        stat.seconds = time.perf_counter() - t0
        tl.stats.append(stat)
        current, prev_lam, prev_x = chosen, lam, x
    return tl


def adaptive_timeline(ctx: GpuContext, types: Sequence[core.WorkloadType], actual: Sequence[Sequence[int]],
                      window: int = 50, **kw) -> Timeline:
    """orch::build_adaptive_timeline entry point over observed per-span
    counts: Holt forecasts (forecast_series, orchestrate.cpp:75-92, host
    C++ in liboserve_gpu) feed the per-window loop above."""
    from ._native import forecast_series
    return build_adaptive_timeline(ctx, types, forecast_series(actual, window), **kw)


def _same(a: core.Deployment, b: core.Deployment) -> bool:
    return [(sorted(r.device_ids), r.tp, r.pp) for r in a.replicas] == \
        [(sorted(r.device_ids), r.tp, r.pp) for r in b.replicas]
