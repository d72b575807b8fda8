"""oserve::search (proj/include/oserve/deploysearch.hpp) on the GPU path.

Same names, argument meaning and exceptions as the reference:

    evaluate_deployment(dep, ctx)                deploysearch.cpp:138-151
    best_strategies(sizes, ctx)                  deploysearch.cpp:153-229
    exhaustive(cluster, model, types, span, span_seconds, params, parallel)
                                                 deploysearch.cpp:436-466
    min_feasible_group(cluster, model)           deploysearch.cpp:77-87

plus the full-space round the reference cannot run at D >= 64:

    scheduling_round(ctx, mode, sizes)           SURVEY §8d (configs 2, 3, 5)

Every call goes through include/oserve_gpu.h into the sm_100a kernels.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

from . import _abi as A
from . import core
from ._native import GpuContext


@dataclass
class EvalContext:
    """deploysearch.hpp:45-54 (the GPU context owns copies, never references)."""
    cluster: core.ClusterSpec
    model: core.ModelSpec
    types: List[core.WorkloadType]
    span: core.TraceSpan
    span_seconds: float
    params: core.ProfileParams = field(default_factory=core.ProfileParams)
    parallel: bool = True
    device: int = 0

    def gpu(self) -> GpuContext:
        key = (id(self.cluster), id(self.model), self.device)
        g = _CTX_CACHE.get(key)
        if g is None or g.cluster is not self.cluster or g.model is not self.model or g.params != self.params:
            g = GpuContext(self.cluster, self.model, self.params, self.device)
            _CTX_CACHE[key] = g
        g.set_workload(self.types, self.span.counts, self.span_seconds)
        return g


_CTX_CACHE: Dict[Tuple[int, int, int], GpuContext] = {}


def min_feasible_group(cluster: core.ClusterSpec, model: core.ModelSpec, device: int = 0) -> int:
    return GpuContext(cluster, model, device=device).min_feasible_group()


def evaluate_deployment(dep: core.Deployment, ctx: EvalContext) -> int:
    if not dep.replicas:
        return 0
    return ctx.gpu().evaluate_deployments([dep])[0]


def best_strategies(sizes: Sequence[int], ctx: EvalContext) -> core.StrategyChoice:
    return ctx.gpu().best_strategies(list(sizes))


def exhaustive(cluster: core.ClusterSpec, model: core.ModelSpec, types: Sequence[core.WorkloadType],
               span: core.TraceSpan, span_seconds: float, params: Optional[core.ProfileParams] = None,
               parallel: bool = True, device: int = 0) -> core.SearchState:
    g = GpuContext(cluster, model, params or core.ProfileParams(), device)
    g.set_workload(list(types), span.counts, span_seconds)
    return g.exhaustive()


def search(cluster: core.ClusterSpec, model: core.ModelSpec, types: Sequence[core.WorkloadType],
           span: core.TraceSpan, span_seconds: float, params: Optional[core.ProfileParams] = None,
           seed: int = 0, max_iters: int = 500, stale_limit: int = 20, mutation_retries: int = 8,
           warm_start: Optional[core.Deployment] = None, device: int = 0):
    """search::search (deploysearch.cpp:341-417): flow-guided mutate / enumerate
    / revert loop; returns (SearchState, log rows (iteration, op, accepted,
    throughput, devices))."""
    g = GpuContext(cluster, model, params or core.ProfileParams(), device)
    g.set_workload(list(types), span.counts, span_seconds)
    return g.search(seed, max_iters, stale_limit, mutation_retries, warm_start)


def scheduling_round(ctx: EvalContext, mode: int = A.SPACE_ORDERED, sizes: Sequence[int] = ()) -> core.SearchState:
    """Argmin over a whole plan space (no D <= 16 guard)."""
    return ctx.gpu().round(mode, list(sizes))
