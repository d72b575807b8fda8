"""oserve::cost on the GPU path (costmodel.hpp).

  build_capacity_table(dep, types, model, cluster, params, span_s)
      costmodel.cpp:94-116: the (replica, class) cells n/e/latency of one
      deployment from the K0 cost tables (cells bit-identical to the
      reference; `GpuContext.plan_detail`).
  build_capacity_tables(deps, ...)
      the same for many deployments against one context (one K0 upload).

Contexts are cached per (cluster, model, params, device) and the workload
(class centroids, span) is re-uploaded only when it changes, like the C++
shim's `cached_context` (include/oserve_gpu.hpp).
"""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence

from . import core
from ._native import GpuContext

_cache: Dict[tuple, list] = {}  # key -> [context, workload key]


def _ctx(types: Sequence[core.WorkloadType], model: core.ModelSpec, cluster: core.ClusterSpec,
         params: core.ProfileParams, span_s: float, device: int) -> GpuContext:
    key = (repr(cluster), repr(model), repr(params), device)
    ent = _cache.get(key)
    if ent is None:
        if len(_cache) > 8:
            _cache.pop(next(iter(_cache)))
        ent = _cache[key] = [GpuContext(cluster, model, params, device), None]
    wkey = (repr(list(types)), float(span_s))
    if ent[1] != wkey:  # the cells do not depend on the demand counts
        ent[0].set_workload(list(types), [0] * len(types), span_s)
        ent[1] = wkey
    return ent[0]


def build_capacity_table(dep: core.Deployment, types: Sequence[core.WorkloadType], model: core.ModelSpec,
                         cluster: core.ClusterSpec, params: Optional[core.ProfileParams] = None,
                         span_s: float = 60.0, device: int = 0) -> core.CapacityTable:
    g = _ctx(types, model, cluster, params or core.ProfileParams(), span_s, device)
    table, _ = g.plan_detail(dep)
    return table


def build_capacity_tables(deps: Sequence[core.Deployment], types: Sequence[core.WorkloadType],
                          model: core.ModelSpec, cluster: core.ClusterSpec,
                          params: Optional[core.ProfileParams] = None, span_s: float = 60.0,
                          device: int = 0) -> List[core.CapacityTable]:
    g = _ctx(types, model, cluster, params or core.ProfileParams(), span_s, device)
    return [g.plan_detail(d)[0] for d in deps]
