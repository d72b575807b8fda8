"""oserve::cost::build_capacity_table (costmodel.cpp:94-116) on the GPU path
(cost kernel K0a; cells bit-identical to the reference)."""
from __future__ import annotations

from typing import Optional, Sequence

from . import core
from ._native import GpuContext


def build_capacity_table(dep: core.Deployment, types: Sequence[core.WorkloadType], model: core.ModelSpec,
                         cluster: core.ClusterSpec, params: Optional[core.ProfileParams] = None,
                         span_s: float = 60.0, device: int = 0) -> core.CapacityTable:
    g = GpuContext(cluster, model, params or core.ProfileParams(), device)
    g.set_workload(list(types), [0] * len(types), span_s)
    table, _ = g.plan_detail(dep)
    return table
