"""oserve::switchplan (switchplan.cpp:40-140) on the GPU path (K2).

`layout(dep, model)` is lazy: the byte-range layout is computed on the device
inside `greedy_plan`, which returns the reference's transfer list in its
order (fragment-major, destination ascending) and the estimate."""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Sequence

from . import core
from ._native import GpuContext


@dataclass
class ShardLayout:
    deployment: core.Deployment
    model: core.ModelSpec


def layout(dep: core.Deployment, model: core.ModelSpec) -> ShardLayout:
    return ShardLayout(dep, model)


def greedy_plan(src: ShardLayout, dst: ShardLayout, cluster: core.ClusterSpec, device: int = 0) -> core.SwitchPlan:
    g = GpuContext(cluster, src.model, device=device)
    return g.switch_plan(src.deployment, dst.deployment)


def estimate_time(plan: core.SwitchPlan, cluster: core.ClusterSpec) -> float:
    return plan.est_seconds


def switch_cost_batch(current: core.Deployment, candidates: Sequence[core.Deployment], model: core.ModelSpec,
                      cluster: core.ClusterSpec, device: int = 0) -> List[float]:
    """est_seconds from `current` to every candidate, one CTA per pair."""
    g = GpuContext(cluster, model, device=device)
    return g.switch_cost_batch(current, list(candidates))[0]
