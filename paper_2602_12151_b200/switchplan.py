"""oserve::switchplan on the GPU path (switchplan.hpp:34-61).

  layout(dep, model)            switchplan::layout (switchplan.cpp:40-63):
                                shards computed on the device (k_layout), `held`
                                coalesced per device as the reference does
  greedy_plan(src, dst, cluster)  switchplan::greedy_plan over two ShardLayouts
                                (switchplan.cpp:65-131): fragments, per-target
                                holder choice and link loads on the device
                                (k_switch_held); transfers in the reference's order
  estimate_time(plan, cluster)  switchplan::estimate_time (switchplan.cpp:133-140)
                                on the device (k_link_time)
  switch_cost_batch             layout + greedy_plan + estimate_time fused for one
                                current deployment and many candidates (K2, one
                                CTA per pair)
Contexts are cached per cluster (and per model for the fused path).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Sequence, Tuple

from . import core
from ._native import GpuContext

_NONE_MODEL = core.ModelSpec("none", 1, 1, 1, 1, 1)
_cache: Dict[tuple, GpuContext] = {}


def _ctx(cluster: core.ClusterSpec, model: core.ModelSpec = _NONE_MODEL, device: int = 0) -> GpuContext:
    key = (repr(cluster), repr(model), device)
    g = _cache.get(key)
    if g is None:
        if len(_cache) > 8:
            _cache.pop(next(iter(_cache)))
        g = _cache[key] = GpuContext(cluster, model, device=device)
    return g


@dataclass
class Shard:
    """switchplan::ShardLayout::Shard (switchplan.hpp:24-28)."""
    shard_id: int
    range: core.ByteRange
    holder: int


@dataclass
class ShardLayout:
    """switchplan::ShardLayout (switchplan.hpp:22-31)."""
    shards: List[Shard] = field(default_factory=list)
    held: Dict[int, List[Tuple[int, int]]] = field(default_factory=dict)  # device -> sorted disjoint ranges


def _coalesce(ranges: List[Tuple[int, int]]) -> List[Tuple[int, int]]:
    """switchplan.cpp:17-29."""
    out: List[Tuple[int, int]] = []
    for b, e in sorted(ranges):
        if b == e:
            continue
        if out and b <= out[-1][1]:
            out[-1] = (out[-1][0], max(out[-1][1], e))
        else:
            out.append((b, e))
    return out


def layout(dep: core.Deployment, model: core.ModelSpec, device: int = 0) -> ShardLayout:
    g = _ctx(core.cluster(1, 1), device=device)
    out = ShardLayout()
    for sid, b, e, h in g.layout_shards(dep, model.param_bytes):
        out.shards.append(Shard(sid, core.ByteRange(b, e), h))
        out.held.setdefault(h, []).append((b, e))
    out.held = {d: _coalesce(r) for d, r in sorted(out.held.items())}
    return out


def greedy_plan(src: ShardLayout, dst: ShardLayout, cluster: core.ClusterSpec, device: int = 0) -> core.SwitchPlan:
    return _ctx(cluster, device=device).greedy_plan_held(src.held, dst.held)


def link_load(plan: core.SwitchPlan) -> Dict[Tuple[int, int], int]:
    """SwitchPlan::link_load (switchplan.hpp:44) from the transfers."""
    ll: Dict[Tuple[int, int], int] = {}
    for t in plan.transfers:
        ll[(t.src, t.dst)] = ll.get((t.src, t.dst), 0) + t.range.len()
    return ll


def estimate_time(plan: core.SwitchPlan, cluster: core.ClusterSpec, device: int = 0) -> float:
    return _ctx(cluster, device=device).estimate_time([(s, d, b) for (s, d), b in sorted(link_load(plan).items())])


def switch_cost_batch(current: core.Deployment, candidates: Sequence[core.Deployment], model: core.ModelSpec,
                      cluster: core.ClusterSpec, device: int = 0) -> List[float]:
    """est_seconds from `current` to every candidate, one CTA per pair (K2)."""
    return _ctx(cluster, model, device).switch_cost_batch(current, list(candidates))[0]
