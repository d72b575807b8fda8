"""Domain types of the scheduling round — Python mirror of the reference's
L0/L1/L2 value types.

    ClusterSpec / MachineSpec / ModelSpec / ReplicaConfig / Deployment /
    WorkloadType / TraceSpan      proj/include/oserve/core.hpp:11-95
    ProfileParams                 proj/include/oserve/costmodel.hpp:14-22
    SolveOptions                  proj/include/oserve/flowassign.hpp:97-101
    exceptions                    proj/include/oserve/errors.hpp:9-82

Plain value types with the same field names and defaults; placement helpers
(`machine_index`, `same_machine`, `stage_devices`) follow core.cpp:29-54.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence

KGB = 1_000_000_000


# ---- errors (errors.hpp:9-82) ------------------------------------------------
class OServeError(RuntimeError):
    """oserve::Error"""


class InfeasibleReplica(OServeError):
    pass


class ModelTooLarge(OServeError):
    pass


class TooLarge(OServeError):
    pass


class EmptyDeployment(OServeError):
    pass


class UnsourcedFragment(OServeError):
    pass


class LcmOverflow(OServeError):
    """oserve::LcmOverflow (errors.hpp:39): flow::normalize past 2^62."""


class Unsupported(OServeError):
    """Input outside the GPU path's documented limits."""


class CudaError(OServeError):
    pass


class LogicError(RuntimeError):
    """std::logic_error (check_constraints, flowassign.cpp:521-554)."""


# ---- core types (core.hpp) -------------------------------------------------
@dataclass
class MachineSpec:
    machine_id: str
    device_ids: List[int]
    device_mem: int  # bytes per device


@dataclass
class ClusterSpec:
    machines: List[MachineSpec]
    intra_bw: float = 0.0
    inter_bw: float = 0.0

    def device_count(self) -> int:
        return sum(len(m.device_ids) for m in self.machines)

    def all_devices(self) -> List[int]:
        return sorted(d for m in self.machines for d in m.device_ids)

    def machine_index(self, d: int) -> int:
        for i, m in enumerate(self.machines):
            if d in m.device_ids:
                return i
        return -1

    def same_machine(self, a: int, b: int) -> bool:
        ma = self.machine_index(a)
        return ma >= 0 and ma == self.machine_index(b)


@dataclass
class ModelSpec:
    name: str = "model"
    param_bytes: int = 0
    num_layers: int = 0
    bytes_per_token_kv: int = 0
    flops_per_token_prefill: int = 0
    min_mem_bytes: int = 0


@dataclass
class ReplicaConfig:
    device_ids: List[int]
    tp: int = 1
    pp: int = 1

    def device_count(self) -> int:
        return len(self.device_ids)

    def stage_devices(self, s: int) -> List[int]:
        srt = sorted(self.device_ids)
        return srt[s * self.tp:(s + 1) * self.tp]


@dataclass
class Deployment:
    replicas: List[ReplicaConfig] = field(default_factory=list)

    def replica_count(self) -> int:
        return len(self.replicas)

    def device_count(self) -> int:
        return sum(r.device_count() for r in self.replicas)

    def shapes(self):
        return [(r.device_count(), r.tp, r.pp) for r in self.replicas]


@dataclass
class WorkloadType:
    type_id: int = 0
    centroid_in: float = 1.0
    centroid_out: float = 1.0


@dataclass
class TraceSpan:
    span_index: int = 0
    counts: List[int] = field(default_factory=list)


@dataclass
class ProfileParams:
    prefill_coeff: float = 6e-6
    decode_coeff: float = 1e-6
    tp_efficiency: float = 0.75
    pp_comm_cost: float = 5e-4
    mem_bw_penalty: float = 0.05


@dataclass
class SolveOptions:
    exact_demand_limit: int = 400
    exact_cell_limit: int = 20
    node_budget: int = 8_000_000


@dataclass
class AssignmentMatrix:
    x: List[List[int]]
    objective: int


@dataclass
class CapacityTable:
    n: List[List[int]]
    e: List[List[int]]
    latency: List[List[float]]

    def replicas(self) -> int:
        return len(self.n)

    def types(self) -> int:
        return len(self.n[0]) if self.n else 0


@dataclass
class LowerLevel:
    assignment: AssignmentMatrix
    M: List[int]
    unit: List[List[int]]
    used: List[int]


@dataclass
class SearchState:
    deployment: Deployment
    throughput: int = 0
    iterations: int = 0
    # GPU-round extras: selection key fields and the plan-space size.
    key: int = 0
    partition_index: int = 0
    local_rank: int = 0
    sum_pp: int = 0
    plans: int = 0


@dataclass
class StrategyChoice:
    deployment: Deployment
    objective: int = 0


@dataclass
class ByteRange:
    begin: int
    end: int

    def len(self) -> int:
        return self.end - self.begin


@dataclass
class Transfer:
    range: ByteRange
    src: int
    dst: int


@dataclass
class SwitchPlan:
    transfers: List[Transfer]
    est_seconds: float = 0.0


@dataclass
class InflightRequest:
    """switchplan::InflightRequest (switchplan.hpp:63-68)."""
    request_id: int
    generated_tokens: int
    kv_bytes: int
    source_replica: int


@dataclass
class KvTransfer:
    """switchplan::KvTransfer (switchplan.hpp:70-77)."""
    request_id: int
    kv_bytes: int
    src: int
    dst: int


@dataclass
class KvPlan:
    """switchplan::KvPlan (switchplan.hpp:79-84)."""
    drained: List[int] = field(default_factory=list)
    migrated: List[KvTransfer] = field(default_factory=list)
    buffer_bytes: int = 0


# ---- fixtures (proj/tests/fixtures.hpp:20-73), used by tests and configs ----
def cluster(machines: int, devices_per_machine: int, mem_per_device: int = 80 * KGB,
            intra_bw: float = 400e9, inter_bw: float = 200e9) -> ClusterSpec:
    ms, dev = [], 0
    for m in range(machines):
        ids = list(range(dev, dev + devices_per_machine))
        dev += devices_per_machine
        ms.append(MachineSpec(f"m{m}", ids, mem_per_device))
    return ClusterSpec(ms, intra_bw, inter_bw)


def small_model() -> ModelSpec:
    return ModelSpec("artifact-26b", 26 * KGB, 40, 80_000, 52_000_000_000, 40 * KGB)


def large_model() -> ModelSpec:
    return ModelSpec("artifact-110b", 110 * KGB, 80, 80_000, 220_000_000_000, 120 * KGB)


def model_140gb() -> ModelSpec:
    return ModelSpec("artifact-70b", 140 * KGB, 80, 160_000, 280_000_000_000, 140 * KGB)


def model_14gb() -> ModelSpec:
    """7B-class model used by config 3 (builder-defined)."""
    return ModelSpec("artifact-7b", 14 * KGB, 32, 32_000, 14_000_000_000, 14 * KGB)


def short_type() -> WorkloadType:
    return WorkloadType(0, 2000.0, 50.0)


def long_type() -> WorkloadType:
    return WorkloadType(1, 100.0, 3000.0)


def canonical_deployment(cl: ClusterSpec, sizes: Sequence[int], tps: Sequence[int],
                         pps: Optional[Sequence[int]] = None) -> Deployment:
    """Deployment on canonical_blocks (deploysearch.cpp:89-103)."""
    devs = cl.all_devices()
    dep, pos = Deployment(), 0
    for i, s in enumerate(sizes):
        tp = tps[i]
        pp = pps[i] if pps is not None else s // tp
        dep.replicas.append(ReplicaConfig(devs[pos:pos + s], tp, pp))
        pos += s
    return dep
