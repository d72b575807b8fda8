"""ctypes mirror of include/oserve_gpu.h (structs and marshalling helpers).

Shared by the product binding (`_native.py`) and the test-only oracle
loader; no compute lives here.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Sequence

from . import core

MAX_REPLICAS = 128
MAX_CLASSES = 16
MAX_DEVICES = 1024

OK = 0
ERR_INVALID_ARGUMENT = 1
ERR_INFEASIBLE_REPLICA = 2
ERR_MODEL_TOO_LARGE = 3
ERR_TOO_LARGE = 4
ERR_EMPTY_DEPLOYMENT = 5
ERR_UNSOURCED_FRAGMENT = 6
ERR_LOGIC = 7
ERR_UNSUPPORTED = 8
ERR_CUDA = 9
ERR_NO_DEVICE = 10
ERR_NCCL = 11
ERR_LCM_OVERFLOW = 12

SPACE_ORDERED = 0
SPACE_CANONICAL = 1


class ClusterDesc(C.Structure):
    _fields_ = [("num_machines", C.c_int), ("machine_num_devices", C.POINTER(C.c_int)),
                ("device_ids", C.POINTER(C.c_int)), ("device_mem", C.POINTER(C.c_uint64)),
                ("intra_bw", C.c_double), ("inter_bw", C.c_double)]


class ModelDesc(C.Structure):
    _fields_ = [("param_bytes", C.c_uint64), ("num_layers", C.c_uint32),
                ("bytes_per_token_kv", C.c_uint64), ("flops_per_token_prefill", C.c_uint64),
                ("min_mem_bytes", C.c_uint64)]


class Profile(C.Structure):
    _fields_ = [("prefill_coeff", C.c_double), ("decode_coeff", C.c_double),
                ("tp_efficiency", C.c_double), ("pp_comm_cost", C.c_double),
                ("mem_bw_penalty", C.c_double)]


class ClassDesc(C.Structure):
    _fields_ = [("type_id", C.c_int), ("centroid_in", C.c_double), ("centroid_out", C.c_double)]


class SolveOptionsDesc(C.Structure):
    _fields_ = [("exact_demand_limit", C.c_int64), ("exact_cell_limit", C.c_int),
                ("node_budget", C.c_int64)]


class DeploymentDesc(C.Structure):
    _fields_ = [("num_replicas", C.c_int), ("replica_num_devices", C.POINTER(C.c_int)),
                ("device_ids", C.POINTER(C.c_int)), ("tp", C.POINTER(C.c_int)),
                ("pp", C.POINTER(C.c_int))]


class Plan(C.Structure):
    _fields_ = [("num_replicas", C.c_int), ("num_devices", C.c_int),
                ("replica_num_devices", C.c_int * MAX_REPLICAS), ("tp", C.c_int * MAX_REPLICAS),
                ("pp", C.c_int * MAX_REPLICAS), ("device_ids", C.c_int * MAX_DEVICES)]


class SpaceDesc(C.Structure):
    _fields_ = [("mode", C.c_int), ("num_sizes", C.c_int), ("sizes", C.POINTER(C.c_int)),
                ("max_devices", C.c_int)]


class RoundResult(C.Structure):
    _fields_ = [("objective", C.c_int64), ("key", C.c_uint64), ("partitions", C.c_int64),
                ("plans", C.c_uint64), ("partition_index", C.c_int64), ("local_rank", C.c_uint64),
                ("sum_pp", C.c_int), ("plan", Plan)]


class TransferDesc(C.Structure):
    _fields_ = [("begin", C.c_uint64), ("end", C.c_uint64), ("src", C.c_int), ("dst", C.c_int)]


class ShardDesc(C.Structure):  # oserve_shard (switchplan::ShardLayout::Shard)
    _fields_ = [("shard_id", C.c_int), ("begin", C.c_uint64), ("end", C.c_uint64), ("holder", C.c_int)]


class HeldRangeDesc(C.Structure):  # oserve_held_range (one ShardLayout::held entry)
    _fields_ = [("device", C.c_int), ("begin", C.c_uint64), ("end", C.c_uint64)]


class LinkLoadDesc(C.Structure):  # oserve_link_load (SwitchPlan::link_load entry)
    _fields_ = [("src", C.c_int), ("dst", C.c_int), ("bytes", C.c_uint64)]


class FlowEdgeDesc(C.Structure):
    _fields_ = [("from_", C.c_int), ("to", C.c_int), ("cap", C.c_int64)]


def flow_edge_dtype():
    """numpy layout of oserve_flow_edge."""
    import numpy as np
    return np.dtype([("from", "<i4"), ("to", "<i4"), ("cap", "<i8")], align=True)


def flow_edges(edges, keep: "Keep"):
    """(from, to, cap) tuples or a flow_edge_dtype array -> oserve_flow_edge*."""
    import numpy as np
    if not isinstance(edges, np.ndarray):
        a = np.zeros(len(edges), flow_edge_dtype())
        if len(edges):
            t = np.asarray(edges, dtype=np.int64).reshape(-1, 3)
            a["from"], a["to"], a["cap"] = t[:, 0], t[:, 1], t[:, 2]
        edges = a
    a = keep(np.ascontiguousarray(edges, dtype=flow_edge_dtype()))
    if not len(a):
        return keep((FlowEdgeDesc * 1)())
    return C.cast(a.ctypes.data, C.POINTER(FlowEdgeDesc))


class InflightDesc(C.Structure):
    _fields_ = [("request_id", C.c_int64), ("generated_tokens", C.c_int64), ("kv_bytes", C.c_uint64),
                ("source_replica", C.c_int)]


class KvTransferDesc(C.Structure):
    _fields_ = [("request_id", C.c_int64), ("kv_bytes", C.c_uint64), ("src", C.c_int), ("dst", C.c_int)]


def inflight_dtype():
    """numpy layout of oserve_inflight (a structured array may be passed
    wherever a list of InflightRequest is accepted)."""
    import numpy as np
    return np.dtype([("request_id", "<i8"), ("generated_tokens", "<i8"), ("kv_bytes", "<u8"),
                     ("source_replica", "<i4")], align=True)


def inflight_arr(reqs, keep: "Keep"):
    import numpy as np
    if isinstance(reqs, np.ndarray):
        a = keep(np.ascontiguousarray(reqs, dtype=inflight_dtype()))
        assert a.dtype.itemsize == C.sizeof(InflightDesc)
        return C.cast(a.ctypes.data, C.POINTER(InflightDesc)) if len(a) else (InflightDesc * 1)()
    arr = (InflightDesc * max(1, len(reqs)))()
    for i, r in enumerate(reqs):
        arr[i] = InflightDesc(r.request_id, r.generated_tokens, r.kv_bytes, r.source_replica)
    return keep(arr)


def kv_arrays(drained, nd: int, mig, nm: int, buffer_bytes: int):
    """kv_plan outputs as numpy: drained ids [nd], migrated rows [nm, 4] =
    (request_id, kv_bytes, src, dst), buffer bytes."""
    import numpy as np
    d = np.ctypeslib.as_array(drained)[:nd].copy()
    rec = np.dtype([("request_id", "<i8"), ("kv_bytes", "<u8"), ("src", "<i4"), ("dst", "<i4")])
    raw = np.frombuffer(mig, dtype=rec, count=nm) if nm else np.zeros(0, rec)
    m = np.stack([raw["request_id"], raw["kv_bytes"].astype(np.int64), raw["src"], raw["dst"]], axis=1) \
        if nm else np.zeros((0, 4), np.int64)
    return d, m, buffer_bytes


def transfer_arr(plan, keep: "Keep"):
    tr = [] if plan is None else plan.transfers
    arr = (TransferDesc * max(1, len(tr)))()
    for i, t in enumerate(tr):
        arr[i] = TransferDesc(t.range.begin, t.range.end, t.src, t.dst)
    return keep(arr), len(tr)


class SearchOptionsDesc(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("max_iters", C.c_int), ("stale_limit", C.c_int),
                ("mutation_retries", C.c_int), ("warm_start", C.POINTER(DeploymentDesc))]


class SearchLogRow(C.Structure):
    _fields_ = [("iteration", C.c_int), ("accepted", C.c_int), ("throughput", C.c_int64), ("devices", C.c_int),
                ("op", C.c_char * 120)]


class SearchResult(C.Structure):
    _fields_ = [("throughput", C.c_int64), ("rng_seed", C.c_uint64), ("stale_iters", C.c_int),
                ("iterations", C.c_int), ("log_count", C.c_int), ("deployment", Plan)]


def search_options(seed=0, max_iters=500, stale_limit=20, mutation_retries=8, warm_start=None, keep=None):
    keep = keep or Keep()
    ws = None
    if warm_start is not None and warm_start.replicas:
        ws = C.pointer(keep(deployment_desc(warm_start, keep)))
    return SearchOptionsDesc(seed, max_iters, stale_limit, mutation_retries, ws)


def search_outcome(res: SearchResult, log, n: int):
    rows = [(log[i].iteration, log[i].op.decode(), bool(log[i].accepted), log[i].throughput, log[i].devices)
            for i in range(min(n, len(log)))]
    st = core.SearchState(plan_to_deployment(res.deployment), res.throughput, res.iterations)
    st.stale_iters = res.stale_iters
    st.rng_seed = res.rng_seed
    return st, rows


class ProblemDesc(C.Structure):
    """oracle_problem (oracle/oracle_api.h) — test infrastructure only."""
    _fields_ = [("cluster", ClusterDesc), ("model", ModelDesc), ("profile", Profile),
                ("num_classes", C.c_int), ("classes", C.POINTER(ClassDesc)),
                ("lambda_", C.POINTER(C.c_int64)), ("span_seconds", C.c_double)]


def _arr(ctype, values):
    values = list(values)
    return (ctype * max(1, len(values)))(*values)


class Keep:
    """Holds ctypes buffers alive alongside the struct that points at them."""

    def __init__(self):
        self.refs = []

    def __call__(self, obj):
        self.refs.append(obj)
        return obj


def cluster_desc(cl: core.ClusterSpec, keep: Keep) -> ClusterDesc:
    nd = keep(_arr(C.c_int, [len(m.device_ids) for m in cl.machines]))
    ids = keep(_arr(C.c_int, [d for m in cl.machines for d in m.device_ids]))
    mem = keep(_arr(C.c_uint64, [m.device_mem for m in cl.machines]))
    return ClusterDesc(len(cl.machines), nd, ids, mem, float(cl.intra_bw), float(cl.inter_bw))


def model_desc(m: core.ModelSpec) -> ModelDesc:
    return ModelDesc(m.param_bytes, m.num_layers, m.bytes_per_token_kv, m.flops_per_token_prefill,
                     m.min_mem_bytes)


def profile_desc(p: core.ProfileParams) -> Profile:
    return Profile(p.prefill_coeff, p.decode_coeff, p.tp_efficiency, p.pp_comm_cost, p.mem_bw_penalty)


def classes_arr(types: Sequence[core.WorkloadType], keep: Keep):
    arr = (ClassDesc * max(1, len(types)))()
    for i, t in enumerate(types):
        arr[i] = ClassDesc(t.type_id, float(t.centroid_in), float(t.centroid_out))
    return keep(arr)


def deployment_desc(dep: core.Deployment, keep: Keep) -> DeploymentDesc:
    nd = keep(_arr(C.c_int, [r.device_count() for r in dep.replicas]))
    ids = keep(_arr(C.c_int, [d for r in dep.replicas for d in r.device_ids]))
    tp = keep(_arr(C.c_int, [r.tp for r in dep.replicas]))
    pp = keep(_arr(C.c_int, [r.pp for r in dep.replicas]))
    return DeploymentDesc(dep.replica_count(), nd, ids, tp, pp)


def deployment_desc_array(deps: Sequence[core.Deployment], keep: Keep):
    """A DeploymentDesc array for many deployments: the replica fields of all
    of them packed into four int arrays, the descriptors' pointers filled by
    numpy offset arithmetic (no per-deployment ctypes arrays)."""
    import numpy as np
    n = len(deps)
    nrep = np.fromiter((len(d.replicas) for d in deps), np.int64, n)
    reps = [r for d in deps for r in d.replicas]
    nd = keep(np.fromiter((len(r.device_ids) for r in reps), np.int32, len(reps)))
    tp = keep(np.fromiter((r.tp for r in reps), np.int32, len(reps)))
    pp = keep(np.fromiter((r.pp for r in reps), np.int32, len(reps)))
    ids = keep(np.fromiter((x for r in reps for x in r.device_ids), np.int32, int(nd.sum())))
    roff = np.zeros(n, np.int64)
    roff[1:] = np.cumsum(nrep)[:-1]
    doff = np.zeros(len(reps) + 1, np.int64)
    doff[1:] = np.cumsum(nd)
    dt = np.dtype({"names": ["num_replicas", "rnd", "ids", "tp", "pp"],
                   "formats": ["<i4", "<u8", "<u8", "<u8", "<u8"],
                   "offsets": [0, 8, 16, 24, 32], "itemsize": C.sizeof(DeploymentDesc)})
    a = keep(np.zeros(max(1, n), dt))
    a["num_replicas"][:n] = nrep
    a["rnd"][:n] = nd.ctypes.data + 4 * roff
    a["ids"][:n] = ids.ctypes.data + 4 * doff[roff]
    a["tp"][:n] = tp.ctypes.data + 4 * roff
    a["pp"][:n] = pp.ctypes.data + 4 * roff
    return C.cast(a.ctypes.data, C.POINTER(DeploymentDesc))


def space_desc(mode: int, sizes: Sequence[int] = (), max_devices: int = 0, keep: Keep = None) -> SpaceDesc:
    keep = keep or Keep()
    sz = keep(_arr(C.c_int, sizes))
    return SpaceDesc(mode, len(sizes), sz if sizes else None, max_devices)


def plan_to_deployment(p: Plan) -> core.Deployment:
    dep, pos = core.Deployment(), 0
    for r in range(p.num_replicas):
        n = p.replica_num_devices[r]
        dep.replicas.append(core.ReplicaConfig(list(p.device_ids[pos:pos + n]), p.tp[r], p.pp[r]))
        pos += n
    return dep


def result_to_state(res: RoundResult) -> core.SearchState:
    return core.SearchState(plan_to_deployment(res.plan), res.objective, res.partitions, res.key,
                            res.partition_index, res.local_rank, res.sum_pp, res.plans)


_EXC = {
    ERR_INVALID_ARGUMENT: ValueError,
    ERR_INFEASIBLE_REPLICA: core.InfeasibleReplica,
    ERR_MODEL_TOO_LARGE: core.ModelTooLarge,
    ERR_TOO_LARGE: core.TooLarge,
    ERR_EMPTY_DEPLOYMENT: core.EmptyDeployment,
    ERR_UNSOURCED_FRAGMENT: core.UnsourcedFragment,
    ERR_LOGIC: core.LogicError,
    ERR_UNSUPPORTED: core.Unsupported,
    ERR_CUDA: core.CudaError,
    ERR_NO_DEVICE: core.CudaError,
    ERR_NCCL: core.CudaError,
    ERR_LCM_OVERFLOW: core.LcmOverflow,
}


def raise_for(status: int, msg: str):
    if status != OK:
        raise _EXC.get(status, core.OServeError)(msg)


def problem_desc(cl, model, profile, types, lam, span_s, keep: Keep) -> ProblemDesc:
    return ProblemDesc(cluster_desc(cl, keep), model_desc(model), profile_desc(profile), len(types),
                       classes_arr(types, keep), keep(_arr(C.c_int64, lam)), float(span_s))


def i64_rows(flat: Sequence[int], R: int, J: int) -> List[List[int]]:
    return [list(flat[k * J:(k + 1) * J]) for k in range(R)]
