"""ctypes binding of liboserve_gpu.so (include/oserve_gpu.h).

The product path: every call goes through the C-ABI into the sm_100a kernels.
There is no CPU fallback — if the in-tree library is missing or no CUDA
device is present the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _abi as A
from . import core

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OSERVE_GPU_LIB", os.path.join(HERE, "liboserve_gpu.so"))

EXPORTS = [
    "oserve_gpu_create", "oserve_gpu_destroy", "oserve_gpu_last_error", "oserve_gpu_status_name",
    "oserve_gpu_set_workload", "oserve_gpu_set_solve_options", "oserve_gpu_set_shard", "oserve_gpu_set_stream",
    "oserve_gpu_min_feasible_group", "oserve_gpu_prepare_space", "oserve_gpu_launch_round_async",
    "oserve_gpu_decode_key", "oserve_gpu_round", "oserve_gpu_exhaustive", "oserve_gpu_best_strategies",
    "oserve_gpu_evaluate_ranks", "oserve_gpu_evaluate_deployments", "oserve_gpu_plan_detail",
    "oserve_gpu_solve_batch", "oserve_gpu_switch_cost_batch", "oserve_gpu_switch_plan",
    "oserve_gpu_launch_count", "oserve_gpu_copy_bytes",
    "oserve_shard_count", "oserve_shard_global_rank", "oserve_key_layout",
    "oserve_gpu_round_topk", "oserve_gpu_switch_cost_keys", "oserve_gpu_switch_cost_keys_async",
    "oserve_gpu_search", "oserve_gpu_kv_plan", "oserve_forecast_series",
    "oserve_gpu_max_flow_batch", "oserve_gpu_flow_assign_batch", "oserve_gpu_extract_assignment_batch",
    "oserve_gpu_solve_fractional_batch",
    "oserve_gpu_create_multi", "oserve_nccl_unique_id", "oserve_gpu_join", "oserve_gpu_world",
    "oserve_gpu_layout", "oserve_gpu_greedy_plan_layouts", "oserve_gpu_estimate_time",
    "oserve_gpu_normalize_batch", "oserve_gpu_check_constraints_batch",
]

_lib = None


def load_library() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                           " (make -C paper_2602_12151_b200/csrc); there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    P = C.POINTER
    vp = C.c_void_p
    L.oserve_gpu_create.argtypes = [C.c_int, P(A.ClusterDesc), P(A.ModelDesc), P(A.Profile), P(vp)]
    L.oserve_gpu_destroy.argtypes = [vp]
    L.oserve_gpu_create_multi.argtypes = [P(C.c_int), C.c_int, P(A.ClusterDesc), P(A.ModelDesc), P(A.Profile), P(vp)]
    L.oserve_nccl_unique_id.argtypes = [vp]
    L.oserve_gpu_join.argtypes = [vp, vp, C.c_int, C.c_int]
    L.oserve_gpu_world.argtypes = [vp, P(C.c_int), P(C.c_int), P(C.c_int)]
    L.oserve_gpu_layout.argtypes = [vp, P(A.DeploymentDesc), C.c_uint64, C.c_int, P(A.ShardDesc), P(C.c_int)]
    L.oserve_gpu_greedy_plan_layouts.argtypes = [vp, C.c_int, P(A.HeldRangeDesc), C.c_int, P(A.HeldRangeDesc),
                                                 C.c_int, P(A.TransferDesc), P(C.c_int), P(C.c_double)]
    L.oserve_gpu_estimate_time.argtypes = [vp, C.c_int, P(A.LinkLoadDesc), P(C.c_double)]
    L.oserve_gpu_normalize_batch.argtypes = [vp, C.c_int, C.c_int, P(C.c_int64), C.c_int, P(C.c_int64),
                                             P(C.c_int64), P(C.c_int)]
    L.oserve_gpu_check_constraints_batch.argtypes = [vp, C.c_int, C.c_int, C.c_int] + [P(C.c_int64)] * 4 + \
        [P(C.c_int)] * 3
    L.oserve_gpu_last_error.argtypes = [vp]
    L.oserve_gpu_last_error.restype = C.c_char_p
    L.oserve_gpu_status_name.restype = C.c_char_p
    L.oserve_gpu_set_workload.argtypes = [vp, C.c_int, P(A.ClassDesc), P(C.c_int64), C.c_double]
    L.oserve_gpu_set_solve_options.argtypes = [vp, P(A.SolveOptionsDesc)]
    L.oserve_gpu_set_shard.argtypes = [vp, C.c_int, C.c_int]
    L.oserve_gpu_set_stream.argtypes = [vp, vp]
    L.oserve_gpu_min_feasible_group.argtypes = [vp, P(C.c_int)]
    L.oserve_gpu_prepare_space.argtypes = [vp, P(A.SpaceDesc), P(C.c_int64), P(C.c_uint64)]
    L.oserve_gpu_launch_round_async.argtypes = [vp, vp]
    L.oserve_gpu_decode_key.argtypes = [vp, C.c_uint64, P(A.RoundResult)]
    L.oserve_gpu_round.argtypes = [vp, P(A.SpaceDesc), P(A.RoundResult)]
    L.oserve_gpu_exhaustive.argtypes = [vp, P(A.RoundResult)]
    L.oserve_gpu_best_strategies.argtypes = [vp, C.c_int, P(C.c_int), P(A.RoundResult)]
    L.oserve_gpu_evaluate_ranks.argtypes = [vp, C.c_uint64, C.c_uint64, P(C.c_int64), P(C.c_int32)]
    L.oserve_gpu_evaluate_deployments.argtypes = [vp, C.c_int, P(A.DeploymentDesc), P(C.c_int64)]
    L.oserve_gpu_plan_detail.argtypes = [vp, P(A.DeploymentDesc)] + [P(C.c_int64)] * 2 + [P(C.c_double)] + \
        [P(C.c_int64)] * 5
    L.oserve_gpu_solve_batch.argtypes = [vp, C.c_int, C.c_int, C.c_int] + [P(C.c_int64)] * 8
    L.oserve_gpu_switch_cost_batch.argtypes = [vp, P(A.DeploymentDesc), C.c_int, P(A.DeploymentDesc),
                                               P(C.c_double), P(C.c_uint64)]
    L.oserve_gpu_switch_plan.argtypes = [vp, P(A.DeploymentDesc), P(A.DeploymentDesc), C.c_int,
                                         P(A.TransferDesc), P(C.c_int), P(C.c_double)]
    L.oserve_gpu_launch_count.argtypes = [vp]
    L.oserve_gpu_launch_count.restype = C.c_uint64
    L.oserve_gpu_copy_bytes.argtypes = [vp, P(C.c_uint64), P(C.c_uint64)]
    L.oserve_gpu_round_topk.argtypes = [vp, C.c_int, vp, vp]
    L.oserve_gpu_switch_cost_keys.argtypes = [vp, P(A.DeploymentDesc), C.c_int, vp, P(C.c_double), P(C.c_uint64)]
    L.oserve_gpu_switch_cost_keys_async.argtypes = [vp, P(A.DeploymentDesc), C.c_int, vp, vp]
    L.oserve_gpu_search.argtypes = [vp, P(A.SearchOptionsDesc), P(A.SearchResult), P(A.SearchLogRow), C.c_int]
    L.oserve_gpu_kv_plan.argtypes = [vp, C.c_int, P(A.InflightDesc), C.c_int64, P(A.DeploymentDesc),
                                     P(A.DeploymentDesc), C.c_double, C.c_int, P(A.TransferDesc), P(C.c_int64),
                                     P(C.c_int), P(A.KvTransferDesc), P(C.c_int), P(C.c_uint64)]
    L.oserve_gpu_max_flow_batch.argtypes = [vp, C.c_int, P(C.c_int), P(C.c_int64), P(A.FlowEdgeDesc), P(C.c_int),
                                            P(C.c_int), P(C.c_int64), P(C.c_int64)]
    L.oserve_gpu_flow_assign_batch.argtypes = [vp, C.c_int, C.c_int, C.c_int] + [P(C.c_int64)] * 7
    L.oserve_gpu_extract_assignment_batch.argtypes = [vp, C.c_int, C.c_int, C.c_int] + [P(C.c_int64)] * 6
    L.oserve_gpu_solve_fractional_batch.argtypes = [vp, C.c_int, C.c_int, C.c_int] + [P(C.c_int64)] * 3 + \
        [P(C.c_double)] * 2
    L.oserve_forecast_series.argtypes = [C.c_int, C.c_int, P(C.c_int64), C.c_int, C.c_double, C.c_double,
                                         P(C.c_int64)]
    L.oserve_shard_count.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_int]
    L.oserve_shard_count.restype = C.c_uint64
    L.oserve_shard_global_rank.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_int]
    L.oserve_shard_global_rank.restype = C.c_uint64
    L.oserve_key_layout.argtypes = [C.c_int64, C.c_int64, C.c_int, C.c_uint64, P(C.c_int), P(C.c_int), P(C.c_int),
                                    P(C.c_uint64)]
    _lib = L
    return L


SHARD_CHUNK = 4096


def forecast_series(counts: Sequence[Sequence[int]], window: int = 50, alpha: float = 0.45,
                    beta: float = 0.25) -> List[List[int]]:
    """orch::forecast_series (orchestrate.cpp:75-92) with HoltForecaster
    (workload.cpp:204-222): per-span demand from the actual counts [T][J]."""
    T = len(counts)
    J = len(counts[0]) if T else 1
    flat = A._arr(C.c_int64, [int(v) for row in counts for v in row])
    out = (C.c_int64 * max(1, T * J))()
    A.raise_for(load_library().oserve_forecast_series(J, T, flat, window, alpha, beta, out),
                "forecast_series: invalid arguments")
    return A.i64_rows(out, T, J)


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId for oserve_gpu_join (rank 0 makes it)."""
    buf = C.create_string_buffer(128)
    A.raise_for(load_library().oserve_nccl_unique_id(buf), "ncclGetUniqueId failed")
    return buf.raw


def shard_count(total: int, rank: int, world: int, chunk: int = SHARD_CHUNK) -> int:
    """Plans of shard `rank` (C++ host logic, no device needed)."""
    return int(load_library().oserve_shard_count(total, chunk, rank, world))


def shard_global_rank(local: int, rank: int, world: int, chunk: int = SHARD_CHUNK) -> int:
    return int(load_library().oserve_shard_global_rank(local, chunk, rank, world))


def key_layout(total_demand: int, partitions: int, devices: int, max_plans: int):
    """(sh_obj, sh_part, sh_spp, obj_max) of the packed selection key."""
    a, b, c, m = C.c_int(), C.c_int(), C.c_int(), C.c_uint64()
    st = load_library().oserve_key_layout(total_demand, partitions, devices, max_plans, C.byref(a), C.byref(b),
                                          C.byref(c), C.byref(m))
    A.raise_for(st, "selection key does not fit 63 bits")
    return a.value, b.value, c.value, m.value


def pack_key(layout, objective: int, partition: int, sum_pp: int, local_rank: int) -> int:
    sh_obj, sh_part, sh_spp, obj_max = layout
    return ((obj_max - objective) << sh_obj) | (partition << sh_part) | (sum_pp << sh_spp) | local_rank


def _np_ptr(a, t):
    return a.ctypes.data_as(C.POINTER(t))


class GpuContext:
    """One oserve_gpu_ctx: a cluster/model/profile bound to one CUDA device.

    Mirrors the reference's EvalContext (deploysearch.hpp:45-54) but owns
    copies of its inputs and the device-resident tables.
    """

    def __init__(self, cluster: core.ClusterSpec, model: core.ModelSpec,
                 params: Optional[core.ProfileParams] = None, device: int = 0,
                 devices: Optional[Sequence[int]] = None):
        """`devices` (several CUDA devices of this process): one context over
        all of them, rounds sharded with an NCCL communicator
        (oserve_gpu_create_multi); otherwise one device."""
        self.lib = load_library()
        self.cluster, self.model = cluster, model
        self.params = params or core.ProfileParams()
        keep = A.Keep()
        cd = A.cluster_desc(cluster, keep)
        md = A.model_desc(model)
        pd = A.profile_desc(self.params)
        h = C.c_void_p()
        self.device = int(devices[0]) if devices else int(device)
        if devices is not None and len(devices) > 1:
            devs = A._arr(C.c_int, list(devices))
            st = self.lib.oserve_gpu_create_multi(devs, len(devices), C.byref(cd), C.byref(md), C.byref(pd),
                                                  C.byref(h))
        else:
            dev = devices[0] if devices else device
            st = self.lib.oserve_gpu_create(dev, C.byref(cd), C.byref(md), C.byref(pd), C.byref(h))
        if st != A.OK:
            A.raise_for(st, f"oserve_gpu_create: {self.lib.oserve_gpu_status_name(st).decode()}")
        self.h = h
        self.types: List[core.WorkloadType] = []
        self.lam: List[int] = []
        self.span_s = 60.0

    def close(self):
        if getattr(self, "h", None):
            self.lib.oserve_gpu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, st: int):
        if st != A.OK:
            A.raise_for(st, self.lib.oserve_gpu_last_error(self.h).decode())

    # -- configuration -------------------------------------------------------
    def set_workload(self, types: Sequence[core.WorkloadType], lam: Sequence[int], span_s: float = 60.0):
        keep = A.Keep()
        cls = A.classes_arr(types, keep)
        self._chk(self.lib.oserve_gpu_set_workload(self.h, len(types), cls, A._arr(C.c_int64, lam), float(span_s)))
        self.types, self.lam, self.span_s = list(types), [int(v) for v in lam], float(span_s)

    def set_solve_options(self, opts: core.SolveOptions):
        self._chk(self.lib.oserve_gpu_set_solve_options(
            self.h, C.byref(A.SolveOptionsDesc(opts.exact_demand_limit, opts.exact_cell_limit, opts.node_budget))))

    def set_shard(self, rank: int, world: int):
        self._chk(self.lib.oserve_gpu_set_shard(self.h, rank, world))

    def join(self, uid: bytes, rank: int, world: int):
        """Join a multi-process world (one GPU per process): rounds shard over
        it and the library runs the NCCL exchange (oserve_gpu_join)."""
        buf = C.create_string_buffer(bytes(uid), 128)
        self._chk(self.lib.oserve_gpu_join(self.h, buf, int(rank), int(world)))

    def world(self):
        """(global rank of the first local device, world size, local devices)."""
        r, w, n = C.c_int(), C.c_int(), C.c_int()
        self._chk(self.lib.oserve_gpu_world(self.h, C.byref(r), C.byref(w), C.byref(n)))
        return r.value, w.value, n.value

    def set_stream(self, stream_ptr: int):
        self._chk(self.lib.oserve_gpu_set_stream(self.h, C.c_void_p(stream_ptr)))

    def launch_count(self) -> int:
        return int(self.lib.oserve_gpu_launch_count(self.h))

    def copy_bytes(self):
        """(host->device, device->host) bytes this context has copied."""
        a, b = C.c_uint64(), C.c_uint64()
        self._chk(self.lib.oserve_gpu_copy_bytes(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def min_feasible_group(self) -> int:
        g = C.c_int()
        self._chk(self.lib.oserve_gpu_min_feasible_group(self.h, C.byref(g)))
        return g.value

    # -- scheduling round ------------------------------------------------------
    def prepare_space(self, mode: int = A.SPACE_ORDERED, sizes: Sequence[int] = (), max_devices: int = 0):
        keep = A.Keep()
        sd = A.space_desc(mode, sizes, max_devices, keep)
        parts, plans = C.c_int64(), C.c_uint64()
        self._chk(self.lib.oserve_gpu_prepare_space(self.h, C.byref(sd), C.byref(parts), C.byref(plans)))
        return parts.value, plans.value

    def launch_round_async(self, d_key_ptr: int):
        self._chk(self.lib.oserve_gpu_launch_round_async(self.h, C.c_void_p(d_key_ptr)))

    def decode_key(self, key: int) -> core.SearchState:
        res = A.RoundResult()
        self._chk(self.lib.oserve_gpu_decode_key(self.h, C.c_uint64(key), C.byref(res)))
        return A.result_to_state(res)

    def round(self, mode: int = A.SPACE_ORDERED, sizes: Sequence[int] = (), max_devices: int = 0) -> core.SearchState:
        keep = A.Keep()
        sd = A.space_desc(mode, sizes, max_devices, keep)
        res = A.RoundResult()
        self._chk(self.lib.oserve_gpu_round(self.h, C.byref(sd), C.byref(res)))
        return A.result_to_state(res)

    def round_topk(self, K: int, d_keys_ptr: int, d_best_ptr: int = 0):
        """Top-K packed keys of this shard into device memory (uint64[K])."""
        self._chk(self.lib.oserve_gpu_round_topk(self.h, int(K), C.c_void_p(d_keys_ptr),
                                                 C.c_void_p(d_best_ptr) if d_best_ptr else None))

    def switch_cost_keys(self, current: core.Deployment, d_keys_ptr: int, count: int):
        """Switching cost current -> plan(key) for `count` device-resident keys."""
        keep = A.Keep()
        s = A.deployment_desc(current, keep)
        est = (C.c_double * max(1, count))()
        mb = (C.c_uint64 * max(1, count))()
        self._chk(self.lib.oserve_gpu_switch_cost_keys(self.h, C.byref(s), int(count), C.c_void_p(d_keys_ptr), est, mb))
        return list(est[:count]), list(mb[:count])

    def switch_cost_keys_async(self, current: core.Deployment, d_keys_ptr: int, count: int, d_est_ptr: int):
        """Asynchronous K2 on the context stream; est written to device memory."""
        keep = A.Keep()
        s = A.deployment_desc(current, keep)
        self._chk(self.lib.oserve_gpu_switch_cost_keys_async(self.h, C.byref(s), int(count), C.c_void_p(d_keys_ptr),
                                                             C.c_void_p(d_est_ptr)))

    def search(self, seed: int = 0, max_iters: int = 500, stale_limit: int = 20, mutation_retries: int = 8,
               warm_start: Optional[core.Deployment] = None, log_capacity: int = 1024):
        """search::search (deploysearch.cpp:341-417) -> (SearchState, log rows)."""
        keep = A.Keep()
        o = A.search_options(seed, max_iters, stale_limit, mutation_retries, warm_start, keep)
        res = A.SearchResult()
        log = (A.SearchLogRow * log_capacity)()
        self._chk(self.lib.oserve_gpu_search(self.h, C.byref(o), C.byref(res), log, log_capacity))
        return A.search_outcome(res, log, res.log_count)

    def exhaustive(self) -> core.SearchState:
        res = A.RoundResult()
        self._chk(self.lib.oserve_gpu_exhaustive(self.h, C.byref(res)))
        return A.result_to_state(res)

    def best_strategies(self, sizes: Sequence[int]) -> core.StrategyChoice:
        res = A.RoundResult()
        self._chk(self.lib.oserve_gpu_best_strategies(self.h, len(sizes), A._arr(C.c_int, sizes), C.byref(res)))
        return core.StrategyChoice(A.plan_to_deployment(res.plan), res.objective)

    def evaluate_ranks(self, first: int, count: int) -> Tuple[np.ndarray, np.ndarray]:
        obj = np.zeros(count, np.int64)
        spp = np.zeros(count, np.int32)
        self._chk(self.lib.oserve_gpu_evaluate_ranks(self.h, C.c_uint64(first), C.c_uint64(count),
                                                     _np_ptr(obj, C.c_int64), _np_ptr(spp, C.c_int32)))
        return obj, spp

    def evaluate_deployments(self, deps: Sequence[core.Deployment]) -> List[int]:
        keep = A.Keep()
        arr = A.deployment_desc_array(deps, keep)
        out = (C.c_int64 * max(1, len(deps)))()
        self._chk(self.lib.oserve_gpu_evaluate_deployments(self.h, len(deps), arr, out))
        return list(out[:len(deps)])

    def plan_detail(self, dep: core.Deployment):
        R, J = dep.replica_count(), len(self.types)
        keep = A.Keep()
        d = A.deployment_desc(dep, keep)
        n, e, x, unit = [(C.c_int64 * max(1, R * J))() for _ in range(4)]
        lat = (C.c_double * max(1, R * J))()
        M, used = (C.c_int64 * max(1, R))(), (C.c_int64 * max(1, R))()
        obj = C.c_int64()
        self._chk(self.lib.oserve_gpu_plan_detail(self.h, C.byref(d), n, e, lat, x, M, unit, used, C.byref(obj)))
        table = core.CapacityTable(A.i64_rows(n, R, J), A.i64_rows(e, R, J),
                                   [list(lat[k * J:(k + 1) * J]) for k in range(R)])
        lower = core.LowerLevel(core.AssignmentMatrix(A.i64_rows(x, R, J), obj.value), list(M[:R]),
                                A.i64_rows(unit, R, J), list(used[:R]))
        return table, lower

    def solve_batch(self, n: np.ndarray, e: np.ndarray, lam: np.ndarray):
        """n, e: [count, R, J]; lam: [count, J] -> (x, obj, M, unit, used)."""
        n = np.ascontiguousarray(n, np.int64)
        e = np.ascontiguousarray(e, np.int64)
        lam = np.ascontiguousarray(lam, np.int64)
        cnt, R, J = n.shape
        x = np.zeros((cnt, R, J), np.int64)
        unit = np.zeros((cnt, R, J), np.int64)
        obj = np.zeros(cnt, np.int64)
        M = np.zeros((cnt, R), np.int64)
        used = np.zeros((cnt, R), np.int64)
        P = lambda a: _np_ptr(a, C.c_int64)
        self._chk(self.lib.oserve_gpu_solve_batch(self.h, cnt, R, J, P(n), P(e), P(lam), P(x), P(obj), P(M), P(unit),
                                                  P(used)))
        return x, obj, M, unit, used

    # -- switching ---------------------------------------------------------------
    def switch_cost_batch(self, src: core.Deployment, dsts: Sequence[core.Deployment]):
        keep = A.Keep()
        s = A.deployment_desc(src, keep)
        arr = A.deployment_desc_array(dsts, keep)
        est = (C.c_double * max(1, len(dsts)))()
        mb = (C.c_uint64 * max(1, len(dsts)))()
        self._chk(self.lib.oserve_gpu_switch_cost_batch(self.h, C.byref(s), len(dsts), arr, est, mb))
        return list(est[:len(dsts)]), list(mb[:len(dsts)])

    # -- flow-network formulation (K6, K7) ---------------------------------------
    def max_flow_batch(self, graphs: Sequence[Tuple[int, Sequence[Tuple[int, int, int]]]], sources: Sequence[int],
                       sinks: Sequence[int]):
        """flow::max_flow per graph (num_nodes, [(from, to, cap)]) -> [(value, flows)]."""
        offs = np.zeros(len(graphs) + 1, np.int64)
        offs[1:] = np.cumsum([len(es) for _, es in graphs])
        edges = [e for _, es in graphs for e in es]
        val, fl = self.max_flow_arrays(np.asarray([g[0] for g in graphs], np.int32), offs, edges, sources, sinks)
        return [(int(val[i]), fl[offs[i]:offs[i + 1]].tolist()) for i in range(len(graphs))]

    def max_flow_arrays(self, num_nodes: np.ndarray, edge_offset: np.ndarray, edges, sources, sinks):
        """Array form: num_nodes [G] i32, edge_offset [G+1] i64, edges (flow_edge_dtype or tuples)
        -> (values [G], flows [E])."""
        keep = A.Keep()
        G = len(num_nodes)
        nn = keep(np.ascontiguousarray(num_nodes, dtype=np.int32))
        off = keep(np.ascontiguousarray(edge_offset, dtype=np.int64))
        ed = A.flow_edges(edges, keep)
        E = int(off[-1] - off[0]) if G else 0
        fl = np.empty(max(1, E), np.int64)  # every entry is written
        val = np.empty(max(1, G), np.int64)
        src = keep(np.ascontiguousarray(sources, dtype=np.int32))
        snk = keep(np.ascontiguousarray(sinks, dtype=np.int32))
        self._chk(self.lib.oserve_gpu_max_flow_batch(self.h, G, _np_ptr(nn, C.c_int), _np_ptr(off, C.c_int64), ed,
                                                     _np_ptr(src, C.c_int), _np_ptr(snk, C.c_int),
                                                     _np_ptr(fl, C.c_int64), _np_ptr(val, C.c_int64)))
        return val[:G], fl[:E]

    def flow_assign_batch(self, n: np.ndarray, e: np.ndarray, lam: np.ndarray, edge_flows: bool = False):
        """build_network + max_flow + extract_assignment per instance [count][R][J]."""
        n = np.ascontiguousarray(n, dtype=np.int64)
        e = np.ascontiguousarray(e, dtype=np.int64)
        lam = np.ascontiguousarray(lam, dtype=np.int64)
        cnt, R, J = n.shape
        m = J + 2 * R * J + 2 * R
        x = np.zeros((cnt, R, J), np.int64)
        obj, val = np.zeros(cnt, np.int64), np.zeros(cnt, np.int64)
        fl = np.zeros((cnt, m), np.int64) if edge_flows else None
        p = C.c_int64
        self._chk(self.lib.oserve_gpu_flow_assign_batch(
            self.h, cnt, R, J, _np_ptr(n, p), _np_ptr(e, p), _np_ptr(lam, p), _np_ptr(x, p), _np_ptr(obj, p),
            _np_ptr(val, p), _np_ptr(fl, p) if fl is not None else None))
        return x, obj, val, fl

    def extract_assignment_batch(self, n: np.ndarray, e: np.ndarray, lam: np.ndarray, edge_flow: np.ndarray):
        n = np.ascontiguousarray(n, dtype=np.int64)
        e = np.ascontiguousarray(e, dtype=np.int64)
        lam = np.ascontiguousarray(lam, dtype=np.int64)
        fl = np.ascontiguousarray(edge_flow, dtype=np.int64)
        cnt, R, J = n.shape
        x = np.zeros((cnt, R, J), np.int64)
        obj = np.zeros(cnt, np.int64)
        p = C.c_int64
        self._chk(self.lib.oserve_gpu_extract_assignment_batch(
            self.h, cnt, R, J, _np_ptr(n, p), _np_ptr(e, p), _np_ptr(lam, p), _np_ptr(fl, p), _np_ptr(x, p),
            _np_ptr(obj, p)))
        return x, obj

    def solve_fractional_batch(self, n: np.ndarray, e: np.ndarray, lam: np.ndarray):
        n = np.ascontiguousarray(n, dtype=np.int64)
        e = np.ascontiguousarray(e, dtype=np.int64)
        lam = np.ascontiguousarray(lam, dtype=np.int64)
        cnt, R, J = n.shape
        f = np.zeros((cnt, R, J), np.float64)
        obj = np.zeros(cnt, np.float64)
        p, d = C.c_int64, C.c_double
        self._chk(self.lib.oserve_gpu_solve_fractional_batch(self.h, cnt, R, J, _np_ptr(n, p), _np_ptr(e, p),
                                                             _np_ptr(lam, p), _np_ptr(f, d), _np_ptr(obj, d)))
        return f, obj

    def kv_plan(self, inflight: Sequence[core.InflightRequest], threshold_tokens: int, src: core.Deployment,
                dst: core.Deployment, headroom: float = 0.1, carry: Optional[core.SwitchPlan] = None,
                as_arrays: bool = False):
        """switchplan::kv_plan (switchplan.cpp:142-207) on the device (K5).
        as_arrays: (drained ids, migrated [n,4] int64 rows, buffer_bytes)."""
        keep = A.Keep()
        s, d = A.deployment_desc(src, keep), A.deployment_desc(dst, keep)
        reqs = A.inflight_arr(inflight, keep)
        tr, ntr = A.transfer_arr(carry, keep)
        n = len(inflight)
        # output buffers kept across calls (results are copied out below)
        bufs = getattr(self, "_kv_bufs", None)
        if bufs is None or bufs[0] < n:
            bufs = self._kv_bufs = (max(1, n), (C.c_int64 * max(1, n))(), (A.KvTransferDesc * max(1, n))())
        drained, mig = bufs[1], bufs[2]
        nd, nm, buf = C.c_int(), C.c_int(), C.c_uint64()
        self._chk(self.lib.oserve_gpu_kv_plan(self.h, n, reqs, threshold_tokens, C.byref(s), C.byref(d),
                                              float(headroom), ntr, tr, drained, C.byref(nd), mig, C.byref(nm),
                                              C.byref(buf)))
        if as_arrays:
            return A.kv_arrays(drained, nd.value, mig, nm.value, buf.value)
        return core.KvPlan(list(drained[:nd.value]),
                           [core.KvTransfer(m.request_id, m.kv_bytes, m.src, m.dst) for m in mig[:nm.value]],
                           buf.value)

    # -- reference-signature pieces (switchplan.hpp:34, 57, 61; flowassign.hpp:24-28, 122)
    def layout_shards(self, dep: core.Deployment, param_bytes: int):
        """switchplan::layout shards [(shard_id, begin, end, holder)] (K: k_layout)."""
        keep = A.Keep()
        d = A.deployment_desc(dep, keep)
        n = C.c_int()
        self._chk(self.lib.oserve_gpu_layout(self.h, C.byref(d), int(param_bytes), 0, None, C.byref(n)))
        buf = (A.ShardDesc * max(1, n.value))()
        if n.value:
            self._chk(self.lib.oserve_gpu_layout(self.h, C.byref(d), int(param_bytes), n.value, buf, C.byref(n)))
        return [(b.shard_id, b.begin, b.end, b.holder) for b in buf[:n.value]]

    def greedy_plan_held(self, src_held, dst_held) -> core.SwitchPlan:
        """switchplan::greedy_plan over two `held` maps {device: [(begin, end)]}."""
        def arr(h):
            items = [(d, b, e) for d in sorted(h) for (b, e) in h[d]]
            a = (A.HeldRangeDesc * max(1, len(items)))()
            for i, (d, b, e) in enumerate(items):
                a[i] = A.HeldRangeDesc(int(d), int(b), int(e))
            return a, len(items)
        sa, ns = arr(src_held)
        da, nd = arr(dst_held)
        n, est = C.c_int(), C.c_double()
        self._chk(self.lib.oserve_gpu_greedy_plan_layouts(self.h, ns, sa, nd, da, 0, None, C.byref(n),
                                                          C.byref(est)))
        tr = (A.TransferDesc * max(1, n.value))()
        if n.value:
            self._chk(self.lib.oserve_gpu_greedy_plan_layouts(self.h, ns, sa, nd, da, n.value, tr, C.byref(n),
                                                              C.byref(est)))
        return core.SwitchPlan([core.Transfer(core.ByteRange(t.begin, t.end), t.src, t.dst) for t in tr[:n.value]],
                               est.value)

    def estimate_time(self, links) -> float:
        """switchplan::estimate_time over [(src, dst, bytes)] link loads."""
        a = (A.LinkLoadDesc * max(1, len(links)))()
        for i, (s_, d_, b) in enumerate(links):
            a[i] = A.LinkLoadDesc(int(s_), int(d_), int(b))
        est = C.c_double()
        self._chk(self.lib.oserve_gpu_estimate_time(self.h, len(links), a, C.byref(est)))
        return est.value

    def normalize_batch(self, n: np.ndarray, strict: bool):
        """flow::normalize (strict) / normalize_or_scale per row -> (M, units, scaled)."""
        n = np.ascontiguousarray(n, dtype=np.int64)
        cnt, J = n.shape
        M = np.zeros(cnt, np.int64)
        U = np.zeros((cnt, J), np.int64)
        sc = np.zeros(cnt, np.int32)
        self._chk(self.lib.oserve_gpu_normalize_batch(self.h, cnt, J, _np_ptr(n, C.c_int64), int(strict),
                                                      _np_ptr(M, C.c_int64), _np_ptr(U, C.c_int64),
                                                      _np_ptr(sc, C.c_int)))
        return M, U, sc.astype(bool)

    def check_constraints_batch(self, x: np.ndarray, n: np.ndarray, e: np.ndarray, lam: np.ndarray,
                                raise_first: bool = True):
        """flow::check_constraints per instance -> (kind, replica, type) arrays
        (kind 0 ok, 1 C1, 2 C2, 3 C3 zero-capacity, 4 C3); raises LogicError
        for the first violation unless raise_first is False."""
        x, n, e, lam = (np.ascontiguousarray(v, dtype=np.int64) for v in (x, n, e, lam))
        cnt, R, J = n.shape
        kind, kk, jj = (np.zeros(cnt, np.int32) for _ in range(3))
        st = self.lib.oserve_gpu_check_constraints_batch(self.h, cnt, R, J, _np_ptr(x, C.c_int64),
                                                         _np_ptr(n, C.c_int64), _np_ptr(e, C.c_int64),
                                                         _np_ptr(lam, C.c_int64), _np_ptr(kind, C.c_int),
                                                         _np_ptr(kk, C.c_int), _np_ptr(jj, C.c_int))
        if raise_first or st not in (A.OK, A.ERR_LOGIC):
            self._chk(st)
        return kind, kk, jj

    def switch_plan(self, src: core.Deployment, dst: core.Deployment) -> core.SwitchPlan:
        keep = A.Keep()
        s, d = A.deployment_desc(src, keep), A.deployment_desc(dst, keep)
        ntr, est = C.c_int(), C.c_double()
        cap = 4096  # one call in the common case; the count is reported when it does not fit
        tr = (A.TransferDesc * cap)()
        st = self.lib.oserve_gpu_switch_plan(self.h, C.byref(s), C.byref(d), cap, tr, C.byref(ntr), C.byref(est))
        if st == A.ERR_INVALID_ARGUMENT and ntr.value > cap:
            cap = ntr.value
            tr = (A.TransferDesc * cap)()
            st = self.lib.oserve_gpu_switch_plan(self.h, C.byref(s), C.byref(d), cap, tr, C.byref(ntr), C.byref(est))
        self._chk(st)
        n = ntr.value
        return core.SwitchPlan([core.Transfer(core.ByteRange(t.begin, t.end), t.src, t.dst) for t in tr[:n]],
                               est.value)
