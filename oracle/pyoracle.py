"""TEST INFRASTRUCTURE ONLY — Python loader for the two CPU oracles.

    Oracle("ref")   oracle/_ref/libref_oserve.so — the unmodified reference
                    (/root/reference/proj/src) behind ref_harness.cpp
    Oracle("port")  oracle/liboserve_port.so — oserve_port.cpp, the CPU
                    restatement of the reference algorithm

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may use
this module; the product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional, Sequence

import numpy as np

from paper_2602_12151_b200 import _abi as A
from paper_2602_12151_b200 import core

HERE = os.path.dirname(os.path.abspath(__file__))
PATHS = {"ref": os.path.join(HERE, "_ref", "libref_oserve.so"),
         "port": os.path.join(HERE, "liboserve_port.so")}


def available(kind: str) -> bool:
    return os.path.exists(PATHS[kind])


class Problem:
    """Cluster + model + profile + workload of one span (an EvalContext)."""

    def __init__(self, cluster: core.ClusterSpec, model: core.ModelSpec,
                 types: Sequence[core.WorkloadType], lam: Sequence[int], span_s: float = 60.0,
                 params: Optional[core.ProfileParams] = None):
        self.cluster, self.model, self.types = cluster, model, list(types)
        self.lam, self.span_s = [int(v) for v in lam], float(span_s)
        self.params = params or core.ProfileParams()
        self.keep = A.Keep()
        self.desc = A.problem_desc(cluster, model, self.params, self.types, self.lam, span_s, self.keep)


class Oracle:
    def __init__(self, kind: str = "port"):
        self.kind = kind
        self.lib = C.CDLL(PATHS[kind], mode=C.RTLD_LOCAL)
        L = self.lib
        L.oracle_last_error.restype = C.c_char_p
        P = C.POINTER
        L.oracle_evaluate_ranks.argtypes = [P(A.ProblemDesc), P(A.SpaceDesc), C.c_int64, P(C.c_uint64),
                                            P(C.c_int64), P(C.c_int32), P(C.c_uint64), C.c_int]
        L.oracle_space_info.argtypes = [P(A.ProblemDesc), P(A.SpaceDesc), P(C.c_int64), P(C.c_uint64)]
        L.oracle_space_plan.argtypes = [P(A.ProblemDesc), P(A.SpaceDesc), C.c_uint64, P(A.Plan),
                                        P(C.c_int64), P(C.c_uint64)]
        L.oracle_round.argtypes = [P(A.ProblemDesc), P(A.SpaceDesc), C.c_int, P(A.RoundResult)]
        L.oracle_switch_plan.argtypes = [P(A.ClusterDesc), C.c_uint64, P(A.DeploymentDesc), P(A.DeploymentDesc),
                                         C.c_int, P(A.TransferDesc), P(C.c_int), P(C.c_double), P(C.c_uint64)]
        L.oracle_fit_types.argtypes = [C.c_int64, P(C.c_uint32), P(C.c_uint32), C.c_int, C.c_uint64,
                                       P(C.c_double), P(C.c_double)]
        L.oracle_holt_forecast.argtypes = [C.c_int, C.c_int, P(C.c_int64), C.c_int, P(C.c_int64)]
        L.oracle_kv_plan.argtypes = [P(A.ClusterDesc), C.c_int, P(A.InflightDesc), C.c_int64, P(A.DeploymentDesc),
                                     P(A.DeploymentDesc), C.c_double, C.c_int, P(A.TransferDesc), P(C.c_int64),
                                     P(C.c_int), P(A.KvTransferDesc), P(C.c_int), P(C.c_uint64)]
        L.oracle_adaptive_timeline_json.argtypes = [P(A.ProblemDesc), C.c_int, P(C.c_int64), C.c_uint64, C.c_int,
                                                    C.c_double, C.c_char_p]
        L.oracle_max_flow.argtypes = [C.c_int, C.c_int, P(A.FlowEdgeDesc), C.c_int, C.c_int, P(C.c_int64),
                                      P(C.c_int64)]
        L.oracle_flow_assign.argtypes = [C.c_int, C.c_int, P(C.c_int64), P(C.c_int64), P(C.c_int64),
                                         P(A.SolveOptionsDesc), P(C.c_int64), P(C.c_int64), P(C.c_int64),
                                         P(C.c_int64)]
        L.oracle_solve_fractional.argtypes = [C.c_int, C.c_int, P(C.c_int64), P(C.c_int64), P(C.c_int64),
                                              P(C.c_double), P(C.c_double)]
        L.oracle_to_dot.argtypes = [C.c_int, C.c_int, P(C.c_int64), P(C.c_int64), P(C.c_int64), C.c_int, C.c_char_p,
                                    C.c_int, P(C.c_int)]
        L.oracle_timeline_resave.argtypes = [C.c_char_p, C.c_char_p, P(C.c_int)]
        L.oracle_deployment_resave.argtypes = [C.c_char_p, C.c_char_p, P(C.c_int)]
        L.oracle_solve_assignment.argtypes = [C.c_int, C.c_int, P(C.c_int64), P(C.c_int64), P(C.c_int64),
                                              P(A.SolveOptionsDesc), P(C.c_int64), P(C.c_int64), P(C.c_int64),
                                              P(C.c_int64), P(C.c_int64), P(C.c_uint64)]
        L.oracle_normalize.argtypes = [C.c_int, P(C.c_int64), C.c_int, P(C.c_int64), P(C.c_int64), P(C.c_int)]

    def _chk(self, st):
        A.raise_for(st, self.lib.oracle_last_error().decode())

    # -- L1/L2 --------------------------------------------------------------
    def capacity_table(self, pr: Problem, dep: core.Deployment):
        R, J = dep.replica_count(), len(pr.types)
        keep = A.Keep()
        d = A.deployment_desc(dep, keep)
        n, e, lat = (C.c_int64 * (R * J))(), (C.c_int64 * (R * J))(), (C.c_double * (R * J))()
        self._chk(self.lib.oracle_capacity_table(C.byref(pr.desc), C.byref(d), n, e, lat))
        return core.CapacityTable(A.i64_rows(n, R, J), A.i64_rows(e, R, J),
                                  [list(lat[k * J:(k + 1) * J]) for k in range(R)])

    def normalize(self, row: Sequence[int], strict: bool = False):
        J = len(row)
        M, units, sc = C.c_int64(), (C.c_int64 * J)(), C.c_int()
        self._chk(self.lib.oracle_normalize(J, A._arr(C.c_int64, row), int(strict), C.byref(M), units,
                                            C.byref(sc)))
        return M.value, list(units), bool(sc.value)

    def solve_assignment(self, n, e, lam, opts: Optional[core.SolveOptions] = None):
        R, J = len(n), len(lam)
        x, M, unit, used = (C.c_int64 * (R * J))(), (C.c_int64 * R)(), (C.c_int64 * (R * J))(), (C.c_int64 * R)()
        obj, work = C.c_int64(), C.c_uint64()
        o = None
        if opts is not None:
            o = C.byref(A.SolveOptionsDesc(opts.exact_demand_limit, opts.exact_cell_limit, opts.node_budget))
        self._chk(self.lib.oracle_solve_assignment(
            R, J, A._arr(C.c_int64, [v for r in n for v in r]), A._arr(C.c_int64, [v for r in e for v in r]),
            A._arr(C.c_int64, lam), o, x, C.byref(obj), M, unit, used, C.byref(work)))
        ll = core.LowerLevel(core.AssignmentMatrix(A.i64_rows(x, R, J), obj.value), list(M),
                             A.i64_rows(unit, R, J), list(used))
        ll.work = work.value
        return ll

    def check_constraints(self, x, n, e, lam):
        R, J = len(n), len(lam)
        f = lambda m: A._arr(C.c_int64, [v for r in m for v in r])
        self._chk(self.lib.oracle_check_constraints(R, J, f(x), f(n), f(e), A._arr(C.c_int64, lam)))

    # -- L3 -----------------------------------------------------------------
    def min_feasible_group(self, pr: Problem) -> int:
        g = C.c_int()
        self._chk(self.lib.oracle_min_feasible_group(C.byref(pr.desc), C.byref(g)))
        return g.value

    def evaluate_deployment(self, pr: Problem, dep: core.Deployment) -> int:
        keep = A.Keep()
        d = A.deployment_desc(dep, keep)
        o = C.c_int64()
        self._chk(self.lib.oracle_evaluate_deployment(C.byref(pr.desc), C.byref(d), C.byref(o)))
        return o.value

    def best_strategies(self, pr: Problem, sizes: Sequence[int], parallel: bool = False):
        res = A.RoundResult()
        self._chk(self.lib.oracle_best_strategies(C.byref(pr.desc), len(sizes), A._arr(C.c_int, sizes),
                                                  int(parallel), C.byref(res)))
        return core.StrategyChoice(A.plan_to_deployment(res.plan), res.objective)

    def exhaustive(self, pr: Problem, parallel: bool = False) -> core.SearchState:
        res = A.RoundResult()
        self._chk(self.lib.oracle_exhaustive(C.byref(pr.desc), int(parallel), C.byref(res)))
        return A.result_to_state(res)

    def space_info(self, pr: Problem, mode: int, sizes: Sequence[int] = (), max_devices: int = 0):
        keep = A.Keep()
        s = A.space_desc(mode, sizes, max_devices, keep)
        parts, plans = C.c_int64(), C.c_uint64()
        self._chk(self.lib.oracle_space_info(C.byref(pr.desc), C.byref(s), C.byref(parts), C.byref(plans)))
        return parts.value, plans.value

    def space_plan(self, pr: Problem, mode: int, rank: int, sizes: Sequence[int] = ()):
        keep = A.Keep()
        s = A.space_desc(mode, sizes, 0, keep)
        plan, pi, lr = A.Plan(), C.c_int64(), C.c_uint64()
        self._chk(self.lib.oracle_space_plan(C.byref(pr.desc), C.byref(s), rank, C.byref(plan),
                                             C.byref(pi), C.byref(lr)))
        return A.plan_to_deployment(plan), pi.value, lr.value

    def evaluate_ranks(self, pr: Problem, mode: int, ranks, sizes: Sequence[int] = (), threads: int = 1):
        keep = A.Keep()
        s = A.space_desc(mode, sizes, 0, keep)
        ranks = np.ascontiguousarray(np.asarray(ranks, dtype=np.uint64))
        n = len(ranks)
        obj = np.zeros(n, np.int64)
        spp = np.zeros(n, np.int32)
        work = np.zeros(n, np.uint64)
        P = lambda a, t: a.ctypes.data_as(C.POINTER(t))
        self._chk(self.lib.oracle_evaluate_ranks(C.byref(pr.desc), C.byref(s), n, P(ranks, C.c_uint64),
                                                 P(obj, C.c_int64), P(spp, C.c_int32), P(work, C.c_uint64),
                                                 threads))
        return obj, spp, work

    def round(self, pr: Problem, mode: int, sizes: Sequence[int] = (), threads: int = 1,
              max_devices: int = 0) -> core.SearchState:
        keep = A.Keep()
        s = A.space_desc(mode, sizes, max_devices, keep)
        res = A.RoundResult()
        self._chk(self.lib.oracle_round(C.byref(pr.desc), C.byref(s), threads, C.byref(res)))
        return A.result_to_state(res)

    # -- L3' ----------------------------------------------------------------
    def switch_plan(self, cl: core.ClusterSpec, param_bytes: int, src: core.Deployment, dst: core.Deployment):
        keep = A.Keep()
        c = A.cluster_desc(cl, keep)
        s, d = A.deployment_desc(src, keep), A.deployment_desc(dst, keep)
        ntr = C.c_int()
        est = C.c_double()
        mx = C.c_uint64()
        self._chk(self.lib.oracle_switch_plan(C.byref(c), param_bytes, C.byref(s), C.byref(d), 0, None,
                                              C.byref(ntr), C.byref(est), C.byref(mx)))
        cap = ntr.value
        tr = (A.TransferDesc * max(1, cap))()
        self._chk(self.lib.oracle_switch_plan(C.byref(c), param_bytes, C.byref(s), C.byref(d), cap, tr,
                                              C.byref(ntr), C.byref(est), C.byref(mx)))
        transfers = [core.Transfer(core.ByteRange(t.begin, t.end), t.src, t.dst) for t in tr[:cap]]
        return core.SwitchPlan(transfers, est.value), mx.value

    def search(self, pr: Problem, seed: int = 0, max_iters: int = 500, stale_limit: int = 20,
               mutation_retries: int = 8, warm_start: Optional[core.Deployment] = None, log_capacity: int = 1024):
        keep = A.Keep()
        o = A.search_options(seed, max_iters, stale_limit, mutation_retries, warm_start, keep)
        res = A.SearchResult()
        log = (A.SearchLogRow * log_capacity)()
        self._chk(self.lib.oracle_search(C.byref(pr.desc), C.byref(o), C.byref(res), log, log_capacity))
        return A.search_outcome(res, log, res.log_count)

    def adaptive_timeline(self, pr: Problem, actual, seed: int = 0, max_iters: int = 150, min_gain: float = 0.01):
        """orch::build_adaptive_timeline (reference only) -> list of entries
        (span_index, deployment, x, switch_seconds, n_transfers)."""
        T, J = len(actual), len(actual[0])
        cap = 64
        si = (C.c_int64 * cap)()
        plans = (A.Plan * cap)()
        x = (C.c_int64 * (cap * 128 * J))()
        sw = (C.c_double * cap)()
        ntr = (C.c_int * cap)()
        n = C.c_int()
        flat = A._arr(C.c_int64, [v for row in actual for v in row])
        self._chk(self.lib.oracle_adaptive_timeline(C.byref(pr.desc), T, flat, C.c_uint64(seed), max_iters,
                                                    C.c_double(min_gain), cap, si, plans, x, sw, ntr, C.byref(n)))
        out = []
        for e in range(min(n.value, cap)):
            dep = A.plan_to_deployment(plans[e])
            R = dep.replica_count()
            xs = [list(x[(e * 128 + k) * J:(e * 128 + k + 1) * J]) for k in range(R)]
            out.append((si[e], dep, xs, sw[e], ntr[e]))
        return out

    # -- workload (reference only) -------------------------------------------
    def fit_types(self, input_len, output_len, k: int, seed: int = 0):
        inp = np.ascontiguousarray(np.asarray(input_len, np.uint32))
        out = np.ascontiguousarray(np.asarray(output_len, np.uint32))
        ci, co = (C.c_double * k)(), (C.c_double * k)()
        self._chk(self.lib.oracle_fit_types(C.c_int64(len(inp)), inp.ctypes.data_as(C.POINTER(C.c_uint32)),
                                            out.ctypes.data_as(C.POINTER(C.c_uint32)), k, C.c_uint64(seed),
                                            ci, co))
        return [core.WorkloadType(c, ci[c], co[c]) for c in range(k)]

    def kv_plan(self, cl: core.ClusterSpec, inflight, threshold_tokens: int, src: core.Deployment,
                dst: core.Deployment, headroom: float = 0.1, carry=None, as_arrays: bool = False):
        keep = A.Keep()
        c = A.cluster_desc(cl, keep)
        s, d = A.deployment_desc(src, keep), A.deployment_desc(dst, keep)
        reqs = A.inflight_arr(inflight, keep)
        tr, ntr = A.transfer_arr(carry, keep)
        n = len(inflight)
        drained = (C.c_int64 * max(1, n))()
        mig = (A.KvTransferDesc * max(1, n))()
        nd, nm, buf = C.c_int(), C.c_int(), C.c_uint64()
        self._chk(self.lib.oracle_kv_plan(C.byref(c), n, reqs, threshold_tokens, C.byref(s), C.byref(d),
                                          float(headroom), ntr, tr, drained, C.byref(nd), mig, C.byref(nm),
                                          C.byref(buf)))
        if as_arrays:
            return A.kv_arrays(drained, nd.value, mig, nm.value, buf.value)
        return core.KvPlan(list(drained[:nd.value]),
                           [core.KvTransfer(m.request_id, m.kv_bytes, m.src, m.dst) for m in mig[:nm.value]],
                           buf.value)

    def adaptive_timeline_json(self, pr: Problem, counts, path: str, seed: int = 0, max_iters: int = 150,
                               min_gain: float = 0.01):
        T = len(counts)
        flat = A._arr(C.c_int64, [v for row in counts for v in row])
        self._chk(self.lib.oracle_adaptive_timeline_json(C.byref(pr.desc), T, flat, C.c_uint64(seed), max_iters,
                                                         min_gain, path.encode()))

    def max_flow(self, num_nodes: int, edges, source: int, sink: int, as_array: bool = False):
        keep = A.Keep()
        ed = A.flow_edges(edges, keep)
        fl = np.zeros(max(1, len(edges)), np.int64)
        v = C.c_int64()
        self._chk(self.lib.oracle_max_flow(num_nodes, len(edges), ed, source, sink,
                                           fl.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(v)))
        return v.value, (fl[:len(edges)] if as_array else fl[:len(edges)].tolist())

    def flow_assign(self, n, e, lam, opts=None):
        """build_network + max_flow + extract_assignment -> (x, objective, value, edge flows)."""
        R, J = len(n), len(lam)
        m = J + 2 * R * J + 2 * R
        fn = A._arr(C.c_int64, [v for r in n for v in r])
        fe = A._arr(C.c_int64, [v for r in e for v in r])
        x, fl = (C.c_int64 * (R * J))(), (C.c_int64 * m)()
        obj, val = C.c_int64(), C.c_int64()
        o = C.byref(A.SolveOptionsDesc(opts.exact_demand_limit, opts.exact_cell_limit, opts.node_budget)) \
            if opts else None
        self._chk(self.lib.oracle_flow_assign(R, J, fn, fe, A._arr(C.c_int64, lam), o, x, C.byref(obj),
                                              C.byref(val), fl))
        return A.i64_rows(x, R, J), obj.value, val.value, list(fl)

    def solve_fractional(self, n, e, lam):
        R, J = len(n), len(lam)
        f, obj = (C.c_double * (R * J))(), C.c_double()
        self._chk(self.lib.oracle_solve_fractional(R, J, A._arr(C.c_int64, [v for r in n for v in r]),
                                                   A._arr(C.c_int64, [v for r in e for v in r]),
                                                   A._arr(C.c_int64, lam), f, C.byref(obj)))
        return [list(f[k * J:(k + 1) * J]) for k in range(R)], obj.value

    def to_dot(self, n, e, lam, with_flow: bool) -> str:
        R, J = len(n), len(lam)
        args = (R, J, A._arr(C.c_int64, [v for r in n for v in r]), A._arr(C.c_int64, [v for r in e for v in r]),
                A._arr(C.c_int64, lam), int(with_flow))
        ln = C.c_int()
        self._chk(self.lib.oracle_to_dot(*args, None, 0, C.byref(ln)))
        buf = C.create_string_buffer(ln.value + 1)
        self._chk(self.lib.oracle_to_dot(*args, buf, ln.value + 1, C.byref(ln)))
        return buf.value.decode()

    def timeline_resave(self, src: str, dst: str) -> int:
        n = C.c_int()
        self._chk(self.lib.oracle_timeline_resave(src.encode(), dst.encode(), C.byref(n)))
        return n.value

    def deployment_resave(self, src: str, dst: str) -> int:
        n = C.c_int()
        self._chk(self.lib.oracle_deployment_resave(src.encode(), dst.encode(), C.byref(n)))
        return n.value

    def holt_forecast(self, counts: List[List[int]], window: int = 50) -> List[List[int]]:
        T, J = len(counts), len(counts[0])
        flat = A._arr(C.c_int64, [v for row in counts for v in row])
        out = (C.c_int64 * (T * J))()
        self._chk(self.lib.oracle_holt_forecast(J, T, flat, window, out))
        return A.i64_rows(out, T, J)
