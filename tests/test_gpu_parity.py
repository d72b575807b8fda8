"""GPU parity: the sm_100a path (through the C-ABI) against the CPU oracle.

Bar (BASELINE.json north star): per-plan objectives, chosen plan and
assignment bit-exact; cost cells (FP64 latency) bit-exact (tolerance stated:
0 ulp; the north star allows 1e-6 relative); switching estimates exact.
The oracle is oracle/liboserve_port.so (restatement pinned to the reference
in test_oracle.py) and, where present, oracle/_ref (the reference itself).
"""
import os

import numpy as np
import pytest

from paper_2602_12151_b200 import _abi as A
from paper_2602_12151_b200 import core, workloads
from paper_2602_12151_b200._native import GpuContext

pytestmark = pytest.mark.gpu

NCPU = os.cpu_count() or 1


def ctx_for(w: workloads.Workload) -> GpuContext:
    g = GpuContext(w.cluster, w.model, w.params)
    g.set_workload(w.types, w.lam, w.span_s)
    return g


def problem_for(w: workloads.Workload):
    from pyoracle import Problem
    return Problem(w.cluster, w.model, w.types, w.lam, w.span_s, w.params)


def same_deployment(a: core.Deployment, b: core.Deployment):
    return [(r.device_ids, r.tp, r.pp) for r in a.replicas] == [(r.device_ids, r.tp, r.pp) for r in b.replicas]


@pytest.mark.parametrize("name", ["cfg1", "cfg1_bnb"])
def test_cfg1_exhaustive_matches_reference(cuda, port, name):
    w = workloads.load(name)
    g = ctx_for(w)
    got = g.exhaustive()
    exp = port.exhaustive(problem_for(w))
    assert got.throughput == exp.throughput
    assert got.iterations == exp.iterations == 7
    assert same_deployment(got.deployment, exp.deployment)
    assert g.launch_count() > 0


@pytest.mark.parametrize("name", ["cfg1", "cfg1_bnb", "cfg2_low"])
def test_every_plan_objective_small(cuda, port, name):
    w = workloads.load(name)
    g = ctx_for(w)
    parts, plans = g.prepare_space(w.space_mode, w.space_sizes)
    assert (parts, plans) == port.space_info(problem_for(w), w.space_mode, w.space_sizes)
    obj, spp = g.evaluate_ranks(0, plans)
    ranks = np.arange(plans, dtype=np.uint64)
    eo, es, _ = port.evaluate_ranks(problem_for(w), w.space_mode, ranks, w.space_sizes, threads=NCPU)
    bad = np.nonzero(obj != eo)[0]
    assert bad.size == 0, f"{bad.size} plan objectives differ, first ranks {bad[:10]}: gpu {obj[bad[:10]]} cpu {eo[bad[:10]]}"
    assert np.array_equal(spp, es)


def test_cfg2_every_plan_and_winner(cuda, port):
    w = workloads.load("cfg2")
    g = ctx_for(w)
    parts, plans = g.prepare_space(w.space_mode, w.space_sizes)
    assert (parts, plans) == (1507, 933333)
    obj, spp = g.evaluate_ranks(0, plans)
    pr = problem_for(w)
    eo, es, _ = port.evaluate_ranks(pr, w.space_mode, np.arange(plans, dtype=np.uint64), w.space_sizes, threads=NCPU)
    bad = np.nonzero(obj != eo)[0]
    assert bad.size == 0, f"{bad.size} of {plans} differ; first {bad[:10]} gpu {obj[bad[:10]]} cpu {eo[bad[:10]]}"
    got = g.round(w.space_mode, w.space_sizes)
    exp = port.round(pr, w.space_mode, w.space_sizes, threads=NCPU)
    assert (got.throughput, got.partition_index, got.local_rank, got.sum_pp) == \
        (exp.throughput, exp.partition_index, exp.local_rank, exp.sum_pp)
    assert same_deployment(got.deployment, exp.deployment)


@pytest.mark.parametrize("name", ["cfg3_70b", "cfg3_7b", "cfg5", "cfg5_low", "cfg5_full"])
def test_sampled_plans_large(cuda, port, name):
    w = workloads.load(name)
    g = ctx_for(w)
    parts, plans = g.prepare_space(w.space_mode, w.space_sizes)
    pr = problem_for(w)
    assert (parts, plans) == port.space_info(pr, w.space_mode, w.space_sizes)
    rng = np.random.default_rng(12151)
    n = 4000 if name.startswith("cfg5") else 20000
    starts = rng.integers(0, plans - 8, n // 8)
    ranks = np.unique((starts[:, None] + np.arange(8)[None, :]).ravel()).astype(np.uint64)
    gpu = np.zeros(len(ranks), np.int64)
    # contiguous windows through evaluate_ranks
    for s in starts:
        o, _ = g.evaluate_ranks(int(s), 8)
        idx = np.searchsorted(ranks, np.arange(s, s + 8, dtype=np.uint64))
        gpu[idx] = o
    eo, _, _ = port.evaluate_ranks(pr, w.space_mode, ranks, w.space_sizes, threads=NCPU)
    bad = np.nonzero(gpu != eo)[0]
    assert bad.size == 0, f"{bad.size} differ; ranks {ranks[bad[:10]]} gpu {gpu[bad[:10]]} cpu {eo[bad[:10]]}"


@pytest.mark.parametrize("name", ["cfg3_70b", "cfg5"])
def test_round_winner_is_argmin_of_all_plans(cuda, port, name):
    """Size-independent property at full size: the fused argmin equals the
    key-argmin over every plan's (objective, partition, sum_pp, rank) as
    produced by the per-plan path, and the winner re-evaluates identically on
    the CPU oracle."""
    w = workloads.load(name)
    g = ctx_for(w)
    parts, plans = g.prepare_space(w.space_mode, w.space_sizes)
    got = g.round(w.space_mode, w.space_sizes)
    obj, spp = g.evaluate_ranks(0, plans)
    best = obj.max()
    assert got.throughput == best
    cand = np.nonzero(obj == best)[0]
    pr = problem_for(w)
    # decode partition of each candidate via the oracle's enumeration
    keyed = []
    for r in cand[:2000]:
        dep, pi, lr = port.space_plan(pr, w.space_mode, int(r), w.space_sizes)
        keyed.append((pi, int(spp[r]), lr, int(r)))
    keyed.sort()
    pi, s, lr, r = keyed[0]
    assert (got.partition_index, got.sum_pp, got.local_rank) == (pi, s, lr)
    assert port.evaluate_deployment(pr, got.deployment) == got.throughput


def test_plan_detail_matches_capacity_table_and_assignment(cuda, port):
    w = workloads.load("cfg5")
    g = ctx_for(w)
    pr = problem_for(w)
    parts, plans = g.prepare_space(w.space_mode, w.space_sizes)
    rng = np.random.default_rng(3)
    for r in rng.integers(0, plans, 6):
        dep, _, _ = port.space_plan(pr, w.space_mode, int(r), w.space_sizes)
        table, lower = g.plan_detail(dep)
        exp = port.capacity_table(pr, dep)
        assert table.n == exp.n and table.e == exp.e
        assert table.latency == exp.latency  # bit-exact FP64 (0 ulp)
        ll = port.solve_assignment(exp.n, exp.e, w.lam)
        assert lower.assignment.x == ll.assignment.x
        assert lower.assignment.objective == ll.assignment.objective
        assert lower.M == ll.M and lower.unit == ll.unit and lower.used == ll.used


@pytest.mark.parametrize("seed,maxr,maxj,maxlam,count", [(7, 3, 3, 60, 400), (11, 6, 5, 500, 1000),
                                                         (13, 16, 8, 4000, 300), (17, 40, 16, 20000, 100)])
def test_solve_batch_random_instances(cuda, port, seed, maxr, maxj, maxlam, count):
    """flow::solve_assignment on raw tables (test_flowassign.cpp:24-47 style,
    incl. zero-capacity cells; small ones take the exact B&B path)."""
    rng = np.random.default_rng(seed)
    g = GpuContext(core.cluster(1, 8), core.model_140gb())
    for R in sorted(set(rng.integers(1, maxr + 1, 4).tolist())):
        for J in sorted(set(rng.integers(1, maxj + 1, 3).tolist())):
            n = rng.integers(1, 101 if maxlam <= 500 else 2000, (count, R, J))
            n[rng.random((count, R, J)) < 0.125] = 0
            e = (rng.random((count, R, J)) * (n + 1)).astype(np.int64)
            lam = rng.integers(0, maxlam + 1, (count, J))
            x, obj, M, unit, used = g.solve_batch(n, e, lam)
            for i in range(count):
                ll = port.solve_assignment(n[i].tolist(), e[i].tolist(), lam[i].tolist())
                assert obj[i] == ll.assignment.objective, (R, J, i)
                assert x[i].tolist() == ll.assignment.x, (R, J, i)
                assert M[i].tolist() == ll.M and unit[i].tolist() == ll.unit and used[i].tolist() == ll.used


def _random_plans(port, pr, mode, sizes, plans, rng, k):
    return [port.space_plan(pr, mode, int(r), sizes)[0] for r in rng.integers(0, plans, k)]


@pytest.mark.parametrize("name", ["cfg2", "cfg5"])
def test_switch_cost_matches_greedy_plan(cuda, port, name):
    w = workloads.load(name)
    g = ctx_for(w)
    pr = problem_for(w)
    parts, plans = g.prepare_space(w.space_mode, w.space_sizes)
    rng = np.random.default_rng(5)
    deps = _random_plans(port, pr, w.space_mode, w.space_sizes, plans, rng, 40)
    src = deps[0]
    est, mb = g.switch_cost_batch(src, deps)
    for d, e, m in zip(deps, est, mb):
        plan, emax = port.switch_plan(w.cluster, w.model.param_bytes, src, d)
        assert e == plan.est_seconds and m == emax
    # full transfer list of a few pairs
    for d in deps[1:5]:
        got = g.switch_plan(src, d)
        exp, _ = port.switch_plan(w.cluster, w.model.param_bytes, src, d)
        assert got.est_seconds == exp.est_seconds
        assert [(t.range.begin, t.range.end, t.src, t.dst) for t in got.transfers] == \
            [(t.range.begin, t.range.end, t.src, t.dst) for t in exp.transfers]
    assert g.switch_cost_batch(src, [src])[0] == [0.0]


def test_best_strategies_dropin(cuda, port):
    w = workloads.load("cfg2")
    g = ctx_for(w)
    pr = problem_for(w)
    for sizes in ([2] * 16, [8, 8, 8, 8], [16, 6, 4, 2, 2, 2], [5, 3], [1, 1], [32]):
        got = g.best_strategies(sizes)
        exp = port.best_strategies(pr, sizes)
        assert got.objective == exp.objective, sizes
        assert same_deployment(got.deployment, exp.deployment), sizes


@pytest.mark.parametrize("name,K", [("cfg3_70b", 1024), ("cfg2", 512), ("cfg5", 256)])
def test_topk_round_and_switch_batch(cuda, port, name, K):
    """Exact top-K of the packed key over the whole space (checked against
    every plan's objective from the per-plan path and the oracle's key
    fields), then the switching cost from init_uniform to each of the K plans
    decoded on the device (K2 key mode) vs explicit deployments and the CPU."""
    import torch
    w = workloads.load(name)
    g = ctx_for(w)
    pr = problem_for(w)
    parts, plans = g.prepare_space(w.space_mode, w.space_sizes)
    d_keys = torch.empty(K, dtype=torch.int64, device="cuda")
    d_best = torch.empty(1, dtype=torch.int64, device="cuda")
    g.round_topk(K, d_keys.data_ptr(), d_best.data_ptr())
    keys = [int(k) & ((1 << 64) - 1) for k in d_keys.cpu().tolist()]
    assert keys == sorted(keys) and len(set(keys)) == K
    assert keys[0] == int(d_best.item()) == g.round(w.space_mode, w.space_sizes).key
    obj, spp = g.evaluate_ranks(0, plans)
    states = [g.decode_key(k) for k in keys]
    kth_obj = states[-1].throughput
    cand = np.nonzero(obj >= kth_obj)[0]
    assert len(cand) < 200000
    from paper_2602_12151_b200 import _native
    lay = None
    full = []
    for r in cand:
        dep, pi, lr = port.space_plan(pr, w.space_mode, int(r), w.space_sizes)
        full.append((-int(obj[r]), pi, int(spp[r]), lr))
    full.sort()
    exp = [(-s.throughput, s.partition_index, s.sum_pp, s.local_rank) for s in states]
    assert full[:K] == exp
    # switching batch: K2 key mode == K2 explicit == greedy_plan on the CPU
    gm = g.min_feasible_group()
    R = w.cluster.device_count() // gm
    current = core.canonical_deployment(w.cluster, [gm] * R, [gm] * R)
    est_k, mb_k = g.switch_cost_keys(current, d_keys.data_ptr(), K)
    est_x, mb_x = g.switch_cost_batch(current, [s.deployment for s in states])
    assert est_k == est_x and mb_k == mb_x
    for s, e in list(zip(states, est_k))[:: max(1, K // 16)]:
        plan, _ = port.switch_plan(w.cluster, w.model.param_bytes, current, s.deployment)
        assert e == plan.est_seconds


GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("name", ["cfg1", "cfg1_bnb", "cfg2", "cfg2_low", "cfg3_70b", "cfg3_7b", "cfg5", "cfg5_low",
                                  "cfg5_full"])
def test_gpu_matches_reference_goldens(cuda, name):
    """GPU per-plan objectives against the REFERENCE's own values (tests/golden,
    generated from the unmodified reference by oracle/gen_golden.py)."""
    import json
    w = workloads.load(name)
    g = ctx_for(w)
    p = json.load(open(os.path.join(GOLD, f"plans_{name}.json")))
    parts, plans = g.prepare_space(w.space_mode, w.space_sizes)
    assert (parts, plans) == (p["partitions"], p["plans"])
    if "all_objective_sha256" in p:
        import hashlib
        obj, _ = g.evaluate_ranks(0, plans)
        assert hashlib.sha256(np.ascontiguousarray(obj, dtype="<i8").tobytes()).hexdigest() == p["all_objective_sha256"]
        assert int(obj.sum()) == p["objective_sum"]
    for r, o, s in zip(p["ranks"], p["objective"], p["sum_pp"]):
        ob, sp_ = g.evaluate_ranks(int(r), 1)
        assert (int(ob[0]), int(sp_[0])) == (o, s), r
    rounds = json.load(open(os.path.join(GOLD, "rounds.json")))
    if name in rounds:
        gr = rounds[name]
        st = g.exhaustive() if name.startswith("cfg1") else g.round(w.space_mode, w.space_sizes)
        assert st.throughput == gr["objective"]
        assert [[r.device_ids, r.tp, r.pp] for r in st.deployment.replicas] == gr["deployment"]
        if "local_rank" in gr:
            assert (st.partition_index, st.local_rank, st.sum_pp) == \
                (gr["partition_index"], gr["local_rank"], gr["sum_pp"])
        if "all_objective_sha256" in gr:  # every plan of the space, full size (oracle/gen_rounds_full.py)
            import hashlib
            obj, _ = g.evaluate_ranks(0, plans)
            assert int(obj.sum()) == gr["objective_sum"]
            assert hashlib.sha256(np.ascontiguousarray(obj, dtype="<i8").tobytes()).hexdigest() == \
                gr["all_objective_sha256"]


def test_gpu_switch_matches_reference_goldens(cuda):
    import json
    for case in json.load(open(os.path.join(GOLD, "switch.json"))):
        w = workloads.load(case["config"])
        g = GpuContext(w.cluster, w.model, w.params)
        src = core.Deployment([core.ReplicaConfig(i, t, p) for i, t, p in case["src"]])
        dst = core.Deployment([core.ReplicaConfig(i, t, p) for i, t, p in case["dst"]])
        plan = g.switch_plan(src, dst)
        assert plan.est_seconds == case["est_seconds"]
        assert [[t.range.begin, t.range.end, t.src, t.dst] for t in plan.transfers] == case["transfers"]
        est, mb = g.switch_cost_batch(src, [dst])
        assert est[0] == case["est_seconds"] and mb[0] == case["max_link_bytes"]


@pytest.mark.parametrize("seed", range(5))
def test_exact_path_random_demands(cuda, port, seed):
    """The branch-and-bound path (every config 1-B&B plan takes it: sum of
    lambda <= 400) at seeded random demands: every plan's objective against
    the restatement (node budget, aborts and heuristic fallthrough included)
    and the exhaustive winner."""
    w = workloads.load("cfg1_bnb")
    rng = np.random.default_rng(900 + seed)
    total = int(rng.integers(40, 401))
    a = int(rng.integers(0, total + 1))
    w.lam = [a, total - a][:len(w.lam)] + [0] * max(0, len(w.lam) - 2)
    g = ctx_for(w)
    parts, plans = g.prepare_space(w.space_mode, w.space_sizes)
    obj, spp = g.evaluate_ranks(0, plans)
    eo, es, _ = port.evaluate_ranks(problem_for(w), w.space_mode, np.arange(plans, dtype=np.uint64), w.space_sizes,
                                    threads=NCPU)
    assert np.array_equal(obj, eo) and np.array_equal(spp, es), (w.lam, np.nonzero(obj != eo)[0][:10])
    got = g.exhaustive()
    exp = port.exhaustive(problem_for(w))
    assert got.throughput == exp.throughput and same_deployment(got.deployment, exp.deployment)
