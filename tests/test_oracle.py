"""CPU oracle pinning (no GPU): the restatement (oracle/liboserve_port.so)
against the reference's own golden vectors (tests/golden, generated from the
reference by oracle/gen_golden.py) and, where built, the reference itself.

Mirrors the reference's test strategy: cost-model and LCM KATs
(test_costmodel.cpp, test_flowassign.cpp:64-99), solver on seeded random
instances incl. the exact path (:209-238), constraint checks, and the
unpinned-by-reference layers (enumeration, selection, switching) checked
against the reference library run here.
"""
import json
import os

import numpy as np
import pytest

from paper_2602_12151_b200 import _abi as A
from paper_2602_12151_b200 import core, workloads

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NCPU = min(8, os.cpu_count() or 1)


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def problem_for(w):
    from pyoracle import Problem
    return Problem(w.cluster, w.model, w.types, w.lam, w.span_s, w.params)


def deps_json(d):
    return [[r.device_ids, r.tp, r.pp] for r in d.replicas]


# ---- L1/L2 known answers ----------------------------------------------------
def test_normalize_kats(port):
    for k in gold("kats.json")["normalize"]:
        M, units, scaled = port.normalize(k["n"])
        assert (M, units, scaled) == (k["M"], k["units"], k["scaled"])
    # test_flowassign.cpp:65-85 literal values
    assert port.normalize([80, 50])[:2] == (400, [5, 8])
    assert port.normalize([12, 18, 30])[:2] == (180, [15, 10, 6])
    assert port.normalize([80, 0, 50])[:2] == (400, [5, 0, 8])
    huge = [(1 << 31) - 1, (1 << 31) - 99, (1 << 31) - 365]
    with pytest.raises(ValueError):
        port.normalize(huge, strict=True)
    M, units, scaled = port.normalize(huge)
    assert scaled and all(h - 1 <= M // u <= h for h, u in zip(huge, units))


def test_capacity_kats(port):
    from pyoracle import Problem
    for k in gold("kats.json")["capacity"]:
        cl = core.cluster(*k["cluster"])
        pr = Problem(cl, core.ModelSpec(**k["model"]), [core.WorkloadType(**t) for t in k["types"]], [0, 0],
                     k["span"], core.ProfileParams(**k["params"]))
        dep = core.Deployment([core.ReplicaConfig(ids, tp, pp) for ids, tp, pp in k["deployment"]])
        t = port.capacity_table(pr, dep)
        assert t.n == k["n"] and t.e == k["e"] and t.latency == k["latency"]
    # test_costmodel.cpp:110-116 and :197-211
    caps = gold("kats.json")["capacity"]
    assert caps[0]["n"] == [[80, 50]]
    assert caps[2]["n"] == [[10, 5], [5, 3], [5, 3]]


def test_assignment_kats(port):
    for k in gold("kats.json")["assignment"]:
        ll = port.solve_assignment(k["n"], k["e"], k["lambda"])
        assert ll.assignment.objective == k["objective"] and ll.assignment.x == k["x"]
        if k["expect"] is not None:
            assert ll.assignment.objective == k["expect"]


def test_solver_matches_reference_goldens(port):
    for inst in gold("solve.json"):
        ll = port.solve_assignment(inst["n"], inst["e"], inst["lambda"])
        assert ll.assignment.objective == inst["objective"]
        assert ll.assignment.x == inst["x"]
        assert ll.M == inst["M"] and ll.unit == inst["unit"] and ll.used == inst["used"]
        port.check_constraints(ll.assignment.x, inst["n"], inst["e"], inst["lambda"])


@pytest.mark.parametrize("name", ["exact_budget.json", "exact_budget_wide.json"])
def test_exact_budget_boundary(port, name):
    """The B&B abort boundary fixtures (reference results at budgets N-1, N,
    N/2 around the node count N): the restatement reproduces every one."""
    for c in gold(name):
        lim = c.get("demand_limit", 400)
        for b in c["budgets"]:
            ll = port.solve_assignment(c["n"], c["e"], c["lambda"], core.SolveOptions(lim, 20, b["budget"]))
            assert ll.assignment.objective == b["objective"] and ll.assignment.x == b["x"], (c["nodes"], b)


def test_check_constraints_detects_violations(port):
    n, e = [[80, 50]], [[80, 50]]
    with pytest.raises(core.LogicError):
        port.check_constraints([[81, 0]], n, e, [100, 0])  # C1 / C2
    with pytest.raises(core.LogicError):
        port.check_constraints([[80, 50]], n, [[80, 50]], [100, 100])  # C3 budget


# ---- L3: enumeration + selection ---------------------------------------------
@pytest.mark.parametrize("name", ["cfg1", "cfg1_bnb"])
def test_exhaustive_matches_golden(port, name):
    w = workloads.load(name)
    s = port.exhaustive(problem_for(w))
    g = gold("rounds.json")[name]
    assert (s.throughput, s.iterations, deps_json(s.deployment)) == (g["objective"], g["iterations"], g["deployment"])
    p = gold(f"plans_{name}.json")
    obj, spp, _ = port.evaluate_ranks(problem_for(w), w.space_mode, np.arange(p["plans"], dtype=np.uint64),
                                      threads=NCPU)
    assert obj.tolist() == p["objective"] and spp.tolist() == p["sum_pp"]


@pytest.mark.parametrize("name", ["cfg2", "cfg2_low"])
def test_ordered_round_matches_golden(port, name):
    w = workloads.load(name)
    pr = problem_for(w)
    p = gold(f"plans_{name}.json")
    assert port.space_info(pr, w.space_mode, w.space_sizes) == (p["partitions"], p["plans"])
    obj, spp, _ = port.evaluate_ranks(pr, w.space_mode, np.asarray(p["ranks"], np.uint64), threads=NCPU)
    assert obj.tolist() == p["objective"] and spp.tolist() == p["sum_pp"]
    s = port.round(pr, w.space_mode, w.space_sizes, threads=NCPU)
    g = gold("rounds.json")[name]
    assert (s.throughput, s.partition_index, s.local_rank, s.sum_pp, deps_json(s.deployment)) == \
        (g["objective"], g["partition_index"], g["local_rank"], g["sum_pp"], g["deployment"])


@pytest.mark.parametrize("name", ["cfg3_70b", "cfg3_7b", "cfg5", "cfg5_low", "cfg5_full"])
def test_canonical_plans_match_golden(port, name):
    w = workloads.load(name)
    pr = problem_for(w)
    p = gold(f"plans_{name}.json")
    assert port.space_info(pr, w.space_mode, w.space_sizes) == (p["partitions"], p["plans"])
    obj, spp, _ = port.evaluate_ranks(pr, w.space_mode, np.asarray(p["ranks"], np.uint64), w.space_sizes,
                                      threads=NCPU)
    assert obj.tolist() == p["objective"] and spp.tolist() == p["sum_pp"]


def test_canonical_round_matches_golden(port):
    w = workloads.load("cfg3_70b")
    s = port.round(problem_for(w), w.space_mode, w.space_sizes, threads=NCPU)
    g = gold("rounds.json")["cfg3_70b"]
    assert (s.throughput, s.partition_index, s.local_rank, deps_json(s.deployment)) == \
        (g["objective"], g["partition_index"], g["local_rank"], g["deployment"])


def test_selection_key_equals_reference_comparator(port, ref):
    """best_strategies' comparator (deploysearch.cpp:47-52) vs the packed
    (obj desc, sum_pp asc, rank asc) order, on every D=16 partition."""
    cl = core.cluster(2, 8)
    w = workloads.load("cfg2")
    from pyoracle import Problem
    pr = Problem(cl, w.model, w.types, [v // 2 for v in w.lam], 60.0, w.params)
    s_ref = ref.exhaustive(pr, parallel=True)
    s_port = port.round(pr, A.SPACE_ORDERED, threads=NCPU)
    assert s_ref.throughput == s_port.throughput
    assert deps_json(s_ref.deployment) == deps_json(s_port.deployment)
    for sizes in ([4, 4, 4, 4], [8, 4, 2, 2], [6, 6, 4], [2] * 8):
        a, b = ref.best_strategies(pr, sizes, parallel=True), port.best_strategies(pr, sizes)
        assert a.objective == b.objective and deps_json(a.deployment) == deps_json(b.deployment)


def test_search_errors(port):
    w = workloads.load("cfg1")
    from pyoracle import Problem
    pr = Problem(core.cluster(4, 8), w.model, w.types, w.lam)
    with pytest.raises(core.TooLarge):
        port.exhaustive(pr)  # D > 16 guard (deploysearch.cpp:440-442)
    big = core.ModelSpec("huge", 10_000 * core.KGB, 80, 1, 1, 10_000 * core.KGB)
    with pytest.raises(core.ModelTooLarge):
        port.exhaustive(Problem(core.cluster(1, 8), big, w.types, w.lam))


# ---- L3': switching ----------------------------------------------------------
def test_switch_matches_golden(port):
    for case in gold("switch.json"):
        w = workloads.load(case["config"])
        src = core.Deployment([core.ReplicaConfig(i, t, p) for i, t, p in case["src"]])
        dst = core.Deployment([core.ReplicaConfig(i, t, p) for i, t, p in case["dst"]])
        plan, mx = port.switch_plan(w.cluster, w.model.param_bytes, src, dst)
        assert plan.est_seconds == case["est_seconds"] and mx == case["max_link_bytes"]
        assert [[t.range.begin, t.range.end, t.src, t.dst] for t in plan.transfers] == case["transfers"]


def test_switch_spec_properties(port):
    """SPEC.md acceptance #8c (src == dst -> empty plan) and #9 (140 GB model,
    2x4 cluster: every resharding <= 15 s and < 50 s reload)."""
    cl = core.cluster(2, 4)
    m = core.model_140gb()
    deps = [core.canonical_deployment(cl, s, t) for s, t in
            (([2, 2, 2, 2], [2, 2, 2, 2]), ([4, 4], [4, 4]), ([4, 4], [2, 1]), ([8], [4]), ([8], [2]),
             ([2, 2, 4], [1, 2, 4]))]
    for a in deps:
        plan, _ = port.switch_plan(cl, m.param_bytes, a, a)
        assert plan.transfers == [] and plan.est_seconds == 0.0
        for b in deps:
            plan, _ = port.switch_plan(cl, m.param_bytes, a, b)
            assert plan.est_seconds <= 15.0 < 50.0


def test_reference_and_port_agree_on_random_pairs(port, ref):
    w = workloads.load("cfg5")
    pr = problem_for(w)
    rng = np.random.default_rng(4)
    _, plans = port.space_info(pr, w.space_mode, w.space_sizes)
    deps = [port.space_plan(pr, w.space_mode, int(r), w.space_sizes)[0] for r in rng.integers(0, plans, 8)]
    for a, b in zip(deps[::2], deps[1::2]):
        pa, ma = port.switch_plan(w.cluster, w.model.param_bytes, a, b)
        pb, mb = ref.switch_plan(w.cluster, w.model.param_bytes, a, b)
        assert pa.est_seconds == pb.est_seconds and ma == mb and len(pa.transfers) == len(pb.transfers)


def test_holt_forecast_matches_reference(port, ref):
    c = workloads.load("cfg4").raw
    assert port.holt_forecast(c["actual"]) == ref.holt_forecast(c["actual"]) == c["forecasts"]
