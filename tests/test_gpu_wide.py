"""GPU parity for plans with 65-128 replicas (config 5-7B: 128 devices, 16
classes, 7B-class model so g_min = 1, canonical sizes {1,2,4}: 32..128
replicas per plan).

These reach the paths no other config does: K1 with four replicas per lane
(k_plan_eval<32,4>), K2 with up to 128 source replicas (the QR = 4 holder
search) and plan_detail / solve rows of 96-128 replicas.  Every expectation is
the REFERENCE's own output (tests/golden/plans_cfg5_7b.json, wide.json and
rounds.json["cfg5_7b"], written by oracle/gen_golden.py wide and
oracle/gen_rounds_full.py from oracle/_ref).  Reference: deploysearch.cpp:138-229,
switchplan.cpp:40-140, flowassign.cpp:481-503.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from paper_2602_12151_b200 import core, workloads
from paper_2602_12151_b200._native import GpuContext

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NAME = "cfg5_7b"


def dep_of(rows):
    return core.Deployment([core.ReplicaConfig(i, t, p) for i, t, p in rows])


@pytest.fixture(scope="module")
def w():
    return workloads.load(NAME)


@pytest.fixture(scope="module")
def g(cuda, w):
    ctx = GpuContext(w.cluster, w.model, w.params)
    ctx.set_workload(w.types, w.lam, w.span_s)
    return ctx


def test_space_reaches_128_replicas(g, w):
    p = json.load(open(os.path.join(GOLD, f"plans_{NAME}.json")))
    assert g.min_feasible_group() == 1
    assert g.prepare_space(w.space_mode, w.space_sizes) == (p["partitions"], p["plans"])
    R = np.array(p["R"])
    assert R.max() == 128 and (R > 64).sum() >= 3000


def test_wide_plans_match_reference(g, w):
    """Per-plan objective and sum_pp of 3,709 reference plans (3,009 with
    R > 64), through the K1 <32,4> instantiation (rmax = 128)."""
    p = json.load(open(os.path.join(GOLD, f"plans_{NAME}.json")))
    g.prepare_space(w.space_mode, w.space_sizes)
    bad = []
    for r, o, s in zip(p["ranks"], p["objective"], p["sum_pp"]):
        ob, sp_ = g.evaluate_ranks(int(r), 1)
        if (int(ob[0]), int(sp_[0])) != (o, s):
            bad.append((r, int(ob[0]), o))
    assert not bad, f"{len(bad)} plans differ, first {bad[:5]}"
    # contiguous windows too (greedy-prefix reuse inside a group chunk)
    ranks = np.array(p["ranks"], np.uint64)
    obj = dict(zip(p["ranks"], p["objective"]))
    for r0 in ranks[::97]:
        o, _ = g.evaluate_ranks(int(r0), 1)
        assert int(o[0]) == obj[int(r0)]


def test_wide_round_and_all_plan_digest(g, w):
    rounds = json.load(open(os.path.join(GOLD, "rounds.json")))
    if NAME not in rounds:
        pytest.skip("rounds.json has no cfg5_7b entry yet (oracle/gen_rounds_full.py cfg5_7b)")
    gr = rounds[NAME]
    parts, plans = g.prepare_space(w.space_mode, w.space_sizes)
    st = g.round(w.space_mode, w.space_sizes)
    assert st.throughput == gr["objective"]
    assert (st.partition_index, st.local_rank, st.sum_pp) == (gr["partition_index"], gr["local_rank"], gr["sum_pp"])
    assert [[r.device_ids, r.tp, r.pp] for r in st.deployment.replicas] == gr["deployment"]
    obj, _ = g.evaluate_ranks(0, plans)
    assert int(obj.sum()) == gr["objective_sum"]
    assert hashlib.sha256(np.ascontiguousarray(obj, dtype="<i8").tobytes()).hexdigest() == gr["all_objective_sha256"]


def test_wide_round_is_argmin_of_every_plan(g, w):
    """Full-size property: the fused R-bucketed argmin (one <32,1> and one
    <32,4> launch) equals the key-argmin of every plan's per-plan output."""
    parts, plans = g.prepare_space(w.space_mode, w.space_sizes)
    st = g.round(w.space_mode, w.space_sizes)
    obj, spp = g.evaluate_ranks(0, plans)
    assert st.throughput == int(obj.max())
    p = json.load(open(os.path.join(GOLD, f"plans_{NAME}.json")))
    assert st.throughput >= max(p["objective"])


def test_plan_detail_128_replicas(g, w):
    """build_capacity_table + solve_assignment rows for R = 66..128 plans
    against the reference (n, e, x, M, unit, used, objective)."""
    for case in json.load(open(os.path.join(GOLD, "wide.json")))["detail"]:
        dep = dep_of(case["deployment"])
        table, lower = g.plan_detail(dep)
        assert table.n == case["n"] and table.e == case["e"]
        assert lower.assignment.x == case["x"]
        assert lower.assignment.objective == case["objective"] == case["evaluate_deployment"]
        assert lower.M == case["M"] and lower.unit == case["unit"] and lower.used == case["used"]
        assert g.evaluate_deployments([dep]) == [case["evaluate_deployment"]]


def test_switch_128_source_replicas(g, w):
    """greedy_plan + estimate_time with 65-128 source replicas (K2 QR = 4)
    against the reference's transfer lists."""
    cases = json.load(open(os.path.join(GOLD, "wide.json")))["switch"]
    assert max(len(c["src"]) for c in cases) == 128
    assert sum(1 for c in cases if len(c["src"]) > 64 and c["transfers"]) >= 8
    for c in cases:
        src, dst = dep_of(c["src"]), dep_of(c["dst"])
        plan = g.switch_plan(src, dst)
        assert plan.est_seconds == c["est_seconds"]
        assert [[t.range.begin, t.range.end, t.src, t.dst] for t in plan.transfers] == c["transfers"]
        est, mb = g.switch_cost_batch(src, [dst])
        assert est[0] == c["est_seconds"] and mb[0] == c["max_link_bytes"]


def test_switch_keys_from_128_replica_source(g, w):
    """K2 key mode: init_uniform (128 one-device replicas) and an R > 64 plan
    as the current deployment -> the top-K plans decoded on the device, vs the
    explicit-deployment kernel and the reference's transfer planner."""
    import torch
    parts, plans = g.prepare_space(w.space_mode, w.space_sizes)
    K = 128
    d_keys = torch.empty(K, dtype=torch.int64, device="cuda")
    g.round_topk(K, d_keys.data_ptr())
    states = [g.decode_key(int(k) & ((1 << 64) - 1)) for k in d_keys.cpu().tolist()]
    cases = json.load(open(os.path.join(GOLD, "wide.json")))["switch"]
    currents = [core.canonical_deployment(w.cluster, [1] * 128, [1] * 128)]
    currents += [dep_of(c["src"]) for c in cases if 64 < len(c["src"]) < 128][:3]
    for cur in currents:
        est_k, mb_k = g.switch_cost_keys(cur, d_keys.data_ptr(), K)
        est_x, mb_x = g.switch_cost_batch(cur, [s.deployment for s in states])
        assert est_k == est_x and mb_k == mb_x
    # the explicit kernel is pinned to the reference by test_switch_128_source_replicas
