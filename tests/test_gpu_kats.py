"""The reference tests' known answers and seeded solve instances straight
through the GPU path (no restatement in between).

  kats.json   test_costmodel.cpp (lcm_80_50 / appendix_d fixtures: n, e,
              FP64 latency 0 ulp), test_flowassign.cpp (normalize rows,
              demand-limited 11, {{200,100}x2} -> 150, Appendix-D x)
  solve.json  flow::solve_assignment on 260 seeded instances (incl. the B&B
              path), x / M / unit / used / objective
Both were written by oracle/gen_golden.py from the unmodified reference.
"""
import json
import os

import numpy as np
import pytest

from paper_2602_12151_b200 import core
from paper_2602_12151_b200._native import GpuContext

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def gold(name):
    return json.load(open(os.path.join(GOLD, name)))


def test_capacity_kats(cuda):
    """build_capacity_table on the reference fixtures (costmodel.cpp:94-116)."""
    for k in gold("kats.json")["capacity"]:
        machines, per = k["cluster"]
        cl = core.cluster(machines, per)
        g = GpuContext(cl, core.ModelSpec(**k["model"]), core.ProfileParams(**k["params"]))
        types = [core.WorkloadType(**t) for t in k["types"]]
        g.set_workload(types, [0] * len(types), k["span"])
        dep = core.Deployment([core.ReplicaConfig(i, t, p) for i, t, p in k["deployment"]])
        table, _ = g.plan_detail(dep)
        assert table.n == k["n"] and table.e == k["e"], k["fixture"]
        assert table.latency == k["latency"], k["fixture"]  # FP64, 0 ulp


def test_capacity_kats_module(cuda):
    """The same fixtures through cost.build_capacity_table (cached contexts:
    each fixture twice, the second a cache hit)."""
    from paper_2602_12151_b200 import cost
    for _ in range(2):
        for k in gold("kats.json")["capacity"]:
            machines, per = k["cluster"]
            types = [core.WorkloadType(**t) for t in k["types"]]
            dep = core.Deployment([core.ReplicaConfig(i, t, p) for i, t, p in k["deployment"]])
            table = cost.build_capacity_table(dep, types, core.ModelSpec(**k["model"]), core.cluster(machines, per),
                                              core.ProfileParams(**k["params"]), k["span"])
            assert table.n == k["n"] and table.e == k["e"] and table.latency == k["latency"], k["fixture"]
            [t2] = cost.build_capacity_tables([dep], types, core.ModelSpec(**k["model"]),
                                              core.cluster(machines, per), core.ProfileParams(**k["params"]), k["span"])
            assert t2.n == table.n and t2.latency == table.latency


def test_assignment_kats(cuda):
    g = GpuContext(core.cluster(1, 8), core.model_140gb())
    for k in gold("kats.json")["assignment"]:
        n, e, lam = (np.array([v], np.int64) for v in (k["n"], k["e"], k["lambda"]))
        x, obj, _, _, _ = g.solve_batch(n, e, lam)
        assert int(obj[0]) == k["objective"]
        assert x[0].tolist() == k["x"]
        if k["expect"] is not None:
            assert int(obj[0]) == k["expect"]


def test_solve_instances_reference(cuda):
    """solve.json instance by instance (each its own R x J)."""
    g = GpuContext(core.cluster(1, 8), core.model_140gb())
    cases = gold("solve.json")
    groups = {}
    for c in cases:
        groups.setdefault((len(c["n"]), len(c["lambda"])), []).append(c)
    seen = 0
    for (R, J), cs in groups.items():
        n = np.array([c["n"] for c in cs], np.int64)
        e = np.array([c["e"] for c in cs], np.int64)
        lam = np.array([c["lambda"] for c in cs], np.int64)
        x, obj, M, unit, used = g.solve_batch(n, e, lam)
        for i, c in enumerate(cs):
            assert int(obj[i]) == c["objective"], (R, J, i)
            assert x[i].tolist() == c["x"], (R, J, i)
            assert M[i].tolist() == c["M"] and unit[i].tolist() == c["unit"] and used[i].tolist() == c["used"]
            seen += 1
    assert seen == len(cases) == 260


def test_normalize_kats_on_gpu(cuda):
    """flow::normalize / normalize_or_scale rows of test_flowassign.cpp:64-99
    through K0b (kats.json from the reference)."""
    from paper_2602_12151_b200 import flow
    for k in gold("kats.json")["normalize"]:
        r = flow.normalize_or_scale(k["n"])
        assert (r.M, r.units, r.scaled) == (k["M"], k["units"], k["scaled"])
        if k["scaled"]:
            with pytest.raises(core.LcmOverflow):
                flow.normalize(k["n"])
        else:
            r2 = flow.normalize(k["n"])
            assert (r2.M, r2.units, r2.scaled) == (k["M"], k["units"], False)
    with pytest.raises(ValueError):
        flow.normalize([-1, 3])


def test_check_constraints_matches_reference(cuda, port, ref):
    """flow::check_constraints on seeded (often perturbed) assignments: the
    same verdict and the same message as the reference itself
    (flowassign.cpp:529-551, oracle/_ref)."""
    from paper_2602_12151_b200 import flow
    rng = np.random.default_rng(21)
    seen = {0: 0, 1: 0}
    for trial in range(300):
        R, J = int(rng.integers(1, 5)), int(rng.integers(1, 5))
        n = rng.integers(0, 31, (R, J))
        n[rng.random((R, J)) < 0.2] = 0
        e = (rng.random((R, J)) * (n + 1)).astype(np.int64)
        lam = rng.integers(0, 40, J)
        x = np.array(port.solve_assignment(n.tolist(), e.tolist(), lam.tolist()).assignment.x)
        if trial % 2:
            x[rng.integers(0, R), rng.integers(0, J)] += int(rng.integers(1, 4))
        table = core.CapacityTable(n.tolist(), e.tolist(), [[0.1] * J for _ in range(R)])
        try:
            ref.check_constraints(x.tolist(), n.tolist(), e.tolist(), lam.tolist())
            exp = None
        except Exception as ex:  # noqa: BLE001
            exp = str(ex)
        try:
            flow.check_constraints(core.AssignmentMatrix(x.tolist(), 0), table, lam.tolist())
            got = None
        except core.LogicError as ex:
            got = str(ex)
        assert got == exp, (trial, got, exp)
        seen[got is None] += 1
    assert seen[0] > 50 and seen[1] > 50


@pytest.mark.parametrize("name", ["cfg2", "cfg5", "cfg5_7b"])
def test_layout_greedy_plan_estimate_time(cuda, port, name):
    """switchplan::layout / greedy_plan(ShardLayout...) / estimate_time one for
    one (orchestrate.cpp:142-144) against layout+greedy_plan of the CPU oracle;
    layouts from the device are checked against the reference's slicing rule
    (switchplan.cpp:40-63)."""
    from paper_2602_12151_b200 import switchplan, workloads
    from pyoracle import Problem
    w = workloads.load(name)
    pr = Problem(w.cluster, w.model, w.types, w.lam, w.span_s, w.params)
    parts, plans = port.space_info(pr, w.space_mode, w.space_sizes)
    rng = np.random.default_rng(8)
    deps = [port.space_plan(pr, w.space_mode, int(r), w.space_sizes)[0] for r in rng.integers(0, plans, 10)]
    P = w.model.param_bytes
    for d in deps[:3]:
        lay = switchplan.layout(d, w.model)
        sid = 0
        for rep in d.replicas:
            devs = sorted(rep.device_ids)
            for s in range(rep.pp):
                sb, se = P * s // rep.pp, P * (s + 1) // rep.pp
                for i in range(rep.tp):
                    sh = lay.shards[sid]
                    assert (sh.shard_id, sh.range.begin, sh.range.end, sh.holder) == \
                        (sid, sb + (se - sb) * i // rep.tp, sb + (se - sb) * (i + 1) // rep.tp, devs[s * rep.tp + i])
                    sid += 1
        assert sid == len(lay.shards)
    for a, b in zip(deps[::2], deps[1::2]):
        plan = switchplan.greedy_plan(switchplan.layout(a, w.model), switchplan.layout(b, w.model), w.cluster)
        exp, _ = port.switch_plan(w.cluster, P, a, b)
        assert [(t.range.begin, t.range.end, t.src, t.dst) for t in plan.transfers] == \
            [(t.range.begin, t.range.end, t.src, t.dst) for t in exp.transfers]
        assert plan.est_seconds == exp.est_seconds
        assert switchplan.estimate_time(plan, w.cluster) == exp.est_seconds
