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
