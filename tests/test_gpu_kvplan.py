"""switchplan::kv_plan (switchplan.cpp:142-207) on the device (K5), against
the reference's own outputs (tests/golden/kv_plan.json, oracle/gen_golden.py)
and, where oracle/_ref is present, against the reference live."""
import json
import os

import numpy as np
import pytest

from paper_2602_12151_b200 import core, workloads
from paper_2602_12151_b200._native import GpuContext

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = json.load(open(os.path.join(ROOT, "tests", "golden", "kv_plan.json")))


def dep(rows):
    return core.Deployment([core.ReplicaConfig(ids, tp, pp) for ids, tp, pp in rows])


def reqs(rows):
    return [core.InflightRequest(*r) for r in rows]


_CTX = {}


def ctx(name):
    if name not in _CTX:
        w = workloads.load(name)
        _CTX[name] = (GpuContext(w.cluster, w.model, w.params), w)
    return _CTX[name]


def carry_of(case):
    if not case["carry"]:
        return None
    sw = json.load(open(os.path.join(ROOT, "tests", "golden", "switch.json")))
    for pair in sw:
        if pair["src"] == case["src"] and pair["dst"] == case["dst"]:
            return core.SwitchPlan([core.Transfer(core.ByteRange(b, e), s, d) for b, e, s, d in pair["transfers"]])
    raise AssertionError("carry plan not found")


@pytest.mark.parametrize("k", range(len(CASES)))
def test_kv_plan_golden(cuda, k):
    c = CASES[k]
    g, _ = ctx(c["config"])
    kv = g.kv_plan(reqs(c["inflight"]), c["threshold"], dep(c["src"]), dep(c["dst"]), c["headroom"], carry_of(c))
    assert kv.drained == c["drained"]
    assert [[m.request_id, m.kv_bytes, m.src, m.dst] for m in kv.migrated] == c["migrated"]
    assert kv.buffer_bytes == c["buffer_bytes"]


def test_kv_plan_errors(cuda):
    g, w = ctx("cfg1")
    d = core.Deployment([core.ReplicaConfig([0, 1], 1, 2), core.ReplicaConfig([2, 3], 2, 1)])
    with pytest.raises(ValueError):
        g.kv_plan([], 10, d, d, headroom=0.6)
    with pytest.raises(ValueError):
        g.kv_plan([], 10, d, d, headroom=-0.1)
    with pytest.raises(ValueError):  # unknown source replica, even when dst is empty
        g.kv_plan([core.InflightRequest(1, 50, 10, 2)], 10, d, core.Deployment())
    # below the threshold the source replica is never looked at
    kv = g.kv_plan([core.InflightRequest(1, 5, 10, 7)], 10, d, d)
    assert kv.drained == [1] and kv.migrated == [] and kv.buffer_bytes == 0


def test_kv_plan_empty_destination(cuda):
    g, _ = ctx("cfg1")
    d = core.Deployment([core.ReplicaConfig([0, 1], 1, 2)])
    kv = g.kv_plan([core.InflightRequest(i, 100 * i, 1 << 20, 0) for i in range(5)], 150, d, core.Deployment())
    assert kv.drained == [0, 1, 2, 3, 4] and kv.migrated == []


def test_kv_plan_live_reference_random(cuda, ref):
    """Irregular clusters, empty replicas and large in-flight sets against the
    reference itself (skipped where oracle/_ref is not built)."""
    rng = np.random.default_rng(5)
    for cl_rows in ([4, 8, 4], [3, 5, 8], [8] * 8):
        machines, nxt = [], 0
        for m, n in enumerate(cl_rows):
            machines.append(core.MachineSpec(m, list(range(nxt, nxt + n)), 80 * core.KGB))
            nxt += n
        cl = core.ClusterSpec(machines, 300e9, 25e9)
        devs = [d for m in cl.machines for d in m.device_ids]
        g = GpuContext(cl, core.small_model())
        for trial in range(6):
            def rand_dep():
                perm = list(rng.permutation(devs))
                out, pos = [], 0
                while pos < len(perm):
                    n = int(rng.integers(1, 5))
                    out.append(core.ReplicaConfig([int(v) for v in perm[pos:pos + n]], 1, n))
                    pos += n
                if trial == 5:
                    out.append(core.ReplicaConfig([], 1, 1))
                return core.Deployment(out)
            src, dst = rand_dep(), rand_dep()
            inflight = [core.InflightRequest(q, int(rng.integers(0, 100)), int(rng.integers(1, 1 << 36)),
                                             int(rng.integers(0, src.replica_count()))) for q in range(3000)]
            a = g.kv_plan(inflight, 40, src, dst, 0.2)
            b = ref.kv_plan(cl, inflight, 40, src, dst, 0.2)
            assert a == b


def test_kv_plan_wide_target_replicas(cuda, ref):
    """Target replicas of more than 32 devices: the replica-parallel kernel
    keeps its state in HBM (the shared-memory form takes <= 32 devices)."""
    rng = np.random.default_rng(6)
    machines = [core.MachineSpec(m, list(range(8 * m, 8 * m + 8)), 80 * core.KGB) for m in range(8)]
    cl = core.ClusterSpec(machines, 300e9, 25e9)
    g = GpuContext(cl, core.small_model())
    for trial in range(3):
        perm = [int(v) for v in rng.permutation(64)]
        dst = core.Deployment([core.ReplicaConfig(perm[:40], 8, 5), core.ReplicaConfig(perm[40:], 4, 6)])
        perm = [int(v) for v in rng.permutation(64)]
        src = core.Deployment([core.ReplicaConfig(perm[i:i + 4], 1, 4) for i in range(0, 64, 4)])
        inflight = [core.InflightRequest(q, int(rng.integers(0, 100)), int(rng.integers(1, 1 << 36)),
                                         int(rng.integers(0, src.replica_count()))) for q in range(4000)]
        assert g.kv_plan(inflight, 30, src, dst, 0.1) == ref.kv_plan(cl, inflight, 30, src, dst, 0.1)
