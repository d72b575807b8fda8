"""Edge cases and error behaviour of the GPU path (through the C-ABI),
against the CPU oracle: the reference's exception types, irregular clusters
(unequal machine sizes, unaligned blocks), non-uniform device memory, a
single class, D = 16 exhaustive, limits."""
import os

import numpy as np
import pytest

from paper_2602_12151_b200 import _abi as A
from paper_2602_12151_b200 import core, workloads
from paper_2602_12151_b200._native import GpuContext

pytestmark = pytest.mark.gpu
NCPU = os.cpu_count() or 1


def make(cl, model, types, lam, params=None):
    g = GpuContext(cl, model, params or core.ProfileParams())
    g.set_workload(types, lam, 60.0)
    return g


def problem(cl, model, types, lam, params=None):
    from pyoracle import Problem
    return Problem(cl, model, types, lam, 60.0, params or core.ProfileParams())


def shapes(d):
    return [(r.device_ids, r.tp, r.pp) for r in d.replicas]


def test_errors_map_to_reference_exceptions(cuda):
    types = [core.short_type(), core.long_type()]
    g = make(core.cluster(4, 8), core.model_140gb(), types, [700, 300])
    with pytest.raises(core.TooLarge):          # exhaustive guard (deploysearch.cpp:440-442)
        g.exhaustive()
    with pytest.raises(ValueError):             # canonical_blocks (deploysearch.cpp:93-95)
        g.best_strategies([16, 16, 8])
    with pytest.raises(core.InfeasibleReplica):  # build_capacity_table (costmodel.cpp:105-107)
        g.evaluate_deployments([core.canonical_deployment(g.cluster, [1], [1])])
    assert g.evaluate_deployments([core.Deployment()]) == [0]  # empty -> 0 (deploysearch.cpp:139)
    big = core.ModelSpec("huge", 10_000 * core.KGB, 80, 1, 1, 10_000 * core.KGB)
    gb = make(core.cluster(1, 8), big, types, [700, 300])
    with pytest.raises(core.ModelTooLarge):     # min_feasible_group (deploysearch.cpp:86)
        gb.exhaustive()
    with pytest.raises(core.UnsourcedFragment):  # greedy_plan (switchplan.cpp:99-103)
        g.switch_plan(core.Deployment(), core.canonical_deployment(g.cluster, [8], [8]))
    with pytest.raises(core.Unsupported):
        g.set_workload(types, [2 ** 31, 1], 60.0)
    with pytest.raises(ValueError):
        g.set_workload(types, [-1, 1], 60.0)
    with pytest.raises(ValueError):             # normalize (flowassign.cpp:36)
        g.solve_batch(np.array([[[-1, 2]]]), np.array([[[1, 1]]]), np.array([[1, 1]]))
    # best_strategies on an infeasible partition: empty choice, objective 0 (:163, :227)
    ch = g.best_strategies([1, 1])
    assert ch.objective == 0 and ch.deployment.replicas == []


def test_d16_exhaustive_matches_reference(cuda, port):
    w = workloads.load("cfg2")
    cl = core.cluster(2, 8)
    lam = [v // 2 for v in w.lam]
    g = make(cl, w.model, w.types, lam)
    got = g.exhaustive()
    exp = port.exhaustive(problem(cl, w.model, w.types, lam))
    assert (got.throughput, got.iterations, shapes(got.deployment)) == \
        (exp.throughput, exp.iterations, shapes(exp.deployment))


@pytest.mark.parametrize("machines", [[4, 8, 4], [3, 5, 8], [6, 6, 4]])
def test_irregular_cluster_every_plan(cuda, port, machines):
    """Unequal machine sizes: tp groups that straddle a machine boundary must
    be rejected exactly like validate_replica (core.cpp:105-127)."""
    ms, dev = [], 0
    for i, n in enumerate(machines):
        ms.append(core.MachineSpec(f"m{i}", list(range(dev, dev + n)), 80 * core.KGB))
        dev += n
    cl = core.ClusterSpec(ms, 400e9, 200e9)
    w = workloads.load("cfg2")
    lam = [v // 2 for v in w.lam]
    g = make(cl, w.model, w.types, lam)
    parts, plans = g.prepare_space(A.SPACE_ORDERED)
    pr = problem(cl, w.model, w.types, lam)
    assert (parts, plans) == port.space_info(pr, A.SPACE_ORDERED)
    n = min(plans, 200000)
    obj, spp = g.evaluate_ranks(0, n)
    eo, es, _ = port.evaluate_ranks(pr, A.SPACE_ORDERED, np.arange(n, dtype=np.uint64), threads=NCPU)
    assert np.array_equal(obj, eo) and np.array_equal(spp, es)
    got = g.round(A.SPACE_ORDERED)
    exp = port.round(pr, A.SPACE_ORDERED, threads=NCPU)
    assert (got.throughput, got.partition_index, got.local_rank) == (exp.throughput, exp.partition_index,
                                                                     exp.local_rank)


def test_nonuniform_memory_cluster(cuda, port):
    """Machines with different device memory: cost rows keyed by the block's
    total memory (shape = (tp, pp, sum mem))."""
    ms = [core.MachineSpec("a", list(range(0, 8)), 80 * core.KGB),
          core.MachineSpec("b", list(range(8, 16)), 192 * core.KGB)]
    cl = core.ClusterSpec(ms, 400e9, 200e9)
    w = workloads.load("cfg2")
    lam = [v // 3 for v in w.lam]
    g = make(cl, w.model, w.types, lam)
    parts, plans = g.prepare_space(A.SPACE_ORDERED)
    pr = problem(cl, w.model, w.types, lam)
    obj, _ = g.evaluate_ranks(0, plans)
    eo, _, _ = port.evaluate_ranks(pr, A.SPACE_ORDERED, np.arange(plans, dtype=np.uint64), threads=NCPU)
    assert np.array_equal(obj, eo)


def test_single_class_and_sixteen_classes_small(cuda, port):
    cl = core.cluster(1, 8)
    m = core.model_140gb()
    for types, lam in (([core.short_type()], [900]),
                       ([core.WorkloadType(j, 100.0 + 300 * j, 20.0 + 97 * j) for j in range(16)],
                        [60 + 7 * j for j in range(16)])):
        g = make(cl, m, types, lam)
        parts, plans = g.prepare_space(A.SPACE_ORDERED)
        obj, _ = g.evaluate_ranks(0, plans)
        eo, _, _ = port.evaluate_ranks(problem(cl, m, types, lam), A.SPACE_ORDERED,
                                       np.arange(plans, dtype=np.uint64), threads=NCPU)
        assert np.array_equal(obj, eo)


def test_zero_demand(cuda, port):
    cl = core.cluster(2, 8)
    w = workloads.load("cfg2")
    g = make(cl, w.model, w.types, [0, 0, 0, 0])
    st = g.round(A.SPACE_ORDERED)
    exp = port.round(problem(cl, w.model, w.types, [0, 0, 0, 0]), A.SPACE_ORDERED, threads=NCPU)
    assert st.throughput == exp.throughput == 0
    assert shapes(st.deployment) == shapes(exp.deployment)
