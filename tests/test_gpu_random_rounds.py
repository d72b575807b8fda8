"""Seeded random scheduling problems, every plan through the GPU round
against the reference itself (oracle/_ref, the unmodified reference compiled
with its own enumerator harness).

Each case draws a cluster shape (machines x devices per machine, device
memory), a model (7B/13B/70B-class), J in 1..16 workload classes with
random centroids, a demand level from starved to saturated (zero-demand
classes included) and a canonical or ordered plan space, then checks:
  * every plan's objective and sum_pp equal the reference's
    `evaluate_deployment` (deploysearch.cpp:138-151), bit-exact;
  * the fused round's winner (key order: objective desc, partition, sum_pp,
    rank) equals the reference harness's first-wins round;
  * the winner's assignment x equals `flow::solve_assignment`
    (flowassign.cpp:481-503) on the reference's capacity table.
Plan spaces are kept small (<= 30k plans) so the reference finishes in
seconds; the large configs are covered by tests/test_gpu_parity.py.
"""
import os

import numpy as np
import pytest

from paper_2602_12151_b200 import _abi as A
from paper_2602_12151_b200 import core
from paper_2602_12151_b200._native import GpuContext

pytestmark = pytest.mark.gpu

NCPU = os.cpu_count() or 1
GB = 1000 ** 3
MODELS = [
    core.ModelSpec("rand-7b", 14 * GB, 32, 32000, 14 * GB, 14 * GB),
    core.ModelSpec("rand-13b", 26 * GB, 40, 80000, 26 * GB, 26 * GB),
    core.ModelSpec("rand-70b", 140 * GB, 80, 160000, 280 * GB, 140 * GB),
]


def draw_case(ref, seed):
    """A random problem with a plan space of 50..30,000 plans."""
    from pyoracle import Problem
    rng = np.random.default_rng(26020 + seed)
    for _ in range(200):
        per = int(rng.choice([2, 4, 8]))
        machines = int(rng.integers(1, 17))
        mem = int(rng.choice([40, 80, 141])) * GB
        cl = core.cluster(machines, per, mem, float(rng.choice([300e9, 400e9, 900e9])),
                          float(rng.choice([50e9, 200e9])))
        model = MODELS[int(rng.integers(0, len(MODELS)))]
        J = int(rng.integers(1, 17))
        types = [core.WorkloadType(j, float(rng.uniform(16, 7999)), float(rng.uniform(1, 3000))) for j in range(J)]
        canonical = bool(rng.random() < 0.6) or cl.device_count() > 24  # ordered spaces explode past D = 24
        mode = A.SPACE_CANONICAL if canonical else A.SPACE_ORDERED
        sizes = [1 << b for b in range(8) if (1 << b) <= cl.device_count() and rng.random() < 0.7] if canonical else []
        if canonical and not sizes:
            continue
        params = core.ProfileParams()
        probe = Problem(cl, model, types, [10 ** 9] * J, 60.0, params)
        try:
            parts, plans = ref.space_info(probe, mode, sizes)
        except Exception:  # ModelTooLarge and friends: draw again
            continue
        if not (50 <= plans <= 30000):
            continue
        # demand: a fraction of the most any of 256 sampled plans serves at
        # unbounded demand (load near 1 keeps the exchange loop busy)
        sample = np.unique(rng.integers(0, plans, 256)).astype(np.uint64)
        cap = max(1, int(ref.evaluate_ranks(probe, mode, sample, sizes, threads=NCPU)[0].max()))
        load = float(rng.choice([0.3, 0.7, 0.9, 1.0, 1.3, 3.0]))
        share = rng.dirichlet(np.ones(J))
        lam = [int(v) for v in np.round(load * share * cap)]
        for j in range(J):
            if rng.random() < 0.1:
                lam[j] = 0
        return cl, model, types, lam, params, mode, sizes, plans
    raise RuntimeError("no case drawn")


@pytest.mark.parametrize("seed", range(48))
def test_random_problem_every_plan_and_winner(cuda, ref, seed):
    from pyoracle import Problem
    cl, model, types, lam, params, mode, sizes, plans = draw_case(ref, seed)
    pr = Problem(cl, model, types, lam, 60.0, params)
    g = GpuContext(cl, model, params)
    g.set_workload(types, lam, 60.0)
    parts, n = g.prepare_space(mode, sizes)
    assert (parts, n) == ref.space_info(pr, mode, sizes)
    obj, spp = g.evaluate_ranks(0, n)
    eo, es, _ = ref.evaluate_ranks(pr, mode, np.arange(n, dtype=np.uint64), sizes, threads=NCPU)
    bad = np.nonzero(obj != eo)[0]
    assert bad.size == 0, (f"seed {seed} (D={cl.device_count()}, J={len(types)}, {n} plans): {bad.size} differ, "
                           f"ranks {bad[:8]} gpu {obj[bad[:8]]} ref {eo[bad[:8]]}")
    assert np.array_equal(spp, es)
    got = g.round(mode, sizes)
    exp = ref.round(pr, mode, sizes, threads=NCPU)
    assert (got.throughput, got.partition_index, got.local_rank, got.sum_pp) == \
        (exp.throughput, exp.partition_index, exp.local_rank, exp.sum_pp)
    # the winner's assignment against flow::solve_assignment on the reference's table
    table, asg = g.plan_detail(got.deployment)
    tref = ref.capacity_table(pr, got.deployment)
    assert (table.n, table.e) == (tref.n, tref.e)
    lower = ref.solve_assignment(tref.n, tref.e, lam)
    assert asg.assignment.x == lower.assignment.x
    assert asg.assignment.objective == lower.assignment.objective == got.throughput


@pytest.mark.parametrize("seed", range(16))
def test_random_problem_switching(cuda, ref, seed):
    """K2 on random clusters / models: est_seconds and max link bytes of the
    switching batch, and full transfer lists, against the reference's
    switchplan::layout + greedy_plan + estimate_time (switchplan.cpp:40-140)."""
    from pyoracle import Problem
    cl, model, types, lam, params, mode, sizes, plans = draw_case(ref, 100 + seed)
    pr = Problem(cl, model, types, lam, 60.0, params)
    g = GpuContext(cl, model, params)
    g.set_workload(types, lam, 60.0)
    g.prepare_space(mode, sizes)
    rng = np.random.default_rng(seed)
    ranks = rng.integers(0, plans, 48)
    deps = [ref.space_plan(pr, mode, int(r), sizes)[0] for r in ranks]
    for src in (deps[0], g.round(mode, sizes).deployment):
        est, mb = g.switch_cost_batch(src, deps)
        for d, e, m in zip(deps, est, mb):
            plan, emax = ref.switch_plan(cl, model.param_bytes, src, d)
            assert e == plan.est_seconds and m == emax
        for d in deps[:6]:
            got = g.switch_plan(src, d)
            exp, _ = ref.switch_plan(cl, model.param_bytes, src, d)
            assert got.est_seconds == exp.est_seconds
            assert [(t.range.begin, t.range.end, t.src, t.dst) for t in got.transfers] == \
                [(t.range.begin, t.range.end, t.src, t.dst) for t in exp.transfers]


@pytest.mark.parametrize("seed", range(16))
def test_random_problem_search(cuda, ref, seed):
    """search::search (deploysearch.cpp:341-417) on random problems (D <= 32:
    the reference's best_strategies walks ordered combos): final state and
    the whole log (ops, acceptances, throughputs) equal the reference's."""
    from pyoracle import Problem
    s = 200 + seed
    while True:
        cl, model, types, lam, params, mode, sizes, plans = draw_case(ref, s)
        if cl.device_count() <= 32:
            break
        s += 1000
    pr = Problem(cl, model, types, lam, 60.0, params)
    g = GpuContext(cl, model, params)
    g.set_workload(types, lam, 60.0)
    for sd in (seed, 7 * seed + 1):
        st, log = g.search(seed=sd, max_iters=200)
        es, elog = ref.search(pr, seed=sd, max_iters=200)
        assert (st.throughput, st.iterations, st.stale_iters) == (es.throughput, es.iterations, es.stale_iters)
        assert [(r.device_ids, r.tp, r.pp) for r in st.deployment.replicas] == \
            [(r.device_ids, r.tp, r.pp) for r in es.deployment.replicas]
        assert [list(r) for r in log] == [list(r) for r in elog]
