"""Generate tests/golden/*.json from the REFERENCE itself (oracle/_ref).

TEST INFRASTRUCTURE — runs in the build container (needs oracle/_ref built
from /root/reference).  The committed fixtures pin the CPU restatement and
the GPU path on machines without the reference:

  kats.json        the reference tests' known answers (test_costmodel.cpp,
                   test_flowassign.cpp) recomputed through the reference API
  solve.json       solve_assignment on seeded random instances (incl. B&B)
  rounds.json      per-config round winners (exhaustive / ordered / canonical)
  plans_<cfg>.json per-plan objectives: every plan of cfg1 / cfg1_bnb, a
                   seeded sample elsewhere, plus an all-plan checksum for cfg2
  switch.json      greedy_plan/estimate_time on seeded deployment pairs
  kv_plan.json     switchplan::kv_plan on seeded in-flight sets (with and
                   without the parameter plan's link loads as carry)
  flow.json        flow::max_flow on random graphs, build_network +
                   max_flow + extract_assignment and solve_fractional on
                   random instances, to_dot texts
  timeline_cfg4_ref.json  io::save_timeline of orch::build_adaptive_timeline
                   on config 4, the reference's own file
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from paper_2602_12151_b200 import core, workloads  # noqa: E402
from pyoracle import Oracle, Problem  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
THREADS = os.cpu_count() or 1


def problem(w):
    return Problem(w.cluster, w.model, w.types, w.lam, w.span_s, w.params)


def dep_json(d: core.Deployment):
    return [[r.device_ids, r.tp, r.pp] for r in d.replicas]


def objective_digest(obj: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(obj, dtype="<i8").tobytes()).hexdigest()


def random_instances(seed, count, max_r, max_j, max_lam, max_n=100):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        R, J = int(rng.integers(1, max_r + 1)), int(rng.integers(1, max_j + 1))
        n = rng.integers(1, max_n + 1, (R, J))
        n[rng.random((R, J)) < 0.125] = 0
        e = (rng.random((R, J)) * (n + 1)).astype(np.int64)
        lam = rng.integers(0, max_lam + 1, J)
        out.append((n.tolist(), e.tolist(), lam.tolist()))
    return out


def canonical_sample(ref, name):
    """3,000 seeded plans of a canonical space through the reference's
    evaluate_deployment -> plans_<name>.json."""
    w = workloads.load(name)
    pr = problem(w)
    parts, plans = ref.space_info(pr, w.space_mode, w.space_sizes)
    sample = np.unique(np.random.default_rng(12151).integers(0, plans, 3000)).astype(np.uint64)
    obj, spp, _ = ref.evaluate_ranks(pr, w.space_mode, sample, w.space_sizes, threads=THREADS)
    json.dump({"partitions": parts, "plans": plans, "ranks": sample.tolist(), "objective": obj.tolist(),
               "sum_pp": spp.tolist()}, open(os.path.join(OUT, f"plans_{name}.json"), "w"))
    return pr


def main():
    os.makedirs(OUT, exist_ok=True)
    ref = Oracle("ref")

    # ---- KATs (test_costmodel.cpp / test_flowassign.cpp) ----
    kats = {"normalize": [], "capacity": [], "assignment": []}
    for row in ([80, 50], [7], [12, 18, 30], [80, 0, 50],
                [(1 << 31) - 1, (1 << 31) - 99, (1 << 31) - 365]):
        M, units, scaled = ref.normalize(row)
        kats["normalize"].append({"n": row, "M": M, "units": units, "scaled": scaled})
    # lcm_80_50_fixture (fixtures.hpp:85-101) and appendix_d_fixture (:113-129)
    lcm = dict(params=core.ProfileParams(1.0 / 256.0, 1.0 / 512.0, 1.0, 1e-9, 0.0),
               model=core.ModelSpec("lcm-fixture", core.KGB, 1, 1, 1, core.KGB),
               types=[core.WorkloadType(0, 128.0, 64.0), core.WorkloadType(1, 128.0, 256.0)], span=50.0,
               cluster=core.cluster(1, 4), deps=[[([0], 1, 1)], [([0], 1, 1), ([1], 1, 1)]])
    appd = dict(params=core.ProfileParams(0.002, 0.002, 1.0, 0.0004, 0.0),
                model=core.ModelSpec("appendix-d", core.KGB, 1, 1, 1, core.KGB),
                types=[core.WorkloadType(0, 131.0, 48.0), core.WorkloadType(1, 121.0, 196.0)], span=1.0,
                cluster=core.cluster(2, 4), deps=[[([0, 1, 2, 3], 2, 2), ([4, 5], 2, 1), ([6, 7], 2, 1)]])
    for name, f in (("lcm_80_50", lcm), ("appendix_d", appd)):
        pr = Problem(f["cluster"], f["model"], f["types"], [0, 0], f["span"], f["params"])
        for d in f["deps"]:
            dep = core.Deployment([core.ReplicaConfig(ids, tp, pp) for ids, tp, pp in d])
            t = ref.capacity_table(pr, dep)
            kats["capacity"].append({"fixture": name, "deployment": d, "n": t.n, "e": t.e, "latency": t.latency,
                                     "cluster": [len(f["cluster"].machines), len(f["cluster"].machines[0].device_ids)],
                                     "params": f["params"].__dict__, "model": f["model"].__dict__,
                                     "types": [t_.__dict__ for t_ in f["types"]], "span": f["span"]})
    for n, e, lam, expect in (([[80, 50], [80, 50]], [[80, 50], [80, 50]], [7, 4], 11),
                              ([[200, 100], [200, 100]], [[200, 100], [200, 100]], [50, 100], 150),
                              ([[10, 5], [5, 3], [5, 3]], [[10, 5], [5, 3], [5, 3]], [5, 60], None)):
        ll = ref.solve_assignment(n, e, lam)
        kats["assignment"].append({"n": n, "e": e, "lambda": lam, "objective": ll.assignment.objective,
                                   "x": ll.assignment.x, "expect": expect})
    json.dump(kats, open(os.path.join(OUT, "kats.json"), "w"), indent=0)

    # ---- solve_assignment on seeded random instances ----
    solve = []
    for seed, cnt, mr, mj, ml in ((7, 80, 3, 3, 60), (11, 120, 6, 5, 500), (13, 60, 12, 8, 3000)):
        for n, e, lam in random_instances(seed, cnt, mr, mj, ml):
            ll = ref.solve_assignment(n, e, lam)
            solve.append({"seed": seed, "n": n, "e": e, "lambda": lam, "objective": ll.assignment.objective,
                          "x": ll.assignment.x, "M": ll.M, "unit": ll.unit, "used": ll.used})
    json.dump(solve, open(os.path.join(OUT, "solve.json"), "w"))

    # ---- rounds and per-plan objectives ----
    rounds = {}
    for name in ("cfg1", "cfg1_bnb"):
        w = workloads.load(name)
        pr = problem(w)
        s = ref.exhaustive(pr, parallel=True)
        rounds[name] = {"kind": "search::exhaustive", "objective": s.throughput, "iterations": s.iterations,
                        "deployment": dep_json(s.deployment)}
        parts, plans = ref.space_info(pr, w.space_mode, w.space_sizes)
        obj, spp, _ = ref.evaluate_ranks(pr, w.space_mode, np.arange(plans, dtype=np.uint64), w.space_sizes,
                                         threads=THREADS)
        json.dump({"partitions": parts, "plans": plans, "ranks": list(range(plans)), "objective": obj.tolist(),
                   "sum_pp": spp.tolist()}, open(os.path.join(OUT, f"plans_{name}.json"), "w"))
    for name in ("cfg2", "cfg2_low"):
        w = workloads.load(name)
        pr = problem(w)
        s = ref.round(pr, w.space_mode, w.space_sizes, threads=THREADS)
        rounds[name] = {"kind": "partitions_desc + search::best_strategies, first wins", "objective": s.throughput,
                        "partitions": s.iterations, "plans": s.plans, "partition_index": s.partition_index,
                        "local_rank": s.local_rank, "sum_pp": s.sum_pp, "deployment": dep_json(s.deployment)}
        parts, plans = ref.space_info(pr, w.space_mode, w.space_sizes)
        ranks = np.arange(plans, dtype=np.uint64)
        obj, spp, _ = ref.evaluate_ranks(pr, w.space_mode, ranks, w.space_sizes, threads=THREADS)
        sample = np.random.default_rng(12151).integers(0, plans, 2000)
        json.dump({"partitions": parts, "plans": plans, "all_objective_sha256": objective_digest(obj),
                   "objective_sum": int(obj.sum()), "ranks": sample.tolist(), "objective": obj[sample].tolist(),
                   "sum_pp": spp[sample].tolist()}, open(os.path.join(OUT, f"plans_{name}.json"), "w"))
    for name in ("cfg3_70b", "cfg3_7b", "cfg5", "cfg5_low", "cfg5_full"):
        pr = canonical_sample(ref, name)
        w = workloads.load(name)
        if name == "cfg3_70b":
            s = ref.round(pr, w.space_mode, w.space_sizes, threads=THREADS)
            rounds[name] = {"kind": "canonical space through search::evaluate_deployment", "objective": s.throughput,
                            "partitions": s.iterations, "plans": s.plans, "partition_index": s.partition_index,
                            "local_rank": s.local_rank, "sum_pp": s.sum_pp, "deployment": dep_json(s.deployment)}
    rpath = os.path.join(OUT, "rounds.json")  # keep the full-space entries of gen_rounds_full.py
    merged = json.load(open(rpath)) if os.path.exists(rpath) else {}
    merged.update(rounds)
    json.dump(merged, open(rpath, "w"), indent=1)

    # ---- search::search (flow-guided heuristic) with its log ----
    srch = []
    for name, seeds, iters in (("cfg1", range(5), 500), ("cfg1_bnb", range(1), 2), ("cfg2", range(3), 500),
                               ("cfg2_low", range(2), 500)):
        w = workloads.load(name)
        pr = problem(w)
        for seed in seeds:
            st, log = ref.search(pr, seed=seed, max_iters=iters)
            srch.append({"config": name, "seed": seed, "max_iters": iters, "throughput": st.throughput,
                         "iterations": st.iterations, "stale_iters": st.stale_iters,
                         "deployment": dep_json(st.deployment), "log": [list(r) for r in log]})
    # warm-started (build_adaptive_timeline style, orchestrate.cpp:116-123)
    w = workloads.load("cfg2")
    warm = core.canonical_deployment(w.cluster, [4] * 8, [4] * 8)
    st, log = ref.search(problem(w), seed=0, max_iters=150, warm_start=warm)
    srch.append({"config": "cfg2", "seed": 0, "max_iters": 150, "warm_start": dep_json(warm),
                 "throughput": st.throughput, "iterations": st.iterations, "stale_iters": st.stale_iters,
                 "deployment": dep_json(st.deployment), "log": [list(r) for r in log]})
    json.dump(srch, open(os.path.join(OUT, "search.json"), "w"))

    # ---- orch::build_adaptive_timeline on config 4 (24 windows) ----
    w = workloads.load("cfg4")
    tl = ref.adaptive_timeline(problem(w), w.raw["actual"], seed=0, max_iters=150, min_gain=w.raw["min_gain"])
    json.dump([{"span_index": si, "deployment": dep_json(d), "x": x, "switch_seconds": sw, "transfers": n}
               for si, d, x, sw, n in tl], open(os.path.join(OUT, "timeline_cfg4.json"), "w"))

    # ---- switching: greedy_plan + estimate_time on seeded pairs ----
    sw = []
    for name in ("cfg1", "cfg2", "cfg5"):
        w = workloads.load(name)
        pr = problem(w)
        parts, plans = ref.space_info(pr, w.space_mode, w.space_sizes)
        rng = np.random.default_rng(99)
        deps = [ref.space_plan(pr, w.space_mode, int(r), w.space_sizes)[0] for r in rng.integers(0, plans, 12)]
        for a in range(0, len(deps) - 1, 2):
            src, dst = deps[a], deps[a + 1]
            plan, mx = ref.switch_plan(w.cluster, w.model.param_bytes, src, dst)
            sw.append({"config": name, "src": dep_json(src), "dst": dep_json(dst), "est_seconds": plan.est_seconds,
                       "max_link_bytes": mx, "transfers": [[t.range.begin, t.range.end, t.src, t.dst]
                                                           for t in plan.transfers]})
    json.dump(sw, open(os.path.join(OUT, "switch.json"), "w"))
    gen_f3(ref)
    gen_f4(ref)
    gen_exact_budget(ref, Oracle("port"))
    gen_exact_wide(ref, Oracle("port"))
    print("golden fixtures written to", OUT)


def kv_cases(ref, seed=4242):
    """Seeded kv_plan cases on the switch.json deployment pairs."""
    rng = np.random.default_rng(seed)
    sw = json.load(open(os.path.join(OUT, "switch.json")))
    cases = []
    for k, pair in enumerate(sw):
        w = workloads.load(pair["config"])
        src = core.Deployment([core.ReplicaConfig(ids, tp, pp) for ids, tp, pp in pair["src"]])
        dst = core.Deployment([core.ReplicaConfig(ids, tp, pp) for ids, tp, pp in pair["dst"]])
        for variant in range(3):
            n = int(rng.integers(0, 400)) if variant else int(rng.integers(1, 12))
            thr = int(rng.integers(0, 2000))
            reqs = [core.InflightRequest(int(1000 * k + q), int(rng.integers(0, 4000)),
                                         int(rng.integers(1, 1 << 33)), int(rng.integers(0, src.replica_count())))
                    for q in range(n)]
            if variant == 2 and n:  # equal kv sizes stress the lowest-id tie-breaks
                for r in reqs:
                    r.kv_bytes = 1 << 20
            headroom = float(rng.choice([0.0, 0.1, 0.25, 0.5, float(rng.random() * 0.5)]))
            carry = None
            if variant != 1:
                carry = core.SwitchPlan([core.Transfer(core.ByteRange(b, e), s_, d_)
                                         for b, e, s_, d_ in pair["transfers"]])
            kv = ref.kv_plan(w.cluster, reqs, thr, src, dst, headroom, carry)
            cases.append({"config": pair["config"], "src": pair["src"], "dst": pair["dst"], "threshold": thr,
                          "headroom": headroom, "carry": variant != 1,
                          "inflight": [[r.request_id, r.generated_tokens, r.kv_bytes, r.source_replica]
                                       for r in reqs],
                          "drained": kv.drained, "buffer_bytes": kv.buffer_bytes,
                          "migrated": [[m.request_id, m.kv_bytes, m.src, m.dst] for m in kv.migrated]})
    return cases


def gen_f4(ref):
    rng = np.random.default_rng(2602)
    graphs = []
    for trial in range(400):
        nn = int(rng.integers(2, 13 if trial < 200 else 60))
        edges = []
        for _ in range(int(rng.integers(1, 3 * nn + 1))):
            u, v = int(rng.integers(0, nn)), int(rng.integers(0, nn))
            if u == v and trial < 200:
                continue
            edges.append((u, v, int(rng.integers(0, 50 if trial % 3 else 1 << 40))))
        src, snk = (0, nn - 1) if trial % 5 else (nn - 1, 0)
        value, flow = ref.max_flow(nn, edges, src, snk)
        graphs.append({"num_nodes": nn, "edges": edges, "source": src, "sink": snk, "value": value, "flow": flow})
    inst = []
    for seed, cnt, mr, mj, ml in ((7, 120, 3, 3, 60), (11, 160, 6, 5, 500), (13, 80, 12, 8, 3000),
                                  (17, 40, 20, 16, 20000)):
        for n, e, lam in random_instances(seed, cnt, mr, mj, ml):
            x, obj, val, fl = ref.flow_assign(n, e, lam)
            inst.append({"n": n, "e": e, "lambda": lam, "x": x, "objective": obj, "value": val, "flow": fl})
    lps = []
    for seed, cnt, mr, mj, ml in ((19, 60, 3, 3, 60), (23, 30, 6, 5, 500), (29, 6, 12, 8, 3000)):
        for n, e, lam in random_instances(seed, cnt, mr, mj, ml):
            f, obj = ref.solve_fractional(n, e, lam)
            lps.append({"n": n, "e": e, "lambda": lam, "f": f, "objective": obj})
    dots = []
    for n, e, lam in (([[80]], [[80]], [10]), ([[80, 50], [40, 20]], [[80, 50], [40, 20]], [10, 10]),
                      ([[10, 10, 10], [10, 10, 10]], [[10, 10, 10], [10, 10, 10]], [5, 5, 5])):
        for wf in (False, True):
            dots.append({"n": n, "e": e, "lambda": lam, "with_flow": wf, "dot": ref.to_dot(n, e, lam, wf)})
    json.dump({"graphs": graphs, "instances": inst, "lp": lps, "dot": dots}, open(os.path.join(OUT, "flow.json"), "w"))


def gen_flow_big(ref):
    """Graphs and instances past the shared-memory workspace (K6a/K6b HBM
    paths): a batch of 34 similar graphs (interleaved workspace), a ragged
    batch (packed workspace) and R=40, J=10 instances -> flow_big.json
    (per-edge flows as sha256 of their int64 bytes)."""
    import hashlib
    rng = np.random.default_rng(2603)
    digest = lambda fl: hashlib.sha256(np.asarray(fl, "<i8").tobytes()).hexdigest()  # noqa: E731

    def graph(nn, m):
        edges = [(int(rng.integers(0, nn)), int(rng.integers(0, nn)), int(rng.integers(0, 1000))) for _ in range(m)]
        value, fl = ref.max_flow(nn, edges, 0, nn - 1)
        return {"num_nodes": nn, "edges": edges, "source": 0, "sink": nn - 1, "value": value,
                "flow_sha256": digest(fl)}
    similar = [graph(nn, int(rng.integers(2 * nn, 3 * nn))) for nn in rng.integers(700, 801, 34).tolist()]
    ragged = [graph(nn, int(rng.integers(nn, 4 * nn))) for nn in (50, 3000, 100, 1200, 20)]
    inst = []
    for _ in range(6):  # R = 40, J = 10
        n = rng.integers(1, 101, (40, 10))
        n[rng.random((40, 10)) < 0.125] = 0
        e = (rng.random((40, 10)) * (n + 1)).astype(np.int64)
        lam = rng.integers(0, 20001, 10)
        n, e, lam = n.tolist(), e.tolist(), lam.tolist()
        x, obj, val, fl = ref.flow_assign(n, e, lam)
        inst.append({"n": n, "e": e, "lambda": lam, "x": x, "objective": obj, "value": val,
                     "flow_sha256": digest(fl)})
    json.dump({"similar": similar, "ragged": ragged, "instances": inst}, open(os.path.join(OUT, "flow_big.json"), "w"))


def gen_exact_budget(ref, port):
    """B&B abort boundary: budgets N-1 / N around the reference's node count N
    (counted by the restatement, checked here against the reference)."""
    cases = []
    for n, e, lam in random_instances(31, 400, 6, 3, 130):
        R, J = len(n), len(lam)
        if R * J > 20 or sum(lam) > 400:
            continue
        N = port.solve_assignment(n, e, lam).work
        if N < 50:
            continue
        row = {"n": n, "e": e, "lambda": lam, "nodes": N, "budgets": []}
        for b in (N - 1, N, N // 2):
            ll = ref.solve_assignment(n, e, lam, core.SolveOptions(400, 20, b))
            row["budgets"].append({"budget": b, "x": ll.assignment.x, "objective": ll.assignment.objective})
        cases.append(row)
    json.dump(cases, open(os.path.join(OUT, "exact_budget.json"), "w"))


def gen_exact_wide(ref, port):
    """B&B abort boundary on instances whose values need the 64-bit DFS
    table: large request sizes (row LCMs past 2^30) and, with the demand
    limit raised, demands past 2^20 -> exact_budget_wide.json."""
    cases = []
    sets = [(random_instances(77, 300, 5, 3, 130, max_n=20000), core.SolveOptions()),
            (random_instances(78, 60, 2, 2, 3_000_000, max_n=100), core.SolveOptions(4_000_000, 20, 8_000_000))]
    for insts, opts in sets:
        for n, e, lam in insts:
            R, J = len(n), len(lam)
            if R * J > opts.exact_cell_limit or sum(lam) > opts.exact_demand_limit:
                continue
            N = port.solve_assignment(n, e, lam, opts).work
            if N < 30 or N > 4_000_000:
                continue
            row = {"n": n, "e": e, "lambda": lam, "nodes": N, "demand_limit": opts.exact_demand_limit,
                   "budgets": []}
            for b in (N - 1, N, N // 2):
                ll = ref.solve_assignment(n, e, lam, core.SolveOptions(opts.exact_demand_limit, 20, b))
                row["budgets"].append({"budget": b, "x": ll.assignment.x, "objective": ll.assignment.objective})
            cases.append(row)
    json.dump(cases, open(os.path.join(OUT, "exact_budget_wide.json"), "w"))
    print(len(cases), "wide exact cases")


def gen_wide(ref):
    """Config 5-7B (g_min = 1, sizes {1,2,4}: 32-128 replicas per plan) ->
    plans_cfg5_7b.json and wide.json.  The sample is weighted toward plans
    with R > 64 (rare under uniform sampling): 2,000 plans from partitions
    with R > 64, 1,000 uniform, plus each R > 64 partition's first plan.
    wide.json: switching pairs with 128 source replicas (init_uniform -> plans)
    and capacity table + solve_assignment of R = 96 / 128 plans."""
    from math import comb
    name = "cfg5_7b"
    w = workloads.load(name)
    pr = problem(w)
    parts, plans = ref.space_info(pr, w.space_mode, w.space_sizes)
    # partitions_desc order with parts {4,2,1} (a fours, b twos, c ones); the
    # blocks of one size share their candidate list (4: 3 strategies, 2: 2,
    # 1: 1), so a partition holds C(a+2,2) * (b+1) canonical plans
    struct = []
    for a in range(32, -1, -1):
        for b in range((128 - 4 * a) // 2, -1, -1):
            struct.append((a + b + 128 - 4 * a - 2 * b, comb(a + 2, 2) * (b + 1)))
    pre = np.cumsum([0] + [c for _, c in struct])
    assert len(struct) == parts and pre[-1] == plans
    for i in (0, len(struct) // 2, len(struct) - 1):  # structure check against the harness
        d, p, l = ref.space_plan(pr, w.space_mode, int(pre[i]), w.space_sizes)
        assert (p, l, d.replica_count()) == (i, 0, struct[i][0])
    rng = np.random.default_rng(12151)
    wide = [i for i, (R, _) in enumerate(struct) if R > 64]
    wt = np.array([struct[i][1] for i in wide], float)
    pick = rng.choice(wide, 2000, p=wt / wt.sum())
    ranks = [int(pre[i] + rng.integers(0, struct[i][1])) for i in pick]
    ranks += rng.integers(0, plans, 1000).tolist() + [int(pre[i]) for i in wide]
    ranks = np.unique(np.array(ranks, np.uint64))
    obj, spp, _ = ref.evaluate_ranks(pr, w.space_mode, ranks, w.space_sizes, threads=THREADS)
    part_of = np.searchsorted(pre, ranks, side="right") - 1
    json.dump({"partitions": parts, "plans": plans, "ranks": ranks.tolist(), "objective": obj.tolist(),
               "sum_pp": spp.tolist(), "R": [struct[p][0] for p in part_of]},
              open(os.path.join(OUT, f"plans_{name}.json"), "w"))
    # 128-source switching pairs and R = 96 / 128 assignment details
    cur = core.canonical_deployment(w.cluster, [1] * 128, [1] * 128)
    sw, det = [], []
    # the R = 128 plan (last rank), R = 127 / ~100 partitions, and uniform ranks
    targets = [plans - 1, int(pre[-3]), int(pre[-40])] + rng.integers(0, plans, 5).tolist()
    # (every device of the all-ones source holds the whole model, so those
    # pairs move nothing; R > 64 sources with 2-/4-device replicas do)
    plan_at = lambda r: ref.space_plan(pr, w.space_mode, int(r), w.space_sizes)[0]
    pairs = [(cur, plan_at(r), -1, int(r)) for r in targets]
    for a in wide[::len(wide) // 12][:12]:
        ra = int(pre[a] + rng.integers(0, struct[a][1]))
        rb = int(rng.integers(0, plans))
        pairs += [(plan_at(ra), plan_at(rb), ra, rb), (plan_at(rb), plan_at(ra), rb, ra)]
    for src, dst, ra, rb in pairs:
        plan, mx = ref.switch_plan(w.cluster, w.model.param_bytes, src, dst)
        sw.append({"src_rank": ra, "rank": rb, "src": dep_json(src), "dst": dep_json(dst),
                   "est_seconds": plan.est_seconds, "max_link_bytes": mx,
                   "transfers": [[t.range.begin, t.range.end, t.src, t.dst] for t in plan.transfers]})
    for r in (plans - 1, plans - 2, int(pre[-20]), int(pre[-300])):
        dep = ref.space_plan(pr, w.space_mode, r, w.space_sizes)[0]
        t = ref.capacity_table(pr, dep)
        ll = ref.solve_assignment(t.n, t.e, w.lam)
        det.append({"rank": r, "deployment": dep_json(dep), "n": t.n, "e": t.e, "x": ll.assignment.x,
                    "objective": ll.assignment.objective, "M": ll.M, "unit": ll.unit, "used": ll.used,
                    "evaluate_deployment": ref.evaluate_deployment(pr, dep)})
    json.dump({"config": name, "switch": sw, "detail": det}, open(os.path.join(OUT, "wide.json"), "w"))


def gen_f3(ref):
    json.dump(kv_cases(ref), open(os.path.join(OUT, "kv_plan.json"), "w"))
    w = workloads.load("cfg4")
    ref.adaptive_timeline_json(problem(w), w.raw["actual"], os.path.join(OUT, "timeline_cfg4_ref.json"), seed=0,
                               max_iters=150, min_gain=w.raw["min_gain"])


if __name__ == "__main__":
    if sys.argv[1:] == ["f3"]:
        gen_f3(Oracle("ref"))
    elif sys.argv[1:] == ["f4"]:
        gen_f4(Oracle("ref"))
    elif sys.argv[1:] == ["exact"]:
        gen_exact_budget(Oracle("ref"), Oracle("port"))
    elif sys.argv[1:] == ["flow_big"]:
        gen_flow_big(Oracle("ref"))
    elif sys.argv[1:] == ["exact_wide"]:
        gen_exact_wide(Oracle("ref"), Oracle("port"))
    elif sys.argv[1:] == ["wide"]:
        gen_wide(Oracle("ref"))
    elif sys.argv[1:2] == ["sample"]:  # python oracle/gen_golden.py sample cfg5_full
        for nm in sys.argv[2:]:
            canonical_sample(Oracle("ref"), nm)
    else:
        main()
