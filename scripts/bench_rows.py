"""Time every SURVEY §8 row beyond the headline round on one B200, with the
reference's own CPU implementation (oracle/_ref, compiled unmodified) timed
beside it on the same inputs, and check the outputs agree.  Writes one JSON
object (stdout, and --out if given).

    python scripts/bench_rows.py --out profiles/round1_rows.json

Rows: config 4 (24 re-scheduling windows), f1 search() (GPU-backed driver), f2 exact B&B (config 1-B&B
exhaustive), f3 kv_plan, f4 max_flow / build_network+max_flow+
extract_assignment / solve_fractional, and the K2 switching batch.  GPU
times are wall-clock around the public call (host copies included) after
one warm-up call; reference times are the same calls on the host cores.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_12151_b200 import core, orchestrate, workloads  # noqa: E402
from paper_2602_12151_b200._native import GpuContext  # noqa: E402
from pyoracle import Oracle, Problem  # noqa: E402


def timed(fn, reps=1):
    fn()  # warm-up
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps, out


def cpu_timed(fn):
    t = time.perf_counter()
    out = fn()
    return time.perf_counter() - t, out


def row(name, gpu_s, ref_s, same, **kw):
    r = {"row": name, "gpu_s": round(gpu_s, 6), "reference_cpu_s": round(ref_s, 6),
         "speedup": round(ref_s / gpu_s, 2) if gpu_s > 0 else None, "identical": bool(same)}
    r.update(kw)
    print(json.dumps(r), file=sys.stderr)
    return r


def problem(w):
    return Problem(w.cluster, w.model, w.types, w.lam, w.span_s, w.params)


def cpu_timeline(ref, w, forecasts, min_gain, threads):
    """The config-4 window loop on the reference (oracle/_ref): its round over the
    full space, evaluate_deployment for the keep rule, capacity table +
    solve_assignment, greedy_plan/estimate_time."""
    entries, current, prev_lam, prev_x = [], None, None, None
    for s, lam in enumerate(forecasts):
        if entries and lam == prev_lam:
            continue
        pr = Problem(w.cluster, w.model, w.types, lam, w.span_s, w.params)
        found = ref.round(pr, w.space_mode, w.space_sizes, threads=threads)
        chosen = found.deployment
        if current is not None:
            keep = ref.evaluate_deployment(pr, current)
            if float(found.throughput) <= float(keep) * (1.0 + min_gain):
                chosen = current
        t = ref.capacity_table(pr, chosen)
        x = ref.solve_assignment(t.n, t.e, lam).assignment.x
        same = current is not None and orchestrate._same(chosen, current)
        if not entries:
            entries.append((s, chosen.shapes(), x, None))
        elif not same:
            plan, _ = ref.switch_plan(w.cluster, w.model.param_bytes, current, chosen)
            entries.append((s, chosen.shapes(), x, plan.est_seconds))
        elif x != prev_x:
            entries.append((s, chosen.shapes(), x, None))
        current, prev_lam, prev_x = chosen, lam, x
    return entries


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    ref = Oracle("ref")
    threads = os.cpu_count() or 1
    rows = []

    # f1: search() driver on config 2 (seeded, 500 iterations cap)
    w = workloads.load("cfg2")
    g = GpuContext(w.cluster, w.model, w.params)
    g.set_workload(w.types, w.lam, w.span_s)
    gs, (gst, glog) = timed(lambda: g.search(seed=3, max_iters=500))
    rs, (rst, rlog) = cpu_timed(lambda: ref.search(problem(w), seed=3, max_iters=500))
    rows.append(row("f1 search() cfg2 seed 3", gs, rs, gst.throughput == rst.throughput and glog == rlog,
                    iterations=gst.iterations))

    # f2: exact B&B, config 1-B&B exhaustive (61 plans)
    w = workloads.load("cfg1_bnb")
    g = GpuContext(w.cluster, w.model, w.params)
    g.set_workload(w.types, w.lam, w.span_s)
    gs, gst = timed(lambda: g.exhaustive())
    rs1, rst = cpu_timed(lambda: ref.exhaustive(problem(w), parallel=False))
    rsp, _ = cpu_timed(lambda: ref.exhaustive(problem(w), parallel=True))
    rows.append(row("f2 exact B&B cfg1_bnb exhaustive", gs, rs1, gst.throughput == rst.throughput,
                    reference_cpu_parallel_s=round(rsp, 6), reference_threads=threads))

    # f3: kv_plan, 200k in-flight requests across a config-5 resharding
    w = workloads.load("cfg5")
    sw = json.load(open(os.path.join(ROOT, "tests", "golden", "switch.json")))
    pair = [p for p in sw if p["config"] == "cfg5"][0]
    src = core.Deployment([core.ReplicaConfig(i, tp, pp) for i, tp, pp in pair["src"]])
    dst = core.Deployment([core.ReplicaConfig(i, tp, pp) for i, tp, pp in pair["dst"]])
    carry = core.SwitchPlan([core.Transfer(core.ByteRange(b, e), s, d) for b, e, s, d in pair["transfers"]])
    rng = np.random.default_rng(1)
    from paper_2602_12151_b200 import _abi
    reqs = np.zeros(200_000, _abi.inflight_dtype())
    reqs["request_id"] = np.arange(len(reqs))
    reqs["generated_tokens"] = rng.integers(0, 2000, len(reqs))
    reqs["kv_bytes"] = rng.integers(1 << 20, 1 << 30, len(reqs))
    reqs["source_replica"] = rng.integers(0, src.replica_count(), len(reqs))
    g = GpuContext(w.cluster, w.model, w.params)
    gs, a = timed(lambda: g.kv_plan(reqs, 500, src, dst, 0.1, carry, as_arrays=True), reps=3)
    rs, b = cpu_timed(lambda: ref.kv_plan(w.cluster, reqs, 500, src, dst, 0.1, carry, as_arrays=True))
    same = np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]
    rows.append(row("f3 kv_plan 200k requests (cfg5 pair)", gs, rs, same, migrated=len(a[1])))

    # f4: max_flow on 20k random graphs (60 nodes)
    G = 20_000
    nn = rng.integers(20, 61, G).astype(np.int32)
    m = np.array([int(rng.integers(v, 4 * v)) for v in nn], np.int64)
    off = np.zeros(G + 1, np.int64)
    off[1:] = np.cumsum(m)
    edges = np.zeros(int(off[-1]), _abi.flow_edge_dtype())
    owner = np.repeat(np.arange(G), m)
    edges["from"] = (rng.random(len(edges)) * nn[owner]).astype(np.int32)
    edges["to"] = (rng.random(len(edges)) * nn[owner]).astype(np.int32)
    edges["cap"] = rng.integers(0, 1000, len(edges))
    gs, (val, fl) = timed(lambda: g.max_flow_arrays(nn, off, edges, np.zeros(G, np.int32), nn - 1))
    rs, exp = cpu_timed(lambda: [ref.max_flow(int(nn[i]), edges[off[i]:off[i + 1]], 0, int(nn[i]) - 1, True)
                                 for i in range(G)])
    same = all(int(val[i]) == exp[i][0] and np.array_equal(fl[off[i]:off[i + 1]], exp[i][1]) for i in range(G))
    rows.append(row("f4 max_flow 20k graphs (20-60 nodes)", gs, rs, same))

    # f4: build_network + max_flow + extract_assignment, 8192 instances R=16 J=8
    cnt, R, J = 8192, 16, 8
    n = rng.integers(1, 400, (cnt, R, J))
    n[rng.random((cnt, R, J)) < 0.1] = 0
    e = (rng.random((cnt, R, J)) * (n + 1)).astype(np.int64)
    lam = rng.integers(0, 3000, (cnt, J))
    gs, (x, obj, val, _) = timed(lambda: g.flow_assign_batch(n, e, lam), reps=3)
    rs, exp = cpu_timed(lambda: [ref.flow_assign(n[i].tolist(), e[i].tolist(), lam[i].tolist()) for i in range(cnt)])
    same = all(x[i].tolist() == exp[i][0] and int(obj[i]) == exp[i][1] and int(val[i]) == exp[i][2]
               for i in range(cnt))
    rows.append(row("f4 flow_assign 8192 x (R=16, J=8)", gs, rs, same))

    # f4: solve_fractional, 256 instances R=6 J=4
    cnt, R, J = 256, 6, 4
    n = rng.integers(1, 100, (cnt, R, J))
    e = (rng.random((cnt, R, J)) * (n + 1)).astype(np.int64)
    lam = rng.integers(0, 500, (cnt, J))
    gs, (f, fo) = timed(lambda: g.solve_fractional_batch(n, e, lam))
    rs, exp = cpu_timed(lambda: [ref.solve_fractional(n[i].tolist(), e[i].tolist(), lam[i].tolist())
                                 for i in range(cnt)])
    same = all(f[i].tolist() == exp[i][0] and float(fo[i]) == exp[i][1] for i in range(cnt))
    rows.append(row("f4 solve_fractional 256 x (R=6, J=4)", gs, rs, same))

    # K2: switching estimates from one deployment to 1024 config-5 plans
    w = workloads.load("cfg5")
    pr = problem(w)
    parts, plans = ref.space_info(pr, w.space_mode, w.space_sizes)
    deps = [ref.space_plan(pr, w.space_mode, int(r), w.space_sizes)[0] for r in rng.integers(0, plans, 1024)]
    g = GpuContext(w.cluster, w.model, w.params)
    gs, (est, _) = timed(lambda: g.switch_cost_batch(src, deps))
    rs, exp = cpu_timed(lambda: [ref.switch_plan(w.cluster, w.model.param_bytes, src, d)[0].est_seconds
                                 for d in deps])
    rows.append(row("K2 switch_cost_batch 1024 pairs (cfg5)", gs, rs, list(est) == exp))

    # config 4: 24 windows of re-scheduling (orchestrate.py loop: full-space round per window, keep
    # rule, assignment, switch plan) against the same loop over the reference's CPU round
    w = workloads.load("cfg4")
    fc, mg = w.raw["forecasts"], w.raw["min_gain"]
    g = GpuContext(w.cluster, w.model, w.params)
    gs, tl = timed(lambda: orchestrate.build_adaptive_timeline(g, w.types, fc, w.span_s, mg, w.space_mode,
                                                                w.space_sizes))
    got = [(e.span_index, e.deployment.shapes(), e.assignment,
            None if e.switch is None else e.switch_seconds) for e in tl.entries]
    rs, exp = cpu_timed(lambda: cpu_timeline(ref, w, fc, mg, threads))
    rows.append(row("cfg4 temporal: 24 windows (round + keep rule + assignment + switch plan)", gs, rs, got == exp,
                    rounds=tl.rounds, entries=len(tl.entries), ms_per_round_gpu=round(1e3 * gs / max(1, tl.rounds), 3)))

    out = {"device": torch.cuda.get_device_name(0), "host_threads": threads, "rows": rows}
    print(json.dumps(out, indent=1))
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
