"""Config 4 (temporal, 24 windows) and the C++ drop-in, on the GPU.

The per-window loop (paper_2602_12151_b200/orchestrate.py, following
orchestrate.cpp:94-154 with the full-space round) is replayed on the CPU
oracle window by window: round winner, keep rule, assignment x and the greedy
switch plan (transfers + estimate) must be identical."""
import os
import subprocess

import pytest

from paper_2602_12151_b200 import core, orchestrate, workloads
from paper_2602_12151_b200._native import GpuContext

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NCPU = os.cpu_count() or 1


def cpu_timeline(port, w, forecasts, min_gain):
    from pyoracle import Problem
    entries, current, prev_lam, prev_x = [], None, None, None
    for s, lam in enumerate(forecasts):
        if entries and lam == prev_lam:
            continue
        pr = Problem(w.cluster, w.model, w.types, lam, w.span_s, w.params)
        found = port.round(pr, w.space_mode, w.space_sizes, threads=NCPU)
        chosen = found.deployment
        if current is not None:
            keep = port.evaluate_deployment(pr, current)
            if float(found.throughput) <= float(keep) * (1.0 + min_gain):
                chosen = current
        t = port.capacity_table(pr, chosen)
        x = port.solve_assignment(t.n, t.e, lam).assignment.x
        same = current is not None and orchestrate._same(chosen, current)
        if not entries:
            entries.append((s, chosen.shapes(), x, None))
        elif not same:
            plan, _ = port.switch_plan(w.cluster, w.model.param_bytes, current, chosen)
            entries.append((s, chosen.shapes(), x, (plan.est_seconds,
                                                     [(t.range.begin, t.range.end, t.src, t.dst) for t in plan.transfers])))
        elif x != prev_x:
            entries.append((s, chosen.shapes(), x, None))
        current, prev_lam, prev_x = chosen, lam, x
    return entries


def test_cfg4_timeline_matches_cpu(cuda, port):
    w = workloads.load("cfg4")
    fc = w.raw["forecasts"]
    g = GpuContext(w.cluster, w.model, w.params)
    tl = orchestrate.build_adaptive_timeline(g, w.types, fc, w.span_s, w.raw["min_gain"], w.space_mode, w.space_sizes)
    got = [(e.span_index, e.deployment.shapes(), e.assignment,
            None if e.switch is None else (e.switch_seconds, [(t.range.begin, t.range.end, t.src, t.dst)
                                                              for t in e.switch.transfers])) for e in tl.entries]
    exp = cpu_timeline(port, w, fc, w.raw["min_gain"])
    assert got == exp
    assert tl.windows == 24 and tl.rounds >= 1


def test_cpp_dropin(cuda):
    exe = os.path.join(ROOT, "oracle", "_ref", "dropin_test")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/dropin_test not built (needs /root/reference at build time)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "DROPIN OK" in out.stdout


def test_cfg4_reference_adaptive_timeline(cuda):
    """orch::build_adaptive_timeline (orchestrate.cpp:94-154) reproduced on the
    GPU path: warm-started search per window, keep rule, assignment and switch
    plan.  Expected values are the unmodified reference's
    (tests/golden/timeline_cfg4.json)."""
    import json
    w = workloads.load("cfg4")
    g = GpuContext(w.cluster, w.model, w.params)
    tl = orchestrate.build_adaptive_timeline(g, w.types, w.raw["forecasts"], w.span_s, w.raw["min_gain"],
                                             strategy="search", seed=0, search_max_iters=150)
    exp = json.load(open(os.path.join(ROOT, "tests", "golden", "timeline_cfg4.json")))
    got = [{"span_index": e.span_index, "deployment": [[r.device_ids, r.tp, r.pp] for r in e.deployment.replicas],
            "x": e.assignment, "switch_seconds": e.switch_seconds,
            "transfers": 0 if e.switch is None else len(e.switch.transfers)} for e in tl.entries]
    assert got == exp


def test_cfg4_timeline_file_is_the_references(cuda):
    """From the observed counts (Holt forecasts in liboserve_gpu) through the
    GPU search loop to the timeline file: byte-identical to the file the
    reference's build_adaptive_timeline + io::save_timeline wrote."""
    from paper_2602_12151_b200 import json_io
    w = workloads.load("cfg4")
    g = GpuContext(w.cluster, w.model, w.params)
    tl = orchestrate.adaptive_timeline(g, w.types, w.raw["actual"], 50, span_seconds=w.span_s,
                                       min_gain=w.raw["min_gain"], strategy="search", seed=0, search_max_iters=150)
    text = open(os.path.join(ROOT, "tests", "golden", "timeline_cfg4_ref.json")).read()
    assert json_io.dumps(json_io.timeline_json(tl, w.span_s)) == text


def test_cfg4_topk_switch_batch_per_window(cuda, port):
    """every window keeps the exact top-K (1,024) plans
    and costs current -> each of them (K2 key mode); the timeline is the same
    as the plain round's, the batch equals the explicit-deployment K2 and the
    greedy_plan + estimate_time of the CPU oracle on sampled pairs, and the
    chosen pair's plan is the batch's entry for the winner."""
    import numpy as np
    w = workloads.load("cfg4")
    fc = w.raw["forecasts"]
    g = GpuContext(w.cluster, w.model, w.params)
    K = 1024
    tl = orchestrate.build_adaptive_timeline(g, w.types, fc, w.span_s, w.raw["min_gain"], w.space_mode, w.space_sizes,
                                             topk=K)
    base = orchestrate.build_adaptive_timeline(GpuContext(w.cluster, w.model, w.params), w.types, fc, w.span_s,
                                               w.raw["min_gain"], w.space_mode, w.space_sizes)
    assert [(e.span_index, e.deployment.shapes(), e.assignment, e.switch_seconds) for e in tl.entries] == \
        [(e.span_index, e.deployment.shapes(), e.assignment, e.switch_seconds) for e in base.entries]
    assert len(tl.stats) >= 2 and all(len(s.candidate_keys) == K for s in tl.stats)
    rng = np.random.default_rng(4)
    current = None
    checked = 0
    by_window = {e.window: e for e in tl.entries}
    for st in tl.stats:
        g.set_workload(w.types, fc[st.window], w.span_s)
        g.prepare_space(w.space_mode, w.space_sizes)
        if current is not None:
            assert len(st.candidate_switch_seconds) == K
            deps = [g.decode_key(k).deployment for k in st.candidate_keys]
            est_x, _ = g.switch_cost_batch(current, deps)
            assert st.candidate_switch_seconds == est_x
            for i in rng.integers(0, K, 8):
                plan, _ = port.switch_plan(w.cluster, w.model.param_bytes, current, deps[i])
                assert st.candidate_switch_seconds[i] == plan.est_seconds
                checked += 1
            e = by_window.get(st.window)
            if e is not None and e.switch is not None and not e.kept:
                assert e.switch_seconds == st.candidate_switch_seconds[0]  # chosen = top-1 candidate
        e = by_window.get(st.window)
        if e is not None:
            current = e.deployment
    assert checked > 0
