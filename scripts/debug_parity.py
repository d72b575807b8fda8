"""Debug helper: per-plan GPU vs CPU-oracle mismatches with assignment dumps."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_2602_12151_b200 import workloads  # noqa: E402
from paper_2602_12151_b200._native import GpuContext  # noqa: E402
from pyoracle import Oracle, Problem  # noqa: E402

port = Oracle("port")
for name in sys.argv[1:]:
    w = workloads.load(name)
    g = GpuContext(w.cluster, w.model, w.params)
    g.set_workload(w.types, w.lam, w.span_s)
    pr = Problem(w.cluster, w.model, w.types, w.lam, w.span_s, w.params)
    parts, plans = g.prepare_space(w.space_mode, w.space_sizes)
    n = min(plans, 3000)
    obj, _ = g.evaluate_ranks(0, n)
    eo, _, _ = port.evaluate_ranks(pr, w.space_mode, np.arange(n, dtype=np.uint64), w.space_sizes, threads=8)
    bad = np.nonzero(obj != eo)[0]
    print(name, "mismatches", len(bad), "of", n)
    for r in bad[:1]:
        dep, _, _ = port.space_plan(pr, w.space_mode, int(r), w.space_sizes)
        table, lower = g.plan_detail(dep)
        t = port.capacity_table(pr, dep)
        ll = port.solve_assignment(t.n, t.e, w.lam)
        print(" rank", r, "gpu", obj[r], "detail", lower.assignment.objective, "cpu", eo[r], dep.shapes())
        print("  gpu x", lower.assignment.x, "used", lower.used)
        print("  cpu x", ll.assignment.x, "used", ll.used, "M", ll.M, "unit", ll.unit)
        print("  n", t.n, "e", t.e, "gpu n", table.n)
