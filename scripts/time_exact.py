"""Time the exact path: config 1-B&B exhaustive (61 plans, all B&B) on the
GPU vs the reference (oracle/_ref) on the host."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import torch  # noqa: E402

from paper_2602_12151_b200 import workloads  # noqa: E402
from paper_2602_12151_b200._native import GpuContext  # noqa: E402

w = workloads.load("cfg1_bnb")
g = GpuContext(w.cluster, w.model, w.params)
g.set_workload(w.types, w.lam, w.span_s)
for rep in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = g.exhaustive()
    torch.cuda.synchronize()
    print(f"gpu exhaustive: {time.perf_counter() - t:.3f} s obj={r.throughput} launches={g.launch_count()}")
try:
    from pyoracle import Oracle, Problem, available
    if available("ref"):
        ref = Oracle("ref")
        pr = Problem(w.cluster, w.model, w.types, w.lam, w.span_s, w.params)
        for par in (False, True):
            t = time.perf_counter()
            s = ref.exhaustive(pr, parallel=par)
            print(f"reference exhaustive (parallel={par}): {time.perf_counter() - t:.3f} s obj={s.throughput}")
except Exception as e:  # noqa: BLE001
    print("reference timing skipped:", e)
