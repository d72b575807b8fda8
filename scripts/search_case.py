"""Time search::search on one random problem (tests/test_gpu_random_rounds.py
draw_case) on the GPU path and the reference.  Usage:
  python scripts/search_case.py <draw seed> <search seed> [gpu|ref|both]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import pyoracle  # noqa: E402
from test_gpu_random_rounds import draw_case  # noqa: E402

ds, ss = int(sys.argv[1]), int(sys.argv[2])
which = sys.argv[3] if len(sys.argv) > 3 else "both"
ref = pyoracle.Oracle("ref")
cl, model, types, lam, params, mode, sizes, plans = draw_case(ref, ds)
print("D", cl.device_count(), "J", len(types), "lam", lam, "model", model.name, flush=True)
pr = pyoracle.Problem(cl, model, types, lam, 60.0, params)
if which in ("ref", "both"):
    t = time.perf_counter()
    es, elog = ref.search(pr, seed=ss, max_iters=200)
    print("ref  %.3f s" % (time.perf_counter() - t), es.throughput, es.iterations, len(elog), flush=True)
if which in ("gpu", "both"):
    from paper_2602_12151_b200._native import GpuContext
    g = GpuContext(cl, model, params)
    g.set_workload(types, lam, 60.0)
    os.environ.get("OSERVE_DEBUG_EXACT")
    t = time.perf_counter()
    st, log = g.search(seed=ss, max_iters=200)
    print("gpu  %.3f s" % (time.perf_counter() - t), st.throughput, st.iterations, len(log), flush=True)
    for r in log[:40]:
        print("  ", list(r))
