"""Per-call host times of one config-4 window loop (the calls of
orchestrate.build_adaptive_timeline, each followed by a device sync)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_12151_b200 import orchestrate, workloads  # noqa: E402
from paper_2602_12151_b200._native import GpuContext  # noqa: E402

w = workloads.load("cfg4")
ctx = GpuContext(w.cluster, w.model, w.params)
ctx.prepare_space(w.space_mode, w.space_sizes)
fc = w.raw["forecasts"]
orig = {}
acc = {}


def wrap(name):
    f = getattr(ctx, name)

    def g(*a, **k):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize()
        acc[name] = acc.get(name, 0.0) + time.perf_counter() - t
        return r
    setattr(ctx, name, g)


for n in ("set_workload", "prepare_space", "round_topk", "decode_key", "switch_cost_keys", "evaluate_deployments",
          "plan_detail", "switch_plan"):
    wrap(n)
for rep in range(3):
    acc.clear()
    torch.cuda.synchronize()
    t = time.perf_counter()
    orchestrate.build_adaptive_timeline(ctx, w.types, fc, w.span_s, w.raw["min_gain"], w.space_mode, w.space_sizes,
                                        topk=1024)
    torch.cuda.synchronize()
    tot = time.perf_counter() - t
print(f"timeline {tot * 1e3:.1f} ms")
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"  {k:22s} {v * 1e3:7.2f} ms")
