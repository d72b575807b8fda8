"""Per-call wall time of bench.py's e2e round (config 5, one GPU): where the
host-side milliseconds around the device round go.  Each call is followed by
a device synchronize."""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2602_12151_b200 import core, workloads  # noqa: E402
from paper_2602_12151_b200._native import GpuContext  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
    w = workloads.load(name)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    ctx = GpuContext(w.cluster, w.model, w.params, device=0)
    ctx.set_stream(s.cuda_stream)
    ctx.set_workload(w.types, w.lam, w.span_s)
    ctx.prepare_space(w.space_mode, w.space_sizes)
    g = ctx.min_feasible_group()
    R = w.cluster.device_count() // g
    cur = core.canonical_deployment(w.cluster, [g] * R, [g] * R)
    K = 1024
    d_topk = torch.empty(K, dtype=torch.int64, device="cuda")
    d_key = torch.empty(1, dtype=torch.int64, device="cuda")
    parts = {}

    def t(label, fn):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        parts.setdefault(label, []).append(1e3 * (time.perf_counter() - t0))
        return r

    for it in range(6):
        t("prepare_space", lambda: ctx.prepare_space(w.space_mode, w.space_sizes))
        t("set_workload", lambda: ctx.set_workload(w.types, w.lam, w.span_s))
        t("round_topk (K0+K1+top-K)", lambda: ctx.round_topk(K, d_topk.data_ptr()))
        t("launch_round_async (K1 only)", lambda: ctx.launch_round_async(d_key.data_ptr()))
        t("switch_cost_keys x1024", lambda: ctx.switch_cost_keys(cur, d_topk.data_ptr(), K))
        k = t("key D2H", lambda: int(d_topk[0].item()))
        st = t("decode_key", lambda: ctx.decode_key(k))
        t("switch_plan", lambda: ctx.switch_plan(cur, st.deployment))
    for k, v in parts.items():
        print(f"{k:32s} median {statistics.median(v[1:]):8.3f} ms")


if __name__ == "__main__":
    main()
