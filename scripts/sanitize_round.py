"""Small scheduling-round workloads that touch every round kernel: K0a/K0b cost
tables, both K1 buckets (one replica per lane, R <= 32, and two per lane,
R > 32), K2 switching batch and the full switch plan — each on a slice small
enough for a tool's replay.  (compute-sanitizer is closed on the GPU pool, so
the memory-safety evidence is the parity suite plus the kernels' own bounds
checks; this script stays as the minimal per-kernel workload.)

  python scripts/sanitize_round.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2602_12151_b200 import core, workloads  # noqa: E402
from paper_2602_12151_b200._native import GpuContext  # noqa: E402


def main():
    # config 1: full round (K0a, K0b, K1 <G=8/16, KPL=1>)
    w = workloads.load("cfg1")
    g = GpuContext(w.cluster, w.model, w.params, device=0)
    g.set_workload(w.types, w.lam, w.span_s)
    st = g.exhaustive()
    print("cfg1 objective", st.throughput)

    # config 5: a slice of ranks with R <= 32 and one with R > 32 (K1 <32, 1> and <32, 2>)
    w = workloads.load("cfg5")
    g = GpuContext(w.cluster, w.model, w.params, device=0)
    g.set_workload(w.types, w.lam, w.span_s)
    parts, plans = g.prepare_space(w.space_mode, w.space_sizes)
    lo, _ = g.evaluate_ranks(0, 64)              # first partition: 16 x 8-device blocks
    hi, _ = g.evaluate_ranks(plans - 64, 64)     # last partition: 64 x 2-device blocks
    print("cfg5 slices", int(lo.max()), int(hi.max()))

    # switching batch (K2) and one full switch plan: init_uniform -> two canonical candidates
    cur = core.canonical_deployment(w.cluster, [2] * 64, [2] * 64)
    cands = [core.canonical_deployment(w.cluster, [8] * 16, [8] * 16),
             core.canonical_deployment(w.cluster, [4] * 32, [1] * 32)]
    est, mb = g.switch_cost_batch(cur, cands)
    plan = g.switch_plan(cur, cands[0])
    print("switch", est, mb, len(plan.transfers))
    torch.cuda.synchronize()
    print("sanitize workload done")


if __name__ == "__main__":
    main()
