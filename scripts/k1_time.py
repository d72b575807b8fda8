"""Time one device-resident scheduling round (K1 over the whole space) with
CUDA events; prints the median ms and the winner key.  For A/B-ing builds:
OSERVE_GPU_LIB=build/<variant>/liboserve_gpu.so python scripts/k1_time.py"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2602_12151_b200 import workloads  # noqa: E402
from paper_2602_12151_b200._native import GpuContext  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    w = workloads.load(name)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    ctx = GpuContext(w.cluster, w.model, w.params, device=0)
    ctx.set_stream(s.cuda_stream)
    ctx.set_workload(w.types, w.lam, w.span_s)
    parts, plans = ctx.prepare_space(w.space_mode, w.space_sizes)
    key = torch.empty(1, dtype=torch.int64, device="cuda")
    flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
    ctx.launch_round_async(key.data_ptr())
    torch.cuda.synchronize()
    ts = []
    for i in range(reps):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        ctx.launch_round_async(key.data_ptr())
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"{os.environ.get('OSERVE_GPU_LIB', 'default')} {name}: plans {plans} median {statistics.median(ts):.2f} ms "
          f"min {min(ts):.2f} key {int(key.item())}")


if __name__ == "__main__":
    main()
