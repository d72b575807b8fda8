"""One-GPU emulation of the 8-GPU sharded round: the plan space
of a config is dealt into 8 interleaved shards (OSERVE_SHARD_CHUNK = 4096-plan
chunks, oserve_gpu_set_shard(r, 8)); each shard's K1 is timed alone with CUDA
events (median of 3) and the max/mean imbalance reported.  At N = 8 the round
time is the slowest shard's plus the 8-byte all-reduce, so max/mean is the
scaling loss the sharding itself causes.

  python scripts/shard_emulation.py [cfg ...] > profiles/round2_shard8_emulation.json
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2602_12151_b200 import workloads  # noqa: E402
from paper_2602_12151_b200._native import GpuContext  # noqa: E402


def main():
    names = sys.argv[1:] or ["cfg5", "cfg5_full", "cfg5_7b"]
    out = {"device": torch.cuda.get_device_name(0), "shards": 8, "configs": {}}
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    d = torch.empty(1, dtype=torch.int64, device="cuda")
    for name in names:
        w = workloads.load(name)
        g = GpuContext(w.cluster, w.model, w.params)
        g.set_stream(stream.cuda_stream)
        g.set_workload(w.types, w.lam, w.span_s)
        parts, plans = g.prepare_space(w.space_mode, w.space_sizes)

        def timed():
            ms = []
            for _ in range(3):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                g.launch_round_async(d.data_ptr())
                b.record(stream)
                b.synchronize()
                ms.append(a.elapsed_time(b))
            return statistics.median(ms), int(d.item())
        g.launch_round_async(d.data_ptr())  # warm-up
        full_ms, full_key = timed()
        per, keys = [], []
        for r in range(8):
            g.set_shard(r, 8)
            ms, k = timed()
            per.append(ms)
            keys.append(k)
        g.set_shard(0, 1)
        mean = statistics.mean(per)
        out["configs"][name] = {"plans": plans, "partitions": parts, "one_gpu_ms": round(full_ms, 3),
                                "shard_ms": [round(x, 3) for x in per], "max_ms": round(max(per), 3),
                                "mean_ms": round(mean, 3), "max_over_mean": round(max(per) / mean, 4),
                                "emulated_8gpu_speedup": round(full_ms / max(per), 3),
                                "min_shard_key_equals_round_key": min(keys) == full_key}
        print(name, out["configs"][name], file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
