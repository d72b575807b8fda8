import sys, json, os, time
os.environ["OSERVE_DEBUG_KV"] = "1"
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2602_12151_b200 import workloads, core, _abi
from paper_2602_12151_b200._native import GpuContext
w = workloads.load("cfg5")
sw = json.load(open("tests/golden/switch.json"))
pair = [p for p in sw if p["config"] == "cfg5"][0]
src = core.Deployment([core.ReplicaConfig(i, tp, pp) for i, tp, pp in pair["src"]])
dst = core.Deployment([core.ReplicaConfig(i, tp, pp) for i, tp, pp in pair["dst"]])
carry = core.SwitchPlan([core.Transfer(core.ByteRange(b, e), s, d) for b, e, s, d in pair["transfers"]])
rng = np.random.default_rng(1)
reqs = np.zeros(200_000, _abi.inflight_dtype())
reqs["request_id"] = np.arange(len(reqs)); reqs["generated_tokens"] = rng.integers(0, 2000, len(reqs))
reqs["kv_bytes"] = rng.integers(1 << 20, 1 << 30, len(reqs)); reqs["source_replica"] = rng.integers(0, src.replica_count(), len(reqs))
g = GpuContext(w.cluster, w.model, w.params)
print("dst reps", dst.replica_count(), "src reps", src.replica_count())
for _ in range(3): g.kv_plan(reqs, 500, src, dst, 0.1, carry, as_arrays=True)
torch.cuda.synchronize(); t=time.perf_counter()
for _ in range(5): g.kv_plan(reqs, 500, src, dst, 0.1, carry, as_arrays=True)
torch.cuda.synchronize(); print("call ms", (time.perf_counter()-t)/5*1e3)
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    g.kv_plan(reqs, 500, src, dst, 0.1, carry, as_arrays=True); torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12))
