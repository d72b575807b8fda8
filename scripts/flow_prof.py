"""Host/kernel split of max_flow_arrays on the f4 row's 20k graphs (torch profiler)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2602_12151_b200 import _abi, core  # noqa: E402
from paper_2602_12151_b200._native import GpuContext  # noqa: E402

rng = np.random.default_rng(1)
G = 20_000
nn = rng.integers(20, 61, G).astype(np.int32)
m = np.array([int(rng.integers(v, 4 * v)) for v in nn], np.int64)
off = np.zeros(G + 1, np.int64)
off[1:] = np.cumsum(m)
edges = np.zeros(int(off[-1]), _abi.flow_edge_dtype())
owner = np.repeat(np.arange(G), m)
edges["from"] = (rng.random(len(edges)) * nn[owner]).astype(np.int32)
edges["to"] = (rng.random(len(edges)) * nn[owner]).astype(np.int32)
edges["cap"] = rng.integers(0, 1000, len(edges))
g = GpuContext(core.cluster(1, 8), core.model_140gb())
src = np.zeros(G, np.int32)
for _ in range(3):
    g.max_flow_arrays(nn, off, edges, src, nn - 1)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    g.max_flow_arrays(nn, off, edges, src, nn - 1)
torch.cuda.synchronize()
print("call ms", (time.perf_counter() - t) / 5 * 1e3)
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    g.max_flow_arrays(nn, off, edges, src, nn - 1)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=10))
