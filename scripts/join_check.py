"""Multi-process check of oserve_gpu_join (one GPU per process): every rank
joins its context to the world; the sharded round (K1 + NCCL all-reduce MIN
inside the library) and the top-K (all-gather + merge) must equal a
single-device round computed on rank 0.

  torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/join_check.py [cfg]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2602_12151_b200 import workloads  # noqa: E402
from paper_2602_12151_b200._native import GpuContext, nccl_unique_id  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    w = workloads.load(name)
    g = GpuContext(w.cluster, w.model, w.params, device=local)
    uid = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, 0)
    g.join(uid[0], rank, world)
    assert g.world() == (rank, world, 1)
    g.set_workload(w.types, w.lam, w.span_s)
    st = g.round(w.space_mode, w.space_sizes)
    K = 256
    dk = torch.empty(K, dtype=torch.int64, device=f"cuda:{local}")
    g.round_topk(K, dk.data_ptr())
    topk = dk.cpu().tolist()
    res = [None] * world
    dist.all_gather_object(res, (st.key, topk))
    if rank == 0:
        one = GpuContext(w.cluster, w.model, w.params, device=local)
        one.set_workload(w.types, w.lam, w.span_s)
        ref = one.round(w.space_mode, w.space_sizes)
        one.prepare_space(w.space_mode, w.space_sizes)
        dk1 = torch.empty(K, dtype=torch.int64, device=f"cuda:{local}")
        one.round_topk(K, dk1.data_ptr())
        ok = all(k == ref.key and t == dk1.cpu().tolist() for k, t in res)
        print(f"JOIN {'OK' if ok else 'MISMATCH'}: world {world}, key {ref.key}, objective {ref.throughput}",
              flush=True)
        if not ok:
            sys.exit(1)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
