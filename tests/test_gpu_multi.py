"""Multi-GPU round inside the library: one context over several
devices (oserve_gpu_create_multi — interleaved plan shards, NCCL all-reduce
MIN of the packed key, all-gather of the top-K lists) must return exactly the
single-device round.  Needs >= 2 GPUs (gpurun --gpus 2/4); skipped otherwise.
The one-GPU shard emulation (8 shards via set_shard) runs everywhere."""
import numpy as np
import pytest

from paper_2602_12151_b200 import workloads
from paper_2602_12151_b200._native import GpuContext

pytestmark = pytest.mark.gpu


def _ngpu():
    import torch
    return torch.cuda.device_count()


def _ctx(w, devices=None):
    g = GpuContext(w.cluster, w.model, w.params, devices=devices)
    g.set_workload(w.types, w.lam, w.span_s)
    return g


@pytest.mark.parametrize("name", ["cfg2", "cfg3_70b", "cfg5", "cfg5_7b"])
def test_eight_shards_on_one_gpu_cover_the_space(cuda, name):
    """set_shard(r, 8) for r = 0..7: the min of the shard keys is the round key
    and each shard holds its interleaved share of the plans."""
    import torch
    w = workloads.load(name)
    g = _ctx(w)
    parts, plans = g.prepare_space(w.space_mode, w.space_sizes)
    full = g.round(w.space_mode, w.space_sizes).key
    d = torch.empty(1, dtype=torch.int64, device="cuda")
    keys = []
    for r in range(8):
        g.set_shard(r, 8)
        g.launch_round_async(d.data_ptr())  # on the context's own stream
        torch.cuda.synchronize()
        keys.append(int(d.item()) & ((1 << 64) - 1))
    g.set_shard(0, 1)
    assert min(keys) == full


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("name", ["cfg2", "cfg5", "cfg5_7b"])
def test_multi_device_round_equals_single(cuda, name):
    import torch
    w = workloads.load(name)
    n = min(_ngpu(), 4)
    one = _ctx(w)
    multi = _ctx(w, devices=list(range(n)))
    assert multi.world() == (0, n, n)
    a = one.round(w.space_mode, w.space_sizes)
    b = multi.round(w.space_mode, w.space_sizes)
    assert (a.key, a.throughput, a.partition_index, a.local_rank) == (b.key, b.throughput, b.partition_index,
                                                                       b.local_rank)
    assert [(r.device_ids, r.tp, r.pp) for r in a.deployment.replicas] == \
        [(r.device_ids, r.tp, r.pp) for r in b.deployment.replicas]
    K = 512
    ka = torch.empty(K, dtype=torch.int64, device="cuda:0")
    kb = torch.empty(K, dtype=torch.int64, device="cuda:0")
    one.round_topk(K, ka.data_ptr())
    multi.round_topk(K, kb.data_ptr())
    assert ka.cpu().tolist() == kb.cpu().tolist()
    # asynchronous sharded launch: global key on the lead device's stream
    d = torch.empty(1, dtype=torch.int64, device="cuda:0")
    multi.launch_round_async(d.data_ptr())
    torch.cuda.synchronize()
    assert int(d.item()) == a.key


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
def test_multi_device_small_spaces_and_search(cuda):
    """Spaces below the sharding threshold and exact-path spaces run on the
    lead device; search() through a multi-device context matches."""
    for name in ("cfg1", "cfg1_bnb"):
        w = workloads.load(name)
        a = _ctx(w).exhaustive()
        b = _ctx(w, devices=[0, 1]).exhaustive()
        assert (a.throughput, a.iterations) == (b.throughput, b.iterations)
    w = workloads.load("cfg2")
    sa = _ctx(w).search(seed=1, max_iters=80)
    sb = _ctx(w, devices=[0, 1]).search(seed=1, max_iters=80)
    assert sa[0].throughput == sb[0].throughput
    assert [(r.device_ids, r.tp, r.pp) for r in sa[0].deployment.replicas] == \
        [(r.device_ids, r.tp, r.pp) for r in sb[0].deployment.replicas]


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
def test_cpp_dropin_multi_device(cuda):
    """oracle/dropin_main.cpp --devices 0,1[,2,3]: the C-ABI round on one and
    on several devices gives the same key and top-K; search() through the
    shim on the device set equals the reference."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "dropin_test")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/dropin_test not built")
    devs = ",".join(str(i) for i in range(min(_ngpu(), 4)))
    out = subprocess.run([exe, "--devices", devs], capture_output=True, text=True, timeout=900)
    print(out.stdout)
    assert out.returncode == 0 and "DROPIN MULTI OK" in out.stdout, out.stdout + out.stderr


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
def test_multi_process_join(cuda):
    """One process per GPU (oserve_gpu_join over a torchrun world)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    n = min(_ngpu(), 4)
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
                          "--master-addr", "127.0.0.1", "--master-port", "29533",
                          os.path.join(root, "scripts", "join_check.py"), "cfg5"],
                         capture_output=True, text=True, timeout=900)
    print(out.stdout[-3000:])
    assert out.returncode == 0 and "JOIN OK" in out.stdout, out.stdout[-3000:] + out.stderr[-3000:]
