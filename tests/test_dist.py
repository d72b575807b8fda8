"""Multi-rank protocol on CPU (gloo, world_size 2): each rank evaluates its
interleaved shard of the plan order (the C++ shard mapping), packs the
selection key (the C++ key layout), and one all-reduce(min) picks the global
winner — which must equal the single-process round.  The per-plan evaluation
here is the CPU oracle standing in for K1; the GPU path runs the identical
protocol in bench.py over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def case(name):
    """cfg1, or the config-2 classes on a 2x8 cluster at half demand (D=16)."""
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from paper_2602_12151_b200 import core, workloads
    from pyoracle import Problem
    w = workloads.load("cfg1" if name == "cfg1" else "cfg2")
    if name != "cfg1":
        w.cluster = core.cluster(2, 8)
        w.lam = [v // 2 for v in w.lam]
    return w, Problem(w.cluster, w.model, w.types, w.lam, w.span_s, w.params)


def _worker(rank, world, port, name, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2602_12151_b200 import _native
    from pyoracle import Oracle
    w, pr = case(name)
    orc = Oracle("port")
    parts, plans = orc.space_info(pr, w.space_mode, w.space_sizes)
    chunk = 64  # small chunks so every rank gets several
    n = _native.shard_count(plans, rank, world, chunk)
    ranks = np.array([_native.shard_global_rank(i, rank, world, chunk) for i in range(n)], np.uint64)
    obj, spp, _ = orc.evaluate_ranks(pr, w.space_mode, ranks, w.space_sizes, threads=2)
    # partition index / local rank of each plan for the key
    max_count = 0
    keys = []
    for r, o, s in zip(ranks, obj, spp):
        _, pi, lr = orc.space_plan(pr, w.space_mode, int(r), w.space_sizes)
        keys.append((int(o), pi, int(s), lr))
        max_count = max(max_count, lr + 1)
    mc = torch.tensor([max_count], dtype=torch.int64)
    dist.all_reduce(mc, op=dist.ReduceOp.MAX)
    # the layout needs the space's max partition size; use an upper bound
    lay = _native.key_layout(sum(w.lam), parts, w.cluster.device_count(), plans)
    best = min((_native.pack_key(lay, *k) for k in keys), default=(1 << 63) - 1)
    t = torch.tensor([best], dtype=torch.int64)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    cnt = torch.tensor([n], dtype=torch.int64)
    dist.all_reduce(cnt, op=dist.ReduceOp.SUM)
    if rank == 0:
        q.put((int(t.item()), int(cnt.item()), lay, plans))
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["cfg1", "d16"])
def test_two_rank_round_equals_single_process(port, name):
    from paper_2602_12151_b200 import _native
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    port_no = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port_no, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    key, count, lay, plans = q.get(timeout=600)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert count == plans
    w, pr = case(name)
    s = port.round(pr, w.space_mode, w.space_sizes, threads=4)
    assert key == _native.pack_key(lay, s.throughput, s.partition_index, s.sum_pp, s.local_rank)
