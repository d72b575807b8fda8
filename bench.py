"""bench.py — OServe scheduling round on B200 (BASELINE.json metric).

Metric: candidate deployment plans evaluated/sec (+ end-to-end round latency)
on config 5 (128-GPU cluster, 16 request classes, canonical plan space of
13,090,221 plans) unless --config says otherwise.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg5] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1)

One step = one full scheduling round over the whole plan space:
  value : device-resident inputs; K1 (enumerate/unrank -> cost gather -> assign
          -> objective -> argmin) on every rank's shard, NCCL all-reduce(min) of
          the packed key (issued by liboserve_gpu on the round's stream), K2
          switching cost current -> winner (decoded on the device) — no host
          round-trip; CUDA events on the launching stream, max over ranks; L2
          flushed (256 MiB write) between timed iterations.
  e2e   : the public C-ABI from host buffers every step — enumerate + upload the
          space tables, upload the workload, K0 cost kernel, K1 with the exact
          top-K (default 1024) of the packed key (at N > 1 the library
          all-gathers and merges the per-rank lists), K2 switching batch
          current -> each of the K best, key D2H, decode, and the full greedy
          switch plan current -> winner (transfers D2H).  "current" is
          init_uniform (deploysearch.cpp:120-136).
The reference arm (--impl reference) times the reference's own CPU path
(oracle/_ref: /root/reference/proj compiled unmodified; evaluate_deployment per
plan, OpenMP over all host threads) on a bounded sample of the same space.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2602_12151_b200 import _abi as A  # noqa: E402
from paper_2602_12151_b200 import core, workloads  # noqa: E402

METRIC = "candidate deployment plans evaluated/sec and end-to-end scheduling-round latency"
PEAK_LANE_OPS = None  # computed from the device: SMs x 128 lanes x max SM clock
OPS_PER_CELL = 8      # lane-instructions per algorithmic cell-op (fixed)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


_RESULT_FD = None


def emit(line: dict):
    """The one JSON line on the original stdout (libraries' banners, e.g.
    NCCL's version line, are redirected to stderr at the fd level)."""
    os.write(_RESULT_FD if _RESULT_FD is not None else 1, (json.dumps(line) + "\n").encode())


def quiet_stdout():
    global _RESULT_FD
    sys.stdout.flush()
    _RESULT_FD = os.dup(1)
    os.dup2(2, 1)


def init_dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    return rank, world, local


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def start(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx.append(float(p[2]))
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def load_work(name):
    p = os.path.join(ROOT, "paper_2602_12151_b200", "configs", "work.json")
    with open(p) as f:
        return json.load(f)[name]


def init_uniform(w: workloads.Workload, g_min: int) -> core.Deployment:
    """init_uniform (deploysearch.cpp:120-136): D/g_min replicas of g_min
    devices with the most tensor-parallel strategy (tp = g_min here)."""
    R = w.cluster.device_count() // g_min
    return core.canonical_deployment(w.cluster, [g_min] * R, [g_min] * R)


def cpu_reference_sample(w: workloads.Workload, plans: int, target_s: float, threads: int):
    """Time the reference CPU path (oracle/_ref; else the restatement) on a
    bounded uniform sample of the same plan space.  Returns (plans/s, kind, n)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import Oracle, Problem, available
    kind = "reference" if available("ref") else "port"
    orc = Oracle("ref" if kind == "reference" else "port")
    pr = Problem(w.cluster, w.model, w.types, w.lam, w.span_s, w.params)
    rng = np.random.default_rng(2602)
    n = 256
    t = 0.0
    while True:  # grow the sample until it takes ~target_s
        ranks = rng.integers(0, plans, n).astype(np.uint64)
        t0 = time.perf_counter()
        orc.evaluate_ranks(pr, w.space_mode, ranks, w.space_sizes, threads=threads)
        t = time.perf_counter() - t0
        if t >= target_s / 4 or n >= plans:
            break
        n = min(plans, int(n * max(2.0, (target_s / 4) / max(t, 1e-3))))
    # final timed sample ~ target_s
    n2 = min(plans, max(n, int(n * target_s / max(t, 1e-3))))
    ranks = rng.integers(0, plans, n2).astype(np.uint64)
    t0 = time.perf_counter()
    orc.evaluate_ranks(pr, w.space_mode, ranks, w.space_sizes, threads=threads)
    t = time.perf_counter() - t0
    return n2 / t, kind, n2, t


def cpu_model() -> str:
    """lscpu "Model name" of the host, from /proc/cpuinfo."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args, rank, world):
    if rank != 0:
        return
    w = workloads.load(args.config)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import Oracle, Problem, available
    threads = os.cpu_count() or 1
    kind = "reference" if available("ref") else "port"
    orc = Oracle("ref" if kind == "reference" else "port")
    pr = Problem(w.cluster, w.model, w.types, w.lam, w.span_s, w.params)
    parts, plans = orc.space_info(pr, w.space_mode, w.space_sizes)
    # per-step sample sized to ~2 s of CPU work on this host
    rate, _, _, _ = cpu_reference_sample(w, plans, 2.0, threads)
    per_step = int(min(plans, max(64, rate * 2.0)))
    rng = np.random.default_rng(7)
    times = []
    for i in range(args.warmup + args.steps):
        ranks = rng.integers(0, plans, per_step).astype(np.uint64)
        t0 = time.perf_counter()
        orc.evaluate_ranks(pr, w.space_mode, ranks, w.space_sizes, threads=threads)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    tot = sum(times)
    value = per_step * len(times) / tot
    ms = 1e3 * plans / value  # projected full-space round latency
    line = {"metric": METRIC, "value": value, "unit": "plans/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
            "round_latency_ms_projected": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "int64", "data": "synthetic",
            "config": {"workload": f"{w.name}: {w.description}", "plans_in_space": plans, "partitions": parts,
                       "per_step_sample_plans": per_step},
            "cpu_baseline": {"value": value, "unit": "plans/s", "cores": threads, "kind": kind,
                             "cpu_model": cpu_model(),
                             "sample": f"{per_step} uniform random plans of {plans} per step "
                                       f"(evaluate_deployment each, OpenMP dynamic,4 over {threads} threads)"},
            "e2e": {"value": value, "unit": "plans/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


def reference_window_loop(orc, w, forecasts, min_gain, threads):
    """The config-4 window loop on the reference CPU path (oracle/_ref): its
    round over the full ordered space (best_strategies per partition), the
    keep rule's evaluate_deployment, capacity table + solve_assignment and
    layout + greedy_plan (orchestrate.cpp:109-150).  Returns per-window seconds."""
    from pyoracle import Problem
    from paper_2602_12151_b200 import orchestrate
    secs, current, prev_lam = [], None, None
    for lam in forecasts:
        if secs and lam == prev_lam:
            continue
        t0 = time.perf_counter()
        pr = Problem(w.cluster, w.model, w.types, lam, w.span_s, w.params)
        found = orc.round(pr, w.space_mode, w.space_sizes, threads=threads)
        chosen = found.deployment
        if current is not None:
            keep = orc.evaluate_deployment(pr, current)
            if float(found.throughput) <= float(keep) * (1.0 + min_gain):
                chosen = current
        t = orc.capacity_table(pr, chosen)
        orc.solve_assignment(t.n, t.e, lam)
        if current is not None and not orchestrate._same(chosen, current):
            orc.switch_plan(w.cluster, w.model.param_bytes, current, chosen)
        secs.append(time.perf_counter() - t0)
        current, prev_lam = chosen, lam
    return secs


def run_temporal(args, rank, world, local):
    """Config 4: 24 windows of re-scheduling.  One step = the whole timeline
    (orchestrate.build_adaptive_timeline, round strategy): per window K0 + K1
    over the full ordered space (933,333 plans) with the exact top-K (1,024)
    of the packed key, the K2 switching batch current -> each candidate, the
    keep rule, the chosen plan's assignment and the greedy switch plan — all
    through the public API from host buffers (synchronous calls).
    value: plans evaluated per second over the timeline, timed with CUDA
    events on the context's stream; e2e: the same step by the host clock."""
    if rank != 0:
        return
    from paper_2602_12151_b200 import orchestrate
    from paper_2602_12151_b200._native import GpuContext
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    w = workloads.load(args.config)
    fc, mg = w.raw["forecasts"], w.raw["min_gain"]
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx = GpuContext(w.cluster, w.model, w.params, device=local)
    ctx.set_stream(stream.cuda_stream)
    parts, plans = ctx.prepare_space(w.space_mode, w.space_sizes)

    def step():
        return orchestrate.build_adaptive_timeline(ctx, w.types, fc, w.span_s, mg, w.space_mode, w.space_sizes,
                                                   topk=args.topk)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    clocks = Clocks(local)
    clocks.start()
    launches0 = ctx.launch_count()
    bytes0 = ctx.copy_bytes()
    ev_ms, wall_ms, per_window = [], [], []
    tl = None
    for _ in range(args.steps):
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        a_.record(stream)
        tl = step()
        b_.record(stream)
        b_.synchronize()
        wall_ms.append(1e3 * (time.perf_counter() - t0))
        ev_ms.append(a_.elapsed_time(b_))
        per_window.append([1e3 * s_.seconds for s_ in tl.stats])
    clk = clocks.stop()
    launches = (ctx.launch_count() - launches0) // args.steps
    bytes1 = ctx.copy_bytes()
    rounds = tl.rounds
    ms = statistics.mean(ev_ms)
    value = rounds * plans / (ms / 1e3)
    pw = [statistics.median(col) for col in zip(*per_window)]
    cpu = None
    if not args.no_cpu:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        from pyoracle import Oracle, available
        threads = os.cpu_count() or 1
        kind = "reference" if available("ref") else "port"
        orc = Oracle("ref" if kind == "reference" else "port")
        n_win = max(1, min(len(fc), int(args.cpu_seconds)))  # bounded: ~1 s per window on 16 threads
        secs = reference_window_loop(orc, w, fc[:n_win], mg, threads)
        cpu = {"value": len(secs) * plans / sum(secs), "unit": "plans/s", "cores": threads, "kind": kind,
               "sample": f"first {len(secs)} of {rounds} windows of the timeline (reference round over the full "
                         f"ordered space per window + keep rule + assignment + switch plan, {threads} threads)",
               "window_ms": [round(1e3 * x_, 1) for x_ in secs],
               "timeline_s_projected": sum(secs) / len(secs) * rounds}
    line = {"metric": METRIC, "value": value, "unit": "plans/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": f"{w.name}: {w.description}", "windows": len(fc), "rounds_per_step": rounds,
                       "plans_per_round": plans, "partitions": parts, "topk": args.topk,
                       "step": "the whole 24-window timeline"},
            "timeline_ms": ms, "window_ms_median": [round(x_, 3) for x_ in pw],
            "e2e": {"value": rounds * plans / (statistics.mean(wall_ms) / 1e3), "unit": "plans/s",
                    "timeline_ms": statistics.mean(wall_ms),
                    "h2d_bytes_per_step": (bytes1[0] - bytes0[0]) // args.steps,
                    "d2h_bytes_per_step": (bytes1[1] - bytes0[1]) // args.steps},
            "timeline": [{"window": e.window, "deployment": label(e.deployment), "objective": e.objective,
                          "switch_s": e.switch_seconds, "kept": e.kept} for e in tl.entries],
            "cpu_baseline": cpu, "gpu_launches": launches, "clocks": clk}
    emit(line)


def run_ours(args, rank, world, local):
    from paper_2602_12151_b200._native import GpuContext
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    w = workloads.load(args.config)
    stream = torch.cuda.Stream(dev)  # the round, the collective and the events share this stream
    torch.cuda.set_stream(stream)
    ctx = GpuContext(w.cluster, w.model, w.params, device=local)
    ctx.set_stream(stream.cuda_stream)
    if world > 1:
        # the library owns the round's collective: rank 0 makes the NCCL id,
        # every rank joins; rounds then shard over the world inside liboserve_gpu
        from paper_2602_12151_b200._native import nccl_unique_id
        uid = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        ctx.join(bytes(uid.cpu().numpy().tobytes()), rank, world)
    ctx.set_workload(w.types, w.lam, w.span_s)
    parts, plans = ctx.prepare_space(w.space_mode, w.space_sizes)
    g_min = ctx.min_feasible_group()
    current = init_uniform(w, g_min)
    d_key = torch.empty(1, dtype=torch.int64, device=dev)
    d_est = torch.empty(1, dtype=torch.float64, device=dev)
    K = args.topk
    d_topk = torch.empty(K, dtype=torch.int64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)  # > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def device_step():
        # enumerate/unrank -> cost gather -> assign -> objective -> shard argmin (K1),
        # global argmin (NCCL all-reduce MIN issued by the library on the same
        # stream), switching cost current -> winner (K2, key decoded on device)
        ctx.launch_round_async(d_key.data_ptr())
        ctx.switch_cost_keys_async(current, d_key.data_ptr(), 1, d_est.data_ptr())

    # ---- value: device-resident round, per-step events, L2 flushed between ----
    for _ in range(args.warmup):
        device_step()
    barrier()
    launches0 = ctx.launch_count()
    clocks = Clocks(local)
    clocks.start()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    barrier()
    for i in range(args.steps):
        flush.fill_(i)
        starts[i].record(stream)
        device_step()
        ends[i].record(stream)
    barrier()
    clk = clocks.stop()
    launches = ctx.launch_count() - launches0
    step_ms = [s_.elapsed_time(e_) for s_, e_ in zip(starts, ends)]
    t_local = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    total_ms = float(t_local.item())
    ms_per_step = total_ms / args.steps
    value = plans / (ms_per_step / 1e3)
    key = int(d_key.item())
    state = ctx.decode_key(key)
    est_winner = float(d_est.item())

    # ---- dominant kernel alone (K1 on this rank's shard), CUDA events ----
    k_ms = []
    for i in range(3):
        flush.fill_(i)
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_.record(stream)
        ctx.launch_round_async(d_key.data_ptr())
        b_.record(stream)
        b_.synchronize()
        k_ms.append(a_.elapsed_time(b_))
    k_ms = statistics.median(k_ms)
    kt = torch.tensor([k_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(kt, op=dist.ReduceOp.MAX)
    k_ms = float(kt.item())

    # ---- e2e: the public C-ABI from host buffers, every step ----
    e2e_ms = []
    bytes0 = None
    sw_est = []
    for i in range(args.warmup + args.steps):
        barrier()
        if i == args.warmup:
            bytes0 = ctx.copy_bytes()
        t0 = time.perf_counter()
        ctx.prepare_space(w.space_mode, w.space_sizes)             # enumerate + H2D space tables
        ctx.set_workload(w.types, w.lam, w.span_s)                 # H2D workload; K0 cost kernel in the round
        ctx.round_topk(K, d_topk.data_ptr())                       # K0 + K1 + exact top-K; at N > 1 the
                                                                   # library all-gathers + merges the lists
        sw_est, _ = ctx.switch_cost_keys(current, d_topk.data_ptr(), K)  # K2 batch: current -> K best
        extra_h2d = extra_d2h = 0
        k = int(d_topk[0].item())                                  # D2H result key
        st = ctx.decode_key(k)
        plan = ctx.switch_plan(current, st.deployment)             # K2 detail + transfers D2H
        torch.cuda.synchronize(dev)
        dt = (time.perf_counter() - t0) * 1e3
        dtt = torch.tensor([dt], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(dtt, op=dist.ReduceOp.MAX)
        if i >= args.warmup:
            e2e_ms.append(float(dtt.item()))
    e2e_step = statistics.mean(e2e_ms)
    # bytes per step, counted by the C-ABI itself (every cudaMemcpy it issues)
    bytes1 = ctx.copy_bytes()
    h2d = (bytes1[0] - bytes0[0]) // args.steps + extra_h2d
    d2h = (bytes1[1] - bytes0[1]) // args.steps + 8 + extra_d2h  # + the key read (.item()), sharded K2 results
    assert k == key, "e2e and device-resident rounds disagree"

    if rank != 0:
        return
    # ---- roofline: issue-bound ----
    work = load_work(args.config)
    props = torch.cuda.get_device_properties(dev)
    sm_max = clk.get("sm_max_mhz") or 1965.0
    nominal = props.multi_processor_count * 128 * sm_max * 1e6  # lane-ops/s per GPU (4 SMSPs x 32 lanes x clock)
    measured = measured_int_peak()
    peak = measured or nominal
    achieved = work["mean_work"] * OPS_PER_CELL * (plans / world) / (k_ms / 1e3)
    traffic = profile_traffic(args.config)
    executed = k1_executed(args.config)  # ncu thread-instructions of one round's K1 launches
    if executed:
        executed = dict(executed, lane_ops_per_s=executed["thread_inst_per_round"] / world / (k_ms / 1e3))
        executed["frac_of_peak"] = executed["lane_ops_per_s"] / peak
    cpu = None
    if world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        rate, kind, n, t = cpu_reference_sample(w, plans, args.cpu_seconds, threads)
        # the serial run (parallel = false, 1 thread) beside the parallel one
        rate1, _, n1, t1 = cpu_reference_sample(w, plans, max(2.0, args.cpu_seconds / 3), 1)
        cpu = {"value": rate, "unit": "plans/s", "cores": threads, "kind": kind,
               "sample": f"{n} uniform random plans of {plans} ({t:.1f} s; evaluate_deployment each, "
                         f"OpenMP dynamic,4 over {threads} host threads)",
               "round_latency_s_projected": plans / rate, "cpu_model": cpu_model(),
               "serial": {"value": rate1, "unit": "plans/s", "cores": 1,
                          "sample": f"{n1} uniform random plans ({t1:.1f} s, one thread)",
                          "round_latency_s_projected": plans / rate1}}
    line = {
        "metric": METRIC, "value": value, "unit": "plans/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "round_latency_ms": ms_per_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic",
        "config": {"workload": f"{w.name}: {w.description}", "devices": w.cluster.device_count(),
                   "classes": len(w.types), "plans_in_space": plans, "partitions": parts,
                   "space": ("canonical sizes " + str(w.space_sizes)) if w.space_mode else "ordered (reference)",
                   "parallelism": f"plan space sharded x{world} (interleaved 4096-plan chunks); NCCL all-reduce "
                                  f"MIN / all-gather top-K inside liboserve_gpu (oserve_gpu_join)",
                   "l2": "flushed between timed iterations (256 MiB write outside the events)"},
        "winner": {"objective": state.throughput, "key": key, "partition": state.partition_index,
                   "local_rank": state.local_rank, "deployment": label(state.deployment),
                   "switch_from": label(current), "switch_est_seconds": est_winner},
        "e2e": {"value": plans / (e2e_step / 1e3), "unit": "plans/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "round_latency_ms": e2e_step, "topk": K,
                "switch_batch_pairs": K, "switch_est_min_max_s": [min(sw_est), max(sw_est)],
                "winner_switch_est_seconds": plan.est_seconds, "winner_switch_transfers": len(plan.transfers)},
        "roofline": {"bound": "issue", "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "Tlane-op/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "peak_kind": ("measured integer issue peak (profiles/round2_int_peak.json: u64 adds, "
                                   "IADD3+IADD3.X)") if measured else "nominal SMs x 128 lanes x clock",
                     "peak_nominal": nominal / 1e12,
                     "achieved_convention": "SURVEY §8d: algorithmic cell-ops per plan x 8 lane-ops",
                     "executed_ncu": executed,
                     "kernel": "k_plan_eval (K1)", "kernel_ms": k_ms,
                     "work_per_plan": work["mean_work"], "work_kind": work["kind"],
                     "ops_per_cell": OPS_PER_CELL},
        "cpu_baseline": cpu,
        "gpu_launches": launches,
        "clocks": clk,
    }
    emit(line)


def label(dep: core.Deployment) -> str:
    """deployment_label (orchestrate.cpp:34-47): "2x(d4,tp1,pp4)+..."."""
    groups = {}
    for r in dep.replicas:
        k = (r.device_count(), r.tp, r.pp)
        groups[k] = groups.get(k, 0) + 1
    return "+".join(f"{c}x(d{d},tp{t},pp{p})" for (d, t, p), c in sorted(groups.items()))


def measured_int_peak():
    """Measured integer issue peak of this B200 (scripts/int_peak.cu): the
    best of the integer-add kernels, lane-ops/s; None if not measured."""
    p = os.path.join(ROOT, "profiles", "round2_int_peak.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    return max(d.get("int_add_lane_ops_per_s", 0.0), d.get("add64_lane_ops_per_s", 0.0)) or None


def k1_executed(name):
    """ncu thread-instructions executed by one round's K1 launches
    (profiles/round2_k1_ncu.json, the same build's capture)."""
    p = os.path.join(ROOT, "profiles", "round2_k1_ncu.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    return d.get(name)


def profile_traffic(name):
    p = os.path.join(ROOT, "profiles", "k1_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get(name)
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--topk", type=int, default=1024, help="candidates costed by the switching batch (e2e)")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warmup raised to 3 (timing rules)")
        args.warmup = 3
    quiet_stdout()
    rank, world, local = init_dist()
    try:
        if args.impl == "reference":
            run_reference(args, rank, world)
        elif args.config == "cfg4":
            run_temporal(args, rank, world, local)
        else:
            run_ours(args, rank, world, local)
    finally:
        if world > 1 and dist.is_initialized():
            dist.barrier()
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
