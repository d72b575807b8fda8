"""Full-space reference rounds for the canonical configs.

TEST INFRASTRUCTURE — runs the REFERENCE (oracle/_ref: /root/reference/proj
compiled unmodified) over EVERY plan of each space on the host threads
(config 5: 13,090,221 plans, ~18 min on 8 cores; config 5-full: 104.7 M
plans, a few hours) and merges into tests/golden/rounds.json:
  * the round winner, and
  * an all-plan SHA-256 of the per-plan objectives (little-endian int64 in
    rank order) plus their sum, so the GPU's per-plan path can be checked
    bit-exact over the whole space at full size.

One pass: every plan goes through search::evaluate_deployment
(deploysearch.cpp:138-151) once (oracle_evaluate_ranks); the winner is the
minimum of the round's packed key (objective desc, partition, sum_pp, rank)
over those per-plan outputs — the same selection the harness's canonical
round (`oracle_round`) makes, recomputed here from the stored arrays.  With
--round the harness round runs as well and both winners must agree.

Chunks are cached under $OSERVE_DIGEST_CACHE (default /tmp/oserve_digest) so
an interrupted run resumes.

Usage: python oracle/gen_rounds_full.py [--port] [--round] [cfg ...]
  --port: use the CPU restatement (oracle/oserve_port.cpp) instead.
  OSERVE_THREADS overrides the thread count (default: all host threads).
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from gen_golden import OUT, dep_json, objective_digest, problem  # noqa: E402
from paper_2602_12151_b200 import workloads  # noqa: E402
from pyoracle import Oracle  # noqa: E402

THREADS = int(os.environ.get("OSERVE_THREADS", os.cpu_count() or 1))
CACHE = os.environ.get("OSERVE_DIGEST_CACHE", "/tmp/oserve_digest")
STEP = 1 << 21


def all_plans(ref, kind, name, w, pr, plans):
    """Per-plan objectives and sum_pp over ranks [0, plans), chunk-cached."""
    d = os.path.join(CACHE, f"{kind}_{name}")
    os.makedirs(d, exist_ok=True)
    obj = np.empty(plans, np.int64)
    spp = np.empty(plans, np.int32)
    for a in range(0, plans, STEP):
        b = min(plans, a + STEP)
        f = os.path.join(d, f"{a:012d}.npz")
        if os.path.exists(f):
            z = np.load(f)
            obj[a:b], spp[a:b] = z["obj"], z["spp"]
            continue
        t0 = time.time()
        o, s, _ = ref.evaluate_ranks(pr, w.space_mode, np.arange(a, b, dtype=np.uint64), w.space_sizes,
                                     threads=THREADS)
        obj[a:b], spp[a:b] = o, s
        np.savez(f + ".tmp.npz", obj=o, spp=s)
        os.replace(f + ".tmp.npz", f)
        print(f"  {name}: {b}/{plans} ({time.time() - t0:.0f}s/chunk)", flush=True)
    return obj, spp


def winner(ref, w, pr, obj, spp):
    """Minimum packed key over the per-plan outputs: objective desc, then the
    first partition (partitions are contiguous rank ranges in enumeration
    order), then sum_pp asc, then rank asc."""
    best = int(obj.max())
    cand = np.flatnonzero(obj == best)
    _, p0, l0 = ref.space_plan(pr, w.space_mode, int(cand[0]), w.space_sizes)
    same = []
    for r in cand:
        _, p, _ = ref.space_plan(pr, w.space_mode, int(r), w.space_sizes)
        if p != p0:
            break
        same.append(int(r))
    r_win = min(same, key=lambda r: (int(spp[r]), r))
    dep, p, local = ref.space_plan(pr, w.space_mode, r_win, w.space_sizes)
    return best, p, local, int(spp[r_win]), dep


def main():
    args = sys.argv[1:]
    kind = "port" if "--port" in args else "ref"
    also_round = "--round" in args
    names = [a for a in args if not a.startswith("--")] or ["cfg3_7b", "cfg5_low", "cfg5"]
    ref = Oracle(kind)
    path = os.path.join(OUT, "rounds.json")
    for name in names:
        w = workloads.load(name)
        pr = problem(w)
        parts, plans = ref.space_info(pr, w.space_mode, w.space_sizes)
        t0 = time.time()
        obj, spp = all_plans(ref, kind, name, w, pr, plans)
        t1 = time.time()
        best, p, local, s_pp, dep = winner(ref, w, pr, obj, spp)
        if also_round:
            s = ref.round(pr, w.space_mode, w.space_sizes, threads=THREADS)
            assert (s.throughput, s.partition_index, s.local_rank, s.sum_pp) == (best, p, local, s_pp), name
        rounds = json.load(open(path))
        rounds[name] = {"kind": "canonical space, every plan through search::evaluate_deployment" if kind == "ref"
                        else "canonical space through the pinned CPU restatement (oracle/oserve_port.cpp)",
                        "objective": best, "partitions": parts, "plans": plans, "partition_index": p,
                        "local_rank": local, "sum_pp": s_pp, "deployment": dep_json(dep),
                        "all_objective_sha256": objective_digest(obj), "objective_sum": int(obj.sum()),
                        "ref_seconds": {"all_plans": round(t1 - t0, 1), "threads": THREADS}}
        json.dump(rounds, open(path, "w"), indent=1)
        print(name, plans, best, f"all-plans {t1 - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main()
