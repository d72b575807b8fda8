"""Full-space reference rounds for the canonical configs (3-7B, 5, 5-low).

TEST INFRASTRUCTURE — runs the REFERENCE (oracle/_ref: /root/reference/proj
compiled unmodified) over EVERY plan of each space on all host threads
(config 5: 13,090,221 plans, ~10 min on 8 cores) and merges into
tests/golden/rounds.json:
  * the round winner through the harness's canonical-space loop over
    search::evaluate_deployment (same key as the 70B entry), and
  * an all-plan SHA-256 of the per-plan objectives (little-endian int64 in
    rank order) plus their sum, so the GPU's per-plan path can be checked
    bit-exact over the whole space at full size.
Usage: python oracle/gen_rounds_full.py [--port] [cfg ...]
  --port: use the CPU restatement (oracle/oserve_port.cpp, pinned to the
  reference by tests/test_oracle.py; ~4x faster) for spaces the reference
  library would need hours for (config 5-full: 104.7 M plans).
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from gen_golden import OUT, THREADS, dep_json, objective_digest, problem  # noqa: E402
from paper_2602_12151_b200 import workloads  # noqa: E402
from pyoracle import Oracle  # noqa: E402


def main():
    args = sys.argv[1:]
    kind = "port" if "--port" in args else "ref"
    names = [a for a in args if a != "--port"] or ["cfg3_7b", "cfg5_low", "cfg5"]
    ref = Oracle(kind)
    path = os.path.join(OUT, "rounds.json")
    for name in names:
        w = workloads.load(name)
        pr = problem(w)
        t0 = time.time()
        s = ref.round(pr, w.space_mode, w.space_sizes, threads=THREADS)
        t1 = time.time()
        parts, plans = ref.space_info(pr, w.space_mode, w.space_sizes)
        obj = np.empty(plans, np.int64)
        step = 1 << 21
        for a in range(0, plans, step):
            b = min(plans, a + step)
            o, _, _ = ref.evaluate_ranks(pr, w.space_mode, np.arange(a, b, dtype=np.uint64), w.space_sizes,
                                         threads=THREADS)
            obj[a:b] = o
        t2 = time.time()
        assert int(obj.max()) == s.throughput
        rounds = json.load(open(path))
        rounds[name] = {"kind": "canonical space through search::evaluate_deployment" if kind == "ref" else
                        "canonical space through the pinned CPU restatement (oracle/oserve_port.cpp)",
                        "objective": s.throughput,
                        "partitions": s.iterations, "plans": s.plans, "partition_index": s.partition_index,
                        "local_rank": s.local_rank, "sum_pp": s.sum_pp, "deployment": dep_json(s.deployment),
                        "all_objective_sha256": objective_digest(obj), "objective_sum": int(obj.sum()),
                        "ref_seconds": {"round": round(t1 - t0, 1), "all_plans": round(t2 - t1, 1),
                                        "threads": THREADS}}
        json.dump(rounds, open(path, "w"), indent=1)
        print(name, plans, s.throughput, f"round {t1 - t0:.1f}s all-plans {t2 - t1:.1f}s", flush=True)


if __name__ == "__main__":
    main()
