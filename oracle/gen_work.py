"""Algorithmic work per plan W for the roofline figure.

W = R*J (cost cells composed) + greedy visits + exchange probes, counted by
the CPU restatement exactly as the reference loops run
(oserve_port.cpp:heuristic).  Exact sums over the whole space where the CPU
finishes in seconds (configs 1, 2), otherwise a seeded uniform sample of
plans (the mean and its standard error are recorded).

Writes paper_2602_12151_b200/configs/work.json (committed; bench.py reads it).
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from paper_2602_12151_b200 import workloads  # noqa: E402
from pyoracle import Oracle, Problem  # noqa: E402


CONFIGS = (("cfg1", None), ("cfg2", None), ("cfg2_low", None), ("cfg3_70b", 50000), ("cfg3_7b", 50000),
           ("cfg5", 50000), ("cfg5_low", 20000), ("cfg5_full", 50000), ("cfg5_7b", 20000))


def main(only=()):
    port = Oracle("port")
    path = os.path.join(ROOT, "paper_2602_12151_b200", "configs", "work.json")
    out = json.load(open(path)) if only and os.path.exists(path) else {}
    threads = os.cpu_count() or 1
    for name, sample in CONFIGS:
        if only and name not in only:
            continue
        w = workloads.load(name)
        pr = Problem(w.cluster, w.model, w.types, w.lam, w.span_s, w.params)
        parts, plans = port.space_info(pr, w.space_mode, w.space_sizes)
        if sample is None or sample >= plans:
            ranks = np.arange(plans, dtype=np.uint64)
            kind = "exact (all plans)"
        else:
            ranks = np.random.default_rng(2602).integers(0, plans, sample).astype(np.uint64)
            kind = f"sampled ({sample} uniform plans, seed 2602)"
        t = time.time()
        obj, spp, work = port.evaluate_ranks(pr, w.space_mode, ranks, w.space_sizes, threads=threads)
        dt = time.time() - t
        wf = work.astype(np.float64)
        out[name] = {"plans": int(plans), "partitions": int(parts), "mean_work": float(wf.mean()),
                     "stderr": float(wf.std() / np.sqrt(len(wf))), "kind": kind,
                     "cpu_port_seconds": dt, "cpu_threads": threads}
        print(name, out[name])
    with open(path, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main(tuple(sys.argv[1:]))  # python oracle/gen_work.py [cfg ...]  (only those, merged)
