"""Generate the synthetic scheduling-round configs (BASELINE.json configs 1-5).

TEST/CONFIG INFRASTRUCTURE — runs in the build container only (needs the
reference oracle oracle/_ref).  Writes paper_2602_12151_b200/configs/cfg*.json;
those JSON files are the committed inputs of bench.py and the parity tests,
so nothing downstream needs /root/reference.

Usage: python oracle/gen_configs.py [cfg ...]   (default: every config)

Workload recipe:
  * trace: 200k records, seed 2602, two lognormal families mixed 60/40 —
    short-output (in ~ LogN(ln 2048, .6), out ~ LogN(ln 28, .8)) and
    long-output (in ~ LogN(ln 1024, .7), out ~ LogN(ln 230, .6)), clipped to
    input [1, 7999], output [1, 5000];
  * classes: the reference's workload::fit_types(records, k=J, seed=0)
    (workload.cpp:32-162) — J in {4, 8, 16};  J = 2 uses the fixtures'
    short/long types (fixtures.hpp:72-73);
  * lambda_j = round(load * share_j * C), C = objective of init_uniform
    (deploysearch.cpp:120-136) evaluated at lambda_j = 1e9, load 0.9
    (plus a demand-limited load 0.3 variant);
  * config 4: 24 windows, class mix swinging 0.7 -> 0.3 -> 0.7 between the two
    families (cosine), load 0.9, +-10% jitter seed 7; per-window lambda are the
    reference's Holt forecasts (orchestrate.cpp:75-92).
"""
from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from paper_2602_12151_b200 import core  # noqa: E402
from pyoracle import Oracle, Problem  # noqa: E402

OUT = os.path.join(ROOT, "paper_2602_12151_b200", "configs")


def synthetic_trace(n=200_000, seed=2602):
    rng = np.random.default_rng(seed)
    fam = (rng.random(n) >= 0.6).astype(np.int64)  # 0 = short-output (60%), 1 = long-output
    inp = np.where(fam == 0, rng.lognormal(math.log(2048), 0.6, n), rng.lognormal(math.log(1024), 0.7, n))
    out = np.where(fam == 0, rng.lognormal(math.log(28), 0.8, n), rng.lognormal(math.log(230), 0.6, n))
    inp = np.clip(np.rint(inp), 1, 7999).astype(np.uint32)
    out = np.clip(np.rint(out), 1, 5000).astype(np.uint32)
    return inp, out, fam


def assign(types, inp, out):
    """workload::assign_type (workload.cpp:164-179) vectorised."""
    i_min, i_max = float(inp.min()), float(inp.max())
    o_min, o_max = float(out.min()), float(out.max())
    ni = (inp - i_min) / (i_max - i_min)
    no = (out - o_min) / (o_max - o_min)
    ci = np.array([(t.centroid_in - i_min) / (i_max - i_min) for t in types])
    co = np.array([(t.centroid_out - o_min) / (o_max - o_min) for t in types])
    d = (ni[:, None] - ci[None, :]) ** 2 + (no[:, None] - co[None, :]) ** 2
    return np.argmin(d, axis=1)


def cluster_json(machines, dpm, mem=80 * core.KGB, intra=400e9, inter=200e9):
    return {"machines": machines, "devices_per_machine": dpm, "device_mem": mem,
            "intra_bw": intra, "inter_bw": inter}


def model_json(m: core.ModelSpec):
    return {"name": m.name, "param_bytes": m.param_bytes, "num_layers": m.num_layers,
            "bytes_per_token_kv": m.bytes_per_token_kv,
            "flops_per_token_prefill": m.flops_per_token_prefill, "min_mem_bytes": m.min_mem_bytes}


def types_json(types):
    return [{"type_id": t.type_id, "centroid_in": t.centroid_in, "centroid_out": t.centroid_out} for t in types]


def uniform_capacity(ref: Oracle, cl, model, types):
    """C: init_uniform's objective at lambda_j = 1e9."""
    pr = Problem(cl, model, types, [10 ** 9] * len(types))
    g = ref.min_feasible_group(pr)
    R = cl.device_count() // g
    dep = core.canonical_deployment(cl, [g] * R, [g] * R)  # most-TP strategy, blocks in one machine
    return ref.evaluate_deployment(pr, dep)


def main():
    os.makedirs(OUT, exist_ok=True)
    ref = Oracle("ref")
    inp, out, fam = synthetic_trace()
    fitted = {}
    for J in (4, 8, 16):
        fitted[J] = ref.fit_types(inp, out, J, seed=0)
    prof = core.ProfileParams()

    only = [a if a.endswith(".json") else a + ".json" for a in sys.argv[1:]]

    def write(name, cfg):
        if only and name not in only:
            return
        with open(os.path.join(OUT, name), "w") as f:
            json.dump(cfg, f, indent=1)
        print("wrote", name, {k: cfg[k] for k in ("lambda",) if k in cfg})

    base = {"profile": prof.__dict__, "span_seconds": 60.0}

    # config 1: D=8, J=2, 70B-class; heuristic and exact (B&B) demand points
    for name, lam in (("cfg1.json", [700, 300]), ("cfg1_bnb.json", [280, 120])):
        write(name, dict(base, name=name[:-5], description="Single scheduling round, 8-GPU cluster, "
                         "70B-class model, 2 request classes (fixtures short/long)",
                         cluster=cluster_json(1, 8), model=model_json(core.model_140gb()),
                         classes=types_json([core.short_type(), core.long_type()]), **{"lambda": lam},
                         space={"mode": "ordered", "sizes": []}))

    def lam_for(cl, model, types, load):
        lab = assign(types, inp, out)
        share = np.bincount(lab, minlength=len(types)) / len(lab)
        C = uniform_capacity(ref, cl, model, types)
        return [int(round(load * s * C)) for s in share], C

    def emit(name, desc, machines, model, J, space, load=0.9):
        if only and name not in only:
            return
        cl = core.cluster(machines, 8)
        lam, C = lam_for(cl, model, fitted[J], load)
        write(name, dict(base, name=name[:-5], description=desc, cluster=cluster_json(machines, 8),
                         model=model_json(model), classes=types_json(fitted[J]), **{"lambda": lam},
                         load=load, uniform_capacity=C, space=space))

    ordered = {"mode": "ordered", "sizes": []}
    emit("cfg2.json", "32-GPU cluster, 4 request classes, full ordered DP/TP/PP plan space", 4,
         core.model_140gb(), 4, ordered)
    emit("cfg2_low.json", "config 2 at demand-limited load 0.3", 4, core.model_140gb(), 4, ordered, load=0.3)
    p2_70 = [2, 4, 8, 16, 32, 64]
    p2_7 = [1, 2, 4, 8, 16, 32, 64]
    emit("cfg3_70b.json", "64-GPU cluster, 8 classes, 70B-class cost tables, canonical pow2 space", 8,
         core.model_140gb(), 8, {"mode": "canonical", "sizes": p2_70})
    emit("cfg3_7b.json", "64-GPU cluster, 8 classes, 7B-class cost tables, canonical pow2 space", 8,
         core.model_14gb(), 8, {"mode": "canonical", "sizes": p2_7})
    emit("cfg5.json", "128-GPU cluster, 16 classes, canonical plan space sizes {2,4,8}", 16,
         core.model_140gb(), 16, {"mode": "canonical", "sizes": [2, 4, 8]})
    emit("cfg5_low.json", "config 5 at demand-limited load 0.3", 16, core.model_140gb(), 16,
         {"mode": "canonical", "sizes": [2, 4, 8]}, load=0.3)
    emit("cfg5_full.json", "128-GPU cluster, 16 classes, canonical plan space sizes {2,4,...,128} "
         "(every power-of-two block)", 16, core.model_140gb(), 16,
         {"mode": "canonical", "sizes": [2, 4, 8, 16, 32, 64, 128]})
    # 7B-class model on the config-5 cluster: g_min = 1, so plans reach 128
    # replicas (sizes {1,2,4}: R from 32 to 128)
    emit("cfg5_7b.json", "128-GPU cluster, 16 classes, 7B-class cost tables, canonical plan space sizes "
         "{1,2,4} (32-128 replicas per plan)", 16, core.model_14gb(), 16, {"mode": "canonical", "sizes": [1, 2, 4]})

    # config 4: temporal, 24 windows on the config-2 cluster
    if only and "cfg4.json" not in only:
        return
    cl = core.cluster(4, 8)
    types = fitted[4]
    lab = assign(types, inp, out)
    C = uniform_capacity(ref, cl, core.model_140gb(), types)
    share_fam = []
    for f in (0, 1):
        sel = lab[fam == f]
        share_fam.append(np.bincount(sel, minlength=len(types)) / len(sel))
    rng = np.random.Generator(np.random.MT19937(7))
    actual = []
    for w in range(24):
        rho = 0.5 + 0.2 * math.cos(2 * math.pi * w / 24)  # short-family share 0.7 -> 0.3 -> 0.7
        mix = rho * share_fam[0] + (1 - rho) * share_fam[1]
        jit = 1.0 + (2 * rng.random(len(types)) - 1) * 0.1
        actual.append([int(round(0.9 * C * m * j)) for m, j in zip(mix, jit)])
    forecasts = ref.holt_forecast(actual, window=50)
    write("cfg4.json", dict(base, name="cfg4", description="Temporal trace: 24 windows, predicted workload "
                            "shifts, re-scheduling + switching cost per window (config-2 cluster)",
                            cluster=cluster_json(4, 8), model=model_json(core.model_140gb()),
                            classes=types_json(types), actual=actual, forecasts=forecasts,
                            **{"lambda": forecasts[0]}, min_gain=0.01, uniform_capacity=C, space=ordered))


if __name__ == "__main__":
    main()
