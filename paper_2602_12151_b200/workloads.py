"""Synthetic scheduling-round workloads (BASELINE.json configs 1-5).

The JSON files under configs/ are generated once by oracle/gen_configs.py
(reference fit_types on a seeded synthetic trace) and committed; this module
only reads them.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass, field
from typing import List

from . import _abi as A
from . import core

CONFIG_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "configs")


@dataclass
class Workload:
    name: str
    description: str
    cluster: core.ClusterSpec
    model: core.ModelSpec
    types: List[core.WorkloadType]
    lam: List[int]
    span_s: float
    params: core.ProfileParams
    space_mode: int
    space_sizes: List[int] = field(default_factory=list)
    raw: dict = field(default_factory=dict)


def load(name: str) -> Workload:
    with open(os.path.join(CONFIG_DIR, f"{name}.json")) as f:
        c = json.load(f)
    cl = c["cluster"]
    cluster = core.cluster(cl["machines"], cl["devices_per_machine"], cl["device_mem"], cl["intra_bw"],
                           cl["inter_bw"])
    model = core.ModelSpec(**c["model"])
    types = [core.WorkloadType(**t) for t in c["classes"]]
    mode = A.SPACE_ORDERED if c["space"]["mode"] == "ordered" else A.SPACE_CANONICAL
    return Workload(c["name"], c.get("description", ""), cluster, model, types, list(c["lambda"]),
                    float(c["span_seconds"]), core.ProfileParams(**c["profile"]), mode, list(c["space"]["sizes"]), c)


def names() -> List[str]:
    return sorted(f[:-5] for f in os.listdir(CONFIG_DIR) if f.endswith(".json"))
