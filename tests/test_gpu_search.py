"""search::search (deploysearch.cpp:341-417) on the GPU path: the reference's
mutate / enumerate / revert loop in the C++ host runtime with every
best_strategies and capacity-table/assignment step on the device.  The final
deployment, throughput, iteration count and the whole search log (op strings,
acceptances) must equal the unmodified reference's (tests/golden/search.json,
generated from oracle/_ref by oracle/gen_golden.py)."""
import json
import os

import pytest

from paper_2602_12151_b200 import core, workloads
from paper_2602_12151_b200._native import GpuContext

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def cases():
    return json.load(open(os.path.join(GOLD, "search.json")))


@pytest.mark.parametrize("case", cases(), ids=lambda c: f"{c['config']}-seed{c['seed']}-{len(c['log'])}it")
def test_search_matches_reference(cuda, case):
    w = workloads.load(case["config"])
    g = GpuContext(w.cluster, w.model, w.params)
    g.set_workload(w.types, w.lam, w.span_s)
    warm = None
    if "warm_start" in case:
        warm = core.Deployment([core.ReplicaConfig(i, t, p) for i, t, p in case["warm_start"]])
    st, log = g.search(seed=case["seed"], max_iters=case.get("max_iters", 500), warm_start=warm)
    assert st.throughput == case["throughput"]
    assert st.iterations == case["iterations"] and st.stale_iters == case["stale_iters"]
    assert [[r.device_ids, r.tp, r.pp] for r in st.deployment.replicas] == case["deployment"]
    assert [list(r) for r in log] == case["log"]
