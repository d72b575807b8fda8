"""§8(f4) flow-network formulation on the device (K6a/K6b/K7) against the
reference's own outputs (tests/golden/flow.json, oracle/gen_golden.py):
per-edge max-flows, extracted assignments, LP relaxations and DOT text,
plus the reference tests' known answers (test_flowassign.cpp:100-322)."""
import json
import os

import numpy as np
import pytest

from paper_2602_12151_b200 import core, flow
from paper_2602_12151_b200._native import GpuContext

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "flow.json")))


def table(n, e):
    return core.CapacityTable(n, e, [[0.1] * len(n[0]) for _ in n])


def g(nn, edges):
    return flow.Graph(nn, [flow.Edge(a, b, c) for a, b, c in edges])


def test_max_flow_golden_batch(cuda):
    gs = GOLD["graphs"]
    out = flow.max_flow_batch([g(x["num_nodes"], x["edges"]) for x in gs], [x["source"] for x in gs],
                              [x["sink"] for x in gs])
    for x, r in zip(gs, out):
        assert r.value == x["value"] and r.flow == x["flow"]


def test_max_flow_known_answers(cuda):
    r = flow.max_flow(g(5, [(0, 1, 10), (1, 2, 80), (2, 3, 80), (3, 4, 80)]), 0, 4)
    assert r.value == 10 and r.flow == [10, 10, 10, 10]
    assert flow.max_flow(g(4, [(0, 1, 10), (1, 2, 10)]), 0, 3).value == 0


def test_max_flow_errors(cuda):
    with pytest.raises(ValueError):
        flow.max_flow(g(3, [(0, 1, 1)]), 0, 0)
    with pytest.raises(ValueError):
        flow.max_flow(g(3, [(0, 1, 1)]), 0, 3)
    with pytest.raises(ValueError):
        flow.max_flow(g(3, [(0, 1, -1)]), 0, 2)


def test_flow_assign_golden(cuda):
    by_shape = {}
    for x in GOLD["instances"]:
        by_shape.setdefault((len(x["n"]), len(x["lambda"])), []).append(x)
    for (R, J), xs in by_shape.items():
        got, vals, fl = flow.flow_assign_batch([x["n"] for x in xs], [x["e"] for x in xs],
                                               [x["lambda"] for x in xs], edge_flows=True)
        for i, x in enumerate(xs):
            assert got[i].x == x["x"] and got[i].objective == x["objective"], (R, J, i)
            assert vals[i] == x["value"] and fl[i].tolist() == x["flow"]


def test_extract_assignment_of_given_flow(cuda):
    for x in GOLD["instances"][:60]:
        net = flow.build_network(x["lambda"], table(x["n"], x["e"]))
        a = flow.extract_assignment(net, flow.FlowResult(x["value"], x["flow"]))
        assert a.x == x["x"] and a.objective == x["objective"]


def test_network_assembly_known_answers(cuda):
    net = flow.build_network([10], table([[80]], [[80]]))
    assert net.node_count() == 6 and len(net.graph.edges) == 5
    assert net.graph.edges[net.edge_source(0)].cap == 10 and net.unit[0][0] == 1
    for q in (net.edge_w_i(0, 0), net.edge_i_c(0, 0), net.edge_node(0), net.edge_out(0)):
        assert net.graph.edges[q].cap == 80
    net = flow.build_network([10, 10], table([[80, 50], [40, 20]], [[80, 50], [40, 20]]))
    assert net.node_count() == 12 and len(net.graph.edges) == 14
    assert net.graph.edges[net.edge_w_i(0, 1)].cap == 400 and net.graph.edges[net.edge_node(0)].cap == 400
    with pytest.raises(core.EmptyDeployment):
        flow.build_network([], core.CapacityTable([], [], []))
    # the device network is the host network: flows of max_flow(net.graph) equal the fused path's
    fr = flow.max_flow(net.graph, net.source(), net.sink())
    _, vals, fl = flow.flow_assign_batch([net.n], [net.e], [net.lam], edge_flows=True)
    assert fr.value == vals[0] and fr.flow == fl[0].tolist()


def test_extraction_known_answers(cuda):
    net = flow.build_network([100, 50], table([[80, 50]], [[80, 50]]))
    a = flow.extract_assignment(net, flow.max_flow(net.graph, net.source(), net.sink()))
    assert a.objective == 80 and a.x == [[80, 0]]  # the IP optimum (test_flowassign.cpp:186-195)
    assert flow.max_flow(net.graph, net.source(), net.sink()).value == 150


def test_solve_fractional_golden(cuda):
    by_shape = {}
    for x in GOLD["lp"]:
        by_shape.setdefault((len(x["n"]), len(x["lambda"])), []).append(x)
    for xs in by_shape.values():
        gctx = flow._gpu(None)
        f, obj = gctx.solve_fractional_batch(np.asarray([x["n"] for x in xs]), np.asarray([x["e"] for x in xs]),
                                             np.asarray([x["lambda"] for x in xs]))
        for i, x in enumerate(xs):
            assert f[i].tolist() == x["f"] and float(obj[i]) == x["objective"]  # bit-identical FP64


def test_fractional_bounds_integral(cuda):
    for x in GOLD["instances"][:80]:
        lp = flow.solve_fractional(table(x["n"], x["e"]), x["lambda"])
        assert lp.objective >= x["objective"] - 1e-6


def test_to_dot_text(cuda):
    for d in GOLD["dot"]:
        net = flow.build_network(d["lambda"], table(d["n"], d["e"]))
        fr = flow.max_flow(net.graph, net.source(), net.sink()) if d["with_flow"] else None
        assert flow.to_dot(net, fr) == d["dot"]


BIG = json.load(open(os.path.join(ROOT, "tests", "golden", "flow_big.json")))


def _sha(fl):
    import hashlib
    return hashlib.sha256(np.asarray(fl, "<i8").tobytes()).hexdigest()


@pytest.mark.parametrize("batch", ["similar", "ragged"])
def test_max_flow_past_shared_memory(cuda, batch):
    """Graphs whose workspace exceeds the shared-memory slice: the HBM kernel,
    interleaved (34 similar graphs) and packed (a ragged batch)."""
    gs = BIG[batch]
    out = flow.max_flow_batch([g(x["num_nodes"], x["edges"]) for x in gs], [x["source"] for x in gs],
                              [x["sink"] for x in gs])
    for x, r in zip(gs, out):
        assert r.value == x["value"] and _sha(r.flow) == x["flow_sha256"]


def test_flow_assign_past_shared_memory(cuda):
    """R = 40, J = 10 instances (workspace past the shared-memory slice)."""
    gctx = GpuContext(core.cluster(1, 8), core.model_140gb())
    cs = BIG["instances"]
    x, obj, val, fl = gctx.flow_assign_batch(np.asarray([c["n"] for c in cs]), np.asarray([c["e"] for c in cs]),
                                             np.asarray([c["lambda"] for c in cs]), edge_flows=True)
    for i, c in enumerate(cs):
        assert x[i].tolist() == c["x"] and int(obj[i]) == c["objective"] and int(val[i]) == c["value"]
        assert _sha(fl[i]) == c["flow_sha256"]
