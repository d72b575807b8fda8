"""oserve::flow on the GPU path.

solve_assignment (flowassign.cpp:481-503): LCM normalisation (K0b) +
greedy/exchange (K1) or branch-and-bound (K4), batched over raw tables.

The flow-network formulation (flowassign.cpp:67-245, 505-519, 559-645):
Graph / FlowResult / FlowNetwork mirror the reference types; max_flow runs
the FIFO push-relabel on the device (K6a, one lane per graph, the
reference's per-edge flows), build_network + max_flow + extract_assignment
run fused per instance (K6b), solve_fractional is the dense simplex (K7).
build_network's bookkeeping and to_dot's text are host-side."""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import core
from ._native import GpuContext

_ctx: Optional[GpuContext] = None


def _gpu(opts: Optional[core.SolveOptions]) -> GpuContext:
    global _ctx
    if _ctx is None:
        _ctx = GpuContext(core.cluster(1, 1), core.ModelSpec("none", 1, 1, 1, 1, 1))
    _ctx.set_solve_options(opts or core.SolveOptions())
    return _ctx


def solve_assignment(table: core.CapacityTable, lam: Sequence[int],
                     opts: Optional[core.SolveOptions] = None) -> core.LowerLevel:
    if len(lam) != table.types():
        raise ValueError("solve_assignment: lambda size mismatch")
    return solve_assignment_batch([table.n], [table.e], [list(lam)], opts)[0]


def solve_assignment_batch(n: Sequence, e: Sequence, lam: Sequence,
                           opts: Optional[core.SolveOptions] = None) -> List[core.LowerLevel]:
    """Many independent instances of equal shape [count][R][J]."""
    x, obj, M, unit, used = _gpu(opts).solve_batch(np.asarray(n), np.asarray(e), np.asarray(lam))
    return [core.LowerLevel(core.AssignmentMatrix(x[i].tolist(), int(obj[i])), M[i].tolist(), unit[i].tolist(),
                            used[i].tolist()) for i in range(len(obj))]


@dataclass
class NormalizedRow:
    """flow::NormalizedRow (flowassign.hpp:16-20)."""
    M: int
    units: List[int]
    scaled: bool = False


def normalize(n_row: Sequence[int]) -> NormalizedRow:
    """flow::normalize (flowassign.cpp:31-46) on the device (K0b); raises
    core.LcmOverflow when the LCM exceeds 2^62."""
    if not len(n_row):
        return NormalizedRow(1, [], False)
    M, U, sc = _gpu(None).normalize_batch(np.asarray([list(n_row)]), strict=True)
    return NormalizedRow(int(M[0]), U[0].tolist(), bool(sc[0]))


def normalize_or_scale(n_row: Sequence[int]) -> NormalizedRow:
    """flow::normalize_or_scale (flowassign.cpp:48-62) on the device (K0b)."""
    if not len(n_row):
        return NormalizedRow(1, [], False)
    M, U, sc = _gpu(None).normalize_batch(np.asarray([list(n_row)]), strict=False)
    return NormalizedRow(int(M[0]), U[0].tolist(), bool(sc[0]))


def check_constraints(a: core.AssignmentMatrix, table: core.CapacityTable, lam: Sequence[int]) -> None:
    """flow::check_constraints (flowassign.cpp:529-551) on the device: raises
    core.LogicError naming the first violated constraint (C1, C2 or C3)."""
    if not table.n:
        return
    _gpu(None).check_constraints_batch(np.asarray([a.x]), np.asarray([table.n]), np.asarray([table.e]),
                                       np.asarray([list(lam)]))


# ---- flow-network formulation ------------------------------------------------
INT64_MAX = (1 << 63) - 1


@dataclass
class Edge:
    """flow::Graph::Edge (flowassign.hpp:32-36)."""
    from_: int
    to: int
    cap: int


@dataclass
class Graph:
    num_nodes: int = 0
    edges: List[Edge] = field(default_factory=list)


@dataclass
class FlowResult:
    value: int = 0
    flow: List[int] = field(default_factory=list)


@dataclass
class FlowNetwork:
    """flow::FlowNetwork (flowassign.hpp:52-79): node layout S, w_j, i_kj
    (k-major), c_k^in, c_k^out, T; edge classes in that order."""
    R: int
    J: int
    lam: List[int]
    e: List[List[int]]
    n: List[List[int]]
    unit: List[List[int]]
    M: List[int]
    graph: Graph

    def source(self): return 0
    def sink(self): return 1 + self.J + self.R * self.J + 2 * self.R
    def node_w(self, j): return 1 + j
    def node_i(self, k, j): return 1 + self.J + k * self.J + j
    def node_c_in(self, k): return 1 + self.J + self.R * self.J + k
    def node_c_out(self, k): return 1 + self.J + self.R * self.J + self.R + k
    def node_count(self): return 2 + self.J + self.R * self.J + 2 * self.R
    def edge_source(self, j): return j
    def edge_w_i(self, k, j): return self.J + 2 * (k * self.J + j)
    def edge_i_c(self, k, j): return self.J + 2 * (k * self.J + j) + 1
    def edge_node(self, k): return self.J + 2 * self.R * self.J + k
    def edge_out(self, k): return self.J + 2 * self.R * self.J + self.R + k
    def edge_count(self): return self.J + 2 * self.R * self.J + 2 * self.R


def build_network(counts: Sequence[int], table: core.CapacityTable) -> FlowNetwork:
    """flow::build_network (flowassign.cpp:152-199); M/unit come from the
    device normalisation (K0b)."""
    R = table.replicas()
    if R == 0:
        raise core.EmptyDeployment("build_network: deployment has no replicas")
    J = table.types()
    if len(counts) != J:
        raise ValueError(f"build_network: span has {len(counts)} type counts but table has {J}")
    ll = solve_assignment(table, list(counts))
    net = FlowNetwork(R, J, [int(v) for v in counts], [list(r) for r in table.e], [list(r) for r in table.n],
                      ll.unit, ll.M, Graph(2 + J + R * J + 2 * R))
    g = net.graph.edges
    for j in range(J):
        g.append(Edge(net.source(), net.node_w(j), net.lam[j]))
    for k in range(R):
        for j in range(J):
            cap = 0
            u = net.unit[k][j]
            if u > 0:
                ekj = min(net.e[k][j], net.n[k][j])
                cap = net.M[k] if ekj > net.M[k] // u else ekj * u
            g.append(Edge(net.node_w(j), net.node_i(k, j), cap))
            g.append(Edge(net.node_i(k, j), net.node_c_in(k), cap))
    for k in range(R):
        g.append(Edge(net.node_c_in(k), net.node_c_out(k), net.M[k]))
    for k in range(R):
        jj = max(J, 1)
        cap = INT64_MAX if net.M[k] > INT64_MAX // jj else net.M[k] * jj
        g.append(Edge(net.node_c_out(k), net.sink(), cap))
    return net


def max_flow(g: Graph, source: int, sink: int) -> FlowResult:
    """flow::max_flow on the device (K6a)."""
    return max_flow_batch([g], [source], [sink])[0]


def max_flow_batch(graphs: Sequence[Graph], sources: Sequence[int], sinks: Sequence[int]) -> List[FlowResult]:
    out = _gpu(None).max_flow_batch([(g.num_nodes, [(e.from_, e.to, e.cap) for e in g.edges]) for g in graphs],
                                    sources, sinks)
    return [FlowResult(v, f) for v, f in out]


def extract_assignment(net: FlowNetwork, fr: FlowResult,
                       opts: Optional[core.SolveOptions] = None) -> core.AssignmentMatrix:
    """flow::extract_assignment (flowassign.cpp:505-519) on the device."""
    x, obj = _gpu(opts).extract_assignment_batch(np.asarray([net.n]), np.asarray([net.e]), np.asarray([net.lam]),
                                                 np.asarray([fr.flow]))
    return core.AssignmentMatrix(x[0].tolist(), int(obj[0]))


def flow_assign_batch(n, e, lam, opts: Optional[core.SolveOptions] = None, edge_flows: bool = False):
    """build_network -> max_flow -> extract_assignment fused per instance
    (K6b): returns (assignments, flow values, per-edge flows or None)."""
    x, obj, val, fl = _gpu(opts).flow_assign_batch(np.asarray(n), np.asarray(e), np.asarray(lam), edge_flows)
    return [core.AssignmentMatrix(x[i].tolist(), int(obj[i])) for i in range(len(obj))], val.tolist(), fl


def to_dot(net: FlowNetwork, fr: Optional[FlowResult] = None) -> str:
    """flow::to_dot (flowassign.cpp:201-243), the same text."""
    def label(i):
        s = ""
        if fr is not None and i < len(fr.flow):
            s = f"{fr.flow[i]} | "
        return s + str(net.graph.edges[i].cap)
    out = ["digraph flownet {\n  rankdir=LR;\n", "  S [shape=circle];\n  T [shape=doublecircle];\n"]
    out += [f"  w{j} [shape=box];\n" for j in range(net.J)]
    out += [f"  cin{k} [shape=ellipse];\n  cout{k} [shape=ellipse];\n" for k in range(net.R)]
    out += [f'  S -> w{j} [label="{label(net.edge_source(j))}"];\n' for j in range(net.J)]
    for k in range(net.R):
        for j in range(net.J):
            out.append(f'  w{j} -> i{k}_{j} [label="{label(net.edge_w_i(k, j))}"];\n')
            out.append(f'  i{k}_{j} -> cin{k} [label="{label(net.edge_i_c(k, j))}"];\n')
    for k in range(net.R):
        out.append(f'  cin{k} -> cout{k} [label="{label(net.edge_node(k))}"];\n')
        out.append(f'  cout{k} -> T [label="{label(net.edge_out(k))}"];\n')
    out.append("}\n")
    return "".join(out)


@dataclass
class FractionalSolution:
    f: List[List[float]]
    objective: float


def solve_fractional(table: core.CapacityTable, lam: Sequence[int]) -> FractionalSolution:
    """flow::solve_fractional (flowassign.cpp:559-645) on the device (K7)."""
    f, obj = _gpu(None).solve_fractional_batch(np.asarray([table.n]), np.asarray([table.e]), np.asarray([list(lam)]))
    return FractionalSolution(f[0].tolist(), float(obj[0]))
