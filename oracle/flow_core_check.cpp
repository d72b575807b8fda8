// TEST INFRASTRUCTURE — host-compiled check of the product's per-instance
// flow cores (paper_2602_12151_b200/csrc/flow_core.hpp, the code K6 runs one
// GPU thread per graph) against the reference's flow::max_flow and
// extract_assignment, before any GPU time is spent.  Built by `make
// flowcheck`; exits non-zero on the first mismatch.
#include <algorithm>
#include <cstdio>
#include <random>
#include <vector>

#include "oserve/flowassign.hpp"
#include "../paper_2602_12151_b200/csrc/flow_core.hpp"

using namespace oserve;
using oserve_gpu::Strided;

static int failures = 0;

static bool check_max_flow(const flow::Graph &g, int s, int t) {
    const int n = g.num_nodes, m = static_cast<int>(g.edges.size());
    std::vector<int32_t> from(m), to(m), arc_to(2 * m), adj(2 * m), adj_off(n + 1), height(n), cur(n), fifo(n);
    std::vector<int64_t> cap(m), res(2 * m), excess(n);
    std::vector<uint8_t> active(n);
    for (int i = 0; i < m; ++i) {
        from[i] = g.edges[i].from;
        to[i] = g.edges[i].to;
        cap[i] = g.edges[i].cap;
    }
    oserve_gpu::PrGraph pg{n, m, {from.data(), 1}, {to.data(), 1}, {cap.data(), 1}, {res.data(), 1},
                           {excess.data(), 1}, {arc_to.data(), 1}, {adj_off.data(), 1}, {adj.data(), 1},
                           {height.data(), 1}, {cur.data(), 1}, {fifo.data(), 1}, {active.data(), 1}};
    if (!oserve_gpu::pr_build(pg)) return false;
    const int64_t v = oserve_gpu::pr_run(pg, s, t);
    auto r = flow::max_flow(g, s, t);
    if (v != r.value) return false;
    for (int i = 0; i < m; ++i)
        if (cap[i] - res[2 * i] != r.flow[i]) return false;
    return true;
}

int main() {
    std::mt19937_64 rng(42);
    for (int trial = 0; trial < 20000; ++trial) {
        flow::Graph g;
        g.num_nodes = 2 + static_cast<int>(rng() % 40);
        int edges = static_cast<int>(rng() % (4 * g.num_nodes)) + 1;
        for (int i = 0; i < edges; ++i) {
            int u = static_cast<int>(rng() % g.num_nodes), v = static_cast<int>(rng() % g.num_nodes);
            if (u == v && rng() % 4) continue;
            g.edges.push_back({u, v, static_cast<int64_t>(rng() % 50)});
        }
        if (!check_max_flow(g, 0, g.num_nodes - 1)) {
            std::printf("max_flow mismatch at trial %d\n", trial);
            ++failures;
            break;
        }
    }
    // network + extract_assignment (warm heuristic path: exact disabled)
    flow::SolveOptions so;
    so.exact_demand_limit = -1;
    for (int trial = 0; trial < 20000; ++trial) {
        const int R = 1 + static_cast<int>(rng() % 8), J = 1 + static_cast<int>(rng() % 6);
        const int64_t maxl = trial % 2 ? 60 : 3000;
        cost::CapacityTable t;
        t.n.assign(R, std::vector<int64_t>(J));
        t.e.assign(R, std::vector<int64_t>(J));
        t.latency.assign(R, std::vector<double>(J, 0.1));
        std::vector<int64_t> lam(J);
        for (int j = 0; j < J; ++j) lam[j] = static_cast<int64_t>(rng() % (maxl + 1));
        for (int k = 0; k < R; ++k)
            for (int j = 0; j < J; ++j) {
                t.n[k][j] = rng() % 8 == 0 ? 0 : static_cast<int64_t>(1 + rng() % 100);
                t.e[k][j] = t.n[k][j] == 0 ? 0 : static_cast<int64_t>(rng() % (t.n[k][j] + 1));
            }
        TraceSpan span{0, lam};
        auto net = flow::build_network(span, t);
        auto fr = flow::max_flow(net.graph, net.source(), net.sink());
        auto a = flow::extract_assignment(net, fr, so);
        // product cores
        std::vector<int64_t> nf(R * J), ef(R * J), unit(R * J), M(R), xs(R * J), mrem(R);
        std::vector<int32_t> capc(R * J);
        std::vector<uint8_t> order(R * 16), olen(R);
        for (int k = 0; k < R; ++k) {
            auto row = flow::normalize_or_scale(t.n[k]);
            M[k] = row.M;
            std::vector<int> ord;
            for (int j = 0; j < J; ++j) {
                nf[k * J + j] = t.n[k][j];
                ef[k * J + j] = t.e[k][j];
                unit[k * J + j] = row.units[j];
                int64_t c = 0;
                if (row.units[j] > 0) {
                    c = std::min(t.e[k][j], t.n[k][j]);
                    c = std::min(c, row.M / row.units[j]);
                    if (c > 0) ord.push_back(j);
                    else c = 0;
                }
                capc[k * J + j] = static_cast<int32_t>(c);
            }
            std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return row.units[x] < row.units[y]; });
            olen[k] = static_cast<uint8_t>(ord.size());
            for (size_t q = 0; q < ord.size(); ++q) order[k * 16 + q] = static_cast<uint8_t>(ord[q]);
        }
        const int nn = oserve_gpu::net_nodes(R, J), m = oserve_gpu::net_edges(R, J);
        std::vector<int32_t> from(m), to(m), arc_to(2 * m), adj(2 * m), adj_off(nn + 1), height(nn), cur(nn), fifo(nn);
        std::vector<int64_t> cap(m), res(2 * m), excess(nn);
        std::vector<uint8_t> active(nn);
        oserve_gpu::NetInstance in{R, J, {nf.data(), 1}, {ef.data(), 1}, {unit.data(), 1}, {M.data(), 1},
                                   {lam.data(), 1}};
        oserve_gpu::net_build(in, {from.data(), 1}, {to.data(), 1}, {cap.data(), 1});
        bool ok = true;
        for (int i = 0; i < m; ++i)
            ok = ok && net.graph.edges[i].from == from[i] && net.graph.edges[i].to == to[i] &&
                 net.graph.edges[i].cap == cap[i];
        oserve_gpu::PrGraph pg{nn, m, {from.data(), 1}, {to.data(), 1}, {cap.data(), 1}, {res.data(), 1},
                               {excess.data(), 1}, {arc_to.data(), 1}, {adj_off.data(), 1}, {adj.data(), 1},
                               {height.data(), 1}, {cur.data(), 1}, {fifo.data(), 1}, {active.data(), 1}};
        oserve_gpu::pr_build(pg);
        ok = ok && oserve_gpu::pr_run(pg, 0, nn - 1) == fr.value;
        for (int k = 0; k < R; ++k)
            for (int j = 0; j < J; ++j) {
                int64_t v = 0;
                const int q = J + 2 * (k * J + j) + 1;
                if (unit[k * J + j] > 0) v = (cap[q] - res[2 * q]) / unit[k * J + j];
                xs[k * J + j] = std::min<int64_t>(v, capc[k * J + j]);
            }
        oserve_gpu::WarmInstance w{R, J, {unit.data(), 1}, {M.data(), 1}, {lam.data(), 1}, {capc.data(), 1},
                                   {order.data(), 1}, {olen.data(), 1}, {xs.data(), 1}, {mrem.data(), 1}};
        const int64_t cnt = oserve_gpu::warm_solve(w);
        ok = ok && cnt == a.objective;
        for (int k = 0; k < R; ++k)
            for (int j = 0; j < J; ++j) ok = ok && xs[k * J + j] == a.x[k][j];
        if (!ok) {
            std::printf("flow_assign mismatch at trial %d (R=%d J=%d)\n", trial, R, J);
            ++failures;
            break;
        }
    }
    std::printf(failures ? "FLOW CORE CHECK FAILED\n" : "FLOW CORE CHECK OK\n");
    return failures ? 1 : 0;
}
