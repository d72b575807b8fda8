// dropin_main.cpp — TEST INFRASTRUCTURE ONLY.
//
// One process linking the UNMODIFIED reference library (compiled from
// /root/reference/proj/src) and liboserve_gpu.so through the C++ shim
// include/oserve_gpu.hpp: every swapped call site of INTEGRATION.md is run
// both ways on the reference's own fixtures and compared bit for bit.
// Built by `make -C oracle dropin` into oracle/_ref/dropin_test; run on a GPU
// box by tests/test_gpu_parity.py::test_cpp_dropin.
#include <cstdio>
#include <cstdlib>
#include <random>

#include "oserve/core.hpp"
#include "oserve/costmodel.hpp"
#include "oserve/deploysearch.hpp"
#include "oserve/flowassign.hpp"
#include "oserve/switchplan.hpp"
#include "oserve_gpu.hpp"

using namespace oserve;

static int failures = 0;
#define EXPECT(cond, what)                                   \
    do {                                                     \
        if (!(cond)) {                                       \
            std::printf("MISMATCH: %s\n", what);             \
            ++failures;                                      \
        }                                                    \
    } while (0)

static ClusterSpec cluster(int machines, int dpm) {
    ClusterSpec c;
    c.intra_bw = 400e9;
    c.inter_bw = 200e9;
    int dev = 0;
    for (int m = 0; m < machines; ++m) {
        MachineSpec ms;
        ms.machine_id = "m" + std::to_string(m);
        ms.device_mem = 80ull * 1000000000ull;
        for (int d = 0; d < dpm; ++d) ms.device_ids.push_back(dev++);
        c.machines.push_back(ms);
    }
    return c;
}

int main() {
    ModelSpec m{"artifact-70b", 140ull * 1000000000ull, 80, 160000, 280000000000ull, 140ull * 1000000000ull};
    std::vector<WorkloadType> types = {{0, 2000.0, 50.0}, {1, 100.0, 3000.0}};
    cost::ProfileParams params;
    ClusterSpec c8 = cluster(1, 8);
    for (auto lam : {std::vector<int64_t>{700, 300}, std::vector<int64_t>{280, 120}, std::vector<int64_t>{5000, 40}}) {
        TraceSpan span{0, lam};
        auto a = search::exhaustive(c8, m, types, span, 60.0, params, true);
        auto b = oserve_gpu::search::exhaustive(c8, m, types, span, 60.0, params, true);
        EXPECT(a.throughput == b.throughput && a.deployment == b.deployment && a.iterations == b.iterations,
               "search::exhaustive");
        search::ObjectiveCache cache;
        search::EvalContext ctx{c8, m, types, span, 60.0, params, &cache, true};
        for (auto sizes : {std::vector<int>{4, 4}, {2, 2, 2, 2}, {6, 2}, {8}, {3, 3, 2}}) {
            auto x = search::best_strategies(sizes, ctx);
            auto y = oserve_gpu::search::best_strategies(sizes, ctx);
            EXPECT(x.objective == y.objective && x.deployment == y.deployment, "search::best_strategies");
            if (!x.deployment.replicas.empty()) {
                EXPECT(search::evaluate_deployment(x.deployment, ctx) ==
                           oserve_gpu::search::evaluate_deployment(x.deployment, ctx),
                       "search::evaluate_deployment");
                auto t1 = cost::build_capacity_table(x.deployment, types, m, c8, params, 60.0);
                auto t2 = oserve_gpu::cost::build_capacity_table(x.deployment, types, m, c8, params, 60.0);
                EXPECT(t1 == t2, "cost::build_capacity_table");
                auto l1 = flow::solve_assignment(t1, lam);
                auto l2 = oserve_gpu::flow::solve_assignment(t1, lam);
                EXPECT(l1.assignment == l2.assignment && l1.M == l2.M && l1.unit == l2.unit && l1.used == l2.used,
                       "flow::solve_assignment");
            }
        }
    }
    // solve_assignment on the reference test's random instance generator shape
    std::mt19937_64 rng(7);
    for (int trial = 0; trial < 80; ++trial) {
        int R = 1 + static_cast<int>(rng() % 3), J = 1 + static_cast<int>(rng() % 3);
        cost::CapacityTable t;
        t.n.assign(R, std::vector<int64_t>(J));
        t.e.assign(R, std::vector<int64_t>(J));
        t.latency.assign(R, std::vector<double>(J, 0.1));
        std::vector<int64_t> lam(J);
        for (int j = 0; j < J; ++j) lam[j] = static_cast<int64_t>(rng() % 61);
        for (int k = 0; k < R; ++k)
            for (int j = 0; j < J; ++j) {
                t.n[k][j] = (rng() % 8 == 0) ? 0 : static_cast<int64_t>(1 + rng() % 100);
                t.e[k][j] = t.n[k][j] == 0 ? 0 : static_cast<int64_t>(rng() % (t.n[k][j] + 1));
            }
        auto a = flow::solve_assignment(t, lam);
        auto b = oserve_gpu::flow::solve_assignment(t, lam);
        EXPECT(a.assignment == b.assignment && a.used == b.used, "flow::solve_assignment (random, exact path)");
        // flow-network formulation: max_flow, extract_assignment, solve_fractional
        auto net = flow::build_network(TraceSpan{0, lam}, t);
        auto f1 = flow::max_flow(net.graph, net.source(), net.sink());
        auto f2 = oserve_gpu::flow::max_flow(net.graph, net.source(), net.sink());
        EXPECT(f1.value == f2.value && f1.flow == f2.flow, "flow::max_flow");
        EXPECT(flow::extract_assignment(net, f1) == oserve_gpu::flow::extract_assignment(net, f1),
               "flow::extract_assignment");
        auto l1 = flow::solve_fractional(t, lam);
        auto l2 = oserve_gpu::flow::solve_fractional(t, lam);
        EXPECT(l1.f == l2.f && l1.objective == l2.objective, "flow::solve_fractional");
    }
    // switching on a 2x4 cluster (SPEC.md acceptance #9 fixture)
    ClusterSpec c24 = cluster(2, 4);
    auto mk = [&](std::vector<int> sizes, std::vector<int> tps) {
        Deployment d;
        int pos = 0;
        for (size_t i = 0; i < sizes.size(); ++i) {
            ReplicaConfig r;
            for (int q = 0; q < sizes[i]; ++q) r.device_ids.push_back(pos++);
            r.tp = tps[i];
            r.pp = sizes[i] / tps[i];
            d.replicas.push_back(r);
        }
        return d;
    };
    std::vector<Deployment> deps = {mk({2, 2, 2, 2}, {2, 2, 2, 2}), mk({4, 4}, {4, 1}), mk({8}, {4}), mk({2, 2, 4}, {1, 2, 4})};
    for (auto &a : deps)
        for (auto &b : deps) {
            auto p1 = switchplan::greedy_plan(switchplan::layout(a, m), switchplan::layout(b, m), c24);
            auto p2 = oserve_gpu::switchplan::greedy_plan(a, b, m, c24);
            EXPECT(p1.transfers == p2.transfers && p1.link_load == p2.link_load && p1.est_seconds == p2.est_seconds,
                   "switchplan::greedy_plan");
            // kv_plan with the parameter plan as carry (switchplan.cpp:142-207)
            std::vector<switchplan::InflightRequest> inflight;
            for (int q = 0; q < 200; ++q)
                inflight.push_back({q, (q * 37) % 101, static_cast<std::uint64_t>(((q * 7919) % 97 + 1) << 20),
                                    q % a.replica_count()});
            auto k1 = switchplan::kv_plan(inflight, 30, a, b, c24, 0.1, &p1);
            auto k2 = oserve_gpu::switchplan::kv_plan(inflight, 30, a, b, c24, 0.1, &p1);
            EXPECT(k1.drained == k2.drained && k1.migrated == k2.migrated && k1.buffer_bytes == k2.buffer_bytes,
                   "switchplan::kv_plan");
        }
    std::printf(failures ? "DROPIN FAILED (%d)\n" : "DROPIN OK\n", failures);
    return failures ? 1 : 0;
}
