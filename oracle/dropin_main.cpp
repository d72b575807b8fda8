// dropin_main.cpp — TEST INFRASTRUCTURE ONLY.
//
// One process linking the UNMODIFIED reference library (compiled from
// /root/reference/proj/src) and liboserve_gpu.so through the C++ shim
// include/oserve_gpu.hpp: every swapped call site of INTEGRATION.md is run
// both ways on the reference's own fixtures and compared bit for bit.
// Built by `make -C oracle dropin` into oracle/_ref/dropin_test; run on a GPU
// box by tests/test_gpu_parity.py::test_cpp_dropin.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>

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

// Exceptions of a call as (type, message) so both sides can be compared.
template <class F>
static std::string outcome(F &&f) {
    try {
        f();
        return "ok";
    } catch (const LcmOverflow &e) {
        return std::string("LcmOverflow:") + e.what();
    } catch (const UnsourcedFragment &e) {
        return std::string("UnsourcedFragment:") + e.what();
    } catch (const std::logic_error &e) {
        return std::string("logic_error:") + e.what();
    } catch (const std::exception &e) {
        return std::string("exception:") + e.what();
    }
}

static double secs(std::chrono::steady_clock::time_point a) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
}

// orchestrate.cpp:116-145 (build_adaptive_timeline's window body) with every
// call swapped one for one: search, evaluate_deployment (keep rule),
// build_capacity_table + solve_assignment (assignment_for), layout x2 +
// greedy_plan.  Returns a printable trace of the decisions.
struct WindowOut {
    Deployment chosen;
    flow::AssignmentMatrix x;
    switchplan::SwitchPlan plan;
    std::int64_t found = 0;
};

template <bool GPU>
static std::vector<WindowOut> adaptive_windows(const ClusterSpec &cl, const ModelSpec &m,
                                               const std::vector<WorkloadType> &types,
                                               const std::vector<std::vector<std::int64_t>> &lams, int iters) {
    cost::ProfileParams params;
    std::vector<WindowOut> out;
    Deployment current;
    for (size_t w = 0; w < lams.size(); ++w) {
        TraceSpan span{static_cast<std::int64_t>(w), lams[w]};
        search::SearchOptions so;
        so.seed = 0;
        so.max_iters = iters;
        if (!current.replicas.empty()) so.warm_start = &current;
        search::SearchState found = GPU ? oserve_gpu::search::search(cl, m, types, span, 60.0, params, so)
                                        : search::search(cl, m, types, span, 60.0, params, so);
        Deployment chosen = found.deployment;
        if (!current.replicas.empty()) {
            search::ObjectiveCache cache;
            search::EvalContext ctx{cl, m, types, span, 60.0, params, &cache, true};
            std::int64_t keep = GPU ? oserve_gpu::search::evaluate_deployment(current, ctx)
                                    : search::evaluate_deployment(current, ctx);
            if (static_cast<double>(found.throughput) <= static_cast<double>(keep) * 1.01) chosen = current;
        }
        auto table = GPU ? oserve_gpu::cost::build_capacity_table(chosen, types, m, cl, params, 60.0)
                         : cost::build_capacity_table(chosen, types, m, cl, params, 60.0);
        WindowOut o;
        o.chosen = chosen;
        o.found = found.throughput;
        o.x = GPU ? oserve_gpu::flow::solve_assignment(table, lams[w]).assignment
                  : flow::solve_assignment(table, lams[w]).assignment;
        if (!current.replicas.empty() && !(chosen == current)) {
            if (GPU) {
                auto from = oserve_gpu::switchplan::layout(current, m);
                auto to = oserve_gpu::switchplan::layout(chosen, m);
                o.plan = oserve_gpu::switchplan::greedy_plan(from, to, cl);
            } else {
                auto from = switchplan::layout(current, m);
                auto to = switchplan::layout(chosen, m);
                o.plan = switchplan::greedy_plan(from, to, cl);
            }
        }
        out.push_back(o);
        current = chosen;
    }
    return out;
}

// Multi-GPU: the same canonical 128-device round through one context on
// 1 device and on `devs` (sharded, NCCL all-reduce / all-gather inside the
// library) must give the same winner key and top-K list.
static void multi_device_round(const std::vector<int> &devs) {
    ClusterSpec cl = cluster(16, 8);
    oserve_gpu::ClusterBuf cb(cl);
    ModelSpec m{"artifact-70b", 140ull * 1000000000ull, 80, 160000, 280000000000ull, 140ull * 1000000000ull};
    oserve_model_desc md = oserve_gpu::model_desc(m);
    oserve_profile pd = oserve_gpu::profile_desc(cost::ProfileParams{});
    std::vector<oserve_class> cls;
    std::vector<std::int64_t> lam;
    for (int j = 0; j < 16; ++j) {  // 16 classes, short- and long-output families
        cls.push_back({j, 200.0 + 400.0 * (j % 8), j < 8 ? 30.0 + 10.0 * j : 150.0 + 60.0 * (j - 8)});
        lam.push_back(300 + 97 * ((j * 7) % 16));
    }
    const int sizes[3] = {2, 4, 8};
    oserve_space_desc space{OSERVE_SPACE_CANONICAL, 3, sizes, 0};
    auto run = [&](const std::vector<int> &d, std::vector<std::uint64_t> &topk) {
        oserve_gpu_ctx *c = nullptr;
        oserve_gpu::check(d.size() > 1 ? oserve_gpu_create_multi(d.data(), static_cast<int>(d.size()), &cb.desc, &md,
                                                                 &pd, &c)
                                       : oserve_gpu_create(d[0], &cb.desc, &md, &pd, &c),
                          nullptr);
        oserve_gpu::check(oserve_gpu_set_workload(c, 16, cls.data(), lam.data(), 60.0), c);
        auto res = std::make_unique<oserve_round_result>();
        auto t0 = std::chrono::steady_clock::now();
        oserve_gpu::check(oserve_gpu_round(c, &space, res.get()), c);
        const double t_round = secs(t0);
        t0 = std::chrono::steady_clock::now();
        oserve_gpu::check(oserve_gpu_round(c, &space, res.get()), c);
        const double t_round2 = secs(t0);
        void *dk = nullptr;
        cudaSetDevice(d[0]);
        cudaMalloc(&dk, 8 * 256);
        oserve_gpu::check(oserve_gpu_round_topk(c, 256, static_cast<std::uint64_t *>(dk), nullptr), c);
        topk.resize(256);
        cudaMemcpy(topk.data(), dk, 8 * 256, cudaMemcpyDeviceToHost);
        cudaFree(dk);
        int r = 0, w = 0, loc = 0;
        oserve_gpu_world(c, &r, &w, &loc);
        std::printf("  %zu device(s) [world %d, local %d]: plans %llu, key %llu, objective %lld, round %.1f ms "
                    "(first %.1f ms)\n",
                    d.size(), w, loc, static_cast<unsigned long long>(res->plans),
                    static_cast<unsigned long long>(res->key), static_cast<long long>(res->objective),
                    1e3 * t_round2, 1e3 * t_round);
        oserve_gpu_destroy(c);
        return res->key;
    };
    std::vector<std::uint64_t> t1, tn;
    const std::uint64_t k1 = run({devs[0]}, t1);
    const std::uint64_t kn = run(devs, tn);
    EXPECT(k1 == kn, "multi-device round key");
    EXPECT(t1 == tn, "multi-device top-K list");
    // the shim on the device set: a D = 32 search (best_strategies sharded
    // for partitions of >= 65,536 plans) against the reference
    ClusterSpec c32 = cluster(4, 8);
    std::vector<WorkloadType> t4 = {{0, 2048.0, 28.0}, {1, 1024.0, 230.0}, {2, 4000.0, 60.0}, {3, 600.0, 900.0}};
    TraceSpan span{0, {1600, 1200, 800, 400}};
    search::SearchOptions so;
    so.max_iters = 60;
    auto a = search::search(c32, m, t4, span, 60.0, cost::ProfileParams{}, so);
    oserve_gpu::set_devices(devs);
    auto b = oserve_gpu::search::search(c32, m, t4, span, 60.0, cost::ProfileParams{}, so);
    oserve_gpu::set_devices({devs[0]});
    EXPECT(a.throughput == b.throughput && a.deployment == b.deployment && a.iterations == b.iterations,
           "search::search on the device set");
}

int main(int argc, char **argv) {
    if (argc > 2 && std::strcmp(argv[1], "--devices") == 0) {
        std::vector<int> devs;
        for (const char *p = argv[2]; *p;) {
            devs.push_back(std::atoi(p));
            while (*p && *p != ',') ++p;
            if (*p == ',') ++p;
        }
        multi_device_round(devs);
        std::printf(failures ? "DROPIN MULTI FAILED (%d)\n" : "DROPIN MULTI OK\n", failures);
        return failures ? 1 : 0;
    }
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
    // layout / greedy_plan(ShardLayout...) / estimate_time, one for one
    // (orchestrate.cpp:142-144), incl. a hand-made layout with several
    // ranges per device and an unsourced fragment
    for (auto &a : deps)
        for (auto &b : deps) {
            auto la = switchplan::layout(a, m), lb = switchplan::layout(b, m);
            auto ga = oserve_gpu::switchplan::layout(a, m), gb = oserve_gpu::switchplan::layout(b, m);
            bool same = la.held == ga.held && la.shards.size() == ga.shards.size();
            for (size_t i = 0; same && i < la.shards.size(); ++i)
                same = la.shards[i].shard_id == ga.shards[i].shard_id && la.shards[i].range == ga.shards[i].range &&
                       la.shards[i].holder == ga.shards[i].holder;
            EXPECT(same, "switchplan::layout");
            auto p1 = switchplan::greedy_plan(la, lb, c24);
            auto p2 = oserve_gpu::switchplan::greedy_plan(ga, gb, c24);
            EXPECT(p1.transfers == p2.transfers && p1.link_load == p2.link_load && p1.est_seconds == p2.est_seconds,
                   "switchplan::greedy_plan(ShardLayout)");
            EXPECT(switchplan::estimate_time(p1, c24) == oserve_gpu::switchplan::estimate_time(p1, c24),
                   "switchplan::estimate_time");
        }
    {
        switchplan::ShardLayout s1, s2;
        s1.held[0] = {{0, 10}, {20, 30}};
        s1.held[5] = {{5, 25}};
        s1.held[9] = {{30, 40}};
        s2.held[1] = {{0, 40}};
        s2.held[6] = {{0, 5}, {25, 35}};
        auto p1 = switchplan::greedy_plan(s1, s2, c24);
        auto p2 = oserve_gpu::switchplan::greedy_plan(s1, s2, c24);
        EXPECT(p1.transfers == p2.transfers && p1.link_load == p2.link_load && p1.est_seconds == p2.est_seconds,
               "switchplan::greedy_plan(multi-range layouts)");
        s2.held[7] = {{35, 50}};
        EXPECT(outcome([&] { switchplan::greedy_plan(s1, s2, c24); }) ==
                   outcome([&] { oserve_gpu::switchplan::greedy_plan(s1, s2, c24); }),
               "switchplan::greedy_plan UnsourcedFragment");
    }
    // normalize / normalize_or_scale / check_constraints (test_flowassign.cpp rows)
    for (auto row : {std::vector<int64_t>{80, 50}, {7}, {12, 18, 30}, {80, 0, 50},
                     {(1ll << 31) - 1, (1ll << 31) - 99, (1ll << 31) - 365}, {0, 0}, {-1, 3}}) {
        flow::NormalizedRow a1, b1, a2, b2;
        const std::string o1 = outcome([&] { a1 = flow::normalize(row); });
        const std::string o2 = outcome([&] { b1 = oserve_gpu::flow::normalize(row); });
        EXPECT(o1 == o2 && a1.M == b1.M && a1.units == b1.units && a1.scaled == b1.scaled, "flow::normalize");
        const std::string o3 = outcome([&] { a2 = flow::normalize_or_scale(row); });
        const std::string o4 = outcome([&] { b2 = oserve_gpu::flow::normalize_or_scale(row); });
        EXPECT(o3 == o4 && a2.M == b2.M && a2.units == b2.units && a2.scaled == b2.scaled, "flow::normalize_or_scale");
    }
    {
        std::mt19937_64 r2(11);
        for (int trial = 0; trial < 200; ++trial) {
            const int R = 1 + static_cast<int>(r2() % 4), J = 1 + static_cast<int>(r2() % 4);
            cost::CapacityTable t;
            t.n.assign(R, std::vector<int64_t>(J));
            t.e.assign(R, std::vector<int64_t>(J));
            t.latency.assign(R, std::vector<double>(J, 0.1));
            std::vector<int64_t> lam(J);
            for (int j = 0; j < J; ++j) lam[j] = static_cast<int64_t>(r2() % 40);
            for (int k = 0; k < R; ++k)
                for (int j = 0; j < J; ++j) {
                    t.n[k][j] = (r2() % 6 == 0) ? 0 : static_cast<int64_t>(1 + r2() % 30);
                    t.e[k][j] = static_cast<int64_t>(r2() % (t.n[k][j] + 1));
                }
            flow::AssignmentMatrix a = flow::solve_assignment(t, lam).assignment;
            if (trial % 2) {  // perturb: some violate C1 / C2 / C3
                const int k = static_cast<int>(r2() % R), j = static_cast<int>(r2() % J);
                a.x[k][j] += 1 + static_cast<int64_t>(r2() % 3);
            }
            EXPECT(outcome([&] { flow::check_constraints(a, t, lam); }) ==
                       outcome([&] { oserve_gpu::flow::check_constraints(a, t, lam); }),
                   "flow::check_constraints");
        }
    }
    // build_adaptive_timeline's window body (orchestrate.cpp:116-145) with
    // every call swapped, on a 32-device cluster over 4 windows
    {
        ClusterSpec c32 = cluster(4, 8);
        std::vector<WorkloadType> t4 = {{0, 2048.0, 28.0}, {1, 1024.0, 230.0}, {2, 4000.0, 60.0}, {3, 600.0, 900.0}};
        std::vector<std::vector<int64_t>> lams = {{1600, 1200, 800, 400}, {900, 1500, 700, 800},
                                                  {400, 700, 1900, 300}, {1800, 300, 500, 1200}};
        auto t0 = std::chrono::steady_clock::now();
        auto ref = adaptive_windows<false>(c32, m, t4, lams, 40);
        const double t_ref = secs(t0);
        t0 = std::chrono::steady_clock::now();
        auto gpu = adaptive_windows<true>(c32, m, t4, lams, 40);
        const double t_gpu_cold = secs(t0);  // includes context creation + first kernel loads
        t0 = std::chrono::steady_clock::now();
        gpu = adaptive_windows<true>(c32, m, t4, lams, 40);
        const double t_gpu = secs(t0);  // cached contexts (a long-running scheduler's steady state)
        for (size_t w = 0; w < lams.size(); ++w) {
            EXPECT(ref[w].chosen == gpu[w].chosen && ref[w].found == gpu[w].found, "orchestrate window: chosen");
            EXPECT(ref[w].x == gpu[w].x, "orchestrate window: assignment_for");
            EXPECT(ref[w].plan.transfers == gpu[w].plan.transfers && ref[w].plan.est_seconds == gpu[w].plan.est_seconds,
                   "orchestrate window: switch plan");
        }
        std::printf("orchestrate windows (4 x search(max_iters=40) + keep + assignment + switch, D=32, J=4): "
                    "reference %.3f s, GPU through the shim %.3f s (first call, cold contexts %.3f s)\n",
                    t_ref, t_gpu, t_gpu_cold);
        // search() alone on the config-2 shape, warm: the reference vs the shim
        TraceSpan span{0, lams[0]};
        search::SearchOptions so;
        so.seed = 3;
        t0 = std::chrono::steady_clock::now();
        auto sa = search::search(c32, m, t4, span, 60.0, cost::ProfileParams{}, so);
        const double ts_ref = secs(t0);
        oserve_gpu::search::search(c32, m, t4, span, 60.0, cost::ProfileParams{}, so);
        t0 = std::chrono::steady_clock::now();
        auto sb = oserve_gpu::search::search(c32, m, t4, span, 60.0, cost::ProfileParams{}, so);
        const double ts_gpu = secs(t0);
        EXPECT(sa.throughput == sb.throughput && sa.deployment == sb.deployment && sa.iterations == sb.iterations,
               "search::search (D=32)");
        std::printf("search::search D=32 J=4 seed 3 (%d iterations): reference %.4f s, GPU through the shim %.4f s\n",
                    sa.iterations, ts_ref, ts_gpu);
    }
    // search::search one for one (the SPEC's schedule path), log rows included
    for (auto lam : {std::vector<int64_t>{700, 300}, std::vector<int64_t>{5000, 40}}) {
        TraceSpan span{0, lam};
        for (std::uint64_t seed : {0ull, 3ull}) {
            std::vector<search::SearchLogRow> l1, l2;
            search::SearchOptions so;
            so.seed = seed;
            so.log = [&](const search::SearchLogRow &r) { l1.push_back(r); };
            auto a = search::search(c8, m, types, span, 60.0, params, so);
            so.log = [&](const search::SearchLogRow &r) { l2.push_back(r); };
            auto b = oserve_gpu::search::search(c8, m, types, span, 60.0, params, so);
            bool logs = l1.size() == l2.size();
            for (size_t i = 0; logs && i < l1.size(); ++i)
                logs = l1[i].iteration == l2[i].iteration && l1[i].op == l2[i].op &&
                       l1[i].accepted == l2[i].accepted && l1[i].throughput == l2[i].throughput &&
                       l1[i].devices == l2[i].devices;
            EXPECT(a.throughput == b.throughput && a.deployment == b.deployment && a.iterations == b.iterations &&
                       a.stale_iters == b.stale_iters && a.rng_seed == b.rng_seed && logs,
                   "search::search");
        }
    }
    std::printf(failures ? "DROPIN FAILED (%d)\n" : "DROPIN OK\n", failures);
    return failures ? 1 : 0;
}
