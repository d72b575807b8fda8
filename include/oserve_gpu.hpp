// oserve_gpu.hpp — header-only C++ shim: the reference's own scheduler API
// (namespace oserve::, /root/reference/proj/include/oserve/*.hpp) on top of
// the C-ABI in oserve_gpu.h.
//
// A maintainer of the reference includes this header next to the oserve
// headers and swaps the call sites listed in INTEGRATION.md:
//
//   oserve::search::search(...)            -> oserve_gpu::search::search(...)
//   oserve::search::exhaustive(...)        -> oserve_gpu::search::exhaustive(...)
//   oserve::search::best_strategies(...)   -> oserve_gpu::search::best_strategies(...)
//   oserve::search::evaluate_deployment    -> oserve_gpu::search::evaluate_deployment
//   oserve::cost::build_capacity_table     -> oserve_gpu::cost::build_capacity_table
//   oserve::flow::solve_assignment         -> oserve_gpu::flow::solve_assignment
//   oserve::flow::normalize / normalize_or_scale / check_constraints / max_flow /
//     extract_assignment / solve_fractional -> oserve_gpu::flow::...
//   oserve::switchplan::layout / greedy_plan / estimate_time / kv_plan
//                                          -> oserve_gpu::switchplan::...
//
// Same argument meaning, same return types, same exceptions (status codes are
// rethrown as the errors.hpp types).  Requires the reference headers on the
// include path (this header converts their value types).
//
// GPU contexts are cached per host thread, keyed by (cluster, model, profile)
// and the device set: repeated calls — e.g. the up to 500 best_strategies of
// one search() — reuse the device tables; a workload change re-runs only the
// cost kernel (K0).  oserve_gpu::set_devices({0, 1, ...}) makes the cached
// contexts span several GPUs (oserve_gpu_create_multi: sharded rounds, NCCL).
#pragma once

#include <algorithm>
#include <cstring>
#include <functional>
#include <list>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "oserve/core.hpp"
#include "oserve/costmodel.hpp"
#include "oserve/deploysearch.hpp"
#include "oserve/errors.hpp"
#include "oserve/flowassign.hpp"
#include "oserve/switchplan.hpp"
#include "oserve_gpu.h"

namespace oserve_gpu {

// Rethrow a C-ABI status as the reference's exception type.
inline void check(int status, const oserve_gpu_ctx *ctx) {
    if (status == OSERVE_OK) return;
    const std::string msg = ctx ? oserve_gpu_last_error(ctx) : oserve_gpu_status_name(status);
    switch (status) {
        case OSERVE_ERR_INFEASIBLE_REPLICA: throw oserve::InfeasibleReplica(msg);
        case OSERVE_ERR_MODEL_TOO_LARGE: throw oserve::ModelTooLarge(msg);
        case OSERVE_ERR_TOO_LARGE: throw oserve::TooLarge(msg);
        case OSERVE_ERR_EMPTY_DEPLOYMENT: throw oserve::EmptyDeployment(msg);
        case OSERVE_ERR_UNSOURCED_FRAGMENT: throw oserve::UnsourcedFragment(msg);
        case OSERVE_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case OSERVE_ERR_LOGIC: throw std::logic_error(msg);
        case OSERVE_ERR_LCM_OVERFLOW: throw oserve::LcmOverflow(msg);
        default: throw oserve::Error(std::string(oserve_gpu_status_name(status)) + ": " + msg);
    }
}

// Flattened copies of reference value types (kept alive for one call).
struct ClusterBuf {
    std::vector<int> ndev, ids;
    std::vector<uint64_t> mem;
    oserve_cluster_desc desc{};
    explicit ClusterBuf(const oserve::ClusterSpec &c) {
        for (const auto &m : c.machines) {
            ndev.push_back(static_cast<int>(m.device_ids.size()));
            ids.insert(ids.end(), m.device_ids.begin(), m.device_ids.end());
            mem.push_back(m.device_mem);
        }
        desc = {static_cast<int>(c.machines.size()), ndev.data(), ids.data(), mem.data(), c.intra_bw, c.inter_bw};
    }
};

struct DeploymentBuf {
    std::vector<int> ndev, ids, tp, pp;
    oserve_deployment desc{};
    explicit DeploymentBuf(const oserve::Deployment &d) {
        for (const auto &r : d.replicas) {
            ndev.push_back(r.device_count());
            ids.insert(ids.end(), r.device_ids.begin(), r.device_ids.end());
            tp.push_back(r.tp);
            pp.push_back(r.pp);
        }
        desc = {d.replica_count(), ndev.data(), ids.data(), tp.data(), pp.data()};
    }
};

inline oserve_model_desc model_desc(const oserve::ModelSpec &m) {
    return {m.param_bytes, m.num_layers, m.bytes_per_token_kv, m.flops_per_token_prefill, m.min_mem_bytes};
}
inline oserve_profile profile_desc(const oserve::cost::ProfileParams &p) {
    return {p.prefill_coeff, p.decode_coeff, p.tp_efficiency, p.pp_comm_cost, p.mem_bw_penalty};
}

inline oserve::Deployment to_deployment(const oserve_plan &p) {
    oserve::Deployment d;
    int pos = 0;
    for (int r = 0; r < p.num_replicas; ++r) {
        oserve::ReplicaConfig rc;
        rc.device_ids.assign(p.device_ids + pos, p.device_ids + pos + p.replica_num_devices[r]);
        pos += p.replica_num_devices[r];
        rc.tp = p.tp[r];
        rc.pp = p.pp[r];
        d.replicas.push_back(rc);
    }
    return d;
}

// RAII context bound to one (cluster, model, profile, workload).
class Context {
  public:
    Context(const oserve::ClusterSpec &cluster, const oserve::ModelSpec &model,
            const oserve::cost::ProfileParams &params, int device = 0) {
        ClusterBuf cb(cluster);
        oserve_model_desc md = model_desc(model);
        oserve_profile pd = profile_desc(params);
        oserve_gpu_ctx *raw = nullptr;
        check(oserve_gpu_create(device, &cb.desc, &md, &pd, &raw), nullptr);
        ctx_.reset(raw);
    }
    // One context over several GPUs of this process (sharded rounds, NCCL).
    Context(const oserve::ClusterSpec &cluster, const oserve::ModelSpec &model,
            const oserve::cost::ProfileParams &params, const std::vector<int> &devices) {
        ClusterBuf cb(cluster);
        oserve_model_desc md = model_desc(model);
        oserve_profile pd = profile_desc(params);
        oserve_gpu_ctx *raw = nullptr;
        if (devices.size() > 1)
            check(oserve_gpu_create_multi(devices.data(), static_cast<int>(devices.size()), &cb.desc, &md, &pd, &raw),
                  nullptr);
        else
            check(oserve_gpu_create(devices.empty() ? 0 : devices[0], &cb.desc, &md, &pd, &raw), nullptr);
        ctx_.reset(raw);
    }
    void set_workload(const std::vector<oserve::WorkloadType> &types, const std::vector<int64_t> &lambda,
                      double span_s) {
        std::vector<oserve_class> cls;
        for (const auto &t : types) cls.push_back({t.type_id, t.centroid_in, t.centroid_out});
        check(oserve_gpu_set_workload(get(), static_cast<int>(cls.size()), cls.data(), lambda.data(), span_s), get());
    }
    oserve_gpu_ctx *get() const { return ctx_.get(); }

  private:
    struct Del {
        void operator()(oserve_gpu_ctx *c) const { oserve_gpu_destroy(c); }
    };
    std::unique_ptr<oserve_gpu_ctx, Del> ctx_;
};

// ---- per-thread context cache -------------------------------------------
// Devices the cached contexts span (default: CUDA device 0).
inline std::vector<int> &device_set() {
    static std::vector<int> d{0};
    return d;
}
inline std::mutex &device_set_mutex() {
    static std::mutex m;
    return m;
}
inline void set_devices(const std::vector<int> &devices) {
    std::lock_guard<std::mutex> lk(device_set_mutex());
    device_set() = devices.empty() ? std::vector<int>{0} : devices;
}
inline std::vector<int> devices() {
    std::lock_guard<std::mutex> lk(device_set_mutex());
    return device_set();
}

namespace detail {
template <class T>
void put(std::string &k, const T &v) {
    k.append(reinterpret_cast<const char *>(&v), sizeof(v));
}
inline std::string context_key(const oserve::ClusterSpec &c, const oserve::ModelSpec &m,
                               const oserve::cost::ProfileParams &p, const std::vector<int> &devs) {
    std::string k;
    put(k, c.intra_bw);
    put(k, c.inter_bw);
    for (const auto &mc : c.machines) {
        put(k, mc.device_mem);
        put(k, mc.device_ids.size());
        for (int d : mc.device_ids) put(k, d);
    }
    k += '|';
    put(k, m.param_bytes);
    put(k, m.num_layers);
    put(k, m.bytes_per_token_kv);
    put(k, m.flops_per_token_prefill);
    put(k, m.min_mem_bytes);
    put(k, p.prefill_coeff);
    put(k, p.decode_coeff);
    put(k, p.tp_efficiency);
    put(k, p.pp_comm_cost);
    put(k, p.mem_bw_penalty);
    for (int d : devs) put(k, d);
    return k;
}
struct CacheEntry {
    std::string key;
    std::unique_ptr<Context> ctx;
    bool has_workload = false;
    std::vector<oserve::WorkloadType> types;
    std::vector<int64_t> lambda;
    double span = 0.0;
};
}  // namespace detail

// The cached context for (cluster, model, params) on the current device set,
// with `types`/`lambda`/`span_s` as its workload (set only when it changed).
inline Context &cached_context(const oserve::ClusterSpec &cluster, const oserve::ModelSpec &model,
                               const oserve::cost::ProfileParams &params) {
    thread_local std::list<detail::CacheEntry> cache;  // most recent first
    const std::vector<int> devs = devices();
    const std::string key = detail::context_key(cluster, model, params, devs);
    for (auto it = cache.begin(); it != cache.end(); ++it)
        if (it->key == key) {
            cache.splice(cache.begin(), cache, it);
            return *cache.front().ctx;
        }
    detail::CacheEntry e;
    e.key = key;
    e.ctx = std::make_unique<Context>(cluster, model, params, devs);
    cache.push_front(std::move(e));
    constexpr size_t kMaxEntries = 8;
    while (cache.size() > kMaxEntries) cache.pop_back();
    return *cache.front().ctx;
}

inline Context &cached_context(const oserve::ClusterSpec &cluster, const oserve::ModelSpec &model,
                               const oserve::cost::ProfileParams &params,
                               const std::vector<oserve::WorkloadType> &types, const std::vector<int64_t> &lambda,
                               double span_s) {
    Context &c = cached_context(cluster, model, params);
    // workload memo lives next to the context (keyed by its handle)
    thread_local std::vector<std::pair<const oserve_gpu_ctx *, detail::CacheEntry>> memo;
    detail::CacheEntry *w = nullptr;
    for (auto &m : memo)
        if (m.first == c.get()) w = &m.second;
    if (!w) {
        if (memo.size() > 16) memo.erase(memo.begin());
        memo.emplace_back(c.get(), detail::CacheEntry{});
        w = &memo.back().second;
    }
    auto same_types = [&] {
        if (w->types.size() != types.size()) return false;
        for (size_t j = 0; j < types.size(); ++j)
            if (w->types[j].type_id != types[j].type_id || w->types[j].centroid_in != types[j].centroid_in ||
                w->types[j].centroid_out != types[j].centroid_out)
                return false;
        return true;
    };
    if (!w->has_workload || !same_types() || w->lambda != lambda || w->span != span_s) {
        c.set_workload(types, lambda, span_s);
        w->has_workload = true;
        w->types = types;
        w->lambda = lambda;
        w->span = span_s;
    }
    return c;
}

namespace detail {
// A one-device context for calls that need no cluster (raw-table solves,
// flow networks, normalisation), cached per thread.
inline Context &scratch() {
    oserve::ClusterSpec cl;
    cl.machines.push_back({"m0", {0}, 1});
    cl.intra_bw = cl.inter_bw = 1.0;
    return cached_context(cl, oserve::ModelSpec{}, oserve::cost::ProfileParams{});
}
}  // namespace detail

inline Context &make_context(const oserve::search::EvalContext &ctx) {
    return cached_context(ctx.cluster, ctx.model, ctx.params, ctx.types, ctx.span.counts, ctx.span_seconds);
}

namespace search {

// oserve::search::evaluate_deployment (deploysearch.cpp:138-151).
inline std::int64_t evaluate_deployment(const oserve::Deployment &dep, const oserve::search::EvalContext &ctx) {
    if (dep.replicas.empty()) return 0;
    Context &c = make_context(ctx);
    DeploymentBuf db(dep);
    int64_t obj = 0;
    check(oserve_gpu_evaluate_deployments(c.get(), 1, &db.desc, &obj), c.get());
    return obj;
}

// oserve::search::best_strategies (deploysearch.cpp:153-229).
inline oserve::search::StrategyChoice best_strategies(const std::vector<int> &sizes,
                                                      const oserve::search::EvalContext &ctx) {
    Context &c = make_context(ctx);
    auto res = std::make_unique<oserve_round_result>();
    check(oserve_gpu_best_strategies(c.get(), static_cast<int>(sizes.size()), sizes.data(), res.get()), c.get());
    oserve::search::StrategyChoice out;
    out.deployment = to_deployment(res->plan);
    out.objective = res->objective;
    return out;
}

// oserve::search::exhaustive (deploysearch.cpp:436-466).  `parallel` is
// accepted for signature compatibility (the GPU path is always parallel).
inline oserve::search::SearchState exhaustive(const oserve::ClusterSpec &cluster, const oserve::ModelSpec &model,
                                              const std::vector<oserve::WorkloadType> &types,
                                              const oserve::TraceSpan &span, double span_seconds,
                                              const oserve::cost::ProfileParams &params, bool /*parallel*/ = true) {
    Context &c = cached_context(cluster, model, params, types, span.counts, span_seconds);
    auto res = std::make_unique<oserve_round_result>();
    check(oserve_gpu_exhaustive(c.get(), res.get()), c.get());
    oserve::search::SearchState s;
    s.deployment = to_deployment(res->plan);
    s.throughput = res->objective;
    s.iterations = static_cast<int>(res->partitions);
    return s;
}

// oserve::search::search (deploysearch.cpp:341-417): the reference's
// mutate / enumerate / revert loop with the identical mt19937_64 stream;
// every best_strategies and capacity-table + assignment step on the GPU.
// `opts.parallel` is accepted for signature compatibility.
inline oserve::search::SearchState search(const oserve::ClusterSpec &cluster, const oserve::ModelSpec &model,
                                          const std::vector<oserve::WorkloadType> &types,
                                          const oserve::TraceSpan &span, double span_seconds,
                                          const oserve::cost::ProfileParams &params,
                                          const oserve::search::SearchOptions &opts = {}) {
    Context &c = cached_context(cluster, model, params, types, span.counts, span_seconds);
    std::unique_ptr<DeploymentBuf> warm;
    if (opts.warm_start) warm = std::make_unique<DeploymentBuf>(*opts.warm_start);
    oserve_search_options so{opts.seed, opts.max_iters, opts.stale_limit, opts.mutation_retries,
                             warm ? &warm->desc : nullptr};
    const int cap = opts.log ? opts.max_iters + 1 : 0;
    std::vector<oserve_search_log_row> rows(static_cast<size_t>(cap > 0 ? cap : 1));
    auto res = std::make_unique<oserve_search_result>();
    check(oserve_gpu_search(c.get(), &so, res.get(), opts.log ? rows.data() : nullptr, cap), c.get());
    if (opts.log)
        for (int i = 0; i < std::min(res->log_count, cap); ++i)
            opts.log(oserve::search::SearchLogRow{rows[i].iteration, rows[i].op, rows[i].accepted != 0,
                                                  rows[i].throughput, rows[i].devices});
    oserve::search::SearchState s;
    s.deployment = to_deployment(res->deployment);
    s.throughput = res->throughput;
    s.rng_seed = res->rng_seed;
    s.stale_iters = res->stale_iters;
    s.iterations = res->iterations;
    return s;
}

}  // namespace search

namespace cost {

// oserve::cost::build_capacity_table (costmodel.cpp:94-116).
inline oserve::cost::CapacityTable build_capacity_table(const oserve::Deployment &dep,
                                                        const std::vector<oserve::WorkloadType> &types,
                                                        const oserve::ModelSpec &model,
                                                        const oserve::ClusterSpec &cluster,
                                                        const oserve::cost::ProfileParams &params, double span_s) {
    Context &c = cached_context(cluster, model, params, types, std::vector<int64_t>(types.size(), 0), span_s);
    DeploymentBuf db(dep);
    const int R = dep.replica_count(), J = static_cast<int>(types.size());
    std::vector<int64_t> n(R * J), e(R * J);
    std::vector<double> lat(R * J);
    check(oserve_gpu_plan_detail(c.get(), &db.desc, n.data(), e.data(), lat.data(), nullptr, nullptr, nullptr,
                                 nullptr, nullptr),
          c.get());
    oserve::cost::CapacityTable t;
    for (int k = 0; k < R; ++k) {
        t.n.emplace_back(n.begin() + k * J, n.begin() + (k + 1) * J);
        t.e.emplace_back(e.begin() + k * J, e.begin() + (k + 1) * J);
        t.latency.emplace_back(lat.begin() + k * J, lat.begin() + (k + 1) * J);
    }
    return t;
}

}  // namespace cost

namespace flow {

// oserve::flow::solve_assignment (flowassign.cpp:481-503) on one table.
inline oserve::flow::LowerLevel solve_assignment(const oserve::cost::CapacityTable &table,
                                                 const std::vector<int64_t> &lambda,
                                                 const oserve::flow::SolveOptions &opts = {},
                                                 oserve_gpu_ctx *ctx = nullptr) {
    const int R = table.replicas(), J = table.types();
    if (static_cast<int>(lambda.size()) != J) throw std::invalid_argument("solve_assignment: lambda size mismatch");
    if (!ctx) ctx = detail::scratch().get();
    oserve_solve_options so{opts.exact_demand_limit, opts.exact_cell_limit, opts.node_budget};
    check(oserve_gpu_set_solve_options(ctx, &so), ctx);
    std::vector<int64_t> n, e, x(R * J), unit(R * J), M(R), used(R);
    for (int k = 0; k < R; ++k) {
        n.insert(n.end(), table.n[k].begin(), table.n[k].end());
        e.insert(e.end(), table.e[k].begin(), table.e[k].end());
    }
    int64_t obj = 0;
    check(oserve_gpu_solve_batch(ctx, 1, R, J, n.data(), e.data(), lambda.data(), x.data(), &obj, M.data(),
                                 unit.data(), used.data()),
          ctx);
    oserve::flow::LowerLevel out;
    out.assignment.objective = obj;
    for (int k = 0; k < R; ++k) {
        out.assignment.x.emplace_back(x.begin() + k * J, x.begin() + (k + 1) * J);
        out.unit.emplace_back(unit.begin() + k * J, unit.begin() + (k + 1) * J);
    }
    out.M = M;
    out.used = used;
    return out;
}

// oserve::flow::normalize (flowassign.cpp:31-46): throws LcmOverflow past 2^62.
inline oserve::flow::NormalizedRow normalize(const std::vector<int64_t> &n_row) {
    oserve::flow::NormalizedRow out;
    out.units.assign(n_row.size(), 0);
    if (n_row.empty()) return out;
    oserve_gpu_ctx *c = detail::scratch().get();
    int sc = 0;
    check(oserve_gpu_normalize_batch(c, 1, static_cast<int>(n_row.size()), n_row.data(), 1, &out.M, out.units.data(),
                                     &sc),
          c);
    out.scaled = sc != 0;
    return out;
}

// oserve::flow::normalize_or_scale (flowassign.cpp:48-62).
inline oserve::flow::NormalizedRow normalize_or_scale(const std::vector<int64_t> &n_row) {
    oserve::flow::NormalizedRow out;
    out.units.assign(n_row.size(), 0);
    if (n_row.empty()) return out;
    oserve_gpu_ctx *c = detail::scratch().get();
    int sc = 0;
    check(oserve_gpu_normalize_batch(c, 1, static_cast<int>(n_row.size()), n_row.data(), 0, &out.M, out.units.data(),
                                     &sc),
          c);
    out.scaled = sc != 0;
    return out;
}

// oserve::flow::check_constraints (flowassign.cpp:529-551): std::logic_error
// naming the first violated constraint.
inline void check_constraints(const oserve::flow::AssignmentMatrix &a, const oserve::cost::CapacityTable &table,
                              const std::vector<int64_t> &lambda) {
    const int R = table.replicas(), J = table.types();
    if (R == 0 || J == 0) return;
    std::vector<int64_t> x, n, e;
    for (int k = 0; k < R; ++k) {
        x.insert(x.end(), a.x[k].begin(), a.x[k].end());
        n.insert(n.end(), table.n[k].begin(), table.n[k].end());
        e.insert(e.end(), table.e[k].begin(), table.e[k].end());
    }
    oserve_gpu_ctx *c = detail::scratch().get();
    check(oserve_gpu_check_constraints_batch(c, 1, R, J, x.data(), n.data(), e.data(), lambda.data(), nullptr, nullptr,
                                             nullptr),
          c);
}

// oserve::flow::max_flow (flowassign.cpp:67-147) on the device (K6a).
inline oserve::flow::FlowResult max_flow(const oserve::flow::Graph &g, int source, int sink) {
    Context *c = &detail::scratch();
    std::vector<oserve_flow_edge> ed;
    for (const auto &e : g.edges) ed.push_back({e.from, e.to, e.cap});
    const int64_t off[2] = {0, static_cast<int64_t>(ed.size())};
    oserve::flow::FlowResult out;
    out.flow.resize(ed.size());
    check(oserve_gpu_max_flow_batch(c->get(), 1, &g.num_nodes, off, ed.data(), &source, &sink, out.flow.data(),
                                    &out.value),
          c->get());
    return out;
}

// oserve::flow::extract_assignment (flowassign.cpp:505-519) on the device (K6b).
inline oserve::flow::AssignmentMatrix extract_assignment(const oserve::flow::FlowNetwork &net,
                                                         const oserve::flow::FlowResult &flow,
                                                         const oserve::flow::SolveOptions &opts = {}) {
    Context *c = &detail::scratch();
    oserve_solve_options so{opts.exact_demand_limit, opts.exact_cell_limit, opts.node_budget};
    check(oserve_gpu_set_solve_options(c->get(), &so), c->get());
    std::vector<int64_t> n, e, x(static_cast<size_t>(net.R) * net.J);
    for (int k = 0; k < net.R; ++k) {
        n.insert(n.end(), net.n[k].begin(), net.n[k].end());
        e.insert(e.end(), net.e[k].begin(), net.e[k].end());
    }
    int64_t obj = 0;
    check(oserve_gpu_extract_assignment_batch(c->get(), 1, net.R, net.J, n.data(), e.data(), net.lambda.data(),
                                              flow.flow.data(), x.data(), &obj),
          c->get());
    oserve::flow::AssignmentMatrix out;
    out.objective = obj;
    for (int k = 0; k < net.R; ++k) out.x.emplace_back(x.begin() + k * net.J, x.begin() + (k + 1) * net.J);
    return out;
}

// oserve::flow::solve_fractional (flowassign.cpp:559-645) on the device (K7).
inline oserve::flow::FractionalSolution solve_fractional(const oserve::cost::CapacityTable &table,
                                                         const std::vector<int64_t> &lambda) {
    Context *c = &detail::scratch();
    const int R = table.replicas(), J = table.types();
    std::vector<int64_t> n, e;
    for (int k = 0; k < R; ++k) {
        n.insert(n.end(), table.n[k].begin(), table.n[k].end());
        e.insert(e.end(), table.e[k].begin(), table.e[k].end());
    }
    std::vector<double> f(static_cast<size_t>(R) * J);
    oserve::flow::FractionalSolution out;
    check(oserve_gpu_solve_fractional_batch(c->get(), 1, R, J, n.data(), e.data(), lambda.data(), f.data(),
                                            &out.objective),
          c->get());
    for (int k = 0; k < R; ++k) out.f.emplace_back(f.begin() + k * J, f.begin() + (k + 1) * J);
    return out;
}

}  // namespace flow

namespace switchplan {

// oserve::switchplan::layout (switchplan.cpp:40-63): shards on the device,
// `held` coalesced per device (sorted disjoint ranges) as the reference does.
inline oserve::switchplan::ShardLayout layout(const oserve::Deployment &dep, const oserve::ModelSpec &model) {
    oserve_gpu_ctx *c = detail::scratch().get();
    DeploymentBuf db(dep);
    int n = 0;
    check(oserve_gpu_layout(c, &db.desc, model.param_bytes, 0, nullptr, &n), c);
    std::vector<oserve_shard> sh(static_cast<size_t>(n));
    if (n) check(oserve_gpu_layout(c, &db.desc, model.param_bytes, n, sh.data(), &n), c);
    oserve::switchplan::ShardLayout out;
    for (const auto &s : sh) {
        out.shards.push_back({s.shard_id, {s.begin, s.end}, s.holder});
        out.held[s.holder].push_back({s.begin, s.end});
    }
    for (auto &[dev, ranges] : out.held) {  // coalesce (switchplan.cpp:17-29)
        std::sort(ranges.begin(), ranges.end());
        std::vector<oserve::switchplan::ByteRange> m;
        for (const auto &r : ranges) {
            if (r.begin == r.end) continue;
            if (!m.empty() && r.begin <= m.back().end) m.back().end = std::max(m.back().end, r.end);
            else m.push_back(r);
        }
        ranges = std::move(m);
    }
    return out;
}

// oserve::switchplan::greedy_plan(const ShardLayout&, const ShardLayout&,
// const ClusterSpec&) (switchplan.cpp:65-131) on the device.
inline oserve::switchplan::SwitchPlan greedy_plan(const oserve::switchplan::ShardLayout &src,
                                                  const oserve::switchplan::ShardLayout &dst,
                                                  const oserve::ClusterSpec &cluster) {
    auto held = [](const oserve::switchplan::ShardLayout &l) {
        std::vector<oserve_held_range> v;
        for (const auto &[dev, ranges] : l.held)
            for (const auto &r : ranges) v.push_back({dev, r.begin, r.end});
        return v;
    };
    const std::vector<oserve_held_range> a = held(src), b = held(dst);
    Context &c = cached_context(cluster, oserve::ModelSpec{}, oserve::cost::ProfileParams{});
    int n = 0;
    double est = 0.0;
    check(oserve_gpu_greedy_plan_layouts(c.get(), static_cast<int>(a.size()), a.data(), static_cast<int>(b.size()),
                                         b.data(), 0, nullptr, &n, &est),
          c.get());
    std::vector<oserve_transfer> tr(static_cast<size_t>(n));
    if (n)
        check(oserve_gpu_greedy_plan_layouts(c.get(), static_cast<int>(a.size()), a.data(),
                                             static_cast<int>(b.size()), b.data(), n, tr.data(), &n, &est),
              c.get());
    oserve::switchplan::SwitchPlan plan;
    for (const auto &t : tr) {
        plan.transfers.push_back({{t.begin, t.end}, t.src, t.dst});
        plan.link_load[{t.src, t.dst}] += t.end - t.begin;
    }
    plan.est_seconds = est;
    return plan;
}

// oserve::switchplan::estimate_time (switchplan.cpp:133-140) on the device.
inline double estimate_time(const oserve::switchplan::SwitchPlan &plan, const oserve::ClusterSpec &cluster) {
    std::vector<oserve_link_load> links;
    for (const auto &[link, bytes] : plan.link_load) links.push_back({link.first, link.second, bytes});
    Context &c = cached_context(cluster, oserve::ModelSpec{}, oserve::cost::ProfileParams{});
    double est = 0.0;
    check(oserve_gpu_estimate_time(c.get(), static_cast<int>(links.size()), links.data(), &est), c.get());
    return est;
}

// layout + greedy_plan + estimate_time (switchplan.cpp:40-140) for one pair
// of deployments, fused in one kernel (K2).
inline oserve::switchplan::SwitchPlan greedy_plan(const oserve::Deployment &from, const oserve::Deployment &to,
                                                  const oserve::ModelSpec &model,
                                                  const oserve::ClusterSpec &cluster) {
    Context &c = cached_context(cluster, model, oserve::cost::ProfileParams{});
    DeploymentBuf a(from), b(to);
    int n = 0;
    double est = 0.0;
    check(oserve_gpu_switch_plan(c.get(), &a.desc, &b.desc, 0, nullptr, &n, &est), c.get());
    std::vector<oserve_transfer> tr(n);
    check(oserve_gpu_switch_plan(c.get(), &a.desc, &b.desc, n, tr.data(), &n, &est), c.get());
    oserve::switchplan::SwitchPlan plan;
    for (const auto &t : tr) {
        plan.transfers.push_back({{t.begin, t.end}, t.src, t.dst});
        plan.link_load[{t.src, t.dst}] += t.end - t.begin;
    }
    plan.est_seconds = est;
    return plan;
}

// kv_plan (switchplan.cpp:142-207) on the device; `carry` may be null.
inline oserve::switchplan::KvPlan kv_plan(const std::vector<oserve::switchplan::InflightRequest> &inflight,
                                          std::int64_t threshold_tokens, const oserve::Deployment &src,
                                          const oserve::Deployment &dst, const oserve::ClusterSpec &cluster,
                                          double headroom, const oserve::switchplan::SwitchPlan *carry = nullptr) {
    oserve::ModelSpec model;
    model.param_bytes = 1;  // the migration plan does not depend on the model
    model.num_layers = 1;
    model.min_mem_bytes = 1;
    Context &c = cached_context(cluster, model, oserve::cost::ProfileParams{});
    DeploymentBuf a(src), b(dst);
    std::vector<oserve_inflight> req;
    for (const auto &r : inflight) req.push_back({r.request_id, r.generated_tokens, r.kv_bytes, r.source_replica});
    std::vector<oserve_transfer> tr;
    if (carry != nullptr)
        for (const auto &t : carry->transfers) tr.push_back({t.range.begin, t.range.end, t.src, t.dst});
    std::vector<int64_t> drained(inflight.size() + 1);
    std::vector<oserve_kv_transfer> mig(inflight.size() + 1);
    int nd = 0, nm = 0;
    uint64_t buf = 0;
    check(oserve_gpu_kv_plan(c.get(), static_cast<int>(req.size()), req.data(), threshold_tokens, &a.desc, &b.desc,
                             headroom, static_cast<int>(tr.size()), tr.data(), drained.data(), &nd, mig.data(), &nm,
                             &buf),
          c.get());
    oserve::switchplan::KvPlan out;
    out.drained.assign(drained.begin(), drained.begin() + nd);
    for (int i = 0; i < nm; ++i) out.migrated.push_back({mig[i].request_id, mig[i].kv_bytes, mig[i].src, mig[i].dst});
    out.buffer_bytes = buf;
    return out;
}

}  // namespace switchplan

}  // namespace oserve_gpu
