// oserve_gpu.hpp — header-only C++ shim: the reference's own scheduler API
// (namespace oserve::, /root/reference/proj/include/oserve/*.hpp) on top of
// the C-ABI in oserve_gpu.h.
//
// A maintainer of the reference includes this header next to the oserve
// headers and swaps the call sites listed in INTEGRATION.md:
//
//   oserve::search::exhaustive(...)        -> oserve_gpu::search::exhaustive(...)
//   oserve::search::best_strategies(...)   -> oserve_gpu::search::best_strategies(...)
//   oserve::search::evaluate_deployment    -> oserve_gpu::search::evaluate_deployment
//   oserve::cost::build_capacity_table     -> oserve_gpu::cost::build_capacity_table
//   oserve::flow::solve_assignment         -> oserve_gpu::flow::solve_assignment
//   layout + greedy_plan + estimate_time   -> oserve_gpu::switchplan::greedy_plan
//
// Same argument meaning, same return types, same exceptions (status codes are
// rethrown as the errors.hpp types).  Requires the reference headers on the
// include path (this header converts their value types).
#pragma once

#include <memory>
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

inline Context make_context(const oserve::search::EvalContext &ctx) {
    Context c(ctx.cluster, ctx.model, ctx.params);
    c.set_workload(ctx.types, ctx.span.counts, ctx.span_seconds);
    return c;
}

namespace search {

// oserve::search::evaluate_deployment (deploysearch.cpp:138-151).
inline std::int64_t evaluate_deployment(const oserve::Deployment &dep, const oserve::search::EvalContext &ctx) {
    if (dep.replicas.empty()) return 0;
    Context c = make_context(ctx);
    DeploymentBuf db(dep);
    int64_t obj = 0;
    check(oserve_gpu_evaluate_deployments(c.get(), 1, &db.desc, &obj), c.get());
    return obj;
}

// oserve::search::best_strategies (deploysearch.cpp:153-229).
inline oserve::search::StrategyChoice best_strategies(const std::vector<int> &sizes,
                                                      const oserve::search::EvalContext &ctx) {
    Context c = make_context(ctx);
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
    Context c(cluster, model, params);
    c.set_workload(types, span.counts, span_seconds);
    auto res = std::make_unique<oserve_round_result>();
    check(oserve_gpu_exhaustive(c.get(), res.get()), c.get());
    oserve::search::SearchState s;
    s.deployment = to_deployment(res->plan);
    s.throughput = res->objective;
    s.iterations = static_cast<int>(res->partitions);
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
    Context c(cluster, model, params);
    c.set_workload(types, std::vector<int64_t>(types.size(), 0), span_s);
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
    std::unique_ptr<Context> own;
    if (!ctx) {
        oserve::ClusterSpec cl;
        cl.machines.push_back({"m0", {0}, 1});
        cl.intra_bw = cl.inter_bw = 1.0;
        own = std::make_unique<Context>(cl, oserve::ModelSpec{}, oserve::cost::ProfileParams{});
        ctx = own->get();
    }
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

namespace detail {
inline std::unique_ptr<Context> scratch_context() {
    oserve::ClusterSpec cl;
    cl.machines.push_back({"m0", {0}, 1});
    cl.intra_bw = cl.inter_bw = 1.0;
    return std::make_unique<Context>(cl, oserve::ModelSpec{}, oserve::cost::ProfileParams{});
}
}  // namespace detail

// oserve::flow::max_flow (flowassign.cpp:67-147) on the device (K6a).
inline oserve::flow::FlowResult max_flow(const oserve::flow::Graph &g, int source, int sink) {
    auto c = detail::scratch_context();
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
    auto c = detail::scratch_context();
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
    auto c = detail::scratch_context();
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

// layout + greedy_plan + estimate_time (switchplan.cpp:40-140) for one pair.
inline oserve::switchplan::SwitchPlan greedy_plan(const oserve::Deployment &from, const oserve::Deployment &to,
                                                  const oserve::ModelSpec &model,
                                                  const oserve::ClusterSpec &cluster) {
    Context c(cluster, model, oserve::cost::ProfileParams{});
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
    Context c(cluster, model, oserve::cost::ProfileParams{});
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
