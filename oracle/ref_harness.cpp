// ref_harness.cpp — TEST INFRASTRUCTURE ONLY.
//
// C-ABI (oracle_api.h) over the UNMODIFIED reference library compiled from
// /root/reference/proj/src (see oracle/Makefile).  Every entry point calls the
// reference's public API:
//   cost::build_capacity_table      costmodel.cpp:94-116
//   flow::normalize(_or_scale)       flowassign.cpp:31-62
//   flow::solve_assignment           flowassign.cpp:481-503
//   flow::check_constraints          flowassign.cpp:521-554
//   search::min_feasible_group       deploysearch.cpp:77-87
//   search::canonical_blocks         deploysearch.cpp:89-103
//   search::strategy_candidates      deploysearch.cpp:105-118
//   search::evaluate_deployment      deploysearch.cpp:138-151
//   search::best_strategies          deploysearch.cpp:153-229
//   search::exhaustive               deploysearch.cpp:436-466
//   switchplan::layout/greedy_plan   switchplan.cpp:40-131
//   workload::fit_types, HoltForecaster, orch::forecast_series
// The only harness-side logic is the space enumeration (space_enum.hpp),
// which restates the reference's anonymous-namespace partitions_desc.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "oserve/core.hpp"
#include "oserve/costmodel.hpp"
#include "oserve/deploysearch.hpp"
#include "oserve/errors.hpp"
#include "oserve/flowassign.hpp"
#include "oserve/json_io.hpp"
#include "oserve/orchestrate.hpp"
#include "oserve/switchplan.hpp"
#include "oserve/workload.hpp"

#include "oracle_api.h"
#include "space_enum.hpp"

using namespace oserve;

namespace {

thread_local std::string g_err;

oserve::ClusterSpec to_cluster(const oserve_cluster_desc &c) {
    ClusterSpec out;
    out.intra_bw = c.intra_bw;
    out.inter_bw = c.inter_bw;
    int pos = 0;
    for (int m = 0; m < c.num_machines; ++m) {
        MachineSpec ms;
        ms.machine_id = "m" + std::to_string(m);
        ms.device_mem = c.device_mem[m];
        for (int i = 0; i < c.machine_num_devices[m]; ++i) ms.device_ids.push_back(c.device_ids[pos++]);
        out.machines.push_back(ms);
    }
    return out;
}

ModelSpec to_model(const oserve_model_desc &m) {
    ModelSpec out;
    out.name = "model";
    out.param_bytes = m.param_bytes;
    out.num_layers = m.num_layers;
    out.bytes_per_token_kv = m.bytes_per_token_kv;
    out.flops_per_token_prefill = m.flops_per_token_prefill;
    out.min_mem_bytes = m.min_mem_bytes;
    return out;
}

cost::ProfileParams to_params(const oserve_profile &p) {
    cost::ProfileParams out;
    out.prefill_coeff = p.prefill_coeff;
    out.decode_coeff = p.decode_coeff;
    out.tp_efficiency = p.tp_efficiency;
    out.pp_comm_cost = p.pp_comm_cost;
    out.mem_bw_penalty = p.mem_bw_penalty;
    return out;
}

std::vector<WorkloadType> to_types(const oracle_problem &p) {
    std::vector<WorkloadType> t;
    for (int j = 0; j < p.num_classes; ++j)
        t.push_back({p.classes[j].type_id, p.classes[j].centroid_in, p.classes[j].centroid_out});
    return t;
}

Deployment to_dep(const oserve_deployment &d) {
    Deployment dep;
    int pos = 0;
    for (int r = 0; r < d.num_replicas; ++r) {
        ReplicaConfig rc;
        for (int i = 0; i < d.replica_num_devices[r]; ++i) rc.device_ids.push_back(d.device_ids[pos++]);
        rc.tp = d.tp[r];
        rc.pp = d.pp[r];
        dep.replicas.push_back(rc);
    }
    return dep;
}

void from_dep(const Deployment &dep, oserve_plan *out) {
    std::memset(out, 0, sizeof(*out));
    out->num_replicas = dep.replica_count();
    int pos = 0;
    for (int r = 0; r < dep.replica_count(); ++r) {
        const auto &rc = dep.replicas[r];
        out->replica_num_devices[r] = rc.device_count();
        out->tp[r] = rc.tp;
        out->pp[r] = rc.pp;
        for (int d : rc.device_ids) out->device_ids[pos++] = d;
    }
    out->num_devices = pos;
}

struct Problem {
    ClusterSpec cluster;
    ModelSpec model;
    cost::ProfileParams params;
    std::vector<WorkloadType> types;
    TraceSpan span;
    double span_s = 60.0;
    explicit Problem(const oracle_problem &p)
        : cluster(to_cluster(p.cluster)), model(to_model(p.model)), params(to_params(p.profile)),
          types(to_types(p)), span{0, std::vector<int64_t>(p.lambda, p.lambda + p.num_classes)},
          span_s(p.span_seconds) {}
    search::EvalContext ctx(bool parallel, search::ObjectiveCache *cache = nullptr) const {
        return search::EvalContext{cluster, model, types, span, span_s, params, cache, parallel};
    }
};

template <class F>
int guarded(F &&f) {
    try {
        f();
        return OSERVE_OK;
    } catch (const InfeasibleReplica &e) {
        g_err = e.what();
        return OSERVE_ERR_INFEASIBLE_REPLICA;
    } catch (const ModelTooLarge &e) {
        g_err = e.what();
        return OSERVE_ERR_MODEL_TOO_LARGE;
    } catch (const TooLarge &e) {
        g_err = e.what();
        return OSERVE_ERR_TOO_LARGE;
    } catch (const EmptyDeployment &e) {
        g_err = e.what();
        return OSERVE_ERR_EMPTY_DEPLOYMENT;
    } catch (const UnsourcedFragment &e) {
        g_err = e.what();
        return OSERVE_ERR_UNSOURCED_FRAGMENT;
    } catch (const std::invalid_argument &e) {
        g_err = e.what();
        return OSERVE_ERR_INVALID_ARGUMENT;
    } catch (const std::logic_error &e) {
        g_err = e.what();
        return OSERVE_ERR_LOGIC;
    } catch (const std::overflow_error &e) {
        g_err = e.what();
        return OSERVE_ERR_TOO_LARGE;
    } catch (const std::exception &e) {
        g_err = e.what();
        return OSERVE_ERR_INVALID_ARGUMENT;
    }
}

oracle_space::Space build_space(const Problem &pr, const oserve_space_desc &s) {
    const int D = pr.cluster.device_count();
    if (s.max_devices > 0 && D > s.max_devices) {
        throw TooLarge("exhaustive enumeration guarded to " + std::to_string(s.max_devices) +
                       " devices, cluster has " + std::to_string(D));
    }
    const int g_min = search::min_feasible_group(pr.cluster, pr.model);
    std::vector<int> sizes(s.sizes, s.sizes + s.num_sizes);
    std::vector<DeviceId> devs = pr.cluster.all_devices();
    return oracle_space::build(D, g_min, s.mode == OSERVE_SPACE_CANONICAL, sizes, [&](int off, int d) {
        std::vector<DeviceId> block(devs.begin() + off, devs.begin() + off + d);
        return search::strategy_candidates(block, pr.cluster, pr.model);
    });
}

Deployment plan_deployment(const Problem &pr, const oracle_space::Space &sp, int64_t p,
                           const std::vector<int> &picks) {
    const auto &part = sp.parts[p];
    auto blocks = search::canonical_blocks(pr.cluster, part.sizes);
    Deployment dep;
    for (size_t r = 0; r < part.sizes.size(); ++r) {
        auto [tp, pp] = part.cands[r][picks[r]];
        dep.replicas.push_back({blocks[r], tp, pp});
    }
    return dep;
}

void fill_result(const Problem &pr, const oracle_space::Space &sp, const oracle_space::Best &b,
                 oserve_round_result *out) {
    std::memset(out, 0, sizeof(*out));
    out->partitions = static_cast<int64_t>(sp.parts.size());
    out->plans = sp.total;
    if (!b.valid) {
        out->objective = -1;
        return;
    }
    out->objective = b.obj;
    out->partition_index = b.part;
    out->local_rank = b.local;
    out->sum_pp = b.sum_pp;
    int64_t p;
    uint64_t local;
    std::vector<int> picks;
    oracle_space::unrank(sp, sp.prefix[b.part] + b.local, p, local, picks);
    from_dep(plan_deployment(pr, sp, p, picks), &out->plan);
}

}  // namespace

extern "C" {

const char *oracle_last_error(void) { return g_err.c_str(); }
int oracle_is_reference(void) { return 1; }

int oracle_min_feasible_group(const oracle_problem *p, int *g_min) {
    return guarded([&] {
        Problem pr(*p);
        *g_min = search::min_feasible_group(pr.cluster, pr.model);
    });
}

int oracle_capacity_table(const oracle_problem *p, const oserve_deployment *dep, int64_t *n,
                          int64_t *e, double *latency) {
    return guarded([&] {
        Problem pr(*p);
        cost::CapacityTable t =
            cost::build_capacity_table(to_dep(*dep), pr.types, pr.model, pr.cluster, pr.params, pr.span_s);
        const int R = t.replicas(), J = static_cast<int>(pr.types.size());
        for (int k = 0; k < R; ++k)
            for (int j = 0; j < J; ++j) {
                if (n) n[k * J + j] = t.n[k][j];
                if (e) e[k * J + j] = t.e[k][j];
                if (latency) latency[k * J + j] = t.latency[k][j];
            }
    });
}

int oracle_normalize(int J, const int64_t *n_row, int strict, int64_t *M, int64_t *units, int *scaled) {
    return guarded([&] {
        std::vector<int64_t> row(n_row, n_row + J);
        flow::NormalizedRow r = strict ? flow::normalize(row) : flow::normalize_or_scale(row);
        *M = r.M;
        for (int j = 0; j < J; ++j) units[j] = r.units[j];
        if (scaled) *scaled = r.scaled ? 1 : 0;
    });
}

int oracle_solve_assignment(int R, int J, const int64_t *n, const int64_t *e, const int64_t *lambda,
                            const oserve_solve_options *opts, int64_t *x, int64_t *objective, int64_t *M,
                            int64_t *unit, int64_t *used, uint64_t *work) {
    return guarded([&] {
        cost::CapacityTable t;
        t.n.assign(R, std::vector<int64_t>(J));
        t.e.assign(R, std::vector<int64_t>(J));
        t.latency.assign(R, std::vector<double>(J, 0.1));
        for (int k = 0; k < R; ++k)
            for (int j = 0; j < J; ++j) {
                t.n[k][j] = n[k * J + j];
                t.e[k][j] = e[k * J + j];
            }
        flow::SolveOptions so;
        if (opts) {
            so.exact_demand_limit = opts->exact_demand_limit;
            so.exact_cell_limit = opts->exact_cell_limit;
            so.node_budget = opts->node_budget;
        }
        flow::LowerLevel ll = flow::solve_assignment(t, std::vector<int64_t>(lambda, lambda + J), so);
        for (int k = 0; k < R; ++k) {
            for (int j = 0; j < J; ++j) {
                if (x) x[k * J + j] = ll.assignment.x[k][j];
                if (unit) unit[k * J + j] = ll.unit[k][j];
            }
            if (M) M[k] = ll.M[k];
            if (used) used[k] = ll.used[k];
        }
        if (objective) *objective = ll.assignment.objective;
        if (work) *work = 0;
    });
}

int oracle_check_constraints(int R, int J, const int64_t *x, const int64_t *n, const int64_t *e,
                             const int64_t *lambda) {
    return guarded([&] {
        cost::CapacityTable t;
        flow::AssignmentMatrix a;
        t.n.assign(R, std::vector<int64_t>(J));
        t.e.assign(R, std::vector<int64_t>(J));
        t.latency.assign(R, std::vector<double>(J, 0.1));
        a.x.assign(R, std::vector<int64_t>(J));
        for (int k = 0; k < R; ++k)
            for (int j = 0; j < J; ++j) {
                t.n[k][j] = n[k * J + j];
                t.e[k][j] = e[k * J + j];
                a.x[k][j] = x[k * J + j];
            }
        flow::check_constraints(a, t, std::vector<int64_t>(lambda, lambda + J));
    });
}

int oracle_evaluate_deployment(const oracle_problem *p, const oserve_deployment *dep, int64_t *objective) {
    return guarded([&] {
        Problem pr(*p);
        *objective = search::evaluate_deployment(to_dep(*dep), pr.ctx(false));
    });
}

int oracle_best_strategies(const oracle_problem *p, int R, const int *sizes, int parallel,
                           oserve_round_result *out) {
    return guarded([&] {
        Problem pr(*p);
        search::ObjectiveCache cache;
        search::StrategyChoice c =
            search::best_strategies(std::vector<int>(sizes, sizes + R), pr.ctx(parallel != 0, &cache));
        std::memset(out, 0, sizeof(*out));
        out->objective = c.objective;
        from_dep(c.deployment, &out->plan);
        int spp = 0;
        for (const auto &r : c.deployment.replicas) spp += r.pp;
        out->sum_pp = spp;
    });
}

int oracle_exhaustive(const oracle_problem *p, int parallel, oserve_round_result *out) {
    return guarded([&] {
        Problem pr(*p);
        search::SearchState s = search::exhaustive(pr.cluster, pr.model, pr.types, pr.span, pr.span_s,
                                                   pr.params, parallel != 0);
        std::memset(out, 0, sizeof(*out));
        out->objective = s.throughput;
        out->partitions = s.iterations;
        from_dep(s.deployment, &out->plan);
        int spp = 0;
        for (const auto &r : s.deployment.replicas) spp += r.pp;
        out->sum_pp = spp;
    });
}

int oracle_space_info(const oracle_problem *p, const oserve_space_desc *s, int64_t *partitions,
                      uint64_t *plans) {
    return guarded([&] {
        Problem pr(*p);
        auto sp = build_space(pr, *s);
        *partitions = static_cast<int64_t>(sp.parts.size());
        *plans = sp.total;
    });
}

int oracle_space_plan(const oracle_problem *p, const oserve_space_desc *s, uint64_t rank, oserve_plan *plan,
                      int64_t *partition_index, uint64_t *local_rank) {
    return guarded([&] {
        Problem pr(*p);
        auto sp = build_space(pr, *s);
        if (rank >= sp.total) throw std::invalid_argument("rank out of range");
        int64_t pi;
        uint64_t local;
        std::vector<int> picks;
        oracle_space::unrank(sp, rank, pi, local, picks);
        from_dep(plan_deployment(pr, sp, pi, picks), plan);
        if (partition_index) *partition_index = pi;
        if (local_rank) *local_rank = local;
    });
}

int oracle_evaluate_ranks(const oracle_problem *p, const oserve_space_desc *s, int64_t count,
                          const uint64_t *ranks, int64_t *objective, int32_t *sum_pp, uint64_t *work,
                          int threads) {
    return guarded([&] {
        Problem pr(*p);
        auto sp = build_space(pr, *s);
        for (int64_t i = 0; i < count; ++i)
            if (ranks[i] >= sp.total) throw std::invalid_argument("rank out of range");
        std::atomic<int> status{0};
        std::mutex mu;
        std::string err;
#pragma omp parallel for schedule(dynamic, 4) num_threads(threads > 0 ? threads : 1)
        for (int64_t i = 0; i < count; ++i) {
            try {
                int64_t pi;
                uint64_t local;
                std::vector<int> picks;
                oracle_space::unrank(sp, ranks[i], pi, local, picks);
                Deployment dep = plan_deployment(pr, sp, pi, picks);
                objective[i] = search::evaluate_deployment(dep, pr.ctx(false));
                if (sum_pp) {
                    int spp = 0;
                    for (const auto &r : dep.replicas) spp += r.pp;
                    sum_pp[i] = spp;
                }
                if (work) work[i] = 0;
            } catch (const std::exception &e) {
                std::lock_guard<std::mutex> g(mu);
                err = e.what();
                status = 1;
            }
        }
        if (status) throw std::runtime_error(err);
    });
}

int oracle_round(const oracle_problem *p, const oserve_space_desc *s, int threads, oserve_round_result *out) {
    return guarded([&] {
        Problem pr(*p);
        auto sp = build_space(pr, *s);
        oracle_space::Best best;
        if (s->mode == OSERVE_SPACE_ORDERED) {
            // The reference's own per-partition argmin: best_strategies
            // (deploysearch.cpp:153-229), first-wins across partitions
            // (exhaustive, :452-460).  The key fields are recovered from the
            // returned deployment.
#ifdef _OPENMP
            if (threads > 0) omp_set_num_threads(threads);
#endif
            search::ObjectiveCache cache;
            auto ctx = pr.ctx(threads > 1, &cache);
            for (size_t pi = 0; pi < sp.parts.size(); ++pi) {
                const auto &part = sp.parts[pi];
                if (part.count == 0) continue;
                search::StrategyChoice c = search::best_strategies(part.sizes, ctx);
                if (c.deployment.replicas.empty()) continue;
                if (best.valid && c.objective <= best.obj) continue;
                std::vector<int> picks;
                int spp = 0;
                for (size_t r = 0; r < part.sizes.size(); ++r) {
                    const auto &rc = c.deployment.replicas[r];
                    int idx = -1;
                    for (size_t q = 0; q < part.cands[r].size(); ++q)
                        if (part.cands[r][q].first == rc.tp) idx = static_cast<int>(q);
                    picks.push_back(idx);
                    spp += rc.pp;
                }
                best.valid = true;
                best.obj = c.objective;
                best.part = static_cast<int64_t>(pi);
                best.sum_pp = spp;
                best.local = oracle_space::rank_of(part, picks);
            }
        } else {
            // Canonical space: every plan through evaluate_deployment
            // (deploysearch.cpp:138-151), OpenMP dynamic,4 like :203.
            const int nt = threads > 0 ? threads : 1;
            std::vector<oracle_space::Best> local_best(nt);
            uint64_t total = sp.total;
#pragma omp parallel num_threads(nt)
            {
                int tid = 0;
#ifdef _OPENMP
                tid = omp_get_thread_num();
#endif
                oracle_space::Best lb;
#pragma omp for schedule(dynamic, 4)
                for (int64_t g = 0; g < static_cast<int64_t>(total); ++g) {
                    int64_t pi;
                    uint64_t local;
                    std::vector<int> picks;
                    oracle_space::unrank(sp, static_cast<uint64_t>(g), pi, local, picks);
                    Deployment dep = plan_deployment(pr, sp, pi, picks);
                    int64_t obj = search::evaluate_deployment(dep, pr.ctx(false));
                    int spp = 0;
                    for (const auto &r : dep.replicas) spp += r.pp;
                    lb.offer(obj, pi, spp, local);
                }
                local_best[tid] = lb;
            }
            for (const auto &lb : local_best)
                if (lb.valid) best.offer(lb.obj, lb.part, lb.sum_pp, lb.local);
        }
        if (!best.valid) throw ModelTooLarge("round: no feasible deployment");
        fill_result(pr, sp, best, out);
    });
}

int oracle_switch_plan(const oserve_cluster_desc *c, uint64_t param_bytes, const oserve_deployment *src,
                       const oserve_deployment *dst, int capacity, oserve_transfer *transfers,
                       int *num_transfers, double *est_seconds, uint64_t *max_link_bytes) {
    return guarded([&] {
        ClusterSpec cluster = to_cluster(*c);
        ModelSpec model;
        model.param_bytes = param_bytes;
        auto from = switchplan::layout(to_dep(*src), model);
        auto to = switchplan::layout(to_dep(*dst), model);
        switchplan::SwitchPlan plan = switchplan::greedy_plan(from, to, cluster);
        int n = static_cast<int>(plan.transfers.size());
        if (num_transfers) *num_transfers = n;
        if (transfers) {
            for (int i = 0; i < std::min(n, capacity); ++i) {
                const auto &t = plan.transfers[i];
                transfers[i] = {t.range.begin, t.range.end, t.src, t.dst};
            }
        }
        if (est_seconds) *est_seconds = switchplan::estimate_time(plan, cluster);
        if (max_link_bytes) {
            uint64_t m = 0;
            for (const auto &[link, bytes] : plan.link_load) m = std::max(m, bytes);
            *max_link_bytes = m;
        }
    });
}

int oracle_search(const oracle_problem *p, const oserve_search_options *o, oserve_search_result *out,
                  oserve_search_log_row *log, int log_capacity) {
    return guarded([&] {
        Problem pr(*p);
        search::SearchOptions so;
        so.seed = o->seed;
        so.max_iters = o->max_iters;
        so.stale_limit = o->stale_limit;
        so.mutation_retries = o->mutation_retries;
        so.parallel = true;
        Deployment warm;
        if (o->warm_start) {
            warm = to_dep(*o->warm_start);
            so.warm_start = &warm;
        }
        int n = 0;
        so.log = [&](const search::SearchLogRow &r) {
            if (log && n < log_capacity) {
                oserve_search_log_row &row = log[n];
                row.iteration = r.iteration;
                row.accepted = r.accepted ? 1 : 0;
                row.throughput = r.throughput;
                row.devices = r.devices;
                std::snprintf(row.op, sizeof(row.op), "%s", r.op.c_str());
            }
            ++n;
        };
        search::SearchState st = search::search(pr.cluster, pr.model, pr.types, pr.span, pr.span_s, pr.params, so);
        std::memset(out, 0, sizeof(*out));
        out->throughput = st.throughput;
        out->rng_seed = st.rng_seed;
        out->stale_iters = st.stale_iters;
        out->iterations = st.iterations;
        out->log_count = n;
        from_dep(st.deployment, &out->deployment);
    });
}

int oracle_adaptive_timeline(const oracle_problem *p, int T, const int64_t *counts, uint64_t seed, int max_iters,
                             double min_gain, int capacity, int64_t *span_index, oserve_plan *plans, int64_t *x,
                             double *switch_seconds, int *transfers, int *count) {
    return guarded([&] {
        Problem pr(*p);
        const int J = p->num_classes;
        workload::SpanSeries series;
        series.span_seconds = static_cast<int>(pr.span_s);
        for (int t = 0; t < T; ++t)
            series.spans.push_back({t, std::vector<int64_t>(counts + t * J, counts + (t + 1) * J)});
        workload::TypeModel tm;
        tm.k = J;
        tm.centroids = pr.types;
        orch::OrchestrateOptions oo;
        oo.seed = seed;
        oo.span_seconds = static_cast<int>(pr.span_s);
        oo.k = J;
        oo.min_gain = min_gain;
        oo.search_max_iters = max_iters;
        oo.parallel = true;
        sim::StrategyTimeline tl = orch::build_adaptive_timeline(series, tm, pr.cluster, pr.model, pr.params, oo);
        int n = static_cast<int>(tl.entries.size());
        *count = n;
        for (int e = 0; e < std::min(n, capacity); ++e) {
            const auto &en = tl.entries[e];
            span_index[e] = en.start_span;
            from_dep(en.deployment, &plans[e]);
            for (size_t k = 0; k < en.assignment.x.size(); ++k)
                for (int j = 0; j < J; ++j) x[(static_cast<size_t>(e) * 128 + k) * J + j] = en.assignment.x[k][j];
            switch_seconds[e] = en.switch_seconds;
            transfers[e] = static_cast<int>(en.plan.transfers.size());
        }
    });
}

int oracle_fit_types(int64_t n, const uint32_t *input_len, const uint32_t *output_len, int k, uint64_t seed,
                     double *centroid_in, double *centroid_out) {
    return guarded([&] {
        std::vector<TraceRecord> recs(n);
        for (int64_t i = 0; i < n; ++i) recs[i] = {static_cast<uint64_t>(i), input_len[i], output_len[i]};
        workload::TypeModel m = workload::fit_types(recs, k, seed);
        for (int c = 0; c < k; ++c) {
            centroid_in[c] = m.centroids[c].centroid_in;
            centroid_out[c] = m.centroids[c].centroid_out;
        }
    });
}

int oracle_holt_forecast(int J, int T, const int64_t *counts, int window, int64_t *lambda_out) {
    // orch::forecast_series (orchestrate.cpp:75-92) with the default Holt
    // predictor (workload.cpp:204-222); counts is [T][J]; output [T][J].
    return guarded([&] {
        workload::SpanSeries series;
        for (int t = 0; t < T; ++t) {
            TraceSpan s{t, std::vector<int64_t>(counts + t * J, counts + (t + 1) * J)};
            series.spans.push_back(s);
        }
        workload::HoltForecaster predictor;
        auto f = orch::forecast_series(series, predictor, window);
        for (int t = 0; t < T; ++t)
            for (int j = 0; j < J; ++j) lambda_out[t * J + j] = f[t][j];
    });
}

int oracle_kv_plan(const oserve_cluster_desc *c, int n_inflight, const oserve_inflight *inflight,
                   int64_t threshold_tokens, const oserve_deployment *src, const oserve_deployment *dst,
                   double headroom, int n_carry, const oserve_transfer *carry, int64_t *drained, int *n_drained,
                   oserve_kv_transfer *migrated, int *n_migrated, uint64_t *buffer_bytes) {
    return guarded([&] {
        ClusterSpec cl = to_cluster(*c);
        std::vector<switchplan::InflightRequest> reqs;
        for (int q = 0; q < n_inflight; ++q)
            reqs.push_back({inflight[q].request_id, inflight[q].generated_tokens, inflight[q].kv_bytes,
                            inflight[q].source_replica});
        switchplan::SwitchPlan cp;
        for (int i = 0; i < n_carry; ++i) {
            switchplan::Transfer t;
            t.range.begin = carry[i].begin;
            t.range.end = carry[i].end;
            t.src = carry[i].src;
            t.dst = carry[i].dst;
            cp.transfers.push_back(t);
            cp.link_load[{t.src, t.dst}] += t.range.len();
        }
        auto kv = switchplan::kv_plan(reqs, threshold_tokens, to_dep(*src), to_dep(*dst), cl, headroom,
                                      n_carry > 0 ? &cp : nullptr);
        *n_drained = static_cast<int>(kv.drained.size());
        for (size_t i = 0; i < kv.drained.size(); ++i) drained[i] = kv.drained[i];
        *n_migrated = static_cast<int>(kv.migrated.size());
        for (size_t i = 0; i < kv.migrated.size(); ++i)
            migrated[i] = {kv.migrated[i].request_id, kv.migrated[i].kv_bytes, kv.migrated[i].src,
                           kv.migrated[i].dst};
        *buffer_bytes = kv.buffer_bytes;
    });
}

int oracle_adaptive_timeline_json(const oracle_problem *p, int T, const int64_t *counts, uint64_t seed,
                                  int max_iters, double min_gain, const char *path) {
    return guarded([&] {
        Problem pr(*p);
        const int J = p->num_classes;
        workload::SpanSeries series;
        series.span_seconds = static_cast<int>(pr.span_s);
        for (int t = 0; t < T; ++t)
            series.spans.push_back({t, std::vector<int64_t>(counts + t * J, counts + (t + 1) * J)});
        workload::TypeModel tm;
        tm.k = J;
        tm.centroids = pr.types;
        orch::OrchestrateOptions oo;
        oo.seed = seed;
        oo.span_seconds = static_cast<int>(pr.span_s);
        oo.k = J;
        oo.min_gain = min_gain;
        oo.search_max_iters = max_iters;
        oo.parallel = true;
        io::save_timeline(path, orch::build_adaptive_timeline(series, tm, pr.cluster, pr.model, pr.params, oo));
    });
}

int oracle_timeline_resave(const char *in_path, const char *out_path, int *entries) {
    return guarded([&] {
        auto tl = io::load_timeline(in_path);
        *entries = static_cast<int>(tl.entries.size());
        io::save_timeline(out_path, tl);
    });
}

int oracle_deployment_resave(const char *in_path, const char *out_path, int *replicas) {
    return guarded([&] {
        auto d = io::load_deployment(in_path);
        *replicas = d.replica_count();
        io::save_deployment(out_path, d);
    });
}

static cost::CapacityTable raw_table(int R, int J, const int64_t *n, const int64_t *e) {
    cost::CapacityTable t;
    t.n.assign(R, std::vector<int64_t>(J));
    t.e.assign(R, std::vector<int64_t>(J));
    t.latency.assign(R, std::vector<double>(J, 0.1));
    for (int k = 0; k < R; ++k)
        for (int j = 0; j < J; ++j) {
            t.n[k][j] = n[k * J + j];
            t.e[k][j] = e[k * J + j];
        }
    return t;
}

int oracle_max_flow(int num_nodes, int num_edges, const oserve_flow_edge *edges, int source, int sink,
                    int64_t *flow, int64_t *value) {
    return guarded([&] {
        flow::Graph g;
        g.num_nodes = num_nodes;
        for (int i = 0; i < num_edges; ++i) g.edges.push_back({edges[i].from, edges[i].to, edges[i].cap});
        auto r = flow::max_flow(g, source, sink);
        for (int i = 0; i < num_edges; ++i) flow[i] = r.flow[i];
        *value = r.value;
    });
}

int oracle_flow_assign(int R, int J, const int64_t *n, const int64_t *e, const int64_t *lambda,
                       const oserve_solve_options *opts, int64_t *x, int64_t *objective, int64_t *flow_value,
                       int64_t *edge_flow) {
    return guarded([&] {
        auto t = raw_table(R, J, n, e);
        TraceSpan span{0, std::vector<int64_t>(lambda, lambda + J)};
        auto net = flow::build_network(span, t);
        auto fr = flow::max_flow(net.graph, net.source(), net.sink());
        flow::SolveOptions so;
        if (opts) {
            so.exact_demand_limit = opts->exact_demand_limit;
            so.exact_cell_limit = opts->exact_cell_limit;
            so.node_budget = opts->node_budget;
        }
        auto a = flow::extract_assignment(net, fr, so);
        for (int k = 0; k < R; ++k)
            for (int j = 0; j < J; ++j) x[k * J + j] = a.x[k][j];
        *objective = a.objective;
        if (flow_value) *flow_value = fr.value;
        if (edge_flow)
            for (size_t i = 0; i < fr.flow.size(); ++i) edge_flow[i] = fr.flow[i];
    });
}

int oracle_solve_fractional(int R, int J, const int64_t *n, const int64_t *e, const int64_t *lambda, double *f,
                            double *objective) {
    return guarded([&] {
        auto t = raw_table(R, J, n, e);
        auto lp = flow::solve_fractional(t, std::vector<int64_t>(lambda, lambda + J));
        for (int k = 0; k < R; ++k)
            for (int j = 0; j < J; ++j) f[k * J + j] = lp.f[k][j];
        *objective = lp.objective;
    });
}

int oracle_to_dot(int R, int J, const int64_t *n, const int64_t *e, const int64_t *lambda, int with_flow,
                  char *buf, int cap, int *len) {
    return guarded([&] {
        auto t = raw_table(R, J, n, e);
        TraceSpan span{0, std::vector<int64_t>(lambda, lambda + J)};
        auto net = flow::build_network(span, t);
        std::string d;
        if (with_flow) {
            auto fr = flow::max_flow(net.graph, net.source(), net.sink());
            d = flow::to_dot(net, &fr);
        } else {
            d = flow::to_dot(net);
        }
        *len = static_cast<int>(d.size());
        if (buf && cap > 0) {
            const int c = std::min(cap - 1, *len);
            std::memcpy(buf, d.data(), c);
            buf[c] = 0;
        }
    });
}

}  // extern "C"
