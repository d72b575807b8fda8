// oserve_port.cpp — TEST INFRASTRUCTURE ONLY: a CPU restatement of the
// reference scheduling round, used as the parity checker of the GPU path.
//
// Parity pinned against the unmodified reference (oracle/_ref) and the golden
// vectors in tests/golden (tests/test_oracle.py).  Each function cites the
// reference file:line it restates (paths under /root/reference/proj).
// Additionally counts the algorithmic work W of SURVEY §8(d):
//   W = R*J (cost cells) + greedy visits + exchange probes.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <mutex>
#include <numeric>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "oracle_api.h"
#include "space_enum.hpp"

namespace {

thread_local std::string g_err;

struct Status : std::runtime_error {
    int code;
    Status(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void fail(int code, const std::string &m) { throw Status(code, m); }

template <class F>
int guarded(F &&f) {
    try {
        f();
        return OSERVE_OK;
    } catch (const Status &s) {
        g_err = s.what();
        return s.code;
    } catch (const std::overflow_error &e) {
        g_err = e.what();
        return OSERVE_ERR_TOO_LARGE;
    } catch (const std::exception &e) {
        g_err = e.what();
        return OSERVE_ERR_INVALID_ARGUMENT;
    }
}

// ---------------------------------------------------------------- cluster --
// ClusterSpec helpers, core.cpp:17-45.
struct Cluster {
    std::vector<int> dev_sorted;        // all_devices(), core.cpp:23-28
    std::map<int, int> machine_of;      // device -> machine index (core.cpp:29-35)
    std::vector<uint64_t> mem;          // per machine
    double intra = 0, inter = 0;
    explicit Cluster(const oserve_cluster_desc &c) : intra(c.intra_bw), inter(c.inter_bw) {
        int pos = 0;
        for (int m = 0; m < c.num_machines; ++m) {
            mem.push_back(c.device_mem[m]);
            for (int i = 0; i < c.machine_num_devices[m]; ++i) {
                int d = c.device_ids[pos++];
                dev_sorted.push_back(d);
                machine_of.emplace(d, m);  // first machine wins, like the linear scan
            }
        }
        std::sort(dev_sorted.begin(), dev_sorted.end());
    }
    int machine(int d) const {
        auto it = machine_of.find(d);
        return it == machine_of.end() ? -1 : it->second;
    }
    uint64_t device_mem(int d) const {
        int m = machine(d);
        return m < 0 ? 0 : mem[m];
    }
    bool same_machine(int a, int b) const {
        int ma = machine(a);
        return ma >= 0 && ma == machine(b);
    }
    int size() const { return static_cast<int>(dev_sorted.size()); }
};

struct Replica {
    std::vector<int> devs;  // as given
    int tp = 1, pp = 1;
};

// validate_replica (core.cpp:105-127) as a predicate (replica_valid :129-136).
bool placement_ok(const Replica &r, const Cluster &c) {
    if (r.tp < 1 || r.pp < 1 || r.devs.empty()) return false;
    if (r.tp * r.pp != static_cast<int>(r.devs.size())) return false;
    std::vector<int> s = r.devs;
    std::sort(s.begin(), s.end());
    if (std::adjacent_find(s.begin(), s.end()) != s.end()) return false;
    for (int d : s)
        if (c.machine(d) < 0) return false;
    for (int st = 0; st < r.pp; ++st) {
        int head = s[st * r.tp];
        for (int i = 1; i < r.tp; ++i)
            if (!c.same_machine(head, s[st * r.tp + i])) return false;
    }
    return true;
}

// ------------------------------------------------------------- cost model --
struct Model {
    uint64_t P, min_mem, kvb;
    double L;
};

// memory_feasible, costmodel.cpp:48-62.
bool mem_feasible(const Replica &r, const Model &m, const Cluster &c) {
    if (r.devs.empty()) return false;
    uint64_t total = 0, min_dev = std::numeric_limits<uint64_t>::max();
    for (int d : r.devs) {
        uint64_t mm = c.device_mem(d);
        if (mm == 0) return false;
        total += mm;
        min_dev = std::min(min_dev, mm);
    }
    if (total < m.min_mem) return false;
    uint64_t shards = static_cast<uint64_t>(r.tp) * static_cast<uint64_t>(r.pp);
    return (m.P + shards - 1) / shards <= min_dev;
}

// service time: prefill (costmodel.cpp:28-33) + decode (:35-40), summed as in
// request_service_time (:42-46).  Operand order kept; no FMA (-ffp-contract=off).
double service_time(int tp, int pp, const Model &m, const oserve_profile &pr, double in, double out) {
    double speedup = tp * std::pow(pr.tp_efficiency, std::log2(static_cast<double>(tp)));  // :22-24
    double prefill = in * m.L * pr.prefill_coeff / speedup + (pp - 1) * pr.pp_comm_cost;
    double penalty = 1.0 + pr.mem_bw_penalty * (tp - 1);                                   // :26
    double decode = out * m.L * pr.decode_coeff * penalty / tp + (pp - 1) * pr.pp_comm_cost * out;
    return prefill + decode;
}

struct Cells {
    std::vector<int64_t> n, e;  // [R*J]
    std::vector<double> lat;
};

// build_capacity_table, costmodel.cpp:94-116 (with capacity :74-82,
// edge_capacity :84-92, replica_kv_budget :64-68, kv_bytes_per_request :70-72).
Cells cost_cells(const std::vector<Replica> &dep, const oracle_problem &p, const Model &m, const Cluster &c) {
    const int R = static_cast<int>(dep.size()), J = p.num_classes;
    Cells t;
    t.n.assign(R * J, 0);
    t.e.assign(R * J, 0);
    t.lat.assign(R * J, 0.0);
    for (int k = 0; k < R; ++k) {
        const Replica &r = dep[k];
        if (!mem_feasible(r, m, c))
            fail(OSERVE_ERR_INFEASIBLE_REPLICA, "replica " + std::to_string(k) + " cannot host model");
        uint64_t total = 0;
        for (int d : r.devs) total += c.device_mem(d);
        uint64_t budget = total > m.P ? total - m.P : 0;
        for (int j = 0; j < J; ++j) {
            const oserve_class &w = p.classes[j];
            double svc = service_time(r.tp, r.pp, m, p.profile, w.centroid_in, w.centroid_out);
            int64_t n = static_cast<int64_t>(std::floor(p.span_seconds * r.pp / svc));
            double per_req = (w.centroid_in + w.centroid_out) * static_cast<double>(m.kvb);
            double capd = std::floor(static_cast<double>(budget) / per_req);
            t.n[k * J + j] = n;
            t.e[k * J + j] = capd >= static_cast<double>(n) ? n : static_cast<int64_t>(capd);
            t.lat[k * J + j] = svc;
        }
    }
    return t;
}

// ---------------------------------------------------------- normalization --
constexpr int64_t kLimit = int64_t{1} << 62;  // flowassign.cpp:19-21

// normalize / normalize_or_scale, flowassign.cpp:22-62.
bool lcm_row(const int64_t *n, int J, int64_t &M, int64_t *units) {
    int64_t acc = 1;
    for (int j = 0; j < J; ++j) {
        if (n[j] < 0) fail(OSERVE_ERR_INVALID_ARGUMENT, "normalize: negative capacity");
        if (n[j] == 0) continue;
        int64_t g = std::gcd(acc, n[j]);
        int64_t q = acc / g;
        if (q > kLimit / n[j]) return false;
        acc = q * n[j];
    }
    M = acc;
    for (int j = 0; j < J; ++j) units[j] = n[j] > 0 ? acc / n[j] : 0;
    return true;
}

bool normalize_row(const int64_t *n, int J, int64_t &M, int64_t *units) {
    if (lcm_row(n, J, M, units)) return false;
    M = kLimit;  // rescaling fallback
    for (int j = 0; j < J; ++j) units[j] = n[j] > 0 ? (kLimit + n[j] - 1) / n[j] : 0;
    return true;
}

// ------------------------------------------------------------ assignment --
struct Inst {
    int R = 0, J = 0;
    std::vector<int64_t> cap, unit, M, lam;  // cap/unit [R*J]
    std::vector<std::vector<int>> order;
    int64_t c(int k, int j) const { return cap[k * J + j]; }
    int64_t u(int k, int j) const { return unit[k * J + j]; }
};

// make_instance, flowassign.cpp:267-294.
Inst instance(const int64_t *n, const int64_t *e, const std::vector<int64_t> &unit, const std::vector<int64_t> &M,
              const int64_t *lam, int R, int J) {
    Inst in;
    in.R = R;
    in.J = J;
    in.unit = unit;
    in.M = M;
    in.lam.assign(lam, lam + J);
    in.cap.assign(R * J, 0);
    in.order.resize(R);
    for (int k = 0; k < R; ++k) {
        for (int j = 0; j < J; ++j) {
            int64_t u = unit[k * J + j];
            if (u <= 0) continue;
            int64_t cc = std::min(std::min(e[k * J + j], n[k * J + j]), M[k] / u);
            if (cc > 0) {
                in.cap[k * J + j] = cc;
                in.order[k].push_back(j);
            }
        }
        std::stable_sort(in.order[k].begin(), in.order[k].end(),
                         [&](int a, int b) { return unit[k * J + a] < unit[k * J + b]; });
    }
    return in;
}

// Branch and bound, flowassign.cpp:296-369 (greedy_suffix :298-311).
struct BnB {
    const Inst &in;
    std::vector<int64_t> lam, mrem, x, best_x;
    int64_t count = 0, best = -1, nodes = 0, budget;
    bool aborted = false;
    BnB(const Inst &i, int64_t b) : in(i), lam(i.lam), mrem(i.M), x(i.R * i.J, 0), best_x(i.R * i.J, 0), budget(b) {}

    int64_t suffix_bound(int k, size_t pos, std::vector<int64_t> l, int64_t mr) const {
        int64_t cnt = 0;
        for (size_t i = pos; i < in.order[k].size(); ++i) {
            int j = in.order[k][i];
            int64_t t = std::min(std::min(in.c(k, j), l[j]), mr / in.u(k, j));
            if (t > 0) {
                cnt += t;
                l[j] -= t;
                mr -= t * in.u(k, j);
            }
        }
        return cnt;
    }

    void visit(int k, size_t pos) {
        if (aborted) return;
        if (++nodes > budget) {
            aborted = true;
            return;
        }
        if (k == in.R) {
            if (count > best) {
                best = count;
                best_x = x;
            }
            return;
        }
        if (pos == in.order[k].size()) {
            visit(k + 1, 0);
            return;
        }
        int64_t lam_total = 0;
        for (int64_t v : lam) lam_total += v;
        int64_t bound = suffix_bound(k, pos, lam, mrem[k]);
        for (int k2 = k + 1; k2 < in.R; ++k2) bound += suffix_bound(k2, 0, lam, in.M[k2]);
        if (count + std::min(lam_total, bound) <= best) return;
        int j = in.order[k][pos];
        int64_t u = in.u(k, j);
        int64_t hi = std::min(std::min(in.c(k, j), lam[j]), mrem[k] / u);
        for (int64_t v = hi; v >= 0; --v) {
            x[k * in.J + j] = v;
            lam[j] -= v;
            mrem[k] -= v * u;
            count += v;
            visit(k, pos + 1);
            count -= v;
            mrem[k] += v * u;
            lam[j] += v;
            x[k * in.J + j] = 0;
            if (aborted) return;
        }
    }
};

struct Solved {
    std::vector<int64_t> x;
    int64_t obj = 0;
    uint64_t work = 0;  // greedy visits + exchange probes (or B&B nodes)
};

// greedy_fill (flowassign.cpp:393-406) + exchange_improve (:411-448).
void heuristic(const Inst &in, Solved &s) {
    const int R = in.R, J = in.J;
    std::vector<int64_t> lam = in.lam, mrem = in.M;
    s.x.assign(R * J, 0);
    int64_t count = 0;
    uint64_t work = 0;
    for (int k = 0; k < R; ++k) {
        for (int j : in.order[k]) {
            ++work;
            int64_t u = in.u(k, j);
            int64_t t = std::min(std::min(in.c(k, j) - s.x[k * J + j], lam[j]), mrem[k] / u);
            if (t > 0) {
                s.x[k * J + j] += t;
                lam[j] -= t;
                mrem[k] -= t * u;
                count += t;
            }
        }
    }
    // Exchange: first improving move in (j, k, direct | (j2, k2)) order,
    // restarting from j = 0 after every move.
    for (bool moved = true; moved;) {
        moved = false;
        for (int j = 0; j < J && !moved; ++j) {
            if (lam[j] <= 0) continue;
            for (int k = 0; k < R && !moved; ++k) {
                ++work;
                int64_t ukj = in.u(k, j);
                if (ukj <= 0 || s.x[k * J + j] >= in.c(k, j)) continue;
                if (mrem[k] >= ukj) {
                    s.x[k * J + j] += 1;
                    lam[j] -= 1;
                    mrem[k] -= ukj;
                    count += 1;
                    moved = true;
                    break;
                }
                for (int j2 = 0; j2 < J && !moved; ++j2) {
                    ++work;
                    if (j2 == j || s.x[k * J + j2] <= 0) continue;
                    if (mrem[k] + in.u(k, j2) < ukj) continue;
                    for (int k2 = 0; k2 < R && !moved; ++k2) {
                        ++work;
                        if (k2 == k || in.u(k2, j2) <= 0) continue;
                        if (s.x[k2 * J + j2] >= in.c(k2, j2)) continue;
                        if (mrem[k2] < in.u(k2, j2)) continue;
                        s.x[k * J + j2] -= 1;
                        mrem[k] += in.u(k, j2);
                        s.x[k2 * J + j2] += 1;
                        mrem[k2] -= in.u(k2, j2);
                        s.x[k * J + j] += 1;
                        mrem[k] -= ukj;
                        lam[j] -= 1;
                        count += 1;
                        moved = true;
                    }
                }
            }
        }
    }
    s.obj = count;
    s.work = work;
}

// solve_instance, flowassign.cpp:450-477 (use_exact :450-453).
Solved solve(const Inst &in, const oserve_solve_options &o) {
    Solved s;
    int64_t total = 0;
    for (int64_t v : in.lam) total += v;
    if (total <= o.exact_demand_limit && in.R * in.J <= o.exact_cell_limit) {
        BnB b(in, o.node_budget);
        b.visit(0, 0);
        if (!b.aborted) {
            s.x = b.best_x;
            s.obj = b.best;
            s.work = static_cast<uint64_t>(b.nodes);
            return s;
        }
    }
    heuristic(in, s);
    return s;
}

constexpr oserve_solve_options kDefaultOpts{400, 20, 8000000};

// solve_assignment, flowassign.cpp:481-503.
Solved solve_table(int R, int J, const int64_t *n, const int64_t *e, const int64_t *lam,
                   const oserve_solve_options &o, std::vector<int64_t> *M_out = nullptr,
                   std::vector<int64_t> *unit_out = nullptr) {
    std::vector<int64_t> M(R), unit(R * J);
    for (int k = 0; k < R; ++k) normalize_row(n + k * J, J, M[k], unit.data() + k * J);
    Inst in = instance(n, e, unit, M, lam, R, J);
    Solved s = solve(in, o);
    if (M_out) *M_out = M;
    if (unit_out) *unit_out = unit;
    return s;
}

Model to_model(const oserve_model_desc &m) {
    return Model{m.param_bytes, m.min_mem_bytes, m.bytes_per_token_kv, static_cast<double>(m.num_layers)};
}

std::vector<Replica> to_dep(const oserve_deployment &d) {
    std::vector<Replica> out;
    int pos = 0;
    for (int r = 0; r < d.num_replicas; ++r) {
        Replica rep;
        rep.devs.assign(d.device_ids + pos, d.device_ids + pos + d.replica_num_devices[r]);
        pos += d.replica_num_devices[r];
        rep.tp = d.tp[r];
        rep.pp = d.pp[r];
        out.push_back(rep);
    }
    return out;
}

void to_plan(const std::vector<Replica> &dep, oserve_plan *out) {
    std::memset(out, 0, sizeof(*out));
    out->num_replicas = static_cast<int>(dep.size());
    int pos = 0;
    for (size_t r = 0; r < dep.size(); ++r) {
        out->replica_num_devices[r] = static_cast<int>(dep[r].devs.size());
        out->tp[r] = dep[r].tp;
        out->pp[r] = dep[r].pp;
        for (int d : dep[r].devs) out->device_ids[pos++] = d;
    }
    out->num_devices = pos;
}

// evaluate_deployment, deploysearch.cpp:138-151 (no memo: the memo only
// changes results on clusters with non-uniform device memory).
int64_t evaluate(const std::vector<Replica> &dep, const oracle_problem &p, const Model &m, const Cluster &c,
                 uint64_t *work = nullptr) {
    if (dep.empty()) return 0;
    const int R = static_cast<int>(dep.size()), J = p.num_classes;
    Cells t = cost_cells(dep, p, m, c);
    Solved s = solve_table(R, J, t.n.data(), t.e.data(), p.lambda, kDefaultOpts);
    if (work) *work = static_cast<uint64_t>(R) * J + s.work;
    return s.obj;
}

// min_feasible_group, deploysearch.cpp:77-87.
int g_min_of(const Cluster &c, const Model &m) {
    uint64_t min_dev = std::numeric_limits<uint64_t>::max();
    for (uint64_t v : c.mem) min_dev = std::min(min_dev, v);
    for (int g = 1; g <= c.size(); ++g) {
        bool total_ok = static_cast<uint64_t>(g) * min_dev >= m.min_mem;
        bool shard_ok = (m.P + g - 1) / g <= min_dev;
        if (total_ok && shard_ok) return g;
    }
    fail(OSERVE_ERR_MODEL_TOO_LARGE, "model does not fit on the cluster");
}

// strategy_candidates, deploysearch.cpp:105-118.
oracle_space::Cands candidates(const std::vector<int> &block, const Cluster &c, const Model &m) {
    oracle_space::Cands out;
    const int d = static_cast<int>(block.size());
    for (int tp = d; tp >= 1; --tp) {
        if (d % tp) continue;
        Replica r{block, tp, d / tp};
        if (placement_ok(r, c) && mem_feasible(r, m, c)) out.emplace_back(tp, d / tp);
    }
    return out;
}

oracle_space::Space space_of(const oracle_problem &p, const oserve_space_desc &s, const Cluster &c, const Model &m) {
    if (s.max_devices > 0 && c.size() > s.max_devices) fail(OSERVE_ERR_TOO_LARGE, "exhaustive guard");
    const int g = g_min_of(c, m);
    std::vector<int> sizes(s.sizes, s.sizes + s.num_sizes);
    return oracle_space::build(c.size(), g, s.mode == OSERVE_SPACE_CANONICAL, sizes, [&](int off, int d) {
        std::vector<int> block(c.dev_sorted.begin() + off, c.dev_sorted.begin() + off + d);
        return candidates(block, c, m);
    });
}

std::vector<Replica> plan_of(const oracle_space::Space &sp, const Cluster &c, int64_t pi, const std::vector<int> &picks) {
    const auto &part = sp.parts[pi];
    std::vector<Replica> dep;
    for (size_t r = 0; r < part.sizes.size(); ++r) {
        Replica rep;
        rep.devs.assign(c.dev_sorted.begin() + part.offsets[r], c.dev_sorted.begin() + part.offsets[r] + part.sizes[r]);
        rep.tp = part.cands[r][picks[r]].first;
        rep.pp = part.cands[r][picks[r]].second;
        dep.push_back(rep);
    }
    return dep;
}

// best_strategies, deploysearch.cpp:153-229 — with the reference's
// comparator ComboResult::better_than (:47-52) verbatim in meaning.
struct Combo {
    int64_t obj = -1;
    int sum_pp = std::numeric_limits<int>::max();
    std::vector<int> tps, pps;
    std::vector<Replica> dep;
    bool better_than(const Combo &o) const {
        if (obj != o.obj) return obj > o.obj;
        if (sum_pp != o.sum_pp) return sum_pp < o.sum_pp;
        if (tps != o.tps) return tps > o.tps;
        return pps < o.pps;
    }
};

Combo best_of_partition(std::vector<int> sizes, const oracle_problem &p, const Model &m, const Cluster &c) {
    std::sort(sizes.begin(), sizes.end(), std::greater<int>());
    const int R = static_cast<int>(sizes.size());
    int total = std::accumulate(sizes.begin(), sizes.end(), 0);
    if (total > c.size()) fail(OSERVE_ERR_INVALID_ARGUMENT, "canonical_blocks: sizes exceed cluster device count");
    std::vector<std::vector<int>> blocks;
    std::vector<oracle_space::Cands> cands;
    int off = 0;
    uint64_t combos = 1;
    for (int s : sizes) {
        blocks.emplace_back(c.dev_sorted.begin() + off, c.dev_sorted.begin() + off + s);
        off += s;
        cands.push_back(candidates(blocks.back(), c, m));
        if (cands.back().empty()) return Combo{};
        combos *= cands.back().size();
    }
    Combo best;
    for (uint64_t idx = 0; idx < combos; ++idx) {
        Combo cur;
        uint64_t rest = idx;
        std::vector<int> pick(R);
        for (int r = R - 1; r >= 0; --r) {
            pick[r] = static_cast<int>(rest % cands[r].size());
            rest /= cands[r].size();
        }
        cur.sum_pp = 0;
        for (int r = 0; r < R; ++r) {
            auto [tp, pp] = cands[r][pick[r]];
            cur.dep.push_back(Replica{blocks[r], tp, pp});
            cur.tps.push_back(tp);
            cur.pps.push_back(pp);
            cur.sum_pp += pp;
        }
        cur.obj = evaluate(cur.dep, p, m, c);
        if (cur.better_than(best)) best = std::move(cur);
    }
    return best;
}

struct Ctx {
    Cluster c;
    Model m;
    explicit Ctx(const oracle_problem &p) : c(p.cluster), m(to_model(p.model)) {}
};

}  // namespace

extern "C" {

const char *oracle_last_error(void) { return g_err.c_str(); }
int oracle_is_reference(void) { return 0; }

int oracle_min_feasible_group(const oracle_problem *p, int *g_min) {
    return guarded([&] {
        Ctx x(*p);
        *g_min = g_min_of(x.c, x.m);
    });
}

int oracle_capacity_table(const oracle_problem *p, const oserve_deployment *dep, int64_t *n, int64_t *e,
                          double *latency) {
    return guarded([&] {
        Ctx x(*p);
        Cells t = cost_cells(to_dep(*dep), *p, x.m, x.c);
        for (size_t i = 0; i < t.n.size(); ++i) {
            if (n) n[i] = t.n[i];
            if (e) e[i] = t.e[i];
            if (latency) latency[i] = t.lat[i];
        }
    });
}

int oracle_normalize(int J, const int64_t *n_row, int strict, int64_t *M, int64_t *units, int *scaled) {
    return guarded([&] {
        bool sc = normalize_row(n_row, J, *M, units);
        if (sc && strict) fail(OSERVE_ERR_INVALID_ARGUMENT, "normalize: LCM exceeds 2^62");
        if (scaled) *scaled = sc ? 1 : 0;
    });
}

int oracle_solve_assignment(int R, int J, const int64_t *n, const int64_t *e, const int64_t *lambda,
                            const oserve_solve_options *opts, int64_t *x, int64_t *objective, int64_t *M,
                            int64_t *unit, int64_t *used, uint64_t *work) {
    return guarded([&] {
        std::vector<int64_t> Mv, uv;
        Solved s = solve_table(R, J, n, e, lambda, opts ? *opts : kDefaultOpts, &Mv, &uv);
        for (int k = 0; k < R; ++k) {
            int64_t u = 0;
            for (int j = 0; j < J; ++j) {
                if (x) x[k * J + j] = s.x[k * J + j];
                if (unit) unit[k * J + j] = uv[k * J + j];
                u += s.x[k * J + j] * uv[k * J + j];
            }
            if (M) M[k] = Mv[k];
            if (used) used[k] = u;
        }
        if (objective) *objective = s.obj;
        if (work) *work = s.work;
    });
}

// check_constraints, flowassign.cpp:521-554.
int oracle_check_constraints(int R, int J, const int64_t *x, const int64_t *n, const int64_t *e,
                             const int64_t *lambda) {
    return guarded([&] {
        for (int j = 0; j < J; ++j) {
            int64_t tot = 0;
            for (int k = 0; k < R; ++k) tot += x[k * J + j];
            if (tot > lambda[j]) fail(OSERVE_ERR_LOGIC, "C1 violated for type " + std::to_string(j));
        }
        for (int k = 0; k < R; ++k)
            for (int j = 0; j < J; ++j)
                if (x[k * J + j] > e[k * J + j]) fail(OSERVE_ERR_LOGIC, "C2 violated");
        std::vector<int64_t> units(J);
        for (int k = 0; k < R; ++k) {
            int64_t M;
            normalize_row(n + k * J, J, M, units.data());
            int64_t used = 0;
            for (int j = 0; j < J; ++j) {
                if (x[k * J + j] > 0 && units[j] == 0) fail(OSERVE_ERR_LOGIC, "C3 violated: zero-capacity type");
                used += x[k * J + j] * units[j];
            }
            if (used > M) fail(OSERVE_ERR_LOGIC, "C3 violated at replica " + std::to_string(k));
        }
    });
}

int oracle_evaluate_deployment(const oracle_problem *p, const oserve_deployment *dep, int64_t *objective) {
    return guarded([&] {
        Ctx x(*p);
        *objective = evaluate(to_dep(*dep), *p, x.m, x.c);
    });
}

int oracle_best_strategies(const oracle_problem *p, int R, const int *sizes, int, oserve_round_result *out) {
    return guarded([&] {
        Ctx x(*p);
        Combo b = best_of_partition(std::vector<int>(sizes, sizes + R), *p, x.m, x.c);
        std::memset(out, 0, sizeof(*out));
        out->objective = std::max<int64_t>(b.obj, 0);
        to_plan(b.dep, &out->plan);
        out->sum_pp = b.dep.empty() ? 0 : b.sum_pp;
    });
}

// exhaustive, deploysearch.cpp:436-466.
int oracle_exhaustive(const oracle_problem *p, int, oserve_round_result *out) {
    return guarded([&] {
        Ctx x(*p);
        if (x.c.size() > 16) fail(OSERVE_ERR_TOO_LARGE, "exhaustive enumeration guarded to 16 devices");
        const int g = g_min_of(x.c, x.m);
        int64_t best_obj = -1, parts = 0;
        Combo best;
        std::vector<int> cur;
        oracle_space::partitions_desc(x.c.size(), x.c.size(), g, {}, cur, [&](const std::vector<int> &sizes) {
            Combo cb = best_of_partition(sizes, *p, x.m, x.c);
            ++parts;
            if (cb.dep.empty()) return;
            int64_t o = std::max<int64_t>(cb.obj, 0);
            if (o > best_obj) {
                best_obj = o;
                best = cb;
            }
        });
        if (best_obj < 0) fail(OSERVE_ERR_MODEL_TOO_LARGE, "exhaustive: no feasible deployment");
        std::memset(out, 0, sizeof(*out));
        out->objective = best_obj;
        out->partitions = parts;
        to_plan(best.dep, &out->plan);
        out->sum_pp = best.sum_pp;
    });
}

int oracle_space_info(const oracle_problem *p, const oserve_space_desc *s, int64_t *partitions, uint64_t *plans) {
    return guarded([&] {
        Ctx x(*p);
        auto sp = space_of(*p, *s, x.c, x.m);
        *partitions = static_cast<int64_t>(sp.parts.size());
        *plans = sp.total;
    });
}

int oracle_space_plan(const oracle_problem *p, const oserve_space_desc *s, uint64_t rank, oserve_plan *plan,
                      int64_t *partition_index, uint64_t *local_rank) {
    return guarded([&] {
        Ctx x(*p);
        auto sp = space_of(*p, *s, x.c, x.m);
        if (rank >= sp.total) fail(OSERVE_ERR_INVALID_ARGUMENT, "rank out of range");
        int64_t pi;
        uint64_t local;
        std::vector<int> picks;
        oracle_space::unrank(sp, rank, pi, local, picks);
        to_plan(plan_of(sp, x.c, pi, picks), plan);
        if (partition_index) *partition_index = pi;
        if (local_rank) *local_rank = local;
    });
}

int oracle_evaluate_ranks(const oracle_problem *p, const oserve_space_desc *s, int64_t count, const uint64_t *ranks,
                          int64_t *objective, int32_t *sum_pp, uint64_t *work, int threads) {
    return guarded([&] {
        Ctx x(*p);
        auto sp = space_of(*p, *s, x.c, x.m);
        for (int64_t i = 0; i < count; ++i)
            if (ranks[i] >= sp.total) fail(OSERVE_ERR_INVALID_ARGUMENT, "rank out of range");
        std::mutex mu;
        int status = 0;
        std::string err;
#pragma omp parallel for schedule(dynamic, 4) num_threads(threads > 0 ? threads : 1)
        for (int64_t i = 0; i < count; ++i) {
            try {
                int64_t pi;
                uint64_t local;
                std::vector<int> picks;
                oracle_space::unrank(sp, ranks[i], pi, local, picks);
                auto dep = plan_of(sp, x.c, pi, picks);
                uint64_t w = 0;
                objective[i] = evaluate(dep, *p, x.m, x.c, &w);
                if (work) work[i] = w;
                if (sum_pp) {
                    int spp = 0;
                    for (const auto &r : dep) spp += r.pp;
                    sum_pp[i] = spp;
                }
            } catch (const std::exception &e) {
                std::lock_guard<std::mutex> g(mu);
                status = 1;
                err = e.what();
            }
        }
        if (status) fail(OSERVE_ERR_INVALID_ARGUMENT, err);
    });
}

int oracle_round(const oracle_problem *p, const oserve_space_desc *s, int threads, oserve_round_result *out) {
    return guarded([&] {
        Ctx x(*p);
        auto sp = space_of(*p, *s, x.c, x.m);
        const int nt = threads > 0 ? threads : 1;
        std::vector<oracle_space::Best> lbs(nt);
#pragma omp parallel num_threads(nt)
        {
            int tid = 0;
#ifdef _OPENMP
            tid = omp_get_thread_num();
#endif
            oracle_space::Best lb;
#pragma omp for schedule(dynamic, 4)
            for (int64_t g = 0; g < static_cast<int64_t>(sp.total); ++g) {
                int64_t pi;
                uint64_t local;
                std::vector<int> picks;
                oracle_space::unrank(sp, static_cast<uint64_t>(g), pi, local, picks);
                auto dep = plan_of(sp, x.c, pi, picks);
                int spp = 0;
                for (const auto &r : dep) spp += r.pp;
                lb.offer(evaluate(dep, *p, x.m, x.c), pi, spp, local);
            }
            lbs[tid] = lb;
        }
        oracle_space::Best best;
        for (const auto &lb : lbs)
            if (lb.valid) best.offer(lb.obj, lb.part, lb.sum_pp, lb.local);
        if (!best.valid) fail(OSERVE_ERR_MODEL_TOO_LARGE, "round: no feasible deployment");
        std::memset(out, 0, sizeof(*out));
        out->objective = best.obj;
        out->partitions = static_cast<int64_t>(sp.parts.size());
        out->plans = sp.total;
        out->partition_index = best.part;
        out->local_rank = best.local;
        out->sum_pp = best.sum_pp;
        int64_t pi;
        uint64_t local;
        std::vector<int> picks;
        oracle_space::unrank(sp, sp.prefix[best.part] + best.local, pi, local, picks);
        to_plan(plan_of(sp, x.c, pi, picks), &out->plan);
    });
}

// layout (switchplan.cpp:40-63, coalesce :17-29), greedy_plan (:65-131) and
// estimate_time (:133-140).
int oracle_switch_plan(const oserve_cluster_desc *cd, uint64_t P, const oserve_deployment *src,
                       const oserve_deployment *dst, int capacity, oserve_transfer *transfers, int *num_transfers,
                       double *est_seconds, uint64_t *max_link_bytes) {
    return guarded([&] {
        Cluster c(*cd);
        using Ranges = std::vector<std::pair<uint64_t, uint64_t>>;
        auto lay = [&](const oserve_deployment &d) {
            std::map<int, Ranges> held;
            for (const Replica &r : to_dep(d)) {
                std::vector<int> devs = r.devs;
                std::sort(devs.begin(), devs.end());
                const uint64_t pp = r.pp, tp = r.tp;
                for (uint64_t s = 0; s < pp; ++s) {
                    uint64_t b = P * s / pp, len = P * (s + 1) / pp - b;
                    for (uint64_t i = 0; i < tp; ++i)
                        held[devs[s * tp + i]].push_back({b + len * i / tp, b + len * (i + 1) / tp});
                }
            }
            for (auto &[dev, rs] : held) {
                std::sort(rs.begin(), rs.end());
                Ranges merged;
                for (auto &rg : rs) {
                    if (rg.first == rg.second) continue;
                    if (!merged.empty() && rg.first <= merged.back().second)
                        merged.back().second = std::max(merged.back().second, rg.second);
                    else
                        merged.push_back(rg);
                }
                rs = merged;
            }
            return held;
        };
        auto A = lay(*src), B = lay(*dst);
        auto covers = [](const Ranges &rs, uint64_t b, uint64_t e) {
            for (auto &r : rs)
                if (r.first <= b && e <= r.second) return true;
            return false;
        };
        std::set<uint64_t> cuts;
        for (auto *L : {&A, &B})
            for (auto &[dev, rs] : *L)
                for (auto &r : rs) {
                    cuts.insert(r.first);
                    cuts.insert(r.second);
                }
        std::vector<oserve_transfer> out;
        std::map<std::pair<int, int>, uint64_t> load;
        std::vector<uint64_t> bounds(cuts.begin(), cuts.end());
        for (size_t i = 0; i + 1 < bounds.size(); ++i) {
            uint64_t fb = bounds[i], fe = bounds[i + 1];
            std::vector<int> holders;
            for (auto &[dev, rs] : A)
                if (covers(rs, fb, fe)) holders.push_back(dev);
            for (auto &[t, rs] : B) {
                if (!covers(rs, fb, fe)) continue;
                auto h = A.find(t);
                if (h != A.end() && covers(h->second, fb, fe)) continue;
                if (holders.empty()) fail(OSERVE_ERR_UNSOURCED_FRAGMENT, "fragment has no source holder");
                // argmin over holders of (!intra, load, id)
                int best = -1;
                bool bi = false;
                uint64_t bl = 0;
                for (int s : holders) {
                    bool intra = c.same_machine(s, t);
                    auto it = load.find({s, t});
                    uint64_t l = it == load.end() ? 0 : it->second;
                    if (best < 0 || (intra && !bi) || (intra == bi && (l < bl || (l == bl && s < best)))) {
                        best = s;
                        bi = intra;
                        bl = l;
                    }
                }
                load[{best, t}] += fe - fb;
                out.push_back({fb, fe, best, t});
            }
        }
        double worst = 0.0;
        uint64_t mx = 0;
        for (auto &[link, bytes] : load) {
            double bw = c.same_machine(link.first, link.second) ? c.intra : c.inter;
            worst = std::max(worst, static_cast<double>(bytes) / bw);
            mx = std::max(mx, bytes);
        }
        if (num_transfers) *num_transfers = static_cast<int>(out.size());
        if (transfers)
            for (int i = 0; i < std::min<int>(capacity, static_cast<int>(out.size())); ++i) transfers[i] = out[i];
        if (est_seconds) *est_seconds = worst;
        if (max_link_bytes) *max_link_bytes = mx;
    });
}

int oracle_search(const oracle_problem *, const oserve_search_options *, oserve_search_result *,
                  oserve_search_log_row *, int) {
    g_err = "search: reference-only (use the _ref oracle)";
    return OSERVE_ERR_UNSUPPORTED;
}

int oracle_adaptive_timeline(const oracle_problem *, int, const int64_t *, uint64_t, int, double, int, int64_t *,
                             oserve_plan *, int64_t *, double *, int *, int *) {
    g_err = "adaptive timeline: reference-only (use the _ref oracle)";
    return OSERVE_ERR_UNSUPPORTED;
}

int oracle_fit_types(int64_t, const uint32_t *, const uint32_t *, int, uint64_t, double *, double *) {
    g_err = "fit_types: reference-only (use the _ref oracle)";
    return OSERVE_ERR_UNSUPPORTED;
}

// Holt forecaster (workload.cpp:204-222) through forecast_series
// (orchestrate.cpp:75-92): span 0 uses its own counts, later spans predict
// from the trailing window, llround, clamped at 0.
int oracle_holt_forecast(int J, int T, const int64_t *counts, int window, int64_t *lambda_out) {
    return guarded([&] {
        const double alpha = 0.45, beta = 0.25;
        for (int t = 0; t < T; ++t) {
            for (int j = 0; j < J; ++j) {
                if (t == 0) {
                    lambda_out[j] = counts[j];
                    continue;
                }
                int start = std::max(0, t - window);
                double level = static_cast<double>(counts[start * J + j]), trend = 0.0;
                for (int s = start + 1; s < t; ++s) {
                    double prev = level;
                    level = alpha * static_cast<double>(counts[s * J + j]) + (1.0 - alpha) * (level + trend);
                    trend = beta * (level - prev) + (1.0 - beta) * trend;
                }
                double v = std::max(0.0, std::max(0.0, level + trend));
                lambda_out[t * J + j] = std::max<int64_t>(0, std::llround(v));
            }
        }
    });
}

// kv_plan and the JSON schema checks are reference-only (the restatement
// has no counterpart; the GPU product is checked against _ref directly).
int oracle_kv_plan(const oserve_cluster_desc *, int, const oserve_inflight *, int64_t, const oserve_deployment *,
                   const oserve_deployment *, double, int, const oserve_transfer *, int64_t *, int *,
                   oserve_kv_transfer *, int *, uint64_t *) {
    g_err = "kv_plan: reference-only (use the _ref oracle)";
    return OSERVE_ERR_UNSUPPORTED;
}
int oracle_adaptive_timeline_json(const oracle_problem *, int, const int64_t *, uint64_t, int, double,
                                  const char *) {
    g_err = "adaptive_timeline_json: reference-only";
    return OSERVE_ERR_UNSUPPORTED;
}
int oracle_timeline_resave(const char *, const char *, int *) {
    g_err = "timeline_resave: reference-only";
    return OSERVE_ERR_UNSUPPORTED;
}
int oracle_deployment_resave(const char *, const char *, int *) {
    g_err = "deployment_resave: reference-only";
    return OSERVE_ERR_UNSUPPORTED;
}

int oracle_max_flow(int, int, const oserve_flow_edge *, int, int, int64_t *, int64_t *) {
    g_err = "max_flow: reference-only";
    return OSERVE_ERR_UNSUPPORTED;
}
int oracle_flow_assign(int, int, const int64_t *, const int64_t *, const int64_t *, const oserve_solve_options *,
                       int64_t *, int64_t *, int64_t *, int64_t *) {
    g_err = "flow_assign: reference-only";
    return OSERVE_ERR_UNSUPPORTED;
}
int oracle_solve_fractional(int, int, const int64_t *, const int64_t *, const int64_t *, double *, double *) {
    g_err = "solve_fractional: reference-only";
    return OSERVE_ERR_UNSUPPORTED;
}
int oracle_to_dot(int, int, const int64_t *, const int64_t *, const int64_t *, int, char *, int, int *) {
    g_err = "to_dot: reference-only";
    return OSERVE_ERR_UNSUPPORTED;
}

}  // extern "C"
