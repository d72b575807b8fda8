// oserve_host.cpp — host runtime of the B200 scheduling round (native C++).
//
// Implements the C-ABI of include/oserve_gpu.h: context (cluster/model/profile
// copies, CUDA stream), the plan-space enumerator (partitions, candidate
// lists, runs, prefix table), the shape registry feeding the cost kernel, key
// packing/decoding, and the launch sequences of K0/K1/K4/K2.
//
// Host-side restatements (control plane, no per-plan compute):
//   min_feasible_group   deploysearch.cpp:77-87
//   partitions_desc      deploysearch.cpp:421-432
//   canonical_blocks     deploysearch.cpp:89-103
//   strategy_candidates  deploysearch.cpp:105-118 (+ validate_replica
//                        core.cpp:105-127, memory_feasible costmodel.cpp:48-62)
//   tp_speedup           costmodel.cpp:22-24 (host libm pow/log2, as the reference)
// Every per-plan quantity (cost cells, normalisation, assignment, objective,
// argmin, switching cost) is computed by the kernels.  There is no CPU
// fallback: without a CUDA device every entry point returns
// OSERVE_ERR_NO_DEVICE.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <functional>
#include <limits>
#include <map>
#include <memory>
#include <numeric>
#include <random>
#include <sstream>
#include <set>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "../../include/oserve_gpu.h"
#include "oserve_internal.h"

using namespace oserve_gpu;

namespace {

struct Fail : std::runtime_error {
    int code;
    Fail(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void fail(int code, const std::string &m) { throw Fail(code, m); }

void cuda_ok(cudaError_t e, const char *what) {
    if (e != cudaSuccess) fail(OSERVE_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
void cuda_ok(int e, const char *what) { cuda_ok(static_cast<cudaError_t>(e), what); }

// NCCL, resolved at run time: a process that already holds a libnccl.so.2
// (e.g. the one PyTorch ships) shares it; otherwise the system library loads.
// Only the multi-GPU entry points need it.
struct Nccl {
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t *, int, const int *) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
    bool ok() const { return why.empty(); }
};

const Nccl &nccl() {
    static const Nccl n = [] {
        Nccl r;
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            r.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
            return r;
        }
        auto sym = [&](auto &fp, const char *name) {
            fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
            if (!fp && r.why.empty()) r.why = std::string("NCCL symbol missing: ") + name;
        };
        sym(r.GetUniqueId, "ncclGetUniqueId");
        sym(r.CommInitRank, "ncclCommInitRank");
        sym(r.CommInitAll, "ncclCommInitAll");
        sym(r.CommDestroy, "ncclCommDestroy");
        sym(r.AllReduce, "ncclAllReduce");
        sym(r.AllGather, "ncclAllGather");
        sym(r.GroupStart, "ncclGroupStart");
        sym(r.GroupEnd, "ncclGroupEnd");
        sym(r.GetErrorString, "ncclGetErrorString");
        return r;
    }();
    return n;
}

const Nccl &nccl_or_fail() {
    const Nccl &n = nccl();
    if (!n.ok()) fail(OSERVE_ERR_NCCL, n.why);
    return n;
}

void nccl_ok(ncclResult_t r, const char *what) {
    if (r != ncclSuccess) fail(OSERVE_ERR_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

// Byte counters of the host<->device copies issued by the current call
// (bound to the calling context by guarded()).
thread_local uint64_t *t_h2d = nullptr;
thread_local uint64_t *t_d2h = nullptr;
inline void count_h2d(size_t b) {
    if (t_h2d) *t_h2d += b;
}
inline void count_d2h(size_t b) {
    if (t_d2h) *t_d2h += b;
}
cudaError_t h2d(void *dst, const void *src, size_t bytes, cudaStream_t s) {
    count_h2d(bytes);
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
}
cudaError_t d2h(void *dst, const void *src, size_t bytes, cudaStream_t s) {
    count_d2h(bytes);
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s);
}

// Growable device buffer.
struct DBuf {
    void *p = nullptr;
    size_t cap = 0;
    DBuf() = default;
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
    ~DBuf() {
        if (p) cudaFree(p);
    }
    void *get(size_t bytes) {
        if (bytes == 0) bytes = 16;
        if (bytes > cap) {
            if (p) cudaFree(p);
            p = nullptr;
            cuda_ok(cudaMalloc(&p, bytes), "cudaMalloc");
            cap = bytes;
        }
        return p;
    }
    template <class T>
    T *upload(const T *src, size_t n, cudaStream_t s) {
        T *d = static_cast<T *>(get(n * sizeof(T)));
        if (n) cuda_ok(h2d(d, src, n * sizeof(T), s), "H2D");
        return d;
    }
    template <class T>
    T *upload(const std::vector<T> &v, cudaStream_t s) {
        T *d = static_cast<T *>(get(v.size() * sizeof(T)));
        if (!v.empty()) cuda_ok(h2d(d, v.data(), v.size() * sizeof(T), s), "H2D");
        return d;
    }
};

template <class T>
void download(std::vector<T> &v, const void *d, size_t n, cudaStream_t s) {
    v.resize(n);
    if (n) cuda_ok(d2h(v.data(), d, n * sizeof(T), s), "D2H");
}

int bits_for(uint64_t x) {
    int b = 1;
    while (b < 64 && (x >> b) != 0) ++b;
    return b;
}

uint64_t binom(int n, int k) {
    if (k < 0 || k > n) return 0;
    unsigned __int128 r = 1;
    for (int i = 1; i <= k; ++i) {
        r = r * static_cast<unsigned>(n - k + i) / static_cast<unsigned>(i);
        if (r > (static_cast<unsigned __int128>(1) << 62)) fail(OSERVE_ERR_TOO_LARGE, "plan count exceeds 2^62");
    }
    return static_cast<uint64_t>(r);
}

using Cand = std::pair<int, int>;  // (tp, pp), tp descending

struct Run {
    int start, len, q;
    uint64_t count;
};

struct Partition {
    std::vector<int> sizes, offsets, cand_list;  // cand_list: list id per replica
    std::vector<Run> runs;
    uint64_t count = 0;
};

struct Space {
    bool valid = false;
    int mode = -1;
    std::vector<int> sizes_key;
    int max_devices = 0;
    bool explicit_partition = false;
    std::vector<int> explicit_sizes;
    std::vector<Partition> parts;
    std::vector<uint64_t> prefix;
    uint64_t total = 0, max_count = 0;
    int rmax = 0;
    std::vector<std::vector<Cand>> lists;      // candidate lists
    std::vector<std::vector<int>> list_shapes; // shape id per candidate
    // device copies
    DBuf d_tables, d_exact;  // every table in one allocation (one H2D copy), exact flags
    SpaceTables view{};
    std::vector<uint8_t> exact;  // per partition, for the current workload
    bool any_exact = false;
    // R-buckets: plans with R <= 32 run one replica per lane, the rest two or
    // four (K1 instantiations); each bucket is a list of rank ranges.
    struct Bucket {
        int rmax = 0;
        uint64_t total = 0;
        std::vector<uint64_t> start, prefix;
        const uint64_t *d_start = nullptr, *d_prefix = nullptr;  // inside Space::d_tables
    };
    Bucket buckets[2];
    bool use_buckets = false;
};

}  // namespace

// Per-task arrays of the frontier-parallel exact path (double-buffered for
// the splitting rounds; kept in the context so repeated rounds reuse them).
struct TaskBufs {
    DBuf plan, td, path, g, lb, lbr, m, inc, vis, nodes, cap, done, nch, nz, al, am;
    void bind(ExactTasks &e, uint64_t n) {
        e.aL = static_cast<int32_t *>(al.get(sizeof(int32_t) * n));
        e.amask = static_cast<uint32_t *>(am.get(sizeof(uint32_t) * n));
        e.plan = static_cast<uint32_t *>(plan.get(sizeof(uint32_t) * n));
        e.tdepth = static_cast<uint8_t *>(td.get(n));
        e.path = static_cast<int32_t *>(path.get(sizeof(int32_t) * n * kTaskDepthMax));
        e.g = static_cast<int64_t *>(g.get(sizeof(int64_t) * n));
        e.lb = static_cast<int64_t *>(lb.get(sizeof(int64_t) * n));
        e.lbran = static_cast<int64_t *>(lbr.get(sizeof(int64_t) * n));
        e.m = static_cast<int64_t *>(m.get(sizeof(int64_t) * n));
        e.inc = static_cast<int64_t *>(inc.get(sizeof(int64_t) * n));
        e.vis = static_cast<uint8_t *>(vis.get(n));
        e.nodes = static_cast<int64_t *>(nodes.get(sizeof(int64_t) * n));
        e.capped = static_cast<uint8_t *>(cap.get(n));
        e.done = static_cast<uint8_t *>(done.get(n));
        e.nchild = static_cast<uint32_t *>(nch.get(sizeof(uint32_t) * (n + 1)));  // + the scan's trailing 0
        e.nzero = static_cast<uint8_t *>(nz.get(n));
    }
};

// Raw [count][R][J] rows staged as the shape tables of one call (K0b only).
struct RawRows {
    DBuf dn, de, dM, du, dc, dord, dol, dpp, dsc, dlat, dinv, drank, dpmask;
    ShapeTables t{};
};

struct ExactScratch {
    DBuf depth, nt, off, top, opt, ist, state, bx, run, ranks, newoff, fetch, topn, ubn, lbn, anycap, scan, grow, psum, pmax,
        work;
    TaskBufs bufs[2];
};

struct oserve_gpu_ctx {
    int device = 0;
    int sm_count = 148;
    cudaStream_t own = nullptr, stream = nullptr;
    std::string err;
    uint64_t launches = 0;
    uint64_t h2d_bytes = 0, d2h_bytes = 0;
    // cluster
    std::vector<int> dev_sorted;
    std::map<int, int> machine_of;
    std::map<int, int> slot_of;
    std::vector<uint64_t> machine_mem;
    double intra = 0, inter = 0;
    oserve_model_desc model{};
    oserve_profile profile{};
    oserve_solve_options opts{400, 20, 8000000};
    // workload
    int J = 0;
    std::vector<double> cin, cout;
    std::vector<int64_t> lambda;
    double span = 60.0;
    bool have_workload = false;
    // shapes
    std::map<std::tuple<int, int, uint64_t>, int> shape_id;
    std::vector<ShapeParam> shapes;
    int tables_shapes = -1;  // shapes computed in device tables
    bool tables_dirty = true;
    uint64_t tables_ver = 0;  // bumped whenever K0 recomputes the tables
    // host copies of the shape tables (plan_detail), valid for host_tables_ver
    std::vector<int64_t> h_n, h_e, h_M, h_unit;
    std::vector<double> h_lat;
    uint64_t host_tables_ver = ~0ull;
    DBuf d_param, d_n, d_e, d_lat, d_M, d_unit, d_inv, d_rank, d_pmask, d_cap, d_order, d_olen, d_pp, d_scaled, d_cin,
        d_cout;
    ShapeTables tables{};
    // space
    Space space;
    KeyLayout key{};
    int rank = 0, world = 1;
    uint64_t chunk = OSERVE_SHARD_CHUNK;
    // scratch
    DBuf d_topk, d_topk_meta, d_topk_tmp, d_collect, d_collect_n, d_bad;
    void *cub_temp = nullptr;
    size_t cub_temp_bytes = 0;
    DBuf d_key, d_obj, d_spp, d_x, d_used, d_aborted, d_aborted_n, d_ranks, d_listR, d_listOff, d_listShapes,
        d_listLam, d_sw[12];
    ExactScratch exact;
    // per-call device scratch of the batch entry points, kept across calls
    // (a cudaMalloc / cudaFree pair per buffer per call otherwise)
    RawRows raw;
    DBuf sc_kv[16], sc_fa[10], sc_mf[20], sc_lp[7], sc_sw[14], sc_aux[8];
    // K1 dynamic-chunk counters of this context (oserve_internal.h WorkRing)
    DBuf d_ring;
    WorkRing ring{nullptr, 0, 0};
    // multi-GPU: this context is local shard 0; `subs` are contexts on the
    // other local devices (oserve_gpu_create_multi).  comms[i] is local shard
    // i's NCCL communicator (empty: no communicator); local shard i has global
    // rank g_rank0 + i of g_world.
    std::vector<oserve_gpu_ctx *> subs;
    std::vector<ncclComm_t> comms;
    int g_rank0 = 0, g_world = 1;
    uint64_t space_ver = 0, work_ver = 0;             // bumped by build_space / workload or shape changes
    uint64_t synced_space = ~0ull, synced_work = ~0ull;  // versions a sub last mirrored from the lead
    DBuf d_mkey, d_mtopk, d_mbest, d_mall, d_mtmp;    // per-shard collective scratch

    oserve_gpu_ctx() = default;
    oserve_gpu_ctx(const oserve_gpu_ctx &) = delete;
    oserve_gpu_ctx &operator=(const oserve_gpu_ctx &) = delete;
    ~oserve_gpu_ctx();

    int D() const { return static_cast<int>(dev_sorted.size()); }
    int machine(int d) const {
        auto it = machine_of.find(d);
        return it == machine_of.end() ? -1 : it->second;
    }
    uint64_t device_mem(int d) const {
        int m = machine(d);
        return m < 0 ? 0 : machine_mem[m];
    }
};

oserve_gpu_ctx::~oserve_gpu_ctx() {
    for (oserve_gpu_ctx *s : subs) delete s;  // each on its own device
    subs.clear();
    cudaSetDevice(device);
    for (ncclComm_t cm : comms)
        if (cm && nccl().ok()) nccl().CommDestroy(cm);
    if (own) {
        cudaStreamSynchronize(own);
        cudaStreamDestroy(own);
    }
    if (cub_temp) cudaFree(cub_temp);
    // the DBuf members are freed next, with this context's device current
}

namespace {

// ----------------------------------------------------------- placement ---
bool placement_ok(const oserve_gpu_ctx &c, const std::vector<int> &devs, int tp, int pp) {
    if (tp < 1 || pp < 1 || devs.empty() || tp * pp != static_cast<int>(devs.size())) return false;
    std::vector<int> s = devs;
    std::sort(s.begin(), s.end());
    if (std::adjacent_find(s.begin(), s.end()) != s.end()) return false;
    for (int d : s)
        if (c.machine(d) < 0) return false;
    for (int st = 0; st < pp; ++st)
        for (int i = 1; i < tp; ++i) {
            int m0 = c.machine(s[st * tp]);
            if (m0 < 0 || m0 != c.machine(s[st * tp + i])) return false;
        }
    return true;
}

bool mem_feasible(const oserve_gpu_ctx &c, const std::vector<int> &devs, int tp, int pp, uint64_t *total_out) {
    if (devs.empty()) return false;
    uint64_t total = 0, mn = std::numeric_limits<uint64_t>::max();
    for (int d : devs) {
        uint64_t m = c.device_mem(d);
        if (m == 0) return false;
        total += m;
        mn = std::min(mn, m);
    }
    if (total_out) *total_out = total;
    if (total < c.model.min_mem_bytes) return false;
    uint64_t shards = static_cast<uint64_t>(tp) * static_cast<uint64_t>(pp);
    return (c.model.param_bytes + shards - 1) / shards <= mn;
}

int shape_for(oserve_gpu_ctx &c, int tp, int pp, uint64_t total_mem) {
    uint64_t budget = total_mem > c.model.param_bytes ? total_mem - c.model.param_bytes : 0;
    auto key = std::make_tuple(tp, pp, budget);
    auto it = c.shape_id.find(key);
    if (it != c.shape_id.end()) return it->second;
    ShapeParam sp;
    sp.tp = tp;
    sp.pp = pp;
    sp.kv_budget = budget;
    sp.speedup = tp * std::pow(c.profile.tp_efficiency, std::log2(static_cast<double>(tp)));
    int id = static_cast<int>(c.shapes.size());
    if (id >= 65535) fail(OSERVE_ERR_UNSUPPORTED, "more than 65535 replica shapes");
    c.shapes.push_back(sp);
    c.shape_id.emplace(key, id);
    c.tables_dirty = true;
    ++c.work_ver;
    return id;
}

int g_min_of(const oserve_gpu_ctx &c) {
    uint64_t mn = std::numeric_limits<uint64_t>::max();
    for (uint64_t v : c.machine_mem) mn = std::min(mn, v);
    for (int g = 1; g <= c.D(); ++g) {
        bool total_ok = static_cast<uint64_t>(g) * mn >= c.model.min_mem_bytes;
        bool shard_ok = (c.model.param_bytes + g - 1) / g <= mn;
        if (total_ok && shard_ok) return g;
    }
    fail(OSERVE_ERR_MODEL_TOO_LARGE, "model does not fit on " + std::to_string(c.D()) + " devices");
}

// ------------------------------------------------------- shape tables ---
void ensure_tables(oserve_gpu_ctx &c) {
    if (!c.have_workload) fail(OSERVE_ERR_INVALID_ARGUMENT, "no workload set (oserve_gpu_set_workload)");
    if (!c.tables_dirty && c.tables_shapes == static_cast<int>(c.shapes.size())) return;
    const int S = static_cast<int>(c.shapes.size()), J = c.J;
    cudaStream_t s = c.stream;
    ShapeTables t{};
    t.num_shapes = S;
    t.J = J;
    t.param = c.d_param.upload(c.shapes, s);
    t.n = static_cast<int64_t *>(c.d_n.get(sizeof(int64_t) * S * J));
    t.e = static_cast<int64_t *>(c.d_e.get(sizeof(int64_t) * S * J));
    t.latency = static_cast<double *>(c.d_lat.get(sizeof(double) * S * J));
    t.M = static_cast<int64_t *>(c.d_M.get(sizeof(int64_t) * S));
    t.unit = static_cast<int64_t *>(c.d_unit.get(sizeof(int64_t) * S * J));
    t.inv_unit = static_cast<double *>(c.d_inv.get(sizeof(double) * S * J));
    t.cap = static_cast<int32_t *>(c.d_cap.get(sizeof(int32_t) * S * J));
    t.order = static_cast<uint8_t *>(c.d_order.get(S * kMaxJ));
    t.rank = static_cast<uint8_t *>(c.d_rank.get(S * kMaxJ));
    t.pmask = static_cast<uint16_t *>(c.d_pmask.get(sizeof(uint16_t) * S * kMaxJ));
    t.olen = static_cast<uint8_t *>(c.d_olen.get(S));
    t.scaled = static_cast<uint8_t *>(c.d_scaled.get(S));
    std::vector<uint8_t> pps(S);
    for (int i = 0; i < S; ++i) pps[i] = static_cast<uint8_t>(std::min(c.shapes[i].pp, 255));
    t.pp = c.d_pp.upload(pps, s);
    const double *cin = c.d_cin.upload(c.cin, s);
    const double *cout = c.d_cout.upload(c.cout, s);
    const auto &p = c.profile;
    cuda_ok(launch_cost_tables(t, cin, cout, c.model.num_layers, c.model.bytes_per_token_kv, p.prefill_coeff,
                               p.decode_coeff, p.pp_comm_cost, p.mem_bw_penalty, c.span, s),
            "cost kernel");
    cuda_ok(launch_normalize_rows(t, s), "normalize kernel");
    c.launches += S ? 2 : 0;
    c.tables = t;
    c.tables_shapes = S;
    c.tables_dirty = false;
    ++c.tables_ver;
}

SolveParams solve_params(const oserve_gpu_ctx &c) {
    SolveParams p{};
    p.J = c.J;
    for (int j = 0; j < c.J; ++j) p.lambda[j] = c.lambda[j];
    p.exact_demand_limit = c.opts.exact_demand_limit;
    p.exact_cell_limit = c.opts.exact_cell_limit;
    p.node_budget = c.opts.node_budget;
    return p;
}

bool use_exact(const oserve_gpu_ctx &c, int R) {
    int64_t tot = 0;
    for (int64_t v : c.lambda) tot += v;
    return tot <= c.opts.exact_demand_limit && static_cast<int64_t>(R) * c.J <= c.opts.exact_cell_limit;
}

// --------------------------------------------------------------- space ---
std::vector<Cand> candidates(oserve_gpu_ctx &c, int off, int d, std::vector<int> &shape_ids) {
    std::vector<int> block(c.dev_sorted.begin() + off, c.dev_sorted.begin() + off + d);
    std::vector<Cand> out;
    shape_ids.clear();
    for (int tp = d; tp >= 1; --tp) {
        if (d % tp) continue;
        uint64_t total = 0;
        if (placement_ok(c, block, tp, d / tp) && mem_feasible(c, block, tp, d / tp, &total)) {
            out.emplace_back(tp, d / tp);
            shape_ids.push_back(shape_for(c, tp, d / tp, total));
        }
    }
    if (out.size() > static_cast<size_t>(kMaxCand)) fail(OSERVE_ERR_UNSUPPORTED, "more than 8 strategy candidates");
    return out;
}

void upload_space(oserve_gpu_ctx &c, Space &sp);

void build_space(oserve_gpu_ctx &c, Space &sp, int mode, const std::vector<int> &allowed_sizes,
                 const std::vector<std::vector<int>> *explicit_parts) {
    const int D = c.D();
    sp.parts.clear();
    sp.prefix.clear();
    sp.lists.clear();
    sp.list_shapes.clear();
    sp.total = 0;
    sp.max_count = 0;
    sp.rmax = 0;
    std::map<std::pair<int, int>, int> list_of;  // (offset, size) -> list id
    std::map<std::vector<int>, int> list_dedup;  // shape-id list -> list id
    auto handle = [&](const std::vector<int> &sizes) {
        Partition part;
        part.sizes = sizes;
        int off = 0;
        bool feasible = true;
        for (int s : sizes) {
            part.offsets.push_back(off);
            auto key = std::make_pair(off, s);
            auto it = list_of.find(key);
            int lid;
            if (it == list_of.end()) {
                std::vector<int> ids;
                std::vector<Cand> cands = candidates(c, off, s, ids);
                auto dd = list_dedup.find(ids);
                if (dd == list_dedup.end()) {
                    lid = static_cast<int>(sp.lists.size());
                    sp.lists.push_back(cands);
                    sp.list_shapes.push_back(ids);
                    list_dedup.emplace(ids, lid);
                } else {
                    lid = dd->second;
                }
                list_of.emplace(key, lid);
            } else {
                lid = it->second;
            }
            part.cand_list.push_back(lid);
            if (sp.lists[lid].empty()) feasible = false;
            off += s;
        }
        if (feasible) {
            const int R = static_cast<int>(sizes.size());
            for (int r = 0; r < R;) {
                int e = r + 1;
                if (mode == OSERVE_SPACE_CANONICAL)
                    while (e < R && sizes[e] == sizes[r] && part.cand_list[e] == part.cand_list[r]) ++e;
                Run run{r, e - r, static_cast<int>(sp.lists[part.cand_list[r]].size()), 0};
                run.count = binom(run.len + run.q - 1, run.q - 1);
                part.runs.push_back(run);
                r = e;
            }
            unsigned __int128 cnt = 1;
            for (const auto &run : part.runs) {
                cnt *= run.count;
                if (cnt > (static_cast<unsigned __int128>(1) << 62))
                    fail(OSERVE_ERR_TOO_LARGE, "plans per partition exceed 2^62");
            }
            part.count = static_cast<uint64_t>(cnt);
            sp.rmax = std::max(sp.rmax, R);
        }
        sp.prefix.push_back(sp.total);
        sp.total += part.count;
        if (sp.total > (uint64_t{1} << 62)) fail(OSERVE_ERR_TOO_LARGE, "plan space exceeds 2^62 plans");
        sp.max_count = std::max(sp.max_count, part.count);
        sp.parts.push_back(std::move(part));
    };
    if (explicit_parts) {
        for (const auto &s : *explicit_parts) handle(s);
    } else {
        const int g = g_min_of(c);
        std::vector<char> allowed;
        if (!allowed_sizes.empty()) {
            allowed.assign(D + 1, 0);
            for (int s : allowed_sizes)
                if (s >= 1 && s <= D) allowed[s] = 1;
        }
        std::vector<int> cur;
        std::function<void(int, int)> rec = [&](int remaining, int max_part) {
            if (remaining == 0) {
                handle(cur);
                return;
            }
            for (int p = std::min(remaining, max_part); p >= g; --p) {
                if (!allowed.empty() && !allowed[p]) continue;
                cur.push_back(p);
                rec(remaining - p, p);
                cur.pop_back();
            }
        };
        rec(D, D);
    }
    if (sp.rmax > OSERVE_MAX_REPLICAS) fail(OSERVE_ERR_UNSUPPORTED, "more than 128 replicas per plan");
    sp.prefix.push_back(sp.total);
    ++c.space_ver;
    upload_space(c, sp);
}

// Several host arrays staged into one device allocation with one H2D copy
// (16-byte aligned offsets): per-partition callers (search -> best_strategies)
// would otherwise pay one copy per table.
struct Packer {
    std::vector<unsigned char> h;
    template <class T>
    size_t add(const std::vector<T> &v) {
        const size_t off = (h.size() + 15) & ~size_t(15);
        h.resize(off + v.size() * sizeof(T));
        if (!v.empty()) std::memcpy(h.data() + off, v.data(), v.size() * sizeof(T));
        return off;
    }
    const unsigned char *upload(DBuf &d, cudaStream_t s) { return d.upload(h.data(), h.size(), s); }
};

// Host fields of a space (the enumeration), without its device copies.
void copy_space_host(const Space &a, Space &b) {
    b.mode = a.mode;
    b.sizes_key = a.sizes_key;
    b.max_devices = a.max_devices;
    b.explicit_partition = a.explicit_partition;
    b.explicit_sizes = a.explicit_sizes;
    b.parts = a.parts;
    b.prefix = a.prefix;
    b.total = a.total;
    b.max_count = a.max_count;
    b.rmax = a.rmax;
    b.lists = a.lists;
    b.list_shapes = a.list_shapes;
}

// Flatten the enumerated space into the device tables of context c (its
// device and stream); also the R-buckets.
void upload_space(oserve_gpu_ctx &c, Space &sp) {
    const size_t P = sp.parts.size();
    std::vector<int32_t> R(P), rep_off(P), run_off(P), nruns(P), rep_list, run_start, run_len, run_q;
    std::vector<uint64_t> run_count, run_weight;
    for (size_t i = 0; i < P; ++i) {
        const auto &part = sp.parts[i];
        R[i] = static_cast<int32_t>(part.sizes.size());
        rep_off[i] = static_cast<int32_t>(rep_list.size());
        run_off[i] = static_cast<int32_t>(run_start.size());
        nruns[i] = static_cast<int32_t>(part.runs.size());
        for (int l : part.cand_list) rep_list.push_back(l);
        uint64_t w = 1;
        std::vector<uint64_t> ws(part.runs.size());
        for (int r = static_cast<int>(part.runs.size()) - 1; r >= 0; --r) {
            ws[r] = w;
            w *= part.runs[r].count;
        }
        for (size_t r = 0; r < part.runs.size(); ++r) {
            run_start.push_back(part.runs[r].start);
            run_len.push_back(part.runs[r].len);
            run_q.push_back(part.runs[r].q);
            run_count.push_back(part.runs[r].count);
            run_weight.push_back(ws[r]);
        }
    }
    std::vector<uint8_t> cl_n(sp.lists.size());
    std::vector<uint16_t> cl_shape(sp.lists.size() * kMaxCand, 0);
    for (size_t l = 0; l < sp.lists.size(); ++l) {
        cl_n[l] = static_cast<uint8_t>(sp.lists[l].size());
        for (size_t q = 0; q < sp.list_shapes[l].size(); ++q)
            cl_shape[l * kMaxCand + q] = static_cast<uint16_t>(sp.list_shapes[l][q]);
    }
    cudaStream_t s = c.stream;
    // R-buckets
    for (auto &b : sp.buckets) {
        b.rmax = 0;
        b.total = 0;
        b.start.clear();
        b.prefix.clear();
    }
    for (size_t i = 0; i < P; ++i) {
        const auto &part = sp.parts[i];
        if (part.count == 0) continue;
        const int R = static_cast<int>(part.sizes.size());
        auto &b = sp.buckets[R <= 32 ? 0 : 1];
        b.rmax = std::max(b.rmax, R);
        if (!b.start.empty() && b.start.back() + (b.total - b.prefix.back()) == sp.prefix[i]) {
            // contiguous with the previous range of this bucket: extend it
        } else {
            b.start.push_back(sp.prefix[i]);
            b.prefix.push_back(b.total);
        }
        b.total += part.count;
    }
    sp.use_buckets = sp.buckets[0].total > 0 && sp.buckets[1].total > 0;
    Packer pk;
    size_t o_bs[2] = {0, 0}, o_bp[2] = {0, 0};
    if (sp.use_buckets)
        for (int q = 0; q < 2; ++q) {
            o_bs[q] = pk.add(sp.buckets[q].start);
            o_bp[q] = pk.add(sp.buckets[q].prefix);
        }
    const size_t o_prefix = pk.add(sp.prefix), o_R = pk.add(R), o_rep_off = pk.add(rep_off),
                 o_run_off = pk.add(run_off), o_nruns = pk.add(nruns), o_rep_list = pk.add(rep_list),
                 o_run_start = pk.add(run_start), o_run_len = pk.add(run_len), o_run_q = pk.add(run_q),
                 o_run_count = pk.add(run_count), o_run_weight = pk.add(run_weight), o_cl_n = pk.add(cl_n),
                 o_cl_shape = pk.add(cl_shape);
    const unsigned char *base = pk.upload(sp.d_tables, s);
    auto at = [&](size_t o) { return static_cast<const void *>(base + o); };
    if (sp.use_buckets)
        for (int q = 0; q < 2; ++q) {
            sp.buckets[q].d_start = static_cast<const uint64_t *>(at(o_bs[q]));
            sp.buckets[q].d_prefix = static_cast<const uint64_t *>(at(o_bp[q]));
        }
    SpaceTables v{};
    v.num_parts = static_cast<int64_t>(P);
    v.prefix = static_cast<const uint64_t *>(at(o_prefix));
    v.R = static_cast<const int32_t *>(at(o_R));
    v.rep_off = static_cast<const int32_t *>(at(o_rep_off));
    v.run_off = static_cast<const int32_t *>(at(o_run_off));
    v.nruns = static_cast<const int32_t *>(at(o_nruns));
    v.rep_list = static_cast<const int32_t *>(at(o_rep_list));
    v.run_start = static_cast<const int32_t *>(at(o_run_start));
    v.run_len = static_cast<const int32_t *>(at(o_run_len));
    v.run_q = static_cast<const int32_t *>(at(o_run_q));
    v.run_count = static_cast<const uint64_t *>(at(o_run_count));
    v.run_weight = static_cast<const uint64_t *>(at(o_run_weight));
    v.cl_n = static_cast<const uint8_t *>(at(o_cl_n));
    v.cl_shape = static_cast<const uint16_t *>(at(o_cl_shape));
    sp.view = v;
    sp.valid = true;
}

// Per-partition exact-path flags for the current workload.
void refresh_exact(oserve_gpu_ctx &c, Space &sp) {
    sp.exact.assign(sp.parts.size(), 0);
    sp.any_exact = false;
    for (size_t i = 0; i < sp.parts.size(); ++i) {
        if (sp.parts[i].count && use_exact(c, static_cast<int>(sp.parts[i].sizes.size()))) {
            if (static_cast<int64_t>(sp.parts[i].sizes.size()) * c.J > kMaxExactCells)
                fail(OSERVE_ERR_UNSUPPORTED, "exact path limited to 64 cells");
            sp.exact[i] = 1;
            sp.any_exact = true;
        }
    }
    sp.view.exact = sp.d_exact.upload(sp.exact, c.stream);
}

// Key bit layout: objective (descending) above partition, sum_pp, rank.
bool key_layout(int64_t total_demand, int64_t parts, int devices, uint64_t max_count, KeyLayout &k) {
    const int b_obj = bits_for(static_cast<uint64_t>(total_demand));
    const int b_part = bits_for(parts > 0 ? static_cast<uint64_t>(parts - 1) : 0);
    const int b_spp = bits_for(static_cast<uint64_t>(devices));
    const int b_loc = bits_for(max_count ? max_count - 1 : 0);
    if (b_obj + b_part + b_spp + b_loc > 63) return false;
    k.sh_spp = b_loc;
    k.sh_part = b_loc + b_spp;
    k.sh_obj = b_loc + b_spp + b_part;
    k.obj_max = (uint64_t{1} << b_obj) - 1;
    return true;
}

void make_key_layout(oserve_gpu_ctx &c, const Space &sp) {
    int64_t tot = 0;
    for (int64_t v : c.lambda) tot += v;
    if (!key_layout(tot, static_cast<int64_t>(sp.parts.size()), c.D(), sp.max_count, c.key))
        fail(OSERVE_ERR_TOO_LARGE, "selection key does not fit 63 bits");
}

uint64_t shard_count_of(uint64_t total, uint64_t ch, uint64_t r, uint64_t w) {
    const uint64_t full = total / ch, rem = total % ch;
    uint64_t n = full > r ? ((full - r + w - 1) / w) * ch : 0;
    if (rem && full % w == r) n += rem;
    return n;
}

uint64_t shard_count(const oserve_gpu_ctx &c, uint64_t total) {
    return shard_count_of(total, c.chunk, static_cast<uint64_t>(c.rank), static_cast<uint64_t>(c.world));
}

void unrank_host(const Space &sp, uint64_t rank, int64_t &p, uint64_t &local, std::vector<int> &picks) {
    auto it = std::upper_bound(sp.prefix.begin(), sp.prefix.end() - 1, rank);
    p = static_cast<int64_t>(it - sp.prefix.begin()) - 1;
    local = rank - sp.prefix[p];
    const Partition &part = sp.parts[p];
    picks.assign(part.sizes.size(), 0);
    uint64_t r = local;
    for (int i = static_cast<int>(part.runs.size()) - 1; i >= 0; --i) {
        const Run &run = part.runs[i];
        uint64_t rr = r % run.count;
        r /= run.count;
        int prev = 0;
        for (int pos = 0; pos < run.len; ++pos) {
            for (int v = prev; v < run.q; ++v) {
                uint64_t cnt = binom((run.len - pos - 1) + (run.q - v) - 1, (run.q - v) - 1);
                if (rr < cnt) {
                    picks[run.start + pos] = v;
                    prev = v;
                    break;
                }
                rr -= cnt;
            }
        }
    }
}

void fill_plan(const oserve_gpu_ctx &c, const Space &sp, int64_t p, const std::vector<int> &picks, oserve_plan *out) {
    std::memset(out, 0, sizeof(*out));
    const Partition &part = sp.parts[p];
    out->num_replicas = static_cast<int>(part.sizes.size());
    int pos = 0;
    for (size_t r = 0; r < part.sizes.size(); ++r) {
        const Cand &cd = sp.lists[part.cand_list[r]][picks[r]];
        out->replica_num_devices[r] = part.sizes[r];
        out->tp[r] = cd.first;
        out->pp[r] = cd.second;
        for (int i = 0; i < part.sizes[r]; ++i) out->device_ids[pos++] = c.dev_sorted[part.offsets[r] + i];
    }
    out->num_devices = pos;
}

void decode_key(oserve_gpu_ctx &c, uint64_t key, oserve_round_result *out) {
    const Space &sp = c.space;
    std::memset(out, 0, sizeof(*out));
    out->partitions = static_cast<int64_t>(sp.parts.size());
    out->plans = sp.total;
    out->key = key;
    if (key == kNoKey) {
        out->objective = -1;
        return;
    }
    const uint64_t m_loc = (uint64_t{1} << c.key.sh_spp) - 1;
    const uint64_t m_spp = (uint64_t{1} << (c.key.sh_part - c.key.sh_spp)) - 1;
    const uint64_t m_part = (uint64_t{1} << (c.key.sh_obj - c.key.sh_part)) - 1;
    const uint64_t local = key & m_loc;
    const int spp = static_cast<int>((key >> c.key.sh_spp) & m_spp);
    const int64_t part = static_cast<int64_t>((key >> c.key.sh_part) & m_part);
    const int64_t obj = static_cast<int64_t>(c.key.obj_max - (key >> c.key.sh_obj));
    if (part >= static_cast<int64_t>(sp.parts.size()) || local >= sp.parts[part].count)
        fail(OSERVE_ERR_INVALID_ARGUMENT, "key does not belong to the prepared space");
    out->objective = obj;
    out->partition_index = part;
    out->local_rank = local;
    out->sum_pp = spp;
    int64_t p2;
    uint64_t l2;
    std::vector<int> picks;
    unrank_host(sp, sp.prefix[part] + local, p2, l2, picks);
    fill_plan(c, sp, p2, picks, &out->plan);
}

// The K1 launches covering this shard of the prepared space: one per R-bucket
// (mode 3) when the space mixes R <= 32 and R > 32, else one (mode 0).
template <class F>
void for_each_k1_launch(oserve_gpu_ctx &c, Space &sp, F &&fn) {
    if (sp.use_buckets) {
        for (auto &b : sp.buckets) {
            PlanSource src{};
            src.mode = 3;
            src.count = shard_count_of(b.total, c.chunk, static_cast<uint64_t>(c.rank), static_cast<uint64_t>(c.world));
            src.rank = c.rank;
            src.world = c.world;
            src.chunk = c.chunk;
            src.range_start = b.d_start;
            src.range_prefix = b.d_prefix;
            src.num_ranges = static_cast<int>(b.start.size());
            fn(src, b.rmax);
        }
        return;
    }
    PlanSource src{};
    src.mode = 0;
    src.count = shard_count(c, sp.total);
    src.rank = c.rank;
    src.world = c.world;
    src.chunk = c.chunk;
    fn(src, sp.rmax);
}

// Exact (B&B) path for the plans of `src` that take it: the frontier-parallel
// passes (k_exact_plan / k_exact_task), then the sequential kernel for plans
// whose tree could not be cut within the task caps or whose phase A hit the
// budget.  Plans whose B&B blows the budget are appended to eo.aborted (the
// caller reruns them through K1).
void run_exact(oserve_gpu_ctx &c, const SpaceTables &view, const KeyLayout &key, const PlanSource &src0,
               const PlanOutputs &eo, const SolveParams &prm, const Space *sp) {
    cudaStream_t s = c.stream;
    PlanSource src = src0;
    DBuf &d_exact_ranks = c.exact.ranks;
    if (sp && src.mode == 0) {
        // restrict to this shard's exact-path plans
        std::vector<uint64_t> ranks;
        for (size_t p = 0; p < sp->parts.size(); ++p) {
            if (!sp->exact[p]) continue;
            for (uint64_t g = sp->prefix[p]; g < sp->prefix[p] + sp->parts[p].count; ++g) {
                if ((g / c.chunk) % static_cast<uint64_t>(c.world) != static_cast<uint64_t>(c.rank)) continue;
                ranks.push_back(g);
            }
        }
        src.mode = 1;
        src.first = 0;
        src.count = ranks.size();
        src.ranks = d_exact_ranks.upload(ranks, s);
        if (ranks.empty()) return;
    }
    if (src.count == 0) return;
    const uint64_t P = src.count;
    ExactScratch &xs = c.exact;
    ExactTasks et{};
    et.depth = static_cast<int32_t *>(xs.depth.get(sizeof(int32_t) * P));
    et.ntask = static_cast<uint64_t *>(xs.nt.get(sizeof(uint64_t) * P));
    et.toff = static_cast<uint64_t *>(xs.off.get(sizeof(uint64_t) * P));
    et.top_nodes = static_cast<int64_t *>(xs.top.get(sizeof(int64_t) * P));
    et.opt = static_cast<int64_t *>(xs.opt.get(sizeof(int64_t) * P));
    et.istar = static_cast<int64_t *>(xs.ist.get(sizeof(int64_t) * P));
    et.state = static_cast<uint8_t *>(xs.state.get(P));
    et.bx = static_cast<int32_t *>(xs.bx.get(sizeof(int32_t) * P * kMaxExactCells));
    et.running = static_cast<unsigned long long *>(xs.run.get(sizeof(unsigned long long) * P));
    et.fetch = static_cast<unsigned long long *>(xs.fetch.get(sizeof(unsigned long long)));
    et.topn = static_cast<unsigned long long *>(xs.topn.get(sizeof(unsigned long long) * P));
    et.ubn = static_cast<unsigned long long *>(xs.ubn.get(sizeof(unsigned long long) * P));
    et.lbn = static_cast<unsigned long long *>(xs.lbn.get(sizeof(unsigned long long) * P));
    et.anycap = static_cast<uint8_t *>(xs.anycap.get(P));
    // Phase A runs every task with a lower bound of its entering incumbent,
    // so a plan whose tree is far larger than the node budget (the sequential
    // search aborts after node_budget nodes) would be explored whole: its
    // phase-A nodes over all rounds are capped at kWorkBudgets x node_budget,
    // past which the sequential DFS (<= node_budget nodes) decides it.
    static const int64_t kWorkBudgets = [] {
        const char *e = getenv("OSERVE_EXACT_WORK");
        return e ? static_cast<int64_t>(atoll(e)) : int64_t{16};
    }();
    et.work = static_cast<unsigned long long *>(xs.work.get(sizeof(unsigned long long) * P));
    et.work_limit = kWorkBudgets * prm.node_budget;
    cuda_ok(cudaMemsetAsync(et.work, 0, sizeof(unsigned long long) * P, s), "memset");
    // ~2^21 tasks in flight at most; at least a few thousand per plan when few plans
    const uint64_t budget_tasks = uint64_t{1} << 21;
    static const uint64_t target_env = [] {
        const char *e = getenv("OSERVE_EXACT_TARGET");
        return e ? static_cast<uint64_t>(atoll(e)) : 0ull;
    }();
    et.target = target_env ? target_env : std::max<uint64_t>(64, std::min<uint64_t>(1024, budget_tasks / P));
    et.max_tasks = et.target * 8;
    static const bool dbg = getenv("OSERVE_DEBUG_EXACT") != nullptr;
    TaskBufs *bufs = c.exact.bufs;
    int cur = 0;
    uint64_t total = 0;
    std::vector<uint8_t> state;
    auto lap = [&](const char *what) {
        if (!dbg) return;
        static auto t0 = std::chrono::steady_clock::now();
        cuda_ok(cudaStreamSynchronize(s), "sync");
        const auto t1 = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[exact] %-14s %8.1f ms  (plans %llu, tasks %llu)\n", what,
                     std::chrono::duration<double, std::milli>(t1 - t0).count(), static_cast<unsigned long long>(P),
                     static_cast<unsigned long long>(total));
        t0 = t1;
    };
    uint32_t *d_newoff = nullptr;
    // Rebuild the task list from et.nchild (children of split tasks in
    // preorder, others copied): device scan, split, per-plan ranges.  False
    // when nothing was split.
    auto rebuild = [&]() -> bool {
        cuda_ok(cudaMemsetAsync(et.nchild + total, 0, sizeof(uint32_t), s), "memset");
        d_newoff = static_cast<uint32_t *>(xs.newoff.get(sizeof(uint32_t) * (total + 1)));
        cuda_ok(launch_exact_rescan(et, total, d_newoff, P, &c.cub_temp, &c.cub_temp_bytes, s, &c.launches),
                "exact rescan");
        uint32_t ntot32 = 0;
        cuda_ok(d2h(&ntot32, d_newoff + total, sizeof(uint32_t), s), "D2H");
        cuda_ok(cudaStreamSynchronize(s), "sync");
        const uint64_t ntot = ntot32;
        if (ntot == total) return false;
        ExactTasks ne = et;
        bufs[cur ^ 1].bind(ne, ntot);
        cuda_ok(launch_exact_split(c.tables, view, src, prm, et, ne, d_newoff, total, c.sm_count, s, &c.launches),
                "exact split");
        cuda_ok(launch_exact_ranges(et, d_newoff, P, s, &c.launches), "exact ranges");
        et = ne;
        cur ^= 1;
        total = ntot;
        return true;
    };
    {
        // Frontier built on the device: one root task per exact-path plan,
        // then level by level every task of a plan still below the target
        // count becomes the branches of its root's first decision (preorder
        // kept), unless that would pass the plan's task cap.
        cuda_ok(launch_exact_plan_pass(10, c.tables, view, key, src, eo, prm, et, c.sm_count, s, &c.launches),
                "exact plan pass 10");
        download(state, et.state, P, s);
        cuda_ok(cudaStreamSynchronize(s), "sync");
        std::vector<uint64_t> off(P, 0);
        std::vector<uint32_t> plan_h;
        for (uint64_t i = 0; i < P; ++i) {
            off[i] = plan_h.size();
            if (state[i] == 1) plan_h.push_back(static_cast<uint32_t>(i));
        }
        total = plan_h.size();
        if (total) {
            bufs[cur].bind(et, total);
            cuda_ok(h2d(et.toff, off.data(), sizeof(uint64_t) * P, s), "H2D");
            cuda_ok(h2d(et.plan, plan_h.data(), sizeof(uint32_t) * total, s), "H2D");
            cuda_ok(cudaMemsetAsync(et.tdepth, 0, total, s), "memset");
            cuda_ok(cudaMemsetAsync(et.done, 0, total, s), "memset");
            cuda_ok(cudaMemsetAsync(et.capped, 0, total, s), "memset");
            et.grow = static_cast<uint8_t *>(xs.grow.get(P));
            et.plan_sum = static_cast<uint32_t *>(xs.psum.get(sizeof(uint32_t) * P));
            std::vector<uint64_t> n_h(P, 0);
            for (uint64_t i = 0; i < P; ++i) n_h[i] = state[i] == 1 ? 1 : 0;
            std::vector<uint8_t> grow(P, 0);
            std::vector<uint32_t> psum;
            for (int level = 1; level <= 6; ++level) {
                bool any = false;
                for (uint64_t i = 0; i < P; ++i) {
                    grow[i] = state[i] == 1 && n_h[i] < et.target;
                    any = any || grow[i];
                }
                if (!any) break;
                auto children = [&]() {
                    cuda_ok(h2d(et.grow, grow.data(), P, s), "H2D");
                    cuda_ok(cudaMemsetAsync(et.plan_sum, 0, sizeof(uint32_t) * P, s), "memset");
                    cuda_ok(launch_exact_task_pass(9, c.tables, view, src, prm, et, total, c.sm_count, s,
                                                   &c.launches),
                            "exact task pass 9");
                };
                children();
                download(psum, et.plan_sum, P, s);
                cuda_ok(cudaStreamSynchronize(s), "sync");
                bool redo = false;
                uint64_t tot_new = 0;
                for (uint64_t i = 0; i < P; ++i) {
                    if (grow[i] && psum[i] > et.max_tasks) {  // keep this plan at the previous level
                        grow[i] = 0;
                        redo = true;
                    }
                    tot_new += grow[i] ? psum[i] : n_h[i];
                }
                if (tot_new > 4 * budget_tasks) {  // task buffers full: stop growing
                    std::fill(grow.begin(), grow.end(), 0);
                    redo = true;
                }
                if (redo) children();
                for (uint64_t i = 0; i < P; ++i)
                    if (grow[i]) n_h[i] = psum[i];
                if (!rebuild()) break;
            }
        }
        lap("frontier");
    }
    if (total) {
        // Phase A in rounds: tasks over the round's node cap are split into
        // their children (preorder kept) and rerun; the last round runs with
        // the full budget.
        // Round r caps each task at cap0 * growth^r nodes: a task over the
        // cap wastes the nodes it ran before it is split, so the caps start
        // small and grow (most tasks finish in the first round).  Small caps
        // keep each round's longest task short; the rounds themselves are
        // cheap (device scans for the per-plan prefix maxima, no per-plan
        // loops): config 1-B&B 1,024 x 2: 13 ms, 8,192 x 4: 36 ms.
        static const int kRounds = [] {
            const char *e = getenv("OSERVE_EXACT_ROUNDS");
            return e ? atoi(e) : 14;
        }();
        static const int64_t kCap0 = [] {
            const char *e = getenv("OSERVE_EXACT_CAP0");
            return e ? static_cast<int64_t>(atoll(e)) : int64_t{1} << 10;
        }();
        static const int kGrowth = [] {
            const char *e = getenv("OSERVE_EXACT_GROWTH");
            return e ? atoi(e) : 2;
        }();
        // the replay of the top: exact incumbents, visited tasks and top-node
        // counts (see exact_replay_task)
        auto replay = [&]() {
            cuda_ok(launch_exact_prefix(6, et, total, P, static_cast<int64_t *>(xs.pmax.get(sizeof(int64_t) * total)),
                                        &c.cub_temp, &c.cub_temp_bytes, c.sm_count, s, &c.launches),
                    "exact incumbents");
            cuda_ok(launch_exact_task_pass(6, c.tables, view, src, prm, et, total, c.sm_count, s, &c.launches),
                    "exact task pass 6");
            uint64_t *tmp = static_cast<uint64_t *>(xs.scan.get(sizeof(uint64_t) * 2 * total));
            cuda_ok(launch_alive_scan(et, total, tmp, &c.cub_temp, &c.cub_temp_bytes, c.sm_count, s, &c.launches),
                    "alive scan");
            cuda_ok(launch_exact_task_pass(7, c.tables, view, src, prm, et, total, c.sm_count, s, &c.launches),
                    "exact task pass 7");
        };
        int64_t round_cap = kCap0;
        for (int round = 0;; ++round) {
            const bool last = round == kRounds || total > (uint64_t{1} << 24);
            et.phase_cap = last ? prm.node_budget : round_cap;
            round_cap = std::min<int64_t>(round_cap * kGrowth, int64_t{1} << 22);
            cuda_ok(launch_exact_task_pass(2, c.tables, view, src, prm, et, total, c.sm_count, s, &c.launches),
                    "exact task pass 2");
            cuda_ok(launch_exact_prefix(4, et, total, P, static_cast<int64_t *>(xs.pmax.get(sizeof(int64_t) * total)),
                                        &c.cub_temp, &c.cub_temp_bytes, c.sm_count, s, &c.launches),
                    "exact lower bounds");
            cuda_ok(launch_exact_task_pass(0, c.tables, view, src, prm, et, total, c.sm_count, s, &c.launches),
                    "exact task pass 0");
            cuda_ok(launch_exact_retire(et, P, c.sm_count, s, &c.launches), "exact retire");
            lap("phaseA round");
            if (last) break;
            cuda_ok(launch_exact_task_pass(3, c.tables, view, src, prm, et, total, c.sm_count, s, &c.launches),
                    "exact task pass 3");
            if (!rebuild()) break;  // nothing capped: phase A complete
        }
        replay();  // the exact incumbents, visited tasks and top-node counts (see exact_replay_task)
        cuda_ok(launch_exact_plan_pass(8, c.tables, view, key, src, eo, prm, et, c.sm_count, s, &c.launches),
                "exact plan pass 8");
        lap("top replay");
        cuda_ok(launch_exact_task_pass(1, c.tables, view, src, prm, et, total, c.sm_count, s, &c.launches),
                "exact task pass 1");
        lap("phaseB");
        cuda_ok(launch_exact_plan_pass(3, c.tables, view, key, src, eo, prm, et, c.sm_count, s, &c.launches),
                "exact plan pass 3");
        lap("finish");
        if (dbg) {
            std::vector<int64_t> nodes;
            std::vector<uint8_t> vis;
            download(nodes, et.nodes, total, s);
            download(vis, et.vis, total, s);
            cuda_ok(cudaStreamSynchronize(s), "sync");
            int64_t mx = 0, sum = 0, nv = 0;
            for (uint64_t q = 0; q < total; ++q)
                if (vis[q]) {
                    mx = std::max(mx, nodes[q]);
                    sum += nodes[q];
                    ++nv;
                }
            {  // per plan: phase-A nodes of all its tasks, final state, top nodes
                std::vector<uint64_t> toff, ntk;
                std::vector<uint8_t> st2;
                std::vector<int64_t> topn;
                std::vector<unsigned long long> run, wk;
                download(wk, et.work, P, s);
                download(toff, et.toff, P, s);
                download(ntk, et.ntask, P, s);
                download(st2, et.state, P, s);
                download(topn, et.top_nodes, P, s);
                download(run, et.running, P, s);
                cuda_ok(cudaStreamSynchronize(s), "sync");
                for (uint64_t i = 0; i < P; ++i) {
                    if (st2[i] == 0) continue;
                    int64_t a = 0, v = 0;
                    for (uint64_t q = toff[i]; q < toff[i] + ntk[i] && q < total; ++q) {
                        a += nodes[q];
                        if (vis[q]) v += nodes[q];
                    }
                    if (a > 1000000 || wk[i] > 1000000)
                        std::fprintf(stderr, "[exact]   plan %llu state %d tasks %llu phase-A nodes %lld (visited %lld) "
                                     "top %lld running %llu, all rounds %llu\n",
                                     static_cast<unsigned long long>(i), st2[i], static_cast<unsigned long long>(ntk[i]),
                                     static_cast<long long>(a), static_cast<long long>(v), static_cast<long long>(topn[i]),
                                     static_cast<unsigned long long>(run[i]), wk[i]);
                }
            }
            std::fprintf(stderr, "[exact] tasks %llu visited %lld, phase-A nodes sum (final tasks) %lld max %lld\n",
                         static_cast<unsigned long long>(total), static_cast<long long>(nv),
                         static_cast<long long>(sum), static_cast<long long>(mx));
        }
    }
    download(state, et.state, P, s);
    cuda_ok(cudaStreamSynchronize(s), "sync");  // scratch buffers are freed on return
    std::vector<uint64_t> redo;
    for (uint64_t i = 0; i < P; ++i)
        if (state[i] == 2) redo.push_back(i);
    if (redo.empty()) return;
    if (src.mode == 2 || (src.mode == 0 && (eo.objective || eo.x))) {
        for (uint64_t li : redo) {  // per-plan outputs: one sequential launch per plan (rare)
            PlanSource one = src;
            one.first = src.first + li;
            one.count = 1;
            PlanOutputs o1 = eo;
            if (eo.objective) o1.objective = eo.objective + li;
            if (eo.sum_pp) o1.sum_pp = eo.sum_pp + li;
            if (eo.x) {
                o1.x = eo.x + li * eo.rmax * prm.J;
                o1.used = eo.used + li * eo.rmax;
            }
            cuda_ok(launch_plan_exact(c.tables, view, key, one, o1, prm, c.sm_count, s, &c.launches),
                    "exact kernel (sequential)");
        }
    } else {
        // rank sources: outputs are keyed (argmin); rerun the listed ranks
        std::vector<uint64_t> ranks;
        for (uint64_t li : redo) {
            if (src.mode == 1) {
                uint64_t r = 0;
                cuda_ok(d2h(&r, src.ranks + src.first + li, sizeof(uint64_t), s), "D2H");
                cuda_ok(cudaStreamSynchronize(s), "sync");
                ranks.push_back(r);
            } else {
                ranks.push_back(src.first + li);
            }
        }
        DBuf d_r;
        PlanSource rs{};
        rs.mode = 1;
        rs.count = ranks.size();
        rs.ranks = d_r.upload(ranks, s);
        PlanOutputs o1 = eo;
        o1.objective = nullptr;
        o1.sum_pp = nullptr;
        cuda_ok(launch_plan_exact(c.tables, view, key, rs, o1, prm, c.sm_count, s, &c.launches),
                "exact kernel (sequential)");
    }
    cuda_ok(cudaStreamSynchronize(s), "sync");
}

// Launch K1 (+K4, + heuristic fallback for aborted B&B) over this shard of
// the prepared space; best key -> d_key.
void launch_round(oserve_gpu_ctx &c, uint64_t *d_key) {
    ensure_tables(c);
    Space &sp = c.space;
    refresh_exact(c, sp);
    make_key_layout(c, sp);
    cudaStream_t s = c.stream;
    cuda_ok(cudaMemsetAsync(d_key, 0xff, sizeof(uint64_t), s), "memset key");
    PlanSource src{};
    src.mode = 0;
    src.count = shard_count(c, sp.total);
    src.rank = c.rank;
    src.world = c.world;
    src.chunk = c.chunk;
    PlanOutputs out{};
    out.best_key = d_key;
    SolveParams prm = solve_params(c);
    count_h2d(sizeof(int64_t) * c.J);  // the demand vector travels as a kernel parameter
    for_each_k1_launch(c, sp, [&](const PlanSource &ls, int rmax) {
        cuda_ok(launch_plan_eval(c.tables, sp.view, c.key, ls, out, prm, rmax, c.sm_count, sp.any_exact ? 1 : 0, &c.ring, s,
                                 &c.launches),
                "plan kernel");
    });
    if (sp.any_exact) {
        uint64_t *ab = static_cast<uint64_t *>(c.d_aborted.get(sizeof(uint64_t) * std::max<uint64_t>(src.count, 1)));
        unsigned *abn = static_cast<unsigned *>(c.d_aborted_n.get(sizeof(unsigned)));
        cuda_ok(cudaMemsetAsync(abn, 0, sizeof(unsigned), s), "memset");
        PlanOutputs eo = out;
        eo.aborted = ab;
        eo.aborted_n = abn;
        run_exact(c, sp.view, c.key, src, eo, prm, &sp);
        unsigned n_ab = 0;
        cuda_ok(d2h(&n_ab, abn, sizeof(unsigned), s), "D2H");
        cuda_ok(cudaStreamSynchronize(s), "sync");
        if (n_ab) {
            PlanSource rs{};
            rs.mode = 1;
            rs.count = n_ab;
            rs.ranks = ab;
            cuda_ok(launch_plan_eval(c.tables, sp.view, c.key, rs, out, prm, sp.rmax, c.sm_count, 0, &c.ring, s, &c.launches),
                    "plan kernel (budget fallback)");
        }
    }
}

void prepare(oserve_gpu_ctx &c, const oserve_space_desc &d) {
    if (d.max_devices > 0 && c.D() > d.max_devices)
        fail(OSERVE_ERR_TOO_LARGE, "exhaustive enumeration guarded to " + std::to_string(d.max_devices) +
                                       " devices, cluster has " + std::to_string(c.D()));
    if (d.mode != OSERVE_SPACE_ORDERED && d.mode != OSERVE_SPACE_CANONICAL)
        fail(OSERVE_ERR_INVALID_ARGUMENT, "unknown space mode");
    std::vector<int> sizes(d.sizes, d.sizes + (d.sizes ? d.num_sizes : 0));
    Space &sp = c.space;
    if (sp.valid && !sp.explicit_partition && sp.mode == d.mode && sp.sizes_key == sizes) return;
    sp.valid = false;
    build_space(c, sp, d.mode, sizes, nullptr);
    sp.mode = d.mode;
    sp.sizes_key = sizes;
    sp.explicit_partition = false;
}

template <class F>
int guarded(oserve_gpu_ctx *c, F &&f) {
    if (!c) return OSERVE_ERR_INVALID_ARGUMENT;
    t_h2d = &c->h2d_bytes;
    t_d2h = &c->d2h_bytes;
    try {
        cuda_ok(cudaSetDevice(c->device), "cudaSetDevice");
        f();
        c->err.clear();
        return OSERVE_OK;
    } catch (const Fail &e) {
        c->err = e.what();
        return e.code;
    } catch (const std::bad_alloc &) {
        c->err = "out of host memory";
        return OSERVE_ERR_INVALID_ARGUMENT;
    } catch (const std::exception &e) {
        c->err = e.what();
        return OSERVE_ERR_INVALID_ARGUMENT;
    }
}

// Deployment -> shape ids (evaluate_deployment / build_capacity_table).
std::vector<int> deployment_shapes(oserve_gpu_ctx &c, const oserve_deployment &d) {
    std::vector<int> ids;
    int pos = 0;
    for (int r = 0; r < d.num_replicas; ++r) {
        std::vector<int> devs(d.device_ids + pos, d.device_ids + pos + d.replica_num_devices[r]);
        pos += d.replica_num_devices[r];
        uint64_t total = 0;
        if (!mem_feasible(c, devs, d.tp[r], d.pp[r], &total))
            fail(OSERVE_ERR_INFEASIBLE_REPLICA, "replica " + std::to_string(r) + " cannot host model");
        ids.push_back(shape_for(c, d.tp[r], d.pp[r], total));
    }
    return ids;
}

// Evaluate explicit shape lists; returns objectives (+ x/used when requested).
void eval_lists(oserve_gpu_ctx &c, const std::vector<int32_t> &listR, const std::vector<int32_t> &listOff,
                const std::vector<int32_t> &shapes, const std::vector<int64_t> *lam_per_plan, int rmax,
                std::vector<int64_t> &obj, std::vector<int64_t> *x, std::vector<int64_t> *used,
                const SolveParams &prm, std::vector<uint64_t> *aborted_out = nullptr) {
    cudaStream_t s = c.stream;
    const uint64_t n = listR.size();
    PlanSource src{};
    src.mode = 2;
    src.count = n;
    Packer pk;  // the plan lists in one H2D copy
    const size_t oR = pk.add(listR), oO = pk.add(listOff), oS = pk.add(shapes);
    const size_t oL = lam_per_plan ? pk.add(*lam_per_plan) : 0;
    const unsigned char *base = pk.upload(c.d_listR, s);
    src.list_R = reinterpret_cast<const int32_t *>(base + oR);
    src.list_off = reinterpret_cast<const int32_t *>(base + oO);
    src.list_shapes = reinterpret_cast<const int32_t *>(base + oS);
    if (lam_per_plan) src.list_lambda = reinterpret_cast<const int64_t *>(base + oL);
    PlanOutputs out{};
    out.objective = static_cast<int64_t *>(c.d_obj.get(sizeof(int64_t) * n));
    out.rmax = std::max(rmax, 1);
    if (x) {
        out.x = static_cast<int64_t *>(c.d_x.get(sizeof(int64_t) * n * out.rmax * prm.J));
        out.used = static_cast<int64_t *>(c.d_used.get(sizeof(int64_t) * n * out.rmax));
    }
    // exact-path plans
    bool any_exact = false;
    for (uint64_t i = 0; i < n; ++i) {
        int64_t tot = 0;
        for (int j = 0; j < prm.J; ++j) tot += lam_per_plan ? (*lam_per_plan)[i * prm.J + j] : prm.lambda[j];
        if (tot <= prm.exact_demand_limit && static_cast<int64_t>(listR[i]) * prm.J <= prm.exact_cell_limit) {
            if (static_cast<int64_t>(listR[i]) * prm.J > kMaxExactCells)
                fail(OSERVE_ERR_UNSUPPORTED, "exact path limited to 64 cells");
            any_exact = true;
        }
    }
    SpaceTables none{};
    KeyLayout nk{};
    cuda_ok(launch_plan_eval(c.tables, none, nk, src, out, prm, rmax, c.sm_count, any_exact ? 1 : 0, &c.ring, s, &c.launches),
            "plan kernel");
    if (any_exact) {
        uint64_t *ab = static_cast<uint64_t *>(c.d_aborted.get(sizeof(uint64_t) * n));
        unsigned *abn = static_cast<unsigned *>(c.d_aborted_n.get(sizeof(unsigned)));
        cuda_ok(cudaMemsetAsync(abn, 0, sizeof(unsigned), s), "memset");
        PlanOutputs eo = out;
        eo.aborted = ab;
        eo.aborted_n = abn;
        run_exact(c, none, nk, src, eo, prm, nullptr);
        unsigned n_ab = 0;
        cuda_ok(d2h(&n_ab, abn, sizeof(unsigned), s), "D2H");
        cuda_ok(cudaStreamSynchronize(s), "sync");
        if (n_ab) {
            std::vector<uint64_t> idx;
            download(idx, ab, n_ab, s);
            cuda_ok(cudaStreamSynchronize(s), "sync");
            std::sort(idx.begin(), idx.end());
            if (aborted_out) {
                *aborted_out = idx;
                idx.clear();
            }
            for (uint64_t li : idx) {  // heuristic fallback, one plan per launch (rare)
                PlanSource one = src;
                one.first = li;
                one.count = 1;
                PlanOutputs o1 = out;
                o1.objective = out.objective + li;
                if (x) {
                    o1.x = out.x + li * out.rmax * prm.J;
                    o1.used = out.used + li * out.rmax;
                }
                cuda_ok(launch_plan_eval(c.tables, none, nk, one, o1, prm, rmax, c.sm_count, 0, &c.ring, s, &c.launches),
                        "plan kernel (budget fallback)");
            }
        }
    }
    download(obj, out.objective, n, s);
    if (x) {
        download(*x, out.x, n * out.rmax * prm.J, s);
        download(*used, out.used, n * out.rmax, s);
    }
    cuda_ok(cudaStreamSynchronize(s), "sync");
}

// --------------------------------------------------------------- switch ---
struct SwitchInput {
    std::vector<int32_t> machine, dev_id, dep_rep_off, rep_tp, rep_pp, rep_dev_off, rep_devs;
};

void add_deployment(oserve_gpu_ctx &c, SwitchInput &in, std::map<int, int> &slots, const oserve_deployment &d) {
    in.dep_rep_off.push_back(static_cast<int32_t>(in.rep_tp.size()));
    int pos = 0;
    std::set<int> seen;
    for (int r = 0; r < d.num_replicas; ++r) {
        std::vector<int> devs(d.device_ids + pos, d.device_ids + pos + d.replica_num_devices[r]);
        pos += d.replica_num_devices[r];
        if (d.tp[r] < 1 || d.pp[r] < 1 || d.tp[r] * d.pp[r] != static_cast<int>(devs.size()))
            fail(OSERVE_ERR_INVALID_ARGUMENT, "switch: replica tp*pp must equal its device count");
        std::sort(devs.begin(), devs.end());
        in.rep_tp.push_back(d.tp[r]);
        in.rep_pp.push_back(d.pp[r]);
        in.rep_dev_off.push_back(static_cast<int32_t>(in.rep_devs.size()));
        for (int dv : devs) {
            if (!seen.insert(dv).second)
                fail(OSERVE_ERR_UNSUPPORTED, "switch: a device appears in two replicas of one deployment");
            auto it = slots.find(dv);
            if (it == slots.end()) fail(OSERVE_ERR_INVALID_ARGUMENT, "switch: device slot missing");
            in.rep_devs.push_back(it->second);
        }
    }
}

void run_switch(oserve_gpu_ctx &c, const oserve_deployment *src, int count, const oserve_deployment *dsts,
                std::vector<double> &est, std::vector<uint64_t> &maxb, std::vector<int32_t> &status,
                std::vector<int32_t> *detail, std::vector<uint64_t> *cuts, int *ncuts, SwitchInput *in_out) {
    // device slots: every cluster device plus unknown ids, ascending id
    std::set<int> ids(c.dev_sorted.begin(), c.dev_sorted.end());
    auto collect = [&](const oserve_deployment &d) {
        int n = 0;
        for (int r = 0; r < d.num_replicas; ++r) n += d.replica_num_devices[r];
        for (int i = 0; i < n; ++i) ids.insert(d.device_ids[i]);
    };
    collect(*src);
    for (int i = 0; i < count; ++i) collect(dsts[i]);
    if (ids.size() > 256) fail(OSERVE_ERR_UNSUPPORTED, "switch kernel limited to 256 devices");
    SwitchInput in;
    std::map<int, int> slots;
    for (int id : ids) {
        slots.emplace(id, static_cast<int>(in.dev_id.size()));
        in.dev_id.push_back(id);
        in.machine.push_back(c.machine(id));
    }
    add_deployment(c, in, slots, *src);
    for (int i = 0; i < count; ++i) add_deployment(c, in, slots, dsts[i]);
    in.dep_rep_off.push_back(static_cast<int32_t>(in.rep_tp.size()));
    in.rep_dev_off.push_back(static_cast<int32_t>(in.rep_devs.size()));
    if (in.dep_rep_off[1] - in.dep_rep_off[0] > 128) fail(OSERVE_ERR_UNSUPPORTED, "switch: > 128 source replicas");
    if (c.model.param_bytes >= (uint64_t{1} << 46)) fail(OSERVE_ERR_UNSUPPORTED, "switch: param_bytes >= 2^46");
    cudaStream_t s = c.stream;
    SwitchDeps d{};
    d.count = count;
    d.num_devices = static_cast<int>(in.dev_id.size());
    d.machine = c.d_sw[0].upload(in.machine, s);
    d.dev_id = c.d_sw[1].upload(in.dev_id, s);
    d.dep_rep_off = c.d_sw[2].upload(in.dep_rep_off, s);
    d.rep_tp = c.d_sw[3].upload(in.rep_tp, s);
    d.rep_pp = c.d_sw[4].upload(in.rep_pp, s);
    d.rep_dev_off = c.d_sw[5].upload(in.rep_dev_off, s);
    d.rep_devs = c.d_sw[6].upload(in.rep_devs, s);
    d.P = c.model.param_bytes;
    d.intra_bw = c.intra;
    d.inter_bw = c.inter;
    SwitchOut o{};
    o.est = static_cast<double *>(c.d_sw[7].get(sizeof(double) * count));
    o.max_bytes = static_cast<uint64_t *>(c.d_sw[8].get(sizeof(uint64_t) * count));
    o.status = static_cast<int32_t *>(c.d_sw[9].get(sizeof(int32_t) * count));
    const int maxf = 4 * d.num_devices;
    if (detail) {
        o.max_frags = maxf;
        o.detail_src = static_cast<int32_t *>(c.d_sw[10].get(sizeof(int32_t) * d.num_devices * maxf));
        cuda_ok(cudaMemsetAsync(o.detail_src, 0xff, sizeof(int32_t) * d.num_devices * maxf, s), "memset");
        o.detail_cuts = static_cast<uint64_t *>(c.d_sw[11].get(sizeof(uint64_t) * (maxf + 2)));
        o.detail_ncuts = reinterpret_cast<int32_t *>(o.detail_cuts + maxf + 1);
    }
    cuda_ok(launch_switch_cost(d, o, s, &c.launches), "switch kernel");
    download(est, o.est, count, s);
    download(maxb, o.max_bytes, count, s);
    download(status, o.status, count, s);
    if (detail) {
        download(*detail, o.detail_src, static_cast<size_t>(d.num_devices) * maxf, s);
        std::vector<uint64_t> tmp;
        download(tmp, o.detail_cuts, maxf + 2, s);
        cuda_ok(cudaStreamSynchronize(s), "sync");
        *ncuts = static_cast<int>(reinterpret_cast<int32_t *>(&tmp[maxf + 1])[0]);
        cuts->assign(tmp.begin(), tmp.begin() + std::min(*ncuts, maxf + 1));
    }
    cuda_ok(cudaStreamSynchronize(s), "sync");
    if (in_out) *in_out = std::move(in);
}


// Top-K of this shard (see oserve_gpu_round_topk).
void round_topk(oserve_gpu_ctx &c, int K, uint64_t *d_keys, uint64_t *d_best) {
    if (K < 1 || K > 65536) fail(OSERVE_ERR_INVALID_ARGUMENT, "K must be in [1, 65536]");
    ensure_tables(c);
    Space &sp = c.space;
    refresh_exact(c, sp);
    if (sp.any_exact) fail(OSERVE_ERR_UNSUPPORTED, "top-K round on exact-path (branch-and-bound) plans");
    make_key_layout(c, sp);
    cudaStream_t s = c.stream;
    SolveParams prm = solve_params(c);
    count_h2d(sizeof(int64_t) * c.J);
    std::vector<std::pair<PlanSource, int>> launches;
    for_each_k1_launch(c, sp, [&](const PlanSource &ls, int rmax) { launches.emplace_back(ls, rmax); });
    std::vector<int> lgroups;
    int groups = 0;
    for (auto &[ls, rmax] : launches) {
        const int g = k1_groups(rmax, c.J, c.sm_count, c.tables, ls.count);
        if (g < 0) fail(OSERVE_ERR_CUDA, "K1 geometry");
        lgroups.push_back(g);
        groups += g;
    }
    const size_t nlist = static_cast<size_t>(std::max(groups, 1)) * kTopK;
    uint64_t *best = d_best ? d_best : static_cast<uint64_t *>(c.d_key.get(sizeof(uint64_t)));
    cuda_ok(cudaMemsetAsync(best, 0xff, sizeof(uint64_t), s), "memset");
    PlanOutputs out{};
    out.best_key = best;
    out.topk = static_cast<uint64_t *>(c.d_topk.get(sizeof(uint64_t) * nlist));
    out.topk_meta = static_cast<uint64_t *>(c.d_topk_meta.get(sizeof(uint64_t) * std::max(groups, 1)));
    cuda_ok(cudaMemsetAsync(out.topk, 0xff, sizeof(uint64_t) * nlist, s), "memset");
    cuda_ok(cudaMemsetAsync(out.topk_meta, 0xff, sizeof(uint64_t) * std::max(groups, 1), s), "memset");
    {
        size_t goff = 0;
        for (size_t q = 0; q < launches.size(); ++q) {
            PlanOutputs lo = out;
            lo.topk = out.topk + goff * kTopK;
            lo.topk_meta = out.topk_meta + goff;
            cuda_ok(launch_plan_eval(c.tables, sp.view, c.key, launches[q].first, lo, prm, launches[q].second,
                                     c.sm_count, 0, &c.ring, s, &c.launches),
                    "plan kernel (top-K)");
            goff += static_cast<size_t>(lgroups[q]);
        }
    }
    uint64_t *sorted = static_cast<uint64_t *>(c.d_topk_tmp.get(sizeof(uint64_t) * nlist));
    cuda_ok(sort_keys(out.topk, sorted, static_cast<int>(nlist), &c.cub_temp, &c.cub_temp_bytes, s), "sort");
    ++c.launches;
    const uint64_t *kth = sorted + std::min<size_t>(K, nlist) - 1;
    unsigned *bad = static_cast<unsigned *>(c.d_bad.get(sizeof(unsigned)));
    cuda_ok(cudaMemsetAsync(bad, 0, sizeof(unsigned), s), "memset");
    cuda_ok(launch_topk_check(out.topk_meta, groups, kth, bad, s), "top-K check");
    ++c.launches;
    unsigned nbad = 0;
    cuda_ok(d2h(&nbad, bad, sizeof(unsigned), s), "D2H");
    cuda_ok(cudaStreamSynchronize(s), "sync");
    const uint64_t *final_sorted = sorted;
    size_t final_n = nlist;
    if (nbad) {
        // exact fallback: collect every key <= the candidate K-th (an upper
        // bound of the true K-th), grow the buffer until nothing overflows
        uint64_t thr = kNoKey;
        cuda_ok(d2h(&thr, kth, sizeof(uint64_t), s), "D2H");
        cuda_ok(cudaStreamSynchronize(s), "sync");
        unsigned cap = static_cast<unsigned>(std::max(4 * K, 4096));
        for (;;) {
            PlanOutputs co{};
            co.collect = static_cast<uint64_t *>(c.d_collect.get(sizeof(uint64_t) * cap));
            co.collect_n = static_cast<unsigned *>(c.d_collect_n.get(sizeof(unsigned)));
            co.collect_cap = cap;
            co.collect_thr = thr;
            co.best_key = best;
            cuda_ok(cudaMemsetAsync(co.collect_n, 0, sizeof(unsigned), s), "memset");
            for (auto &[ls, rmax] : launches)
                cuda_ok(launch_plan_eval(c.tables, sp.view, c.key, ls, co, prm, rmax, c.sm_count, 0, &c.ring, s, &c.launches),
                        "plan kernel (threshold collect)");
            unsigned n = 0;
            cuda_ok(d2h(&n, co.collect_n, sizeof(unsigned), s), "D2H");
            cuda_ok(cudaStreamSynchronize(s), "sync");
            if (n <= cap) {
                uint64_t *tmp = static_cast<uint64_t *>(c.d_topk_tmp.get(sizeof(uint64_t) * std::max<size_t>(n, nlist)));
                cuda_ok(sort_keys(co.collect, tmp, static_cast<int>(n), &c.cub_temp, &c.cub_temp_bytes, s), "sort");
                final_sorted = tmp;
                final_n = n;
                break;
            }
            cap = n + 1024;
        }
    }
    cuda_ok(cudaMemsetAsync(d_keys, 0xff, sizeof(uint64_t) * K, s), "memset");
    cuda_ok(cudaMemcpyAsync(d_keys, final_sorted, sizeof(uint64_t) * std::min<size_t>(K, final_n),
                            cudaMemcpyDeviceToDevice, s),
            "D2D");
    cuda_ok(cudaStreamSynchronize(s), "sync");  // synchronous API: d_keys is ready on return
}

void switch_cost_keys(oserve_gpu_ctx &c, const oserve_deployment &current, int count, const uint64_t *d_keys,
                      double *est, uint64_t *maxb, double *d_est_async = nullptr) {
    if (!c.space.valid) fail(OSERVE_ERR_INVALID_ARGUMENT, "no prepared space");
    ensure_tables(c);
    if (c.D() > 256) fail(OSERVE_ERR_UNSUPPORTED, "switch kernel limited to 256 devices");
    // slots = the cluster's sorted devices (the candidates' canonical blocks)
    std::map<int, int> slots;
    SwitchInput in;
    for (int i = 0; i < c.D(); ++i) {
        slots.emplace(c.dev_sorted[i], i);
        in.dev_id.push_back(c.dev_sorted[i]);
        in.machine.push_back(c.machine(c.dev_sorted[i]));
    }
    add_deployment(c, in, slots, current);
    in.dep_rep_off.push_back(static_cast<int32_t>(in.rep_tp.size()));
    in.rep_dev_off.push_back(static_cast<int32_t>(in.rep_devs.size()));
    if (in.dep_rep_off[1] > 128) fail(OSERVE_ERR_UNSUPPORTED, "switch: > 128 source replicas");
    if (c.model.param_bytes >= (uint64_t{1} << 46)) fail(OSERVE_ERR_UNSUPPORTED, "switch: param_bytes >= 2^46");
    make_key_layout(c, c.space);
    cudaStream_t s = c.stream;
    SwitchDeps d{};
    d.count = count;
    d.num_devices = static_cast<int>(in.dev_id.size());
    d.machine = c.d_sw[0].upload(in.machine, s);
    d.dev_id = c.d_sw[1].upload(in.dev_id, s);
    d.dep_rep_off = c.d_sw[2].upload(in.dep_rep_off, s);
    d.rep_tp = c.d_sw[3].upload(in.rep_tp, s);
    d.rep_pp = c.d_sw[4].upload(in.rep_pp, s);
    d.rep_dev_off = c.d_sw[5].upload(in.rep_dev_off, s);
    d.rep_devs = c.d_sw[6].upload(in.rep_devs, s);
    d.P = c.model.param_bytes;
    d.intra_bw = c.intra;
    d.inter_bw = c.inter;
    SwitchOut o{};
    o.est = d_est_async ? d_est_async : static_cast<double *>(c.d_sw[7].get(sizeof(double) * count));
    o.max_bytes = static_cast<uint64_t *>(c.d_sw[8].get(sizeof(uint64_t) * count));
    o.status = static_cast<int32_t *>(c.d_sw[9].get(sizeof(int32_t) * count));
    cuda_ok(launch_switch_cost_keys(d, c.space.view, c.key, c.tables, d_keys, count, nullptr, o, s, &c.launches),
            "switch kernel (keys)");
    if (d_est_async) return;
    std::vector<int32_t> st;
    cuda_ok(d2h(est, o.est, sizeof(double) * count, s), "D2H");
    if (maxb) cuda_ok(d2h(maxb, o.max_bytes, sizeof(uint64_t) * count, s), "D2H");
    download(st, o.status, count, s);
    cuda_ok(cudaStreamSynchronize(s), "sync");
    for (int i = 0; i < count; ++i)
        if (st[i]) fail(OSERVE_ERR_UNSOURCED_FRAGMENT, "required bytes have no source holder");
}

// ----------------------------------------------------------- multi-GPU ---
// A context may own several local shards (oserve_gpu_create_multi: itself
// plus `subs` on the other devices) and/or belong to a multi-process world
// (oserve_gpu_join).  The sharded round: every local shard evaluates its
// interleaved chunks of the plan order (the same tables, mirrored from the
// lead), then one NCCL collective per shard — all-reduce(MIN) of the packed
// key, or all-gather of the top-K lists — on the shards' streams.

struct DeviceScope {
    int prev = -1;
    explicit DeviceScope(int d) {
        cudaGetDevice(&prev);
        cuda_ok(cudaSetDevice(d), "cudaSetDevice");
    }
    ~DeviceScope() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// Temporarily evaluate as shard (rank, world).
struct ShardAs {
    oserve_gpu_ctx &c;
    int r0, w0;
    ShardAs(oserve_gpu_ctx &cc, int r, int w) : c(cc), r0(cc.rank), w0(cc.world) {
        c.rank = r;
        c.world = w;
    }
    ~ShardAs() {
        c.rank = r0;
        c.world = w0;
    }
};

std::vector<oserve_gpu_ctx *> local_shards(oserve_gpu_ctx &c) {
    std::vector<oserve_gpu_ctx *> v{&c};
    v.insert(v.end(), c.subs.begin(), c.subs.end());
    return v;
}

// Bring a sub-context's workload, shape registry and space up to the lead's.
void mirror(oserve_gpu_ctx &lead, oserve_gpu_ctx &s) {
    DeviceScope ds(s.device);
    s.opts = lead.opts;
    s.chunk = lead.chunk;
    if (s.synced_work != lead.work_ver) {
        s.J = lead.J;
        s.cin = lead.cin;
        s.cout = lead.cout;
        s.lambda = lead.lambda;
        s.span = lead.span;
        s.have_workload = lead.have_workload;
        s.shapes = lead.shapes;
        s.shape_id = lead.shape_id;
        s.tables_dirty = true;
        s.synced_work = lead.work_ver;
    }
    if (lead.space.valid && s.synced_space != lead.space_ver) {
        s.space.valid = false;
        copy_space_host(lead.space, s.space);
        upload_space(s, s.space);
        s.synced_space = lead.space_ver;
    }
}

uint64_t shard_min_plans() {
    static const uint64_t v = [] {
        const char *e = getenv("OSERVE_SHARD_MIN");
        return e ? static_cast<uint64_t>(atoll(e)) : (uint64_t{1} << 16);
    }();
    return v;
}

// Shard the prepared space over the world?  Exact-path (branch-and-bound)
// spaces and small spaces run whole on the lead device of every rank.
bool shard_round(oserve_gpu_ctx &c) {
    if (c.g_world <= 1 || c.comms.empty()) return false;
    refresh_exact(c, c.space);
    return !c.space.any_exact && c.space.total >= shard_min_plans();
}

// K1 over every local shard + all-reduce(MIN) of the key; the global best
// key lands in d_key (lead device) on the lead's stream.  Asynchronous.
void sharded_launch_round(oserve_gpu_ctx &c, uint64_t *d_key) {
    auto sh = local_shards(c);
    std::vector<uint64_t *> keys(sh.size());
    for (size_t i = 0; i < sh.size(); ++i) {
        oserve_gpu_ctx &s = *sh[i];
        if (i) mirror(c, s);
        DeviceScope ds(s.device);
        ShardAs as(s, c.g_rank0 + static_cast<int>(i), c.g_world);
        keys[i] = i ? static_cast<uint64_t *>(s.d_mkey.get(sizeof(uint64_t))) : d_key;
        launch_round(s, keys[i]);
    }
    const Nccl &n = nccl_or_fail();
    nccl_ok(n.GroupStart(), "ncclGroupStart");
    for (size_t i = 0; i < sh.size(); ++i)
        nccl_ok(n.AllReduce(keys[i], keys[i], 1, ncclUint64, ncclMin, c.comms[i], sh[i]->stream), "ncclAllReduce");
    nccl_ok(n.GroupEnd(), "ncclGroupEnd");
}

// The round's key: sharded over the world when it pays, else this context's
// own shard (set_shard) — or the whole space when it has a communicator.
void round_key(oserve_gpu_ctx &c, uint64_t *d_key) {
    if (shard_round(c)) {
        sharded_launch_round(c, d_key);
    } else if (!c.comms.empty()) {
        ShardAs as(c, 0, 1);
        launch_round(c, d_key);
    } else {
        launch_round(c, d_key);
    }
}

// Top-K over every local shard (a host thread per device), all-gather of the
// per-shard lists, merge on the lead: sort world*K keys, keep the K smallest.
void sharded_topk(oserve_gpu_ctx &c, int K, uint64_t *d_keys, uint64_t *d_best) {
    auto sh = local_shards(c);
    for (size_t i = 1; i < sh.size(); ++i) mirror(c, *sh[i]);
    const size_t W = static_cast<size_t>(c.g_world);
    std::vector<uint64_t *> lk(sh.size()), all(sh.size());
    for (size_t i = 0; i < sh.size(); ++i) {
        DeviceScope ds(sh[i]->device);
        lk[i] = static_cast<uint64_t *>(sh[i]->d_mtopk.get(sizeof(uint64_t) * K));
        all[i] = static_cast<uint64_t *>(sh[i]->d_mall.get(sizeof(uint64_t) * K * W));
    }
    std::vector<std::exception_ptr> errs(sh.size());
    std::vector<uint64_t> h2d(sh.size(), 0), d2h(sh.size(), 0);
    auto work = [&](size_t i) {
        try {
            t_h2d = &h2d[i];
            t_d2h = &d2h[i];
            cuda_ok(cudaSetDevice(sh[i]->device), "cudaSetDevice");
            ShardAs as(*sh[i], c.g_rank0 + static_cast<int>(i), c.g_world);
            round_topk(*sh[i], K, lk[i], nullptr);
        } catch (...) {
            errs[i] = std::current_exception();
        }
    };
    {
        uint64_t *ch = t_h2d, *cd = t_d2h;
        std::vector<std::thread> th;
        for (size_t i = 1; i < sh.size(); ++i) th.emplace_back(work, i);
        work(0);
        for (auto &t : th) t.join();
        t_h2d = ch;
        t_d2h = cd;
        for (size_t i = 0; i < sh.size(); ++i) {
            count_h2d(h2d[i]);
            count_d2h(d2h[i]);
        }
        cuda_ok(cudaSetDevice(c.device), "cudaSetDevice");
    }
    for (auto &e : errs)
        if (e) std::rethrow_exception(e);
    const Nccl &n = nccl_or_fail();
    nccl_ok(n.GroupStart(), "ncclGroupStart");
    for (size_t i = 0; i < sh.size(); ++i)
        nccl_ok(n.AllGather(lk[i], all[i], static_cast<size_t>(K), ncclUint64, c.comms[i], sh[i]->stream),
                "ncclAllGather");
    nccl_ok(n.GroupEnd(), "ncclGroupEnd");
    cudaStream_t s = c.stream;
    uint64_t *tmp = static_cast<uint64_t *>(c.d_mtmp.get(sizeof(uint64_t) * K * W));
    cuda_ok(sort_keys(all[0], tmp, static_cast<int>(K * W), &c.cub_temp, &c.cub_temp_bytes, s), "sort");
    ++c.launches;
    cuda_ok(cudaMemcpyAsync(d_keys, tmp, sizeof(uint64_t) * K, cudaMemcpyDeviceToDevice, s), "D2D");
    if (d_best) cuda_ok(cudaMemcpyAsync(d_best, tmp, sizeof(uint64_t), cudaMemcpyDeviceToDevice, s), "D2D");
    cuda_ok(cudaStreamSynchronize(s), "sync");
}

void topk_any(oserve_gpu_ctx &c, int K, uint64_t *d_keys, uint64_t *d_best) {
    if (K < 1 || K > 65536) fail(OSERVE_ERR_INVALID_ARGUMENT, "K must be in [1, 65536]");
    if (shard_round(c)) {
        sharded_topk(c, K, d_keys, d_best);
    } else if (!c.comms.empty()) {
        ShardAs as(c, 0, 1);
        round_topk(c, K, d_keys, d_best);
    } else {
        round_topk(c, K, d_keys, d_best);
    }
}

}  // namespace

// ====================================================================== ABI
extern "C" {

const char *oserve_gpu_status_name(int status) {
    switch (status) {
        case OSERVE_OK: return "OK";
        case OSERVE_ERR_INVALID_ARGUMENT: return "INVALID_ARGUMENT";
        case OSERVE_ERR_INFEASIBLE_REPLICA: return "INFEASIBLE_REPLICA";
        case OSERVE_ERR_MODEL_TOO_LARGE: return "MODEL_TOO_LARGE";
        case OSERVE_ERR_TOO_LARGE: return "TOO_LARGE";
        case OSERVE_ERR_EMPTY_DEPLOYMENT: return "EMPTY_DEPLOYMENT";
        case OSERVE_ERR_UNSOURCED_FRAGMENT: return "UNSOURCED_FRAGMENT";
        case OSERVE_ERR_LOGIC: return "LOGIC";
        case OSERVE_ERR_UNSUPPORTED: return "UNSUPPORTED";
        case OSERVE_ERR_CUDA: return "CUDA";
        case OSERVE_ERR_NO_DEVICE: return "NO_DEVICE";
        case OSERVE_ERR_NCCL: return "NCCL";
        case OSERVE_ERR_LCM_OVERFLOW: return "LCM_OVERFLOW";
        default: return "UNKNOWN";
    }
}

int oserve_gpu_create(int cuda_device, const oserve_cluster_desc *cluster, const oserve_model_desc *model,
                      const oserve_profile *profile, oserve_gpu_ctx **out) {
    if (!out || !cluster || !model || !profile) return OSERVE_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return OSERVE_ERR_NO_DEVICE;
    if (cuda_device < 0 || cuda_device >= ndev) return OSERVE_ERR_NO_DEVICE;
    auto c = std::make_unique<oserve_gpu_ctx>();
    c->device = cuda_device;
    int pos = 0;
    for (int m = 0; m < cluster->num_machines; ++m) {
        c->machine_mem.push_back(cluster->device_mem[m]);
        for (int i = 0; i < cluster->machine_num_devices[m]; ++i) {
            int d = cluster->device_ids[pos++];
            c->machine_of.emplace(d, m);  // first machine wins (linear scan, core.cpp:29-35)
            c->dev_sorted.push_back(d);
        }
    }
    std::sort(c->dev_sorted.begin(), c->dev_sorted.end());
    if (c->dev_sorted.empty() || c->dev_sorted.size() > OSERVE_MAX_DEVICES) return OSERVE_ERR_UNSUPPORTED;
    c->intra = cluster->intra_bw;
    c->inter = cluster->inter_bw;
    c->model = *model;
    c->profile = *profile;
    int rc = guarded(c.get(), [&] {
        cuda_ok(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking), "stream");
        c->stream = c->own;
        cudaDeviceProp prop{};
        cuda_ok(cudaGetDeviceProperties(&prop, cuda_device), "props");
        c->sm_count = prop.multiProcessorCount;
        constexpr int kRingSlots = 64;  // one 128-byte line per K1 launch, round robin
        c->ring.base = static_cast<unsigned long long *>(c->d_ring.get(128 * kRingSlots));
        c->ring.slots = kRingSlots;
    });
    if (rc != OSERVE_OK) return rc;
    *out = c.release();
    return OSERVE_OK;
}

int oserve_gpu_create_multi(const int *cuda_devices, int ndev, const oserve_cluster_desc *cluster,
                            const oserve_model_desc *model, const oserve_profile *profile, oserve_gpu_ctx **out) {
    if (!out || !cuda_devices || ndev < 1) return OSERVE_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    for (int i = 0; i < ndev; ++i)
        for (int j = 0; j < i; ++j)
            if (cuda_devices[i] == cuda_devices[j]) return OSERVE_ERR_INVALID_ARGUMENT;
    oserve_gpu_ctx *lead = nullptr;
    int rc = oserve_gpu_create(cuda_devices[0], cluster, model, profile, &lead);
    if (rc != OSERVE_OK) return rc;
    std::unique_ptr<oserve_gpu_ctx> own(lead);
    for (int i = 1; i < ndev; ++i) {
        oserve_gpu_ctx *s = nullptr;
        rc = oserve_gpu_create(cuda_devices[i], cluster, model, profile, &s);
        if (rc != OSERVE_OK) return rc;
        lead->subs.push_back(s);
    }
    if (ndev > 1) {
        rc = guarded(lead, [&] {
            const Nccl &n = nccl_or_fail();
            std::vector<ncclComm_t> comms(ndev, nullptr);
            nccl_ok(n.CommInitAll(comms.data(), ndev, cuda_devices), "ncclCommInitAll");
            lead->comms = comms;
            lead->g_rank0 = 0;
            lead->g_world = ndev;
        });
        if (rc != OSERVE_OK) return rc;
    }
    *out = own.release();
    return OSERVE_OK;
}

int oserve_nccl_unique_id(void *id) {
    if (!id) return OSERVE_ERR_INVALID_ARGUMENT;
    const Nccl &n = nccl();
    if (!n.ok()) return OSERVE_ERR_NCCL;
    ncclUniqueId u;
    if (n.GetUniqueId(&u) != ncclSuccess) return OSERVE_ERR_NCCL;
    std::memcpy(id, &u, sizeof(u));
    return OSERVE_OK;
}

int oserve_gpu_join(oserve_gpu_ctx *ctx, const void *id, int rank, int world) {
    return guarded(ctx, [&] {
        if (!id || world < 1 || rank < 0 || rank >= world) fail(OSERVE_ERR_INVALID_ARGUMENT, "bad rank/world");
        if (!ctx->subs.empty() || !ctx->comms.empty())
            fail(OSERVE_ERR_INVALID_ARGUMENT, "context already has a communicator");
        if (world == 1) return;
        const Nccl &n = nccl_or_fail();
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof(u));
        ncclComm_t cm = nullptr;
        nccl_ok(n.CommInitRank(&cm, world, u, rank), "ncclCommInitRank");
        ctx->comms = {cm};
        ctx->g_rank0 = rank;
        ctx->g_world = world;
    });
}

int oserve_gpu_world(const oserve_gpu_ctx *ctx, int *rank, int *world, int *local_devices) {
    if (!ctx) return OSERVE_ERR_INVALID_ARGUMENT;
    if (rank) *rank = ctx->g_rank0;
    if (world) *world = ctx->g_world;
    if (local_devices) *local_devices = 1 + static_cast<int>(ctx->subs.size());
    return OSERVE_OK;
}

int oserve_gpu_destroy(oserve_gpu_ctx *ctx) {
    delete ctx;
    return OSERVE_OK;
}

const char *oserve_gpu_last_error(const oserve_gpu_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

uint64_t oserve_gpu_launch_count(const oserve_gpu_ctx *ctx) { return ctx ? ctx->launches : 0; }

uint64_t oserve_shard_count(uint64_t total, uint64_t chunk, int rank, int world) {
    if (chunk == 0 || world < 1 || rank < 0 || rank >= world) return 0;
    return shard_count_of(total, chunk, static_cast<uint64_t>(rank), static_cast<uint64_t>(world));
}

uint64_t oserve_shard_global_rank(uint64_t local, uint64_t chunk, int rank, int world) {
    // same mapping as the kernels' shard_rank (oserve_kernels.cu)
    const uint64_t c = local / chunk;
    return (c * static_cast<uint64_t>(world) + static_cast<uint64_t>(rank)) * chunk + (local - c * chunk);
}

int oserve_key_layout(int64_t total_demand, int64_t partitions, int devices, uint64_t max_plans_per_partition,
                      int *sh_obj, int *sh_part, int *sh_spp, uint64_t *obj_max) {
    KeyLayout k{};
    if (!key_layout(total_demand, partitions, devices, max_plans_per_partition, k)) return OSERVE_ERR_TOO_LARGE;
    *sh_obj = k.sh_obj;
    *sh_part = k.sh_part;
    *sh_spp = k.sh_spp;
    *obj_max = k.obj_max;
    return OSERVE_OK;
}

int oserve_gpu_copy_bytes(const oserve_gpu_ctx *ctx, uint64_t *h2d_bytes, uint64_t *d2h_bytes) {
    if (!ctx) return OSERVE_ERR_INVALID_ARGUMENT;
    if (h2d_bytes) *h2d_bytes = ctx->h2d_bytes;
    if (d2h_bytes) *d2h_bytes = ctx->d2h_bytes;
    return OSERVE_OK;
}

int oserve_gpu_set_workload(oserve_gpu_ctx *ctx, int num_classes, const oserve_class *classes, const int64_t *lambda,
                            double span_seconds) {
    return guarded(ctx, [&] {
        if (num_classes < 1 || num_classes > OSERVE_MAX_CLASSES)
            fail(OSERVE_ERR_UNSUPPORTED, "classes must be in [1, 16]");
        int64_t tot = 0;
        for (int j = 0; j < num_classes; ++j) {
            if (lambda[j] < 0) fail(OSERVE_ERR_INVALID_ARGUMENT, "negative demand");
            if (lambda[j] > 0x7fffffffll) fail(OSERVE_ERR_UNSUPPORTED, "demand per class must be < 2^31");
            tot += lambda[j];
        }
        if (tot > 0x7fffffffll) fail(OSERVE_ERR_UNSUPPORTED, "total demand must be < 2^31");
        std::vector<double> ci(num_classes), co(num_classes);
        for (int j = 0; j < num_classes; ++j) {
            ci[j] = classes[j].centroid_in;
            co[j] = classes[j].centroid_out;
        }
        ctx->tables_dirty = true;  // every round re-runs the cost kernel (K0) on its workload
        ++ctx->work_ver;
        ctx->J = num_classes;
        ctx->cin = ci;
        ctx->cout = co;
        ctx->lambda.assign(lambda, lambda + num_classes);
        ctx->span = span_seconds;
        ctx->have_workload = true;
    });
}

int oserve_gpu_set_solve_options(oserve_gpu_ctx *ctx, const oserve_solve_options *opts) {
    return guarded(ctx, [&] {
        if (!opts) fail(OSERVE_ERR_INVALID_ARGUMENT, "null options");
        ctx->opts = *opts;
    });
}

int oserve_gpu_set_shard(oserve_gpu_ctx *ctx, int rank, int world) {
    return guarded(ctx, [&] {
        if (world < 1 || rank < 0 || rank >= world) fail(OSERVE_ERR_INVALID_ARGUMENT, "bad shard");
        ctx->rank = rank;
        ctx->world = world;
    });
}

int oserve_gpu_set_stream(oserve_gpu_ctx *ctx, void *stream) {
    // Exactly the given stream (NULL = the legacy default stream), so callers
    // can order the round with their own work and events.
    return guarded(ctx, [&] { ctx->stream = static_cast<cudaStream_t>(stream); });
}

int oserve_gpu_min_feasible_group(oserve_gpu_ctx *ctx, int *g_min) {
    return guarded(ctx, [&] { *g_min = g_min_of(*ctx); });
}

int oserve_gpu_prepare_space(oserve_gpu_ctx *ctx, const oserve_space_desc *space, int64_t *partitions,
                             uint64_t *plans) {
    return guarded(ctx, [&] {
        ctx->space.valid = false;  // explicit call: always re-enumerate and re-upload
        prepare(*ctx, *space);
        if (partitions) *partitions = static_cast<int64_t>(ctx->space.parts.size());
        if (plans) *plans = ctx->space.total;
    });
}

int oserve_gpu_launch_round_async(oserve_gpu_ctx *ctx, uint64_t *d_key) {
    return guarded(ctx, [&] {
        if (!ctx->space.valid) fail(OSERVE_ERR_INVALID_ARGUMENT, "no prepared space");
        round_key(*ctx, d_key);
    });
}

int oserve_gpu_decode_key(oserve_gpu_ctx *ctx, uint64_t key, oserve_round_result *out) {
    return guarded(ctx, [&] {
        if (!ctx->space.valid) fail(OSERVE_ERR_INVALID_ARGUMENT, "no prepared space");
        decode_key(*ctx, key, out);
    });
}

int oserve_gpu_round(oserve_gpu_ctx *ctx, const oserve_space_desc *space, oserve_round_result *out) {
    return guarded(ctx, [&] {
        prepare(*ctx, *space);
        uint64_t *dk = static_cast<uint64_t *>(ctx->d_key.get(sizeof(uint64_t)));
        round_key(*ctx, dk);
        uint64_t key = kNoKey;
        cuda_ok(d2h(&key, dk, sizeof(key), ctx->stream), "D2H");
        cuda_ok(cudaStreamSynchronize(ctx->stream), "sync");
        decode_key(*ctx, key, out);
        if (key == kNoKey && (ctx->world == 1 || !ctx->comms.empty()))
            fail(OSERVE_ERR_MODEL_TOO_LARGE, "round: no feasible deployment");
    });
}

int oserve_gpu_round_topk(oserve_gpu_ctx *ctx, int K, uint64_t *d_keys, uint64_t *d_best) {
    return guarded(ctx, [&] {
        if (!ctx->space.valid) fail(OSERVE_ERR_INVALID_ARGUMENT, "no prepared space");
        topk_any(*ctx, K, d_keys, d_best);
    });
}

int oserve_gpu_switch_cost_keys(oserve_gpu_ctx *ctx, const oserve_deployment *current, int count,
                                const uint64_t *d_keys, double *est_seconds, uint64_t *max_link_bytes) {
    return guarded(ctx, [&] {
        if (count <= 0) return;
        switch_cost_keys(*ctx, *current, count, d_keys, est_seconds, max_link_bytes);
    });
}

int oserve_gpu_switch_cost_keys_async(oserve_gpu_ctx *ctx, const oserve_deployment *current, int count,
                                      const uint64_t *d_keys, double *d_est) {
    return guarded(ctx, [&] {
        if (count <= 0) return;
        if (!d_est) fail(OSERVE_ERR_INVALID_ARGUMENT, "null d_est");
        switch_cost_keys(*ctx, *current, count, d_keys, nullptr, nullptr, d_est);
    });
}

int oserve_gpu_kv_plan(oserve_gpu_ctx *ctx, int n_inflight, const oserve_inflight *inflight, int64_t threshold_tokens,
                       const oserve_deployment *src, const oserve_deployment *dst, double headroom, int n_carry,
                       const oserve_transfer *carry, int64_t *drained, int *n_drained, oserve_kv_transfer *migrated,
                       int *n_migrated, uint64_t *buffer_bytes) {
    return guarded(ctx, [&] {
        static const bool dbg = getenv("OSERVE_DEBUG_KV") != nullptr;
        auto t0 = std::chrono::steady_clock::now();
        auto lap = [&](const char *what) {
            if (!dbg) return;
            const auto t1 = std::chrono::steady_clock::now();
            std::fprintf(stderr, "[kv] %-10s %7.3f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
            t0 = t1;
        };
        if (headroom < 0.0 || headroom > 0.5) fail(OSERVE_ERR_INVALID_ARGUMENT, "kv_plan: headroom must be in [0, 0.5]");
        int m_tot = 0;  // migrating requests (also the validation pass)
        for (int q = 0; q < n_inflight; ++q) {
            const auto &r = inflight[q];
            if (r.generated_tokens <= threshold_tokens) continue;
            ++m_tot;
            if (r.source_replica < 0 || r.source_replica >= src->num_replicas)
                fail(OSERVE_ERR_INVALID_ARGUMENT, "kv_plan: request " + std::to_string(r.request_id) +
                                                      " names unknown source replica");
        }
        lap("validate");
        // device slots: cluster devices plus any id of the deployments / carry, ascending
        std::set<int> ids(ctx->dev_sorted.begin(), ctx->dev_sorted.end());
        auto add = [&](const oserve_deployment &d) {
            int n = 0;
            for (int r = 0; r < d.num_replicas; ++r) n += d.replica_num_devices[r];
            for (int i = 0; i < n; ++i) ids.insert(d.device_ids[i]);
        };
        add(*src);
        add(*dst);
        for (const oserve_deployment *d : {src, dst})  // an empty replica picks device -1 (switchplan.cpp:170-176)
            for (int r = 0; r < d->num_replicas; ++r)
                if (d->replica_num_devices[r] == 0) ids.insert(-1);
        for (int i = 0; i < n_carry; ++i) {
            ids.insert(carry[i].src);
            ids.insert(carry[i].dst);
        }
        if (ids.size() > 4096) fail(OSERVE_ERR_UNSUPPORTED, "kv_plan limited to 4096 devices");
        std::map<int, int> slot;
        std::vector<int32_t> machine, dev_id;
        for (int id : ids) {
            slot.emplace(id, static_cast<int>(dev_id.size()));
            dev_id.push_back(id);
            machine.push_back(ctx->machine(id));
        }
        const int NS = static_cast<int>(dev_id.size());
        auto flat = [&](const oserve_deployment &d, std::vector<int32_t> &off, std::vector<int32_t> &devs) {
            int pos = 0;
            off.push_back(0);
            for (int r = 0; r < d.num_replicas; ++r) {
                for (int i = 0; i < d.replica_num_devices[r]; ++i) devs.push_back(slot[d.device_ids[pos++]]);
                off.push_back(static_cast<int32_t>(devs.size()));
            }
        };
        std::vector<int32_t> soff, sdev, doff, ddev;
        flat(*src, soff, sdev);
        flat(*dst, doff, ddev);
        lap("slots");
        std::vector<uint64_t> load(static_cast<size_t>(NS) * NS, 0);
        for (int i = 0; i < n_carry; ++i)  // SwitchPlan::link_load from its transfers
            load[static_cast<size_t>(slot[carry[i].src]) * NS + slot[carry[i].dst]] += carry[i].end - carry[i].begin;
        lap("load");
        // Requests migrating to different target replicas are independent
        // (disjoint devices): partition them by target replica (round-robin
        // over the migrated sequence, switchplan.cpp:178-181) for the
        // warp-per-replica kernel, unless a target replica is empty.
        bool par = dst->num_replicas > 1;
        for (int r = 0; r < dst->num_replicas && par; ++r)
            if (dst->replica_num_devices[r] == 0) par = false;
        if (par) {  // replicas must not share a device (the state partition relies on it)
            std::set<int32_t> seen(ddev.begin(), ddev.end());
            if (seen.size() != ddev.size()) par = false;
        }
        cudaStream_t s = ctx->stream;
        DBuf *b = ctx->sc_kv;
        KvPlanIn in{};
        in.n = n_inflight;
        in.threshold = threshold_tokens;
        in.num_slots = NS;
        in.none_slot = slot.count(-1) ? slot[-1] : -1;
        in.src_reps = src->num_replicas;
        in.dst_reps = dst->num_replicas;
        in.n_src_devs = static_cast<int>(sdev.size());
        in.n_dst_devs = static_cast<int>(ddev.size());
        in.h_dst_off = doff.data();
        const int R = dst->num_replicas;
        std::vector<int32_t> goff, gsr, gpos;  // gpos: group position of the m-th migrated request
        std::vector<uint64_t> gkv;
        std::vector<int64_t> gen;
        std::vector<uint64_t> kv;
        std::vector<int32_t> sr;
        if (par) {
            // the m-th migrated request goes to target replica m mod R: group
            // sizes follow from the count, no per-request division
            goff.assign(static_cast<size_t>(R) + 1, 0);
            for (int r = 0; r < R; ++r) goff[r + 1] = goff[r] + m_tot / R + (r < m_tot % R ? 1 : 0);
            gkv.resize(static_cast<size_t>(std::max(m_tot, 1)));
            gsr.resize(gkv.size());
            gpos.resize(gkv.size());
            std::vector<int32_t> fill(goff.begin(), goff.end() - 1);
            int m = 0, r = 0;
            for (int q = 0; q < n_inflight; ++q) {
                if (inflight[q].generated_tokens <= threshold_tokens) continue;
                const int at = fill[r]++;
                r = r + 1 == R ? 0 : r + 1;
                gkv[at] = inflight[q].kv_bytes;
                gsr[at] = inflight[q].source_replica;
                gpos[m++] = at;
            }
        } else {
            gen.resize(n_inflight);
            kv.resize(n_inflight);
            sr.resize(n_inflight);
            for (int q = 0; q < n_inflight; ++q) {
                gen[q] = inflight[q].generated_tokens;
                kv[q] = inflight[q].kv_bytes;
                sr[q] = inflight[q].source_replica;
            }
        }
        lap("host prep");
        in.machine = b[3].upload(machine, s);
        in.dev_id = b[4].upload(dev_id, s);
        in.src_off = b[5].upload(soff, s);
        in.src_devs = b[6].upload(sdev, s);
        in.dst_off = b[7].upload(doff, s);
        in.dst_devs = b[8].upload(ddev, s);
        in.load = b[9].upload(load, s);
        in.inbound = static_cast<uint64_t *>(b[10].get(sizeof(uint64_t) * NS));
        cuda_ok(cudaMemsetAsync(in.inbound, 0, sizeof(uint64_t) * NS, s), "memset");
        if (par) {
            DBuf *pb = ctx->sc_kv + 14;
            in.grp_off = pb[0].upload(goff, s);
            in.grp_kv = b[1].upload(gkv, s);
            in.grp_sr = b[2].upload(gsr, s);
            in.grp_src = static_cast<int32_t *>(b[12].get(sizeof(int32_t) * gkv.size()));
            in.grp_dst = static_cast<int32_t *>(b[13].get(sizeof(int32_t) * gkv.size()));
        } else {
            in.gen = b[0].upload(gen, s);
            in.kv = b[1].upload(kv, s);
            in.srcrep = b[2].upload(sr, s);
            in.kind = static_cast<int32_t *>(b[11].get(sizeof(int32_t) * std::max(n_inflight, 1)));
            in.mig_src = static_cast<int32_t *>(b[12].get(sizeof(int32_t) * std::max(n_inflight, 1)));
            in.mig_dst = static_cast<int32_t *>(b[13].get(sizeof(int32_t) * std::max(n_inflight, 1)));
        }
        lap("upload");
        cuda_ok(launch_kv_plan(in, s, &ctx->launches), "kv_plan kernel");
        if (dbg) cuda_ok(cudaStreamSynchronize(s), "sync");
        lap("kernel");
        std::vector<int32_t> kind, ms, md;
        if (par) {
            download(ms, in.grp_src, static_cast<size_t>(m_tot), s);
            download(md, in.grp_dst, static_cast<size_t>(m_tot), s);
        } else {
            download(kind, in.kind, n_inflight, s);
            download(ms, in.mig_src, n_inflight, s);
            download(md, in.mig_dst, n_inflight, s);
        }
        cuda_ok(cudaStreamSynchronize(s), "sync");
        lap("download");
        int nd = 0, nm = 0;
        uint64_t migrated_bytes = 0;
        for (int q = 0; q < n_inflight; ++q) {
            const bool mig = par ? inflight[q].generated_tokens > threshold_tokens : kind[q] != 0;
            if (!mig) {
                drained[nd++] = inflight[q].request_id;
            } else {
                const size_t at = par ? static_cast<size_t>(gpos[nm]) : static_cast<size_t>(q);
                migrated[nm++] = {inflight[q].request_id, inflight[q].kv_bytes, ms[at], md[at]};
                migrated_bytes += inflight[q].kv_bytes;
            }
        }
        *n_drained = nd;
        *n_migrated = nm;
        *buffer_bytes = static_cast<uint64_t>(std::ceil(static_cast<double>(migrated_bytes) * (1.0 + headroom)));
        lap("assemble");
    });
}

int oserve_forecast_series(int J, int T, const int64_t *counts, int window, double alpha, double beta,
                           int64_t *lambda_out) {
    if (J < 1 || T < 0 || window < 1) return OSERVE_ERR_INVALID_ARGUMENT;
    for (int t = 0; t < T; ++t) {
        for (int j = 0; j < J; ++j) {
            if (t == 0) {  // cold start: the first span's own counts
                lambda_out[j] = counts[j];
                continue;
            }
            // HoltForecaster::predict over the trailing window (workload.cpp:204-222, :231-244)
            const int start = std::max(0, t - window);
            double level = static_cast<double>(counts[static_cast<size_t>(start) * J + j]), trend = 0.0;
            for (int u = start + 1; u < t; ++u) {
                const double prev = level;
                level = alpha * static_cast<double>(counts[static_cast<size_t>(u) * J + j]) +
                        (1.0 - alpha) * (level + trend);
                trend = beta * (level - prev) + (1.0 - beta) * trend;
            }
            const double v = std::max(0.0, std::max(0.0, level + trend));
            lambda_out[static_cast<size_t>(t) * J + j] = std::max<int64_t>(0, std::llround(v));
        }
    }
    return OSERVE_OK;
}

int oserve_gpu_exhaustive(oserve_gpu_ctx *ctx, oserve_round_result *out) {
    oserve_space_desc d{OSERVE_SPACE_ORDERED, 0, nullptr, 16};
    int rc = oserve_gpu_round(ctx, &d, out);
    return rc;
}

int oserve_gpu_best_strategies(oserve_gpu_ctx *ctx, int num_replicas, const int *sizes, oserve_round_result *out) {
    return guarded(ctx, [&] {
        std::vector<int> sz(sizes, sizes + num_replicas);
        std::sort(sz.begin(), sz.end(), std::greater<int>());
        int tot = std::accumulate(sz.begin(), sz.end(), 0);
        if (tot > ctx->D()) fail(OSERVE_ERR_INVALID_ARGUMENT, "canonical_blocks: sizes exceed cluster device count");
        for (int s : sz)
            if (s < 1) fail(OSERVE_ERR_INVALID_ARGUMENT, "replica size must be >= 1");
        Space &sp = ctx->space;
        if (!(sp.valid && sp.explicit_partition && sp.explicit_sizes == sz)) {
            sp.valid = false;
            std::vector<std::vector<int>> parts{sz};
            build_space(*ctx, sp, OSERVE_SPACE_ORDERED, {}, &parts);
            sp.explicit_partition = true;
            sp.explicit_sizes = sz;
            sp.mode = OSERVE_SPACE_ORDERED;
        }
        std::memset(out, 0, sizeof(*out));
        out->partitions = 1;
        if (sp.total == 0) return;  // a block without candidates: empty choice, objective 0
        uint64_t *dk = static_cast<uint64_t *>(ctx->d_key.get(sizeof(uint64_t)));
        round_key(*ctx, dk);
        uint64_t key = kNoKey;
        cuda_ok(d2h(&key, dk, sizeof(key), ctx->stream), "D2H");
        cuda_ok(cudaStreamSynchronize(ctx->stream), "sync");
        decode_key(*ctx, key, out);
        if (out->objective < 0) out->objective = 0;
    });
}

// ---------------------------------------------------------------------------
// search::search (deploysearch.cpp:341-417): the reference's host loop, with
// best_strategies and the per-iteration capacity table + assignment on the
// GPU.  classify (:57-75), mutate_sizes (:240-319), absorb_leftovers
// (:324-337) and init_uniform (:120-136) are restated; the mt19937_64 stream
// and every draw (rng() % n) happen in the reference's order.
namespace {

struct Mutation {
    std::vector<int> sizes;
    std::string op;
};

Mutation mutate_sizes(const std::vector<int> &sizes, const std::vector<int> &pps, const std::vector<int> &over,
                      const std::vector<int> &under, int g_min, std::mt19937_64 &rng) {
    std::vector<int> sz = sizes;
    std::vector<char> alive(sz.size(), 1);
    std::ostringstream ops;
    auto below = [&](uint64_t n) { return rng() % n; };
    auto alive_in = [&](const std::vector<int> &set, int except) {
        std::vector<int> o;
        for (int r : set)
            if (r != except && alive[r]) o.push_back(r);
        return o;
    };
    std::vector<std::pair<int, int>> splits;
    for (int r : over) {
        if (!alive[r]) continue;
        const bool try_merge = below(2) == 0;
        std::vector<int> others = alive_in(over, r);
        std::vector<int> donors;
        for (int u : alive_in(under, -1))
            if (sz[u] > g_min) donors.push_back(u);
        if (try_merge && !others.empty()) {
            const int r2 = others[below(others.size())];
            sz[r] += sz[r2];
            alive[r2] = 0;
            ops << "merge(" << r << "," << r2 << ");";
        } else if (!donors.empty()) {
            const int u = donors[below(donors.size())];
            int delta = std::max(1, sz[u] / std::max(1, pps[u]));
            delta = std::min(delta, sz[u] - g_min);
            if (delta <= 0) continue;
            sz[r] += delta;
            sz[u] -= delta;
            ops << "swap(" << r << "<-" << u << ",d=" << delta << ");";
        } else if (!others.empty()) {
            const int r2 = others[below(others.size())];
            sz[r] += sz[r2];
            alive[r2] = 0;
            ops << "merge(" << r << "," << r2 << ");";
        }
    }
    for (int r : under) {
        if (!alive[r]) continue;
        const bool try_split = below(2) == 0;
        const bool can_split = sz[r] >= 2 * g_min;
        std::vector<int> receivers = alive_in(over, -1);
        int delta = std::max(1, sz[r] / std::max(1, pps[r]));
        delta = std::min(delta, sz[r] - g_min);
        const bool can_swap = !receivers.empty() && delta > 0;
        if (try_split && can_split) {
            splits.emplace_back(r, sz[r] / 2);
            ops << "split(" << r << ");";
        } else if (can_swap) {
            const int o = receivers[below(receivers.size())];
            sz[o] += delta;
            sz[r] -= delta;
            ops << "swap(" << o << "<-" << r << ",d=" << delta << ");";
        } else if (can_split) {
            splits.emplace_back(r, sz[r] / 2);
            ops << "split(" << r << ");";
        }
    }
    Mutation m;
    for (size_t r = 0; r < sz.size(); ++r) {
        if (!alive[r]) continue;
        auto it = std::find_if(splits.begin(), splits.end(), [&](const auto &p) { return p.first == static_cast<int>(r); });
        if (it != splits.end()) {
            m.sizes.push_back(it->second);
            m.sizes.push_back(sz[r] - it->second);
        } else {
            m.sizes.push_back(sz[r]);
        }
    }
    m.op = ops.str();
    return m;
}

std::vector<int> absorb_leftovers(std::vector<int> sizes, int D, int g_min) {
    int left = D - std::accumulate(sizes.begin(), sizes.end(), 0);
    while (left >= g_min) {
        sizes.push_back(g_min);
        left -= g_min;
    }
    while (left > 0 && !sizes.empty()) {
        *std::min_element(sizes.begin(), sizes.end()) += 1;
        --left;
    }
    return sizes;
}

int64_t device_total(const oserve_plan &p) {
    int64_t n = 0;
    for (int r = 0; r < p.num_replicas; ++r) n += p.replica_num_devices[r];
    return n;
}

void check_status(int st, oserve_gpu_ctx *ctx) {
    if (st != OSERVE_OK) fail(st, ctx->err);
}

}  // namespace

int oserve_gpu_search(oserve_gpu_ctx *ctx, const oserve_search_options *opts, oserve_search_result *out,
                      oserve_search_log_row *log, int log_capacity) {
    if (!ctx || !opts || !out) return OSERVE_ERR_INVALID_ARGUMENT;
    std::string err;
    int code = OSERVE_OK;
    try {
        const int g_min = [&] {
            int g = 0;
            check_status(oserve_gpu_min_feasible_group(ctx, &g), ctx);
            return g;
        }();
        const int D = ctx->D();
        std::vector<int> sizes;
        if (opts->warm_start && opts->warm_start->num_replicas > 0) {
            for (int r = 0; r < opts->warm_start->num_replicas; ++r)
                sizes.push_back(opts->warm_start->replica_num_devices[r]);
        } else {
            // init_uniform: D / g_min replicas of g_min devices, each block must
            // have a feasible strategy
            const int R = D / g_min;
            for (int r = 0; r < R; ++r) {
                std::vector<int> ids;
                candidates(*ctx, r * g_min, g_min, ids);
                if (ids.empty())
                    fail(OSERVE_ERR_MODEL_TOO_LARGE, "no feasible strategy for a " + std::to_string(g_min) +
                                                         "-device replica");
                sizes.push_back(g_min);
            }
        }
        sizes = absorb_leftovers(std::move(sizes), D, g_min);
        auto current = std::make_unique<oserve_round_result>();
        check_status(oserve_gpu_best_strategies(ctx, static_cast<int>(sizes.size()), sizes.data(), current.get()), ctx);
        if (current->plan.num_replicas == 0)
            fail(OSERVE_ERR_MODEL_TOO_LARGE, "search: no feasible strategy for the initial deployment");
        std::mt19937_64 rng(opts->seed);
        int stale = 0, iter = 0, nlog = 0;
        auto emit = [&](const std::string &op, bool accepted) {
            if (log && nlog < log_capacity) {
                oserve_search_log_row &row = log[nlog];
                row.iteration = iter;
                row.accepted = accepted ? 1 : 0;
                row.throughput = current->objective;
                row.devices = static_cast<int>(device_total(current->plan));
                std::snprintf(row.op, sizeof(row.op), "%s", op.c_str());
            }
            ++nlog;
        };
        auto candidate = std::make_unique<oserve_round_result>();
        // best_strategies is a pure function of the ordered sizes for this
        // context and workload, and the search revisits the same mutations
        // again and again while the current deployment stands (the reference
        // recomputes them): results are memoised per sizes vector, and the
        // current deployment's classification is redone only when it changes.
        std::map<std::vector<int>, std::unique_ptr<oserve_round_result>> memo;
        bool classified = false;
        std::vector<int> over, under, cur_sizes, cur_pps;
        while (iter < opts->max_iters && stale < opts->stale_limit) {
            ++iter;
            // capacity table + assignment of the current deployment (GPU), classify
            const oserve_plan &cp = current->plan;
            const int R = cp.num_replicas, J = ctx->J;
            if (!classified) {
                oserve_deployment dd{R, cp.replica_num_devices, cp.device_ids, cp.tp, cp.pp};
                std::vector<int64_t> M(R), unit(static_cast<size_t>(R) * J), used(R);
                check_status(oserve_gpu_plan_detail(ctx, &dd, nullptr, nullptr, nullptr, nullptr, M.data(), unit.data(),
                                                    used.data(), nullptr),
                             ctx);
                over.clear();
                under.clear();
                cur_sizes.clear();
                cur_pps.clear();
                for (int k = 0; k < R; ++k) {
                    int64_t min_unit = std::numeric_limits<int64_t>::max();
                    for (int j = 0; j < J; ++j)
                        if (unit[k * J + j] > 0) min_unit = std::min(min_unit, unit[k * J + j]);
                    const bool saturated =
                        min_unit != std::numeric_limits<int64_t>::max() && M[k] - used[k] < min_unit;
                    (saturated ? over : under).push_back(k);
                    cur_sizes.push_back(cp.replica_num_devices[k]);
                    cur_pps.push_back(cp.pp[k]);
                }
                classified = true;
            }
            Mutation mut;
            bool found = false;
            for (int attempt = 0; attempt < opts->mutation_retries && !found; ++attempt) {
                mut = mutate_sizes(cur_sizes, cur_pps, over, under, g_min, rng);
                std::vector<int> a = mut.sizes, b = cur_sizes;
                std::sort(a.begin(), a.end());
                std::sort(b.begin(), b.end());
                found = !mut.op.empty() && a != b;
            }
            if (!found) {
                ++stale;
                emit("stale(no-mutation)", false);
                continue;
            }
            auto hit = memo.find(mut.sizes);
            if (hit != memo.end()) {
                *candidate = *hit->second;
            } else {
                check_status(oserve_gpu_best_strategies(ctx, static_cast<int>(mut.sizes.size()), mut.sizes.data(),
                                                        candidate.get()),
                             ctx);
                memo.emplace(mut.sizes, std::make_unique<oserve_round_result>(*candidate));
            }
            const bool accepted = candidate->plan.num_replicas > 0 && candidate->objective > current->objective;
            if (accepted) {
                std::swap(current, candidate);
                classified = false;
                stale = 0;
            } else {
                ++stale;
            }
            emit(mut.op, accepted);
        }
        std::memset(out, 0, sizeof(*out));
        out->throughput = current->objective;
        out->rng_seed = opts->seed;
        out->stale_iters = stale;
        out->iterations = iter;
        out->log_count = nlog;
        out->deployment = current->plan;
        ctx->err.clear();
    } catch (const Fail &e) {
        code = e.code;
        err = e.what();
    } catch (const std::exception &e) {
        code = OSERVE_ERR_INVALID_ARGUMENT;
        err = e.what();
    }
    if (code != OSERVE_OK) ctx->err = err;
    return code;
}

int oserve_gpu_evaluate_ranks(oserve_gpu_ctx *ctx, uint64_t first, uint64_t count, int64_t *objective,
                              int32_t *sum_pp) {
    return guarded(ctx, [&] {
        Space &sp = ctx->space;
        if (!sp.valid) fail(OSERVE_ERR_INVALID_ARGUMENT, "no prepared space");
        if (first + count > sp.total) fail(OSERVE_ERR_INVALID_ARGUMENT, "rank range out of the space");
        ensure_tables(*ctx);
        refresh_exact(*ctx, sp);
        cudaStream_t s = ctx->stream;
        PlanSource src{};
        src.mode = 0;
        src.first = first;
        src.count = count;
        src.rank = 0;
        src.world = 1;
        src.chunk = ~0ull >> 2;
        PlanOutputs out{};
        out.objective = static_cast<int64_t *>(ctx->d_obj.get(sizeof(int64_t) * count));
        out.sum_pp = static_cast<int32_t *>(ctx->d_spp.get(sizeof(int32_t) * count));
        SolveParams prm = solve_params(*ctx);
        KeyLayout nk{};
        cuda_ok(launch_plan_eval(ctx->tables, sp.view, nk, src, out, prm, sp.rmax, ctx->sm_count, sp.any_exact, &ctx->ring, s,
                                 &ctx->launches),
                "plan kernel");
        if (sp.any_exact) {
            uint64_t *ab = static_cast<uint64_t *>(ctx->d_aborted.get(sizeof(uint64_t) * count));
            unsigned *abn = static_cast<unsigned *>(ctx->d_aborted_n.get(sizeof(unsigned)));
            cuda_ok(cudaMemsetAsync(abn, 0, sizeof(unsigned), s), "memset");
            PlanOutputs eo = out;
            eo.aborted = ab;
            eo.aborted_n = abn;
            run_exact(*ctx, sp.view, nk, src, eo, prm, nullptr);
            unsigned n_ab = 0;
            cuda_ok(d2h(&n_ab, abn, sizeof(unsigned), s), "D2H");
            cuda_ok(cudaStreamSynchronize(s), "sync");
            if (n_ab) {
                std::vector<uint64_t> ranks;
                download(ranks, ab, n_ab, s);
                cuda_ok(cudaStreamSynchronize(s), "sync");
                for (uint64_t g : ranks) {
                    PlanSource one = src;
                    one.first = g;
                    one.count = 1;
                    PlanOutputs o1 = out;
                    o1.objective = out.objective + (g - first);
                    o1.sum_pp = out.sum_pp + (g - first);
                    cuda_ok(launch_plan_eval(ctx->tables, sp.view, nk, one, o1, prm, sp.rmax, ctx->sm_count, 0, &ctx->ring, s,
                                             &ctx->launches),
                            "plan kernel (budget fallback)");
                }
            }
        }
        if (objective)
            cuda_ok(d2h(objective, out.objective, sizeof(int64_t) * count, s), "D2H");
        if (sum_pp)
            cuda_ok(d2h(sum_pp, out.sum_pp, sizeof(int32_t) * count, s), "D2H");
        cuda_ok(cudaStreamSynchronize(s), "sync");
    });
}

int oserve_gpu_evaluate_deployments(oserve_gpu_ctx *ctx, int count, const oserve_deployment *deps,
                                    int64_t *objective) {
    return guarded(ctx, [&] {
        std::vector<int32_t> listR, listOff, shapes;
        std::vector<int> idx;  // non-empty deployments
        int rmax = 1;
        for (int i = 0; i < count; ++i) {
            objective[i] = 0;  // evaluate_deployment: empty -> 0 (deploysearch.cpp:139)
            if (deps[i].num_replicas == 0) continue;
            if (deps[i].num_replicas > OSERVE_MAX_REPLICAS) fail(OSERVE_ERR_UNSUPPORTED, "more than 128 replicas");
            auto ids = deployment_shapes(*ctx, deps[i]);
            listR.push_back(static_cast<int32_t>(ids.size()));
            listOff.push_back(static_cast<int32_t>(shapes.size()));
            shapes.insert(shapes.end(), ids.begin(), ids.end());
            rmax = std::max(rmax, static_cast<int>(ids.size()));
            idx.push_back(i);
        }
        if (idx.empty()) return;
        ensure_tables(*ctx);
        std::vector<int64_t> obj;
        eval_lists(*ctx, listR, listOff, shapes, nullptr, rmax, obj, nullptr, nullptr, solve_params(*ctx));
        for (size_t q = 0; q < idx.size(); ++q) objective[idx[q]] = obj[q];
    });
}

int oserve_gpu_plan_detail(oserve_gpu_ctx *ctx, const oserve_deployment *dep, int64_t *n, int64_t *e, double *latency,
                           int64_t *x, int64_t *M, int64_t *unit, int64_t *used, int64_t *objective) {
    return guarded(ctx, [&] {
        const int R = dep->num_replicas, J = ctx->J;
        if (R == 0) {
            if (objective) *objective = 0;
            return;
        }
        if (R > OSERVE_MAX_REPLICAS) fail(OSERVE_ERR_UNSUPPORTED, "more than 128 replicas");
        auto ids = deployment_shapes(*ctx, *dep);
        ensure_tables(*ctx);
        std::vector<int32_t> listR{R}, listOff{0}, shapes(ids.begin(), ids.end());
        std::vector<int64_t> obj, xs, us;
        eval_lists(*ctx, listR, listOff, shapes, nullptr, R, obj, &xs, &us, solve_params(*ctx));
        // shape rows (n, e, latency, M, unit) from the device tables (host
        // copies refreshed once per K0 run)
        const int S = ctx->tables.num_shapes;
        if (ctx->host_tables_ver != ctx->tables_ver) {
            cudaStream_t s = ctx->stream;
            download(ctx->h_n, ctx->tables.n, S * J, s);
            download(ctx->h_e, ctx->tables.e, S * J, s);
            download(ctx->h_lat, ctx->tables.latency, S * J, s);
            download(ctx->h_M, ctx->tables.M, S, s);
            download(ctx->h_unit, ctx->tables.unit, S * J, s);
            cuda_ok(cudaStreamSynchronize(s), "sync");
            ctx->host_tables_ver = ctx->tables_ver;
        }
        const auto &hn = ctx->h_n, &he = ctx->h_e, &hM = ctx->h_M, &hu = ctx->h_unit;
        const auto &hl = ctx->h_lat;
        for (int k = 0; k < R; ++k) {
            const int sh = ids[k];
            for (int j = 0; j < J; ++j) {
                if (n) n[k * J + j] = hn[sh * J + j];
                if (e) e[k * J + j] = he[sh * J + j];
                if (latency) latency[k * J + j] = hl[sh * J + j];
                if (unit) unit[k * J + j] = hu[sh * J + j];
                if (x) x[k * J + j] = xs[k * J + j];
            }
            if (M) M[k] = hM[sh];
            if (used) used[k] = us[k];
        }
        if (objective) *objective = obj[0];
    });
}

void validate_raw(int count, int R, int J, const int64_t *n, const int64_t *lambda) {
    if (J < 1 || J > OSERVE_MAX_CLASSES) fail(OSERVE_ERR_UNSUPPORTED, "classes must be in [1, 16]");
    if (R < 1 || R > OSERVE_MAX_REPLICAS) fail(OSERVE_ERR_UNSUPPORTED, "replicas must be in [1, 128]");
    const int64_t rows = static_cast<int64_t>(count) * R;
    for (int64_t i = 0; i < rows * J; ++i) {
        if (n[i] < 0) fail(OSERVE_ERR_INVALID_ARGUMENT, "normalize: negative capacity");
    }
    for (int64_t i = 0; i < static_cast<int64_t>(count); ++i) {
        int64_t tot = 0;
        for (int j = 0; j < J; ++j) {
            if (lambda[i * J + j] < 0 || lambda[i * J + j] > 0x7fffffffll)
                fail(OSERVE_ERR_UNSUPPORTED, "demand per class must be in [0, 2^31)");
            tot += lambda[i * J + j];
        }
        if (tot > 0x7fffffffll) fail(OSERVE_ERR_UNSUPPORTED, "total demand must be < 2^31");
    }
}

void stage_raw_rows(oserve_gpu_ctx &c, int64_t rows, int J, const int64_t *n, const int64_t *e, RawRows &rr) {
    cudaStream_t s = c.stream;
    ShapeTables &t = rr.t;
    t.num_shapes = static_cast<int>(rows);
    t.J = J;
    t.n = static_cast<int64_t *>(rr.dn.get(sizeof(int64_t) * rows * J));
    t.e = static_cast<int64_t *>(rr.de.get(sizeof(int64_t) * rows * J));
    cuda_ok(h2d(t.n, n, sizeof(int64_t) * rows * J, s), "H2D");
    cuda_ok(h2d(t.e, e, sizeof(int64_t) * rows * J, s), "H2D");
    t.latency = static_cast<double *>(rr.dlat.get(8));
    t.M = static_cast<int64_t *>(rr.dM.get(sizeof(int64_t) * rows));
    t.unit = static_cast<int64_t *>(rr.du.get(sizeof(int64_t) * rows * J));
    t.inv_unit = static_cast<double *>(rr.dinv.get(sizeof(double) * rows * J));
    t.cap = static_cast<int32_t *>(rr.dc.get(sizeof(int32_t) * rows * J));
    t.order = static_cast<uint8_t *>(rr.dord.get(rows * kMaxJ));
    t.rank = static_cast<uint8_t *>(rr.drank.get(rows * kMaxJ));
    t.pmask = static_cast<uint16_t *>(rr.dpmask.get(sizeof(uint16_t) * rows * kMaxJ));
    t.olen = static_cast<uint8_t *>(rr.dol.get(rows));
    t.scaled = static_cast<uint8_t *>(rr.dsc.get(rows));
    t.pp = static_cast<uint8_t *>(rr.dpp.get(rows));
    cuda_ok(cudaMemsetAsync(t.pp, 1, rows, s), "memset");
    cuda_ok(launch_normalize_rows(t, s), "normalize kernel");
    c.launches += 1;
}

// solve_assignment over the staged rows of instances `which` (each R rows);
// aborted_out (when given) receives the local indices whose B&B blew the
// node budget instead of running the heuristic fallback for them.
void solve_staged(oserve_gpu_ctx &c, RawRows &rr, const std::vector<int> &which, int R, int J,
                  const int64_t *lambda, std::vector<int64_t> &obj, std::vector<int64_t> &xs,
                  std::vector<int64_t> &us, std::vector<uint64_t> *aborted_out) {
    const int cnt = static_cast<int>(which.size());
    std::vector<int32_t> listR(cnt, R), listOff(cnt), shapes(static_cast<size_t>(cnt) * R);
    std::vector<int64_t> lam(static_cast<size_t>(cnt) * J);
    for (int q = 0; q < cnt; ++q) {
        listOff[q] = q * R;
        for (int k = 0; k < R; ++k) shapes[static_cast<size_t>(q) * R + k] = which[q] * R + k;
        for (int j = 0; j < J; ++j) lam[static_cast<size_t>(q) * J + j] = lambda[static_cast<int64_t>(which[q]) * J + j];
    }
    SolveParams prm = solve_params(c);
    prm.J = J;
    ShapeTables saved = c.tables;
    c.tables = rr.t;
    try {
        eval_lists(c, listR, listOff, shapes, &lam, R, obj, &xs, &us, prm, aborted_out);
    } catch (...) {
        c.tables = saved;
        throw;
    }
    c.tables = saved;
}

int oserve_gpu_solve_batch(oserve_gpu_ctx *ctx, int count, int R, int J, const int64_t *n, const int64_t *e,
                           const int64_t *lambda, int64_t *x, int64_t *objective, int64_t *M, int64_t *unit,
                           int64_t *used) {
    return guarded(ctx, [&] {
        if (count <= 0) return;
        validate_raw(count, R, J, n, lambda);
        const int64_t rows = static_cast<int64_t>(count) * R;
        cudaStream_t s = ctx->stream;
        RawRows &rr = ctx->raw;
        stage_raw_rows(*ctx, rows, J, n, e, rr);
        std::vector<int> all(count);
        std::iota(all.begin(), all.end(), 0);
        std::vector<int64_t> obj, xs, us;
        solve_staged(*ctx, rr, all, R, J, lambda, obj, xs, us, nullptr);
        std::vector<int64_t> hM, hu;
        download(hM, rr.t.M, rows, s);
        download(hu, rr.t.unit, rows * J, s);
        cuda_ok(cudaStreamSynchronize(s), "sync");
        for (int i = 0; i < count; ++i) {
            if (objective) objective[i] = obj[i];
            for (int k = 0; k < R; ++k) {
                const int64_t row = static_cast<int64_t>(i) * R + k;
                for (int j = 0; j < J; ++j) {
                    if (x) x[row * J + j] = xs[row * J + j];
                    if (unit) unit[row * J + j] = hu[row * J + j];
                }
                if (M) M[row] = hM[row];
                if (used) used[row] = us[row];
            }
        }
    });
}

namespace {
int flow_assign_impl(oserve_gpu_ctx *ctx, int count, int R, int J, const int64_t *n, const int64_t *e,
                     const int64_t *lambda, const int64_t *flow_in, int64_t *x, int64_t *objective,
                     int64_t *flow_value, int64_t *edge_flow) {
    return guarded(ctx, [&] {
        if (count <= 0) return;
        validate_raw(count, R, J, n, lambda);
        const int64_t rows = static_cast<int64_t>(count) * R;
        cudaStream_t s = ctx->stream;
        RawRows &rr = ctx->raw;
        stage_raw_rows(*ctx, rows, J, n, e, rr);
        // K6b: network, push-relabel, rounded chain flows, warm greedy + exchange
        size_t n32 = 0, n64 = 0, n8 = 0;
        flow_assign_workspace(R, J, count, &n32, &n64, &n8);
        const int m = J + 2 * R * J + 2 * R;
        DBuf &w32 = ctx->sc_fa[0], &w64 = ctx->sc_fa[1], &w8 = ctx->sc_fa[2], &dlam = ctx->sc_fa[3], &dx = ctx->sc_fa[4], &dobj = ctx->sc_fa[5], &dval = ctx->sc_fa[6], &dflow = ctx->sc_fa[7], &dst = ctx->sc_fa[8];
        FlowAssignBatch fb{};
        fb.count = count;
        fb.R = R;
        fb.J = J;
        fb.lambda = dlam.upload(lambda, static_cast<size_t>(count) * J, s);
        fb.ws_i32 = static_cast<int32_t *>(w32.get(sizeof(int32_t) * n32));
        fb.ws_i64 = static_cast<int64_t *>(w64.get(sizeof(int64_t) * n64));
        fb.ws_u8 = static_cast<uint8_t *>(w8.get(n8));
        fb.x = static_cast<int64_t *>(dx.get(sizeof(int64_t) * rows * J));
        fb.objective = static_cast<int64_t *>(dobj.get(sizeof(int64_t) * count));
        fb.value = static_cast<int64_t *>(dval.get(sizeof(int64_t) * count));
        fb.edge_flow = edge_flow ? static_cast<int64_t *>(dflow.get(sizeof(int64_t) * count * m)) : nullptr;
        fb.status = static_cast<int32_t *>(dst.get(sizeof(int32_t) * count));
        DBuf &dfin = ctx->sc_fa[9];
        if (flow_in) fb.flow_in = dfin.upload(flow_in, static_cast<size_t>(count) * m, s);
        cuda_ok(launch_flow_assign(rr.t, fb, s, &ctx->launches), "flow assign kernel");
        std::vector<int64_t> hx, hobj, hval, hflow;
        std::vector<int32_t> hst;
        download(hx, fb.x, rows * J, s);
        download(hobj, fb.objective, count, s);
        download(hval, fb.value, count, s);
        download(hst, fb.status, count, s);
        if (edge_flow) download(hflow, fb.edge_flow, static_cast<size_t>(count) * m, s);
        cuda_ok(cudaStreamSynchronize(s), "sync");
        for (int i = 0; i < count; ++i)
            if (hst[i] != 0) fail(OSERVE_ERR_INVALID_ARGUMENT, "max_flow: negative capacity");
        // solve_instance: the exact path ignores the warm start unless its budget blows
        std::vector<int> exact;
        for (int i = 0; i < count; ++i) {
            int64_t tot = 0;
            for (int j = 0; j < J; ++j) tot += lambda[static_cast<int64_t>(i) * J + j];
            if (tot <= ctx->opts.exact_demand_limit && static_cast<int64_t>(R) * J <= ctx->opts.exact_cell_limit)
                exact.push_back(i);
        }
        if (!exact.empty()) {
            std::vector<int64_t> obj, xs, us;
            std::vector<uint64_t> aborted;
            solve_staged(*ctx, rr, exact, R, J, lambda, obj, xs, us, &aborted);
            std::set<uint64_t> ab(aborted.begin(), aborted.end());
            for (size_t q = 0; q < exact.size(); ++q) {
                if (ab.count(q)) continue;
                const int i = exact[q];
                hobj[i] = obj[q];
                std::copy(xs.begin() + static_cast<int64_t>(q) * R * J, xs.begin() + static_cast<int64_t>(q + 1) * R * J,
                          hx.begin() + static_cast<int64_t>(i) * R * J);
            }
        }
        std::copy(hx.begin(), hx.end(), x);
        std::copy(hobj.begin(), hobj.end(), objective);
        if (flow_value) std::copy(hval.begin(), hval.end(), flow_value);
        if (edge_flow) std::copy(hflow.begin(), hflow.end(), edge_flow);
    });
}
}  // namespace

int oserve_gpu_flow_assign_batch(oserve_gpu_ctx *ctx, int count, int R, int J, const int64_t *n, const int64_t *e,
                                 const int64_t *lambda, int64_t *x, int64_t *objective, int64_t *flow_value,
                                 int64_t *edge_flow) {
    return flow_assign_impl(ctx, count, R, J, n, e, lambda, nullptr, x, objective, flow_value, edge_flow);
}

int oserve_gpu_extract_assignment_batch(oserve_gpu_ctx *ctx, int count, int R, int J, const int64_t *n,
                                        const int64_t *e, const int64_t *lambda, const int64_t *edge_flow,
                                        int64_t *x, int64_t *objective) {
    if (!edge_flow) return OSERVE_ERR_INVALID_ARGUMENT;
    return flow_assign_impl(ctx, count, R, J, n, e, lambda, edge_flow, x, objective, nullptr, nullptr);
}

int oserve_gpu_max_flow_batch(oserve_gpu_ctx *ctx, int count, const int *num_nodes, const int64_t *edge_offset,
                              const oserve_flow_edge *edges, const int *source, const int *sink, int64_t *flow,
                              int64_t *value) {
    return guarded(ctx, [&] {
        if (count <= 0) return;
        std::vector<int64_t> node_off(count + 1, 0), eoff(edge_offset, edge_offset + count + 1);
        for (int g = 0; g < count; ++g) {
            const int nn = num_nodes[g];
            if (source[g] < 0 || source[g] >= nn || sink[g] < 0 || sink[g] >= nn || source[g] == sink[g])
                fail(OSERVE_ERR_INVALID_ARGUMENT, "max_flow: bad source/sink");
            if (eoff[g + 1] < eoff[g]) fail(OSERVE_ERR_INVALID_ARGUMENT, "max_flow: edge offsets must not decrease");
            if (eoff[g + 1] - eoff[g] > (int64_t{1} << 29)) fail(OSERVE_ERR_UNSUPPORTED, "max_flow: too many edges");
            for (int64_t i = eoff[g]; i < eoff[g + 1]; ++i) {
                if (edges[i].from < 0 || edges[i].from >= nn || edges[i].to < 0 || edges[i].to >= nn)
                    fail(OSERVE_ERR_INVALID_ARGUMENT, "max_flow: edge endpoint out of range");
                if (edges[i].cap < 0) fail(OSERVE_ERR_INVALID_ARGUMENT, "max_flow: negative capacity");
            }
            node_off[g + 1] = node_off[g] + nn;
        }
        const int64_t E = eoff[count] - eoff[0], N = node_off[count];
        if (eoff[0] != 0) {
            for (auto &v : eoff) v -= edge_offset[0];
        }
        std::vector<int32_t> nn(num_nodes, num_nodes + count), src(source, source + count), snk(sink, sink + count);
        cudaStream_t s = ctx->stream;
        DBuf *b = ctx->sc_mf;
        MaxFlowBatch mb{};
        mb.count = count;
        mb.num_nodes = b[0].upload(nn, s);
        mb.edge_off = b[1].upload(eoff, s);
        mb.node_off = b[2].upload(node_off, s);
        static_assert(sizeof(oserve_flow_edge) == 16, "oserve_flow_edge: from, to, cap");
        mb.edges32 = reinterpret_cast<const int32_t *>(b[3].upload(edges + edge_offset[0], static_cast<size_t>(E), s));
        mb.source = b[6].upload(src, s);
        mb.sink = b[7].upload(snk, s);
        // graphs of similar size: interleaved workspace padded to the largest
        // (coalesced across a warp's graphs); very uneven batches stay packed
        int64_t n_max = 0, m_max = 0;
        for (int g = 0; g < count; ++g) {
            n_max = std::max<int64_t>(n_max, num_nodes[g]);
            m_max = std::max<int64_t>(m_max, eoff[g + 1] - eoff[g]);
        }
        const bool il = count >= 32 && m_max * count <= 4 * std::max<int64_t>(E, 1) + 64 * count &&
                        (n_max + 1) * count <= 4 * (N + count) + 64 * count;
        const int64_t We = il ? m_max * count : E, Wn = il ? n_max * count : N,
                      Wo = il ? (n_max + 1) * count : N + count;
        mb.interleave = il ? 1 : 0;
        mb.n_max = static_cast<int>(n_max);
        mb.m_max = static_cast<int>(m_max);
        mb.res = static_cast<int64_t *>(b[8].get(sizeof(int64_t) * 2 * We));
        mb.excess = static_cast<int64_t *>(b[9].get(sizeof(int64_t) * Wn));
        mb.arc_to = static_cast<int32_t *>(b[10].get(sizeof(int32_t) * 2 * We));
        mb.adj = static_cast<int32_t *>(b[11].get(sizeof(int32_t) * 2 * We));
        mb.adj_off = static_cast<int32_t *>(b[12].get(sizeof(int32_t) * Wo));
        mb.height = static_cast<int32_t *>(b[13].get(sizeof(int32_t) * Wn));
        mb.cur = static_cast<int32_t *>(b[14].get(sizeof(int32_t) * Wn));
        mb.fifo = static_cast<int32_t *>(b[15].get(sizeof(int32_t) * Wn));
        mb.active = static_cast<uint8_t *>(b[16].get(Wn));
        if (il) {
            mb.il_from = static_cast<int32_t *>(ctx->sc_aux[5].get(sizeof(int32_t) * We));
            mb.il_to = static_cast<int32_t *>(ctx->sc_aux[6].get(sizeof(int32_t) * We));
            mb.il_cap = static_cast<int64_t *>(ctx->sc_aux[7].get(sizeof(int64_t) * We));
        }
        mb.flow = static_cast<int64_t *>(b[17].get(sizeof(int64_t) * E));
        mb.value = static_cast<int64_t *>(b[18].get(sizeof(int64_t) * count));
        mb.status = static_cast<int32_t *>(b[19].get(sizeof(int32_t) * count));
        cuda_ok(launch_max_flow(mb, s, &ctx->launches), "max flow kernel");
        if (E) cuda_ok(d2h(flow, mb.flow, sizeof(int64_t) * E, s), "D2H");
        cuda_ok(d2h(value, mb.value, sizeof(int64_t) * count, s), "D2H");
        cuda_ok(cudaStreamSynchronize(s), "sync");
    });
}

int oserve_gpu_solve_fractional_batch(oserve_gpu_ctx *ctx, int count, int R, int J, const int64_t *n,
                                      const int64_t *e, const int64_t *lambda, double *f, double *objective) {
    return guarded(ctx, [&] {
        if (count <= 0) return;
        if (R < 1 || J < 1) fail(OSERVE_ERR_INVALID_ARGUMENT, "solve_fractional: empty instance");
        const size_t per = simplex_tableau_doubles(R, J) * sizeof(double);
        const size_t budget = size_t{1} << 31;
        if (per > budget) fail(OSERVE_ERR_UNSUPPORTED, "solve_fractional: tableau exceeds 2 GiB");
        const int chunk = static_cast<int>(std::min<size_t>(count, std::max<size_t>(1, budget / per)));
        const int nv = R * J;
        cudaStream_t s = ctx->stream;
        DBuf &dn = ctx->sc_lp[0], &de = ctx->sc_lp[1], &dl = ctx->sc_lp[2], &dt = ctx->sc_lp[3], &df = ctx->sc_lp[4], &dobj = ctx->sc_lp[5], &dst = ctx->sc_lp[6];
        for (int c0 = 0; c0 < count; c0 += chunk) {
            const int cn = std::min(chunk, count - c0);
            LpBatch lb{};
            lb.count = cn;
            lb.R = R;
            lb.J = J;
            lb.n = dn.upload(n + static_cast<int64_t>(c0) * nv, static_cast<size_t>(cn) * nv, s);
            lb.e = de.upload(e + static_cast<int64_t>(c0) * nv, static_cast<size_t>(cn) * nv, s);
            lb.lambda = dl.upload(lambda + static_cast<int64_t>(c0) * J, static_cast<size_t>(cn) * J, s);
            lb.tab = static_cast<double *>(dt.get(per * cn));
            lb.f = static_cast<double *>(df.get(sizeof(double) * cn * nv));
            lb.objective = static_cast<double *>(dobj.get(sizeof(double) * cn));
            lb.status = static_cast<int32_t *>(dst.get(sizeof(int32_t) * cn));
            cuda_ok(launch_simplex(lb, s, &ctx->launches), "simplex kernel");
            std::vector<double> hf, ho;
            std::vector<int32_t> hs;
            download(hf, lb.f, static_cast<size_t>(cn) * nv, s);
            download(ho, lb.objective, cn, s);
            download(hs, lb.status, cn, s);
            cuda_ok(cudaStreamSynchronize(s), "sync");
            for (int i = 0; i < cn; ++i)
                if (hs[i] != 0) fail(OSERVE_ERR_LOGIC, "solve_fractional: unbounded LP (malformed instance)");
            std::copy(hf.begin(), hf.end(), f + static_cast<int64_t>(c0) * nv);
            std::copy(ho.begin(), ho.end(), objective + c0);
        }
    });
}

int oserve_gpu_switch_cost_batch(oserve_gpu_ctx *ctx, const oserve_deployment *src, int count,
                                 const oserve_deployment *dsts, double *est_seconds, uint64_t *max_link_bytes) {
    return guarded(ctx, [&] {
        if (count <= 0) return;
        std::vector<double> est;
        std::vector<uint64_t> mb;
        std::vector<int32_t> st;
        run_switch(*ctx, src, count, dsts, est, mb, st, nullptr, nullptr, nullptr, nullptr);
        for (int i = 0; i < count; ++i) {
            if (st[i]) fail(OSERVE_ERR_UNSOURCED_FRAGMENT, "required bytes have no source holder");
            est_seconds[i] = est[i];
            if (max_link_bytes) max_link_bytes[i] = mb[i];
        }
    });
}

int oserve_gpu_switch_plan(oserve_gpu_ctx *ctx, const oserve_deployment *src, const oserve_deployment *dst,
                           int capacity, oserve_transfer *transfers, int *num_transfers, double *est_seconds) {
    return guarded(ctx, [&] {
        std::vector<double> est;
        std::vector<uint64_t> mb, cuts;
        std::vector<int32_t> st, detail;
        int ncuts = 0;
        SwitchInput in;
        run_switch(*ctx, src, 1, dst, est, mb, st, &detail, &cuts, &ncuts, &in);
        if (st[0]) fail(OSERVE_ERR_UNSOURCED_FRAGMENT, "required bytes have no source holder");
        const int ND = static_cast<int>(in.dev_id.size()), maxf = 4 * ND;
        std::vector<oserve_transfer> tr;
        for (int f = 0; f + 1 < ncuts; ++f)
            for (int t = 0; t < ND; ++t) {
                int sslot = detail[static_cast<size_t>(t) * maxf + f];
                if (sslot >= 0) tr.push_back({cuts[f], cuts[f + 1], in.dev_id[sslot], in.dev_id[t]});
            }
        if (num_transfers) *num_transfers = static_cast<int>(tr.size());
        if (est_seconds) *est_seconds = est[0];
        if (transfers) {
            for (int i = 0; i < std::min<int>(capacity, static_cast<int>(tr.size())); ++i) transfers[i] = tr[i];
            if (static_cast<int>(tr.size()) > capacity) fail(OSERVE_ERR_INVALID_ARGUMENT, "transfer capacity too small");
        }
    });
}


// ---------------------------------------------------------------------------
// Reference-signature pieces of switching and of the assignment (the C++
// shim's layout / greedy_plan(ShardLayout...) / estimate_time / normalize /
// normalize_or_scale / check_constraints).

int oserve_gpu_layout(oserve_gpu_ctx *ctx, const oserve_deployment *dep, uint64_t param_bytes, int capacity,
                      oserve_shard *shards, int *n_shards) {
    return guarded(ctx, [&] {
        if (!dep || !n_shards) fail(OSERVE_ERR_INVALID_ARGUMENT, "layout: null argument");
        const int R = dep->num_replicas;
        std::vector<int32_t> rep_off{0}, dev_off, tp, pp, devs;
        int pos = 0;
        for (int r = 0; r < R; ++r) {
            const int nd = dep->replica_num_devices[r];
            if (dep->tp[r] < 1 || dep->pp[r] < 1) fail(OSERVE_ERR_INVALID_ARGUMENT, "layout: tp and pp must be >= 1");
            if (static_cast<int64_t>(dep->tp[r]) * dep->pp[r] > nd)
                fail(OSERVE_ERR_INVALID_ARGUMENT, "layout: replica " + std::to_string(r) + " has fewer than tp*pp devices");
            std::vector<int> d(dep->device_ids + pos, dep->device_ids + pos + nd);
            std::sort(d.begin(), d.end());  // devices sorted per replica (switchplan.cpp:45-46)
            dev_off.push_back(static_cast<int32_t>(devs.size()));
            devs.insert(devs.end(), d.begin(), d.end());
            pos += nd;
            tp.push_back(dep->tp[r]);
            pp.push_back(dep->pp[r]);
            rep_off.push_back(rep_off.back() + dep->tp[r] * dep->pp[r]);
        }
        const int total = rep_off.back();
        *n_shards = total;
        if (total == 0 || !shards) return;  // count query
        if (capacity < total) fail(OSERVE_ERR_INVALID_ARGUMENT, "layout: shard capacity too small");
        cudaStream_t s = ctx->stream;
        DBuf *b = ctx->sc_aux;
        LayoutIn in{};
        in.R = R;
        in.total = total;
        in.rep_off = b[0].upload(rep_off, s);
        in.dev_off = b[1].upload(dev_off, s);
        in.tp = b[2].upload(tp, s);
        in.pp = b[3].upload(pp, s);
        in.devs_sorted = b[4].upload(devs, s);
        in.P = param_bytes;
        in.begin = static_cast<uint64_t *>(b[5].get(sizeof(uint64_t) * total));
        in.end = static_cast<uint64_t *>(b[6].get(sizeof(uint64_t) * total));
        in.holder = static_cast<int32_t *>(b[7].get(sizeof(int32_t) * total));
        cuda_ok(launch_layout(in, s, &ctx->launches), "layout kernel");
        std::vector<uint64_t> hb, he;
        std::vector<int32_t> hh;
        download(hb, in.begin, total, s);
        download(he, in.end, total, s);
        download(hh, in.holder, total, s);
        cuda_ok(cudaStreamSynchronize(s), "sync");
        for (int g = 0; g < total; ++g) shards[g] = {g, hb[g], he[g], hh[g]};
    });
}

int oserve_gpu_greedy_plan_layouts(oserve_gpu_ctx *ctx, int n_src, const oserve_held_range *src, int n_dst,
                                   const oserve_held_range *dst, int capacity, oserve_transfer *transfers,
                                   int *n_transfers, double *est_seconds) {
    return guarded(ctx, [&] {
        if (n_src < 0 || n_dst < 0) fail(OSERVE_ERR_INVALID_ARGUMENT, "greedy_plan: negative range count");
        std::set<int> ids;
        std::vector<uint64_t> bounds;
        for (int i = 0; i < n_src; ++i) ids.insert(src[i].device);
        for (int i = 0; i < n_dst; ++i) ids.insert(dst[i].device);
        for (const oserve_held_range *v : {src, dst})
            for (int i = 0, n = (v == src ? n_src : n_dst); i < n; ++i) {
                if (v[i].end >= (uint64_t{1} << 54)) fail(OSERVE_ERR_UNSUPPORTED, "greedy_plan: byte offsets >= 2^54");
                bounds.push_back(v[i].begin);
                bounds.push_back(v[i].end);
            }
        if (n_transfers) *n_transfers = 0;
        if (est_seconds) *est_seconds = 0.0;
        if (bounds.size() < 2) return;  // cuts.size() < 2: empty plan (:87)
        if (ids.size() > 256) fail(OSERVE_ERR_UNSUPPORTED, "greedy_plan limited to 256 devices");
        if (bounds.size() > 16384) fail(OSERVE_ERR_UNSUPPORTED, "greedy_plan limited to 8192 held ranges");
        std::vector<int32_t> dev_id(ids.begin(), ids.end()), machine;
        std::map<int, int> slot;
        for (size_t i = 0; i < dev_id.size(); ++i) {
            slot[dev_id[i]] = static_cast<int>(i);
            machine.push_back(ctx->machine(dev_id[i]));
        }
        const int ND = static_cast<int>(dev_id.size());
        auto csr = [&](int n, const oserve_held_range *v, std::vector<int32_t> &off, std::vector<uint64_t> &b,
                       std::vector<uint64_t> &e) {
            std::vector<std::vector<std::pair<uint64_t, uint64_t>>> per(ND);
            for (int i = 0; i < n; ++i) per[slot[v[i].device]].emplace_back(v[i].begin, v[i].end);
            off.assign(1, 0);
            for (int t = 0; t < ND; ++t) {
                for (auto &r : per[t]) {
                    b.push_back(r.first);
                    e.push_back(r.second);
                }
                off.push_back(static_cast<int32_t>(b.size()));
            }
        };
        std::vector<int32_t> soff, doff;
        std::vector<uint64_t> sb, se, db, de;
        csr(n_src, src, soff, sb, se);
        csr(n_dst, dst, doff, db, de);
        cudaStream_t s = ctx->stream;
        DBuf *b = ctx->sc_sw;
        HeldIn in{};
        in.num_devices = ND;
        in.machine = b[0].upload(machine, s);
        in.src_off = b[1].upload(soff, s);
        in.dst_off = b[2].upload(doff, s);
        in.src_b = b[3].upload(sb, s);
        in.src_e = b[4].upload(se, s);
        in.dst_b = b[5].upload(db, s);
        in.dst_e = b[6].upload(de, s);
        in.nbounds = static_cast<int>(bounds.size());
        in.bounds = b[7].upload(bounds, s);
        in.intra_bw = ctx->intra;
        in.inter_bw = ctx->inter;
        HeldOut o{};
        o.max_frags = in.nbounds;
        o.detail = static_cast<int32_t *>(b[8].get(sizeof(int32_t) * ND * o.max_frags));
        cuda_ok(cudaMemsetAsync(o.detail, 0xff, sizeof(int32_t) * ND * o.max_frags, s), "memset");
        o.cuts = static_cast<uint64_t *>(b[9].get(sizeof(uint64_t) * in.nbounds));
        o.ncuts = static_cast<int32_t *>(b[10].get(sizeof(int32_t)));
        o.est = static_cast<double *>(b[11].get(sizeof(double)));
        o.max_bytes = static_cast<unsigned long long *>(b[12].get(sizeof(unsigned long long)));
        cuda_ok(launch_switch_held(in, o, s, &ctx->launches), "greedy_plan kernel");
        std::vector<int32_t> detail, nc;
        std::vector<uint64_t> cuts;
        std::vector<double> est;
        download(detail, o.detail, static_cast<size_t>(ND) * o.max_frags, s);
        download(cuts, o.cuts, in.nbounds, s);
        download(nc, o.ncuts, 1, s);
        download(est, o.est, 1, s);
        cuda_ok(cudaStreamSynchronize(s), "sync");
        std::vector<oserve_transfer> tr;
        for (int f = 0; f + 1 < nc[0]; ++f)
            for (int t = 0; t < ND; ++t) {
                const int v = detail[static_cast<size_t>(t) * o.max_frags + f];
                if (v == -2)
                    fail(OSERVE_ERR_UNSOURCED_FRAGMENT, "bytes [" + std::to_string(cuts[f]) + ", " +
                                                            std::to_string(cuts[f + 1]) + ") required by device " +
                                                            std::to_string(dev_id[t]) + " have no source holder");
                if (v >= 0) tr.push_back({cuts[f], cuts[f + 1], dev_id[v], dev_id[t]});
            }
        if (n_transfers) *n_transfers = static_cast<int>(tr.size());
        if (est_seconds) *est_seconds = est[0];
        if (transfers) {
            for (int i = 0; i < std::min<int>(capacity, static_cast<int>(tr.size())); ++i) transfers[i] = tr[i];
            if (static_cast<int>(tr.size()) > capacity) fail(OSERVE_ERR_INVALID_ARGUMENT, "transfer capacity too small");
        }
    });
}

int oserve_gpu_estimate_time(oserve_gpu_ctx *ctx, int n_links, const oserve_link_load *links, double *est_seconds) {
    return guarded(ctx, [&] {
        if (!est_seconds || n_links < 0) fail(OSERVE_ERR_INVALID_ARGUMENT, "estimate_time: bad arguments");
        *est_seconds = 0.0;
        if (n_links == 0) return;
        std::vector<int32_t> ms(n_links), md(n_links);
        std::vector<uint64_t> by(n_links);
        for (int i = 0; i < n_links; ++i) {
            ms[i] = ctx->machine(links[i].src);
            md[i] = ctx->machine(links[i].dst);
            by[i] = links[i].bytes;
        }
        cudaStream_t s = ctx->stream;
        DBuf *b = ctx->sc_aux;
        LinkIn in{};
        in.n = n_links;
        in.src_machine = b[0].upload(ms, s);
        in.dst_machine = b[1].upload(md, s);
        in.bytes = b[2].upload(by, s);
        in.intra_bw = ctx->intra;
        in.inter_bw = ctx->inter;
        double *d_est = static_cast<double *>(b[3].get(sizeof(double)));
        cuda_ok(launch_link_time(in, d_est, s, &ctx->launches), "estimate_time kernel");
        cuda_ok(d2h(est_seconds, d_est, sizeof(double), s), "D2H");
        cuda_ok(cudaStreamSynchronize(s), "sync");
    });
}

int oserve_gpu_normalize_batch(oserve_gpu_ctx *ctx, int count, int J, const int64_t *n, int strict, int64_t *M,
                               int64_t *units, int *scaled) {
    return guarded(ctx, [&] {
        if (count <= 0) return;
        if (J < 1) fail(OSERVE_ERR_INVALID_ARGUMENT, "normalize: empty row");
        if (J > OSERVE_MAX_CLASSES) fail(OSERVE_ERR_UNSUPPORTED, "normalize: rows limited to 16 entries");
        const int64_t cells = static_cast<int64_t>(count) * J;
        for (int64_t i = 0; i < cells; ++i)
            if (n[i] < 0) fail(OSERVE_ERR_INVALID_ARGUMENT, "normalize: negative capacity");
        RawRows &rr = ctx->raw;
        stage_raw_rows(*ctx, count, J, n, n, rr);  // K0b: checked LCM, 2^62 fallback
        cudaStream_t s = ctx->stream;
        std::vector<int64_t> hM, hu;
        std::vector<uint8_t> hs;
        download(hM, rr.t.M, count, s);
        download(hu, rr.t.unit, cells, s);
        download(hs, rr.t.scaled, count, s);
        cuda_ok(cudaStreamSynchronize(s), "sync");
        for (int i = 0; i < count; ++i) {
            if (strict && hs[i]) fail(OSERVE_ERR_LCM_OVERFLOW, "normalize: LCM exceeds 2^62");
            if (M) M[i] = hM[i];
            if (scaled) scaled[i] = hs[i];
        }
        if (units) std::copy(hu.begin(), hu.end(), units);
    });
}

int oserve_gpu_check_constraints_batch(oserve_gpu_ctx *ctx, int count, int R, int J, const int64_t *x,
                                       const int64_t *n, const int64_t *e, const int64_t *lambda, int *kind,
                                       int *replica, int *type) {
    return guarded(ctx, [&] {
        if (count <= 0) return;
        if (R < 1 || J < 1) fail(OSERVE_ERR_INVALID_ARGUMENT, "check_constraints: empty instance");
        if (J > OSERVE_MAX_CLASSES) fail(OSERVE_ERR_UNSUPPORTED, "check_constraints: J limited to 16");
        const int64_t rows = static_cast<int64_t>(count) * R;
        for (int64_t i = 0; i < rows * J; ++i)
            if (n[i] < 0) fail(OSERVE_ERR_INVALID_ARGUMENT, "normalize: negative capacity");
        RawRows &rr = ctx->raw;
        stage_raw_rows(*ctx, rows, J, n, e, rr);  // normalize_or_scale per row (K0b)
        cudaStream_t s = ctx->stream;
        DBuf *b = ctx->sc_aux;
        CheckIn in{};
        in.count = count;
        in.R = R;
        in.J = J;
        in.x = b[0].upload(x, static_cast<size_t>(rows) * J, s);
        in.e = rr.t.e;
        in.lambda = b[1].upload(lambda, static_cast<size_t>(count) * J, s);
        in.t = rr.t;
        in.kind = static_cast<int32_t *>(b[2].get(sizeof(int32_t) * count));
        in.k = static_cast<int32_t *>(b[3].get(sizeof(int32_t) * count));
        in.j = static_cast<int32_t *>(b[4].get(sizeof(int32_t) * count));
        cuda_ok(launch_check(in, s, &ctx->launches), "check_constraints kernel");
        std::vector<int32_t> hk, hr, hj;
        download(hk, in.kind, count, s);
        download(hr, in.k, count, s);
        download(hj, in.j, count, s);
        cuda_ok(cudaStreamSynchronize(s), "sync");
        for (int i = 0; i < count; ++i) {
            if (kind) kind[i] = hk[i];
            if (replica) replica[i] = hr[i];
            if (type) type[i] = hj[i];
        }
        for (int i = 0; i < count; ++i) {
            const std::string k = std::to_string(hr[i]), j = std::to_string(hj[i]);
            switch (hk[i]) {  // flowassign.cpp:529-551 messages
                case 1: fail(OSERVE_ERR_LOGIC, "C1 violated for type " + j);
                case 2: fail(OSERVE_ERR_LOGIC, "C2 violated at replica " + k + ", type " + j);
                case 3: fail(OSERVE_ERR_LOGIC, "C3 violated at replica " + k + ": zero-capacity type " + j + " assigned");
                case 4: fail(OSERVE_ERR_LOGIC, "C3 violated at replica " + k);
                default: break;
            }
        }
    });
}

}  // extern "C"
