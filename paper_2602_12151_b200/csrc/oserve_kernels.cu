// oserve_kernels.cu — sm_100a kernels of the OServe scheduling round.
//
//   K0a k_cost_cells      per (shape, class) FP64 service time, n, e
//                         (costmodel.cpp:22-116; bit-exact: __dmul_rn/__dadd_rn/
//                         __ddiv_rn keep the reference's operand order, no FMA)
//   K0b k_normalize_rows  per shape LCM normalisation + instance caps + class
//                         order (flowassign.cpp:22-62, :267-294)
//   K1  k_plan_eval       one G-lane group per plan: unrank -> gather shape rows
//                         (smem) -> speculative-parallel greedy_fill -> exchange
//                         (first improving move, restart) -> objective -> packed
//                         key -> group/CTA min -> atomicMin
//                         (deploysearch.cpp:153-229, flowassign.cpp:393-503)
//   K4  k_plan_exact      thread per plan: branch-and-bound exact path
//                         (flowassign.cpp:296-369, :450-477)
//   K2  k_switch_cost     CTA per (current, candidate) pair: layouts, cut points,
//                         warp per target device, lane per source replica
//                         (switchplan.cpp:40-140)
// All integer work runs on the CUDA-core INT/FP32 pipes; there is no dense
// contraction here, so no tensor-core path.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <map>
#include <tuple>
#include <type_traits>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>

#include "oserve_internal.h"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#define OSERVE_MAX_REPLICAS_DEV 128

#ifndef OSERVE_K1_MINB
#define OSERVE_K1_MINB 4  // CTAs of 256 threads per SM the register budget must allow (64 regs; measured 5% faster than 3)
#endif
// exchange-loop per-slot loops: unrolled for one or two slots per lane (config
// 5: 105.5 -> 103.9 ms), rolled for four (instruction-cache footprint: config
// 5-7B 58.9 ms rolled, 61.4 ms unrolled)
#ifndef OSERVE_K1_XUNROLL
#define OSERVE_K1_XUNROLL _Pragma("unroll (KPL <= 2 ? KPL : 1)")
#endif
#ifndef OSERVE_K1_ZUNROLL  // clearing a resumed replica's J classes (config 5: -0.4%)
#define OSERVE_K1_ZUNROLL _Pragma("unroll (KPL <= 2 ? 4 : 1)")
#endif
#ifndef OSERVE_K1_TUNROLL
#define OSERVE_K1_TUNROLL _Pragma("unroll 1")
#endif
#ifndef OSERVE_K1_MINB_4
#define OSERVE_K1_MINB_4 2  // four replicas per lane (KPL = 4, R <= 128): shared memory holds it to 2 CTAs/SM anyway, so no spill at 107 registers (cfg5-7B 63.8 -> 59.0 ms)
#endif
#ifndef OSERVE_K1_MINB_1
#define OSERVE_K1_MINB_1 OSERVE_K1_MINB  // one replica per lane (KPL = 1)
#endif

namespace oserve_gpu {

namespace {

constexpr int64_t kLcmLimit = int64_t{1} << 62;
constexpr int kBinomN = 160;
constexpr int kBinomK = kMaxCand;
__constant__ uint64_t c_binom[kBinomN][kBinomK];  // C(n, k), k < kMaxCand

inline int check(cudaError_t e) { return e == cudaSuccess ? 0 : static_cast<int>(e); }

__device__ __forceinline__ int64_t gcd64(int64_t a, int64_t b) {
    while (b != 0) {
        int64_t t = a % b;
        a = b;
        b = t;
    }
    return a;
}

// ----------------------------------------------------------------- K0a ----
__global__ void k_cost_cells(ShapeTables t, const double *__restrict__ cin, const double *__restrict__ cout,
                             uint32_t num_layers, uint64_t kvb, double pc, double dc, double ppc,
                             double slope, double span) {
    const int J = t.J;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < t.num_shapes * J;
         idx += gridDim.x * blockDim.x) {
        const int s = idx / J, j = idx - (idx / J) * J;
        const ShapeParam sp = t.param[s];
        const double in = cin[j], out = cout[j], L = static_cast<double>(num_layers);
        const double ppm1 = static_cast<double>(sp.pp - 1);
        // prefill_latency (costmodel.cpp:28-33): in*L*pc/speedup + (pp-1)*ppc
        const double prefill = __dadd_rn(__ddiv_rn(__dmul_rn(__dmul_rn(in, L), pc), sp.speedup), __dmul_rn(ppm1, ppc));
        // decode_latency (:35-40): out*L*dc*(1+slope*(tp-1))/tp + (pp-1)*ppc*out
        const double pen = __dadd_rn(1.0, __dmul_rn(slope, static_cast<double>(sp.tp - 1)));
        const double decode = __dadd_rn(
            __ddiv_rn(__dmul_rn(__dmul_rn(__dmul_rn(out, L), dc), pen), static_cast<double>(sp.tp)),
            __dmul_rn(__dmul_rn(ppm1, ppc), out));
        const double svc = __dadd_rn(prefill, decode);  // request_service_time (:42-46)
        // capacity (:74-82) and edge_capacity (:84-92)
        const int64_t n = static_cast<int64_t>(floor(__ddiv_rn(__dmul_rn(span, static_cast<double>(sp.pp)), svc)));
        const double per_req = __dmul_rn(__dadd_rn(in, out), static_cast<double>(kvb));
        const double capd = floor(__ddiv_rn(static_cast<double>(sp.kv_budget), per_req));
        const int64_t e = capd >= static_cast<double>(n) ? n : static_cast<int64_t>(capd);
        t.n[idx] = n;
        t.e[idx] = e;
        t.latency[idx] = svc;
    }
}

// ----------------------------------------------------------------- K0b ----
__global__ void k_normalize_rows(ShapeTables t) {
    const int J = t.J;
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < t.num_shapes; s += gridDim.x * blockDim.x) {
        const int64_t *n = t.n + static_cast<int64_t>(s) * J;
        const int64_t *e = t.e + static_cast<int64_t>(s) * J;
        int64_t *unit = t.unit + static_cast<int64_t>(s) * J;
        int32_t *cap = t.cap + static_cast<int64_t>(s) * J;
        // normalize (flowassign.cpp:31-46) with checked_lcm (:22-27)
        int64_t m = 1;
        bool overflow = false;
        for (int j = 0; j < J && !overflow; ++j) {
            const int64_t nj = n[j];
            if (nj <= 0) continue;
            const int64_t g = gcd64(m, nj);
            const int64_t q = m / g;
            if (q > kLcmLimit / nj) overflow = true;
            else m = q * nj;
        }
        if (overflow) m = kLcmLimit;  // normalize_or_scale fallback (:48-62)
        t.M[s] = m;
        t.scaled[s] = overflow ? 1 : 0;
        uint8_t ord[kMaxJ];
        int ol = 0;
        for (int j = 0; j < J; ++j) {
            const int64_t nj = n[j];
            int64_t u = 0;
            if (nj > 0) u = overflow ? (kLcmLimit + nj - 1) / nj : m / nj;
            unit[j] = u;
            t.inv_unit[static_cast<int64_t>(s) * J + j] = u > 0 ? __drcp_rn(static_cast<double>(u)) : 0.0;
            // make_instance (:278-292): cap = min(e, n, M/unit) where unit > 0
            int64_t c = 0;
            if (u > 0) {
                c = e[j] < nj ? e[j] : nj;
                const int64_t byb = m / u;
                c = c < byb ? c : byb;
            }
            if (c > 0) {
                cap[j] = c > 0x7fffffffll ? 0x7fffffff : static_cast<int32_t>(c);
                // stable insertion by ascending unit (std::stable_sort, :289)
                int pos = ol;
                while (pos > 0 && unit[ord[pos - 1]] > u) {
                    ord[pos] = ord[pos - 1];
                    --pos;
                }
                ord[pos] = static_cast<uint8_t>(j);
                ++ol;
            } else {
                cap[j] = 0;
            }
        }
        for (int i = 0; i < kMaxJ; ++i) {
            t.order[s * kMaxJ + i] = i < ol ? ord[i] : 0;
            t.rank[s * kMaxJ + i] = 0xff;
        }
        uint32_t pm = 0;
        for (int i = 0; i < kMaxJ; ++i) {
            if (i < ol) {
                t.rank[s * kMaxJ + ord[i]] = static_cast<uint8_t>(i);
                pm |= 1u << ord[i];
            }
            t.pmask[s * kMaxJ + i] = static_cast<uint16_t>(pm);
        }
        t.olen[s] = static_cast<uint8_t>(ol);
    }
}

// ------------------------------------------------------- plan resolution --
__device__ __noinline__ uint64_t div64(uint64_t a, uint64_t b) { return a / b; }  // one out-of-line copy
__device__ __forceinline__ uint64_t div_small(uint64_t a, uint64_t b) {
    if ((a >> 32) == 0 && (b >> 32) == 0) return static_cast<uint32_t>(a) / static_cast<uint32_t>(b);
    return div64(a, b);
}

// Largest p with prefix[p] <= g (skips empty partitions automatically).
__device__ __forceinline__ int64_t find_partition(const SpaceTables &sp, uint64_t g) {
    int64_t lo = 0, hi = sp.num_parts - 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (__ldg(sp.prefix + mid) <= g) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ uint64_t shard_rank(const PlanSource &src, uint64_t li) {
    const uint64_t c = div_small(li, src.chunk);
    return (c * static_cast<uint64_t>(src.world) + static_cast<uint64_t>(src.rank)) * src.chunk + (li - c * src.chunk);
}

// Global plan rank of launch-local index li (modes 0, 1, 3).
__device__ __forceinline__ uint64_t source_rank(const PlanSource &src, uint64_t li) {
    if (src.mode == 1) return src.ranks[li];
    const uint64_t b = shard_rank(src, li);
    if (src.mode == 0) return b;
    int lo = 0, hi = src.num_ranges - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(src.range_prefix + mid) <= b) lo = mid;
        else hi = mid - 1;
    }
    return __ldg(src.range_start + lo) + (b - __ldg(src.range_prefix + lo));
}

// source_rank with the current rank range cached (consecutive launch-local
// indices stay inside one range almost always).
#ifdef OSERVE_K1_STATS
__device__ unsigned long long g_k1_stats[4];
#endif
// Group-uniform K1 state carried across plans (shared memory, written by
// lane 0 only; read after the next group sync).
struct K1Carry {
    uint64_t r_lo, r_hi, r_start;  // current rank range (mode 3)
    uint64_t cp_lo, cp_hi;         // current partition's plan-rank interval
    int64_t cpart;
    uint64_t snap_hi;              // snapshot: prefix digits and partition
    int64_t snap_part;
    uint64_t best;                 // group's best key (lane 0 only)
    uint64_t tk_max;               // worst key kept in the top-K list
    int tk_idx;                    // its slot (lane 0 only)
    int lossy;                     // the list dropped a key (lane 0 only)
};
// (rlo, rhi, rst): the carried range, read by the caller before any lane
// of the group may update it.
__device__ __forceinline__ uint64_t source_rank_cached(const PlanSource &src, uint64_t li, K1Carry *c, int gl,
                                                       uint64_t rlo, uint64_t rhi, uint64_t rst) {
    if (src.mode == 1) return src.ranks[li];
    const uint64_t b = shard_rank(src, li);
    if (src.mode == 0) return b;
    if (b < rlo || b >= rhi) {
        int lo = 0, hi = src.num_ranges - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (__ldg(src.range_prefix + mid) <= b) lo = mid;
            else hi = mid - 1;
        }
        rlo = __ldg(src.range_prefix + lo);
        rhi = lo + 1 < src.num_ranges ? __ldg(src.range_prefix + lo + 1) : ~uint64_t{0};
        rst = __ldg(src.range_start + lo);
        if (gl == 0) {
            c->r_lo = rlo;
            c->r_hi = rhi;
            c->r_start = rst;
        }
    }
    return rst + (b - rlo);
}

// Unrank a non-decreasing pick sequence of length len over [0, q) (lex order).
__device__ __forceinline__ void unrank_run(uint64_t r, int len, int q, uint8_t *out) {
    int prev = 0;
    for (int pos = 0; pos < len; ++pos) {
        const int rem = len - pos - 1;
        for (int v = prev; v < q; ++v) {
            const uint64_t c = c_binom[rem + (q - v) - 1][(q - v) - 1];
            if (r < c) {
                out[pos] = static_cast<uint8_t>(v);
                prev = v;
                break;
            }
            r -= c;
        }
    }
}

// floor(m / u) for 0 <= m < 2^63, u >= 1, when the quotient is known to be
// < 2^31 (greedy: m < a*u with a <= INT32_MAX).  The FP64 estimate has
// relative error < 2^-51, i.e. absolute error < 2^-20, so one correction
// step in each direction makes it exact (no 64-bit integer division).
__device__ __forceinline__ int32_t quot_small(int64_t m, int64_t u, double inv_u) {
    int64_t q = static_cast<int64_t>(__dmul_rn(static_cast<double>(m), inv_u));
    const int64_t r = m - q * u;
    if (r < 0) --q;
    else if (r >= u) ++q;
    return static_cast<int32_t>(q);
}


// ------------------------------------------------------------------- K1 ---
// Group of G lanes evaluates one plan; lane gl owns replicas k = gl + G*kk.
template <int G, int KPL>
struct Group {
    static constexpr int RMAX = G * KPL;
    static constexpr int kG = G;
    unsigned mask;
    int gl, base;
    __device__ __forceinline__ Group() {
        const int lane = threadIdx.x & 31;
        gl = lane & (G - 1);
        base = lane - gl;
        mask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << base);
    }
    __device__ __forceinline__ void sync() const { __syncwarp(mask); }
    __device__ __forceinline__ uint32_t ballot(bool p) const {
        const uint32_t b = __ballot_sync(mask, p);
        return (G == 32) ? b : ((b >> base) & ((1u << G) - 1u));
    }
    template <class T>
    __device__ __forceinline__ T bcast(T v, int src) const { return __shfl_sync(mask, v, src, G); }
    __device__ __forceinline__ uint32_t sum(uint32_t v) const { return __reduce_add_sync(mask, v); }
    __device__ __forceinline__ uint32_t or_all(uint32_t v) const { return __reduce_or_sync(mask, v); }
    // inclusive prefix sum of u64 over the first W lanes, saturating at `sat`
    // (sat + sat must not overflow)
    template <int W>
    __device__ __forceinline__ uint64_t scan_sat64(uint64_t v, uint64_t sat) const {
#pragma unroll
        for (int d = 1; d < W; d <<= 1) {
            const uint64_t o = __shfl_up_sync(mask, v, d, G);
            if (gl >= d) {
                v += o;
                v = v < sat ? v : sat;
            }
        }
        return v;
    }
    // inclusive prefix sum, saturating at `sat`
    __device__ __forceinline__ uint32_t scan_sat(uint32_t v, uint32_t sat) const {
#pragma unroll
        for (int d = 1; d < G; d <<= 1) {
            const uint32_t o = __shfl_up_sync(mask, v, d, G);
            if (gl >= d) v = min(v + o, sat);
        }
        return v;
    }
};

// Greedy-prefix reuse (K1): x changes of the exchange since the snapshot,
// one u32 per change ((cell << 1) | was_increment), 3 slots per move.
constexpr int kUndo = 96;
#ifndef OSERVE_K1_CHUNK
#define OSERVE_K1_CHUNK 32
#endif
constexpr uint64_t kGroupChunk = OSERVE_K1_CHUNK;  // plans per contiguous group chunk

// Register-array element by a runtime slot index without dynamic indexing
// (keeps the array in registers): lets the exchange run ONE copy of a body
// in a non-unrolled slot loop instead of KPL inlined copies (instruction-
// cache footprint; the K1 loop body is the whole hot path).
template <int KPL, class T>
__device__ __forceinline__ T rsel(const T (&a)[KPL], int kk) {
    T v = a[0];
#pragma unroll
    for (int q = 1; q < KPL; ++q)
        if (kk == q) v = a[q];
    return v;
}
template <int KPL, class T>
__device__ __forceinline__ void rput(T (&a)[KPL], int kk, T v) {
#pragma unroll
    for (int q = 0; q < KPL; ++q)
        if (kk == q) a[q] = v;
}

// Per-group scratch: the fixed-size arrays first (compile-time offsets from
// one base register), the J-sized assignment x last.
template <int RMAX, int KPL>
__host__ __device__ constexpr size_t group_fixed_bytes() {
    return ((size_t)kTopK * 8 + (size_t)RMAX * 8 + (size_t)kMaxJ * KPL * 4 + (size_t)(RMAX / KPL) * 4 +
            (size_t)RMAX * 8 + (size_t)kUndo * 4 + sizeof(K1Carry) + (size_t)RMAX * 2 + RMAX + 15) &
           ~size_t(15);
}
// Warp-wide groups (G = 32, the large configs) size the assignment x as
// [kMaxJ][RMAX] whatever J is, so a group's scratch — hence every group and
// the shape rows after them — sits at a compile-time offset in shared memory.
// Narrow groups (small plans) keep x at [J][RMAX] and the rows first: there
// the shared-memory footprint, i.e. occupancy, matters more.
template <int G>
__host__ __device__ constexpr bool fixed_layout() {
    return G == 32;
}
template <int G, int KPL>
__host__ __device__ constexpr size_t group_scratch_bytes(int J) {
    constexpr int RMAX = G * KPL;
    return group_fixed_bytes<RMAX, KPL>() +
           (((size_t)(fixed_layout<G>() ? kMaxJ : J) * RMAX * 4 + 15) & ~size_t(15));
}

// Group-uniform unranking of one run of `len` non-decreasing picks over
// [0, q) with rank rr (same order as unrank_run): the count of each value v
// is the largest m with rr < C(rem - m + K, K), K = q - v - 1 (the
// sequences holding >= m copies of v come first); lanes fill the positions.
template <class Grp>
__device__ __forceinline__ void unrank_run_group(const Grp &g, uint64_t rr, int len, int q, uint8_t *out) {
    int rem = len, pos = 0;
    for (int v = 0; v < q - 1 && rem > 0; ++v) {
        const int K = q - v - 1;
        int lo = 0, hi = rem;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (rr < c_binom[rem - mid + K][K]) lo = mid;
            else hi = mid - 1;
        }
        if (lo < rem) rr -= c_binom[rem - lo - 1 + K][K];
#pragma unroll 1
        for (int p = g.gl; p < lo; p += Grp::kG) out[pos + p] = static_cast<uint8_t>(v);
        pos += lo;
        rem -= lo;
    }
#pragma unroll 1
    for (int p = g.gl; p < rem; p += Grp::kG) out[pos + p] = static_cast<uint8_t>(q - 1);
}

// One shape's tables in K1's shared memory (fixed class stride kMaxJ).
struct alignas(16) ShapeRow {
    int64_t unit[kMaxJ];
    double inv[kMaxJ];
    int64_t M;
    int32_t cap[kMaxJ];
    uint16_t pmask[kMaxJ];
    uint8_t order[kMaxJ];
    uint8_t rank[kMaxJ];
    uint8_t olen, pp;
};

// K1 variants: the round (best key only; plan sources 0/1/3), the top-K
// round (+ per-group key lists, threshold collect) and the general kernel
// (explicit shape lists, per-plan objective / sum_pp / x / used).  The round
// kernel carries no per-plan output code: its hot loop is the whole kernel,
// and cold code inside it still costs instruction-cache lines.
enum K1Variant { kK1Round = 0, kK1TopK = 1, kK1General = 2 };

template <int G, int KPL, bool SMEM, int V>
__global__ void __launch_bounds__(256, KPL == 1 ? OSERVE_K1_MINB_1 : (KPL == 4 ? OSERVE_K1_MINB_4 : OSERVE_K1_MINB)) k_plan_eval(ShapeTables t, SpaceTables sp, KeyLayout key,
                                                                   PlanSource src, PlanOutputs out, SolveParams prm,
                                                                   int skip_exact, int gchunk,
                                                                   unsigned long long *work) {
    using Grp = Group<G, KPL>;
    constexpr int RMAX = Grp::RMAX;
    constexpr int GPB = 256 / G;
    constexpr bool kGeneral = V == kK1General;
    constexpr bool kLists = V != kK1Round;  // top-K lists / threshold collect
    extern __shared__ __align__(16) unsigned char smem[];
    const int S = t.num_shapes, J = prm.J;

    // ---- shape tables: staged in shared memory as one fixed-stride row per
    // shape at the start of the dynamic shared window (every field at a
    // compile-time offset from a compile-time base: no table pointers held
    // in, or rematerialised into, registers), or read from the global SoA
    // tables (L1-cached) when they do not fit (solve_batch: a row per instance)
    // layout (fixed): GPB group scratch blocks, the CTA's best keys, the
    // shape rows; (narrow groups) the shape rows, then the groups and keys
    constexpr bool kFixed = fixed_layout<G>();
    const size_t per_group = group_scratch_bytes<G, KPL>(kFixed ? kMaxJ : J);
    const size_t rows_off = kFixed ? ((per_group * GPB + GPB * 8 + 15) & ~size_t(15)) : 0;
    const size_t groups_off = (kFixed || !SMEM) ? 0 : static_cast<size_t>(S) * sizeof(ShapeRow);
    const ShapeRow *rows = reinterpret_cast<const ShapeRow *>(smem + rows_off);
    auto tUnit = [&](int sh, int j) -> int64_t {
        if constexpr (SMEM) return rows[sh].unit[j];
        else return t.unit[sh * J + j];
    };
    auto tInv = [&](int sh, int j) -> double {
        if constexpr (SMEM) return rows[sh].inv[j];
        else return t.inv_unit[sh * J + j];
    };
    auto tCap = [&](int sh, int j) -> int32_t {
        if constexpr (SMEM) return rows[sh].cap[j];
        else return t.cap[sh * J + j];
    };
    auto tOrder = [&](int sh, int p) -> int {
        if constexpr (SMEM) return rows[sh].order[p];
        else return t.order[sh * kMaxJ + p];
    };
    auto tRank = [&](int sh, int j) -> int {
        if constexpr (SMEM) return rows[sh].rank[j];
        else return t.rank[sh * kMaxJ + j];
    };
    auto tPmask = [&](int sh, int p) -> uint32_t {
        if constexpr (SMEM) return rows[sh].pmask[p];
        else return t.pmask[sh * kMaxJ + p];
    };
    auto tM = [&](int sh) -> int64_t {
        if constexpr (SMEM) return rows[sh].M;
        else return t.M[sh];
    };
    auto tOlen = [&](int sh) -> int {
        if constexpr (SMEM) return rows[sh].olen;
        else return t.olen[sh];
    };
    auto tPP = [&](int sh) -> int {
        if constexpr (SMEM) return rows[sh].pp;
        else return t.pp[sh];
    };
    if constexpr (SMEM) {
        ShapeRow *w = reinterpret_cast<ShapeRow *>(smem + rows_off);
        for (int i = threadIdx.x; i < S * kMaxJ; i += blockDim.x) {
            const int sh = i / kMaxJ, j = i - sh * kMaxJ;
            const bool in = j < J;
            w[sh].unit[j] = in ? t.unit[sh * J + j] : 0;
            w[sh].inv[j] = in ? t.inv_unit[sh * J + j] : 0.0;
            w[sh].cap[j] = in ? t.cap[sh * J + j] : 0;
            w[sh].order[j] = t.order[i];
            w[sh].rank[j] = t.rank[i];
            w[sh].pmask[j] = t.pmask[i];
        }
        for (int i = threadIdx.x; i < S; i += blockDim.x) {
            w[i].M = t.M[i];
            w[i].olen = t.olen[i];
            w[i].pp = t.pp[i];
        }
    }

    // ---- per-group scratch ----
    const int gib = threadIdx.x / G;
    unsigned char *gs = smem + groups_off + per_group * gib;
    uint64_t *tks = reinterpret_cast<uint64_t *>(gs);                   // [kTopK] top-K candidate list
    int64_t *snM = reinterpret_cast<int64_t *>(tks + kTopK);            // [KPL][G] snapshot: mrem
    uint32_t *Am = reinterpret_cast<uint32_t *>(snM + RMAX);            // [kMaxJ][KPL] direct-take masks
    int32_t *snL = reinterpret_cast<int32_t *>(Am + kMaxJ * KPL);       // [G] snapshot: lam per class lane
    uint32_t *snH = reinterpret_cast<uint32_t *>(snL + G);              // [KPL][G] snapshot: held
    uint32_t *snA = snH + RMAX;                                         // [KPL][G] snapshot: A words
    uint32_t *ulog = snA + RMAX;                                        // [kUndo] exchange x changes
    K1Carry *cy = reinterpret_cast<K1Carry *>(ulog + kUndo);            // carried lookups / snapshot key
    uint16_t *shpS = reinterpret_cast<uint16_t *>(cy + 1);              // [RMAX] shape per replica
    uint8_t *pick = reinterpret_cast<uint8_t *>(shpS + RMAX);           // [RMAX] candidate pick per replica
    int32_t *xs = reinterpret_cast<int32_t *>(gs + group_fixed_bytes<RMAX, KPL>());  // [kMaxJ][RMAX] assignment x
    unsigned long long *blk_best = reinterpret_cast<unsigned long long *>(smem + groups_off + per_group * GPB);
    __syncthreads();

    const Grp g;
    constexpr int TKE = kTopK / G;  // top-K list entries per lane (shared memory)
    if (kLists)
        for (int e = 0; e < TKE; ++e) tks[g.gl * TKE + e] = kNoKey;
    const uint64_t ngroups = static_cast<uint64_t>(gridDim.x) * GPB;

    // Each group walks contiguous chunks of `gchunk` plans, so consecutive
    // plans of a group usually share their partition and every pick but the
    // last run's: the partition / rank-range lookups are cached, and the
    // greedy state at the start of the last run (a step boundary) is kept as
    // a snapshot that the next plan with the same prefix resumes from (the
    // exchange's x changes since are undone from a log).
#ifdef OSERVE_K1_GCH1
    gchunk = 1;
#endif
    const uint64_t gch = static_cast<uint64_t>(gchunk > 0 ? gchunk : 1);
#ifdef OSERVE_K1_STATS
    if (blockIdx.x == 0 && threadIdx.x == 0)
        printf("K1 stats so far: plans %llu reuse %llu greedy steps %llu moves %llu\n", g_k1_stats[0], g_k1_stats[1],
               g_k1_stats[2], g_k1_stats[3]);
    unsigned long long st_plans = 0, st_reuse = 0, st_steps = 0, st_moves = 0;
#endif
    if (g.gl == 0) {
        cy->r_lo = 1;
        cy->r_hi = 0;
        cy->cp_lo = 1;
        cy->cp_hi = 0;
        cy->cpart = -1;
        cy->snap_part = -1;
        cy->best = kNoKey;
        cy->tk_max = kNoKey;
        cy->tk_idx = 0;
        cy->lossy = 0;
    }
    // x changes logged since the snapshot; -1: no live snapshot
    int nlog = -1;
    g.sync();

    // chunks are handed out dynamically (one atomic per chunk): neighbouring
    // plans have correlated costs, so a static split leaves a long tail.
    // Guided: once fewer than ~2 full chunks per group remain, chunks shrink
    // to a quarter so the last ones finish together.
    const uint64_t tail_from = src.count > 2 * ngroups * gch ? src.count - 2 * ngroups * gch : 0;
    const uint64_t gsmall = gch >= 4 ? gch / 4 : 1;
    for (;;) {
    unsigned long long cb = 0;
    uint64_t csz = gch;
    if (g.gl == 0) {
        const unsigned long long seen = *reinterpret_cast<volatile unsigned long long *>(work);
        if (seen >= tail_from) csz = gsmall;
        cb = atomicAdd(work, static_cast<unsigned long long>(csz));
    }
    cb = g.bcast(cb, 0);
    csz = g.bcast(csz, 0);
    if (cb >= src.count) break;
    for (uint64_t i = cb, ce = (cb + csz < src.count ? cb + csz : src.count); i < ce; ++i) {
        // ---- resolve the plan ----
        int R;
        int shp[KPL];
        int64_t part = 0;
        uint64_t local = 0, hi = 0;
        int P = 0;            // first replica of the partition's last run
        bool reuse = false;   // resume the greedy from the snapshot at P
        const int64_t *lam_src = prm.lambda;
        if (kGeneral && src.mode == 2) {
            const uint64_t li = src.first + i;
            R = src.list_R[li];
            const int32_t *ls = src.list_shapes + src.list_off[li];
#pragma unroll
            for (int kk = 0; kk < KPL; ++kk) {
                const int k = g.gl + G * kk;
                shp[kk] = k < R ? ls[k] : 0;
            }
            if (src.list_lambda) lam_src = src.list_lambda + li * J;
            if (skip_exact) {
                int64_t tot = 0;
                for (int j = 0; j < J; ++j) tot += lam_src[j];
                if (tot <= prm.exact_demand_limit && R * J <= prm.exact_cell_limit) continue;
            }
            nlog = -1;
        } else {
            const uint64_t rlo = cy->r_lo, rhi = cy->r_hi, rst = cy->r_start;
            uint64_t cp_lo = cy->cp_lo;
            const uint64_t cp_hi = cy->cp_hi;
            part = cy->cpart;
            g.sync();  // every lane has read the carry before lane 0 updates it
            const uint64_t gr = source_rank_cached(src, src.first + i, cy, g.gl, rlo, rhi, rst);
            if (gr < cp_lo || gr >= cp_hi) {
                part = find_partition(sp, gr);
                cp_lo = __ldg(sp.prefix + part);
                if (g.gl == 0) {
                    cy->cpart = part;
                    cy->cp_lo = cp_lo;
                    cy->cp_hi = __ldg(sp.prefix + part + 1);
                }
            }
            if (skip_exact && sp.exact[part]) continue;
            local = gr - cp_lo;
            R = sp.R[part];
            const int ro = sp.rep_off[part], runo = sp.run_off[part], nr = sp.nruns[part];
            // the last run with a choice (later runs have one multiset each)
            int lr = runo + nr - 1;
            while (lr > runo && sp.run_count[lr] == 1) --lr;
            P = sp.run_start[lr];
            const uint64_t lc = sp.run_count[lr];
            hi = div_small(local, lc);
            const uint64_t rl = local - hi * lc;  // run lr's own rank (weight 1)
            reuse = nlog >= 0 && part == cy->snap_part && hi == cy->snap_hi;
#ifdef OSERVE_K1_NOREUSE
            reuse = false;
#endif
            if (!reuse) {
                // runs of one replica: lane-parallel; longer runs: group-uniform
                uint32_t longm[KPL];
#pragma unroll
                for (int t = 0; t < KPL; ++t) {
                    const int ri = g.gl + G * t;
                    bool lng = false;
                    if (ri < nr && runo + ri != lr) {
                        const int len = sp.run_len[runo + ri];
                        if (len == 1) {
                            const uint64_t w = sp.run_weight[runo + ri], c = sp.run_count[runo + ri];
                            uint64_t rr = div_small(local, w);
                            rr = rr - div_small(rr, c) * c;
                            pick[sp.run_start[runo + ri]] = static_cast<uint8_t>(rr);
                        } else {
                            lng = true;
                        }
                    }
                    longm[t] = g.ballot(lng);
                }
#pragma unroll
                for (int t = 0; t < KPL; ++t) {
                    while (longm[t]) {
                        const int ri = __ffs(longm[t]) - 1 + G * t;
                        longm[t] &= longm[t] - 1;
                        const uint64_t w = sp.run_weight[runo + ri], c = sp.run_count[runo + ri];
                        uint64_t rr = div_small(local, w);
                        rr = rr - div_small(rr, c) * c;
                        unrank_run_group(g, rr, sp.run_len[runo + ri], sp.run_q[runo + ri],
                                         pick + sp.run_start[runo + ri]);
                    }
                }
            }
            {
                const int len = sp.run_len[lr];
                if (len == 1) {
                    if (g.gl == 0) pick[P] = static_cast<uint8_t>(rl);
                } else {
                    unrank_run_group(g, rl, len, sp.run_q[lr], pick + P);
                }
            }
            g.sync();
#pragma unroll
            for (int kk = 0; kk < KPL; ++kk) {
                const int k = g.gl + G * kk;
                shp[kk] = k < R ? sp.cl_shape[sp.rep_list[ro + k] * kMaxCand + pick[k]] : 0;
            }
        }

        // ---- init: lam (lane j holds class j), x = 0 (or the snapshot) ----
        int32_t lamr;
        int64_t mrem[KPL];
        uint32_t held[KPL];
        uint32_t areg[KPL];  // lane c: A[c] word per ownership slot, built replica by replica
#pragma unroll
        for (int kk = 0; kk < KPL; ++kk) {
            const int k = g.gl + G * kk;
            if (k < R) shpS[k] = static_cast<uint16_t>(shp[kk]);
        }
        if (reuse) {
            // undo the previous plans' exchange moves (+-1 changes commute)
#pragma unroll 1
            for (int e = g.gl; e < nlog; e += G) {
                const uint32_t v = ulog[e];
                if (v != 0xffffffffu) atomicAdd(&xs[v >> 1], (v & 1u) ? -1 : 1);
            }
            g.sync();
            lamr = snL[g.gl];
#pragma unroll
            for (int kk = 0; kk < KPL; ++kk) {
                const int k = g.gl + G * kk;
                mrem[kk] = snM[kk * G + g.gl];
                held[kk] = snH[kk * G + g.gl];
                areg[kk] = snA[kk * G + g.gl];
                if (k >= P && k < R) {
OSERVE_K1_ZUNROLL
                    for (int j = 0; j < J; ++j) xs[j * RMAX + k] = 0;
                }
            }
        } else {
            nlog = -1;
            lamr = g.gl < J ? static_cast<int32_t>(lam_src[g.gl]) : 0;
#pragma unroll
            for (int kk = 0; kk < KPL; ++kk) {
                mrem[kk] = 0;
                held[kk] = 0;
                areg[kk] = 0;
            }
            int4 *xz = reinterpret_cast<int4 *>(xs);
            const int n4 = (J * RMAX) >> 2;  // RMAX is a multiple of 4
#pragma unroll 1
            for (int q = g.gl; q < n4; q += G) xz[q] = make_int4(0, 0, 0, 0);
        }
        if (reuse) nlog = 0;
        g.sync();
#ifdef OSERVE_K1_STATS
        ++st_plans;
        st_reuse += reuse;
#endif

        // ---- greedy_fill (flowassign.cpp:393-406) ----
        // Replicas in order; inside one replica the reference takes
        // min(cap, lam) for a prefix of its ascending-unit class order, one
        // partial class where the budget binds, then nothing (every later
        // class costs >= the binding unit > the budget left).  So one replica
        // is one prefix scan of costs over its order positions (lane = position)
        // plus a ballot for the binding position.  Bit-identical to the
        // sequential fill; no 64-bit division.
        // shape-run boundaries: bit k set when replica k+1 has another shape
        // (or starts the last run: the snapshot point is a step boundary)
        uint32_t bnd[KPL];
#pragma unroll
        for (int kk = 0; kk < KPL; ++kk) {
            const int k = g.gl + G * kk;
            const bool last = k < R && (k + 1 == R || shpS[k + 1] != shpS[k] || k + 1 == P);
            bnd[kk] = g.ballot(last);
        }
        for (int k = reuse ? P : 0; k < R;) {
#ifdef OSERVE_K1_STATS
            ++st_steps;
#endif
            if (k == P && P > 0 && !reuse) {  // snapshot the prefix state
                snL[g.gl] = lamr;
#pragma unroll
                for (int kk = 0; kk < KPL; ++kk) {
                    snM[kk * G + g.gl] = mrem[kk];
                    snH[kk * G + g.gl] = held[kk];
                    snA[kk * G + g.gl] = areg[kk];
                }
                nlog = 0;
                if (g.gl == 0) {
                    cy->snap_part = part;
                    cy->snap_hi = hi;
                }
            }
            const int s = shpS[k];
            const int ol = tOlen(s);
            const bool act = g.gl < ol;
            const int j = act ? tOrder(s, g.gl) : 0;
            const int32_t lamp = g.bcast(lamr, j);
            const int64_t Ms = tM(s);
            int64_t u = 1;
            int32_t a = 0, capj = 0;
            if (act) {
                u = tUnit(s, j);
                capj = tCap(s, j);
                a = min(capj, lamp);
            }
            const uint64_t cost = static_cast<uint64_t>(a) * static_cast<uint64_t>(u);
            // (over min(G, 16) >= J lanes: positions past the shape's order add 0)
            const uint64_t csum = g.template scan_sat64<(G < kMaxJ ? G : kMaxJ)>(cost, static_cast<uint64_t>(Ms) + 1);
            // exclusive prefix from the previous lane: unsaturated up to the
            // binding position (csum - cost is not, once saturated)
            uint64_t excl = __shfl_up_sync(g.mask, csum, 1, G);
            if (g.gl == 0) excl = 0;
            const uint32_t ob = g.ballot(act && csum > static_cast<uint64_t>(Ms));
            const int pb = ob ? __ffs(ob) - 1 : ol;
            int32_t take = 0;
            if (act) {
                if (g.gl < pb) take = a;
                else if (g.gl == pb) take = quot_small(Ms - static_cast<int64_t>(excl), u, tInv(s, j));
            }
            const uint64_t used_l = (g.gl == pb) ? excl + static_cast<uint64_t>(take) * static_cast<uint64_t>(u) : csum;
            const uint64_t used = ol ? g.bcast(used_l, pb < ol ? pb : ol - 1) : 0ull;
            // held classes (low 16 bits) and full classes x == cap (high 16 bits)
            const uint32_t hb = g.or_all((take > 0 ? (1u << j) : 0u) | (act && take >= capj ? (1u << (j + 16)) : 0u));
            const int64_t mfin = Ms - static_cast<int64_t>(used);
            // run-length step: the next c replicas of the same shape take the
            // identical fill while lam_p - i*take_p >= a_p at every position
            // p <= pb with take_p > 0 (then min(cap, lam) is unchanged up to
            // the binding position, hence so are the costs and the fill).
            int run_end = R - 1;
#pragma unroll
            for (int kk = KPL - 1; kk >= 0; --kk) {
                const int lo = k - G * kk;  // first bit of this slot at or after k
                uint32_t m = bnd[kk];
                if (lo >= G) m = 0;
                else if (lo > 0) m &= ~((1u << lo) - 1u);
                if (m) run_end = __ffs(m) - 1 + G * kk;
            }
            int c = 0;
            if (run_end > k) {  // same shape follows: how many can take the identical fill
                // c = min(run length left L, min over positions of (lam_p - a_p) / take_p):
                // the quotient only matters below L, so divide only then
                const uint32_t L = static_cast<uint32_t>(run_end - k);
                uint32_t cb = L;
                if (act && take > 0 && g.gl <= pb) {
                    const uint32_t xq = static_cast<uint32_t>(lamp - a), tq = static_cast<uint32_t>(take);
                    if (static_cast<uint64_t>(L) * tq > xq) cb = xq / tq;
                }
                cb = __reduce_min_sync(g.mask, cb);
                c = static_cast<int>(cb);
            }
            if (act && take) {
OSERVE_K1_TUNROLL
                for (int q = 0; q <= c; ++q) xs[j * RMAX + k + q] = take;
            }
            // direct-take bit of (class at this position, replicas k..k+c)
            const bool abit = act && take < capj && mfin >= u;
            const int rp = g.gl < J ? tRank(s, g.gl) : 0xff;
            const int src_p = rp < G ? rp : 0;
            const int32_t tk = g.bcast(take, src_p);
            const bool ab = g.bcast(abit ? 1 : 0, src_p) != 0;
            if (rp != 0xff) {
                lamr -= tk * (c + 1);
                if (ab) {
#pragma unroll
                    for (int kk = 0; kk < KPL; ++kk) {
                        const int lo = max(k, G * kk) - G * kk, hi = min(k + c, G * kk + G - 1) - G * kk;
                        if (lo <= hi) {
                            const uint32_t span = (hi - lo == 31) ? 0xffffffffu : (((1u << (hi - lo + 1)) - 1u) << lo);
                            areg[kk] |= span;
                        }
                    }
                }
            }
#pragma unroll
            for (int kk = 0; kk < KPL; ++kk) {
                const int kq = g.gl + G * kk;
                if (kq >= k && kq <= k + c) {
                    mrem[kk] = mfin;
                    held[kk] = hb;
                }
            }
            k += c + 1;
        }
        g.sync();

        // ---- exchange_improve (flowassign.cpp:411-448) ----
        // A[j] = replicas able to take one more class-j request directly (one
        // G-bit word per ownership slot kk; lane j is the only writer of class
        // j's words).  (j, k) has a move iff lam_j > 0, unit > 0, x < cap and
        // either mrem >= unit (direct) or some held class j2 != j has
        // A[j2]\{k} non-empty and unit[k][j2] >= unit[k][j] - mrem[k].  The
        // first such (j asc, k asc), then first j2 asc, first k2 asc, is the
        // reference's first move.  F[kk] caches the feasible classes of each
        // owned replica; a move changes only replicas kf, k2 (and lam_jf), so
        // after it F is recomputed for those two and for replicas holding a
        // class whose A set crossed size 2 (the only way A[j2]\{k} can change
        // emptiness for a third replica).
        if (g.gl < J) {
#pragma unroll
            for (int kk = 0; kk < KPL; ++kk) Am[g.gl * KPL + kk] = areg[kk];
        }
        uint32_t lam_mask = g.ballot(g.gl < J && lamr > 0);
        // classes whose A set has >= 2 members / exactly 1 member
        uint32_t M2, M1;
        {
            int pc = 0;
#pragma unroll
            for (int kk = 0; kk < KPL; ++kk) pc += __popc(areg[kk]);
            M2 = g.ballot(g.gl < J && pc >= 2);
            M1 = g.ballot(g.gl < J && pc == 1);
        }
        g.sync();
        // held classes of owned replica kk whose A set minus k is non-empty:
        // |A| >= 2, or |A| == 1 and the member is not k itself
        auto eligible_held = [&](uint32_t hb, int kk) -> uint32_t {
            uint32_t el = hb & M2, h1 = hb & M1;
            while (h1) {
                const int j2 = __ffs(h1) - 1;
                h1 &= h1 - 1;
                if (!((Am[j2 * KPL + kk] >> g.gl) & 1u)) el |= 1u << j2;
            }
            return el;
        };
        // feasible classes of owned replica kk given its eligible held set
        // feasible classes of owned replica kk given its eligible held set:
        // j is feasible iff lam_j > 0, x < cap and u_j <= mrem + max(e(j), 0)
        // (e(j) = largest eligible held unit other than j's own).  Units
        // ascend along the shape's class order, so for j != e1j that is a
        // prefix of the order (binary search + prefix mask); e1j is checked
        // against e2 separately.
        auto feasible_row = [&](int kk, uint32_t el) -> uint32_t {
            const int k = g.gl + G * kk;
            if (k >= R) return 0u;
            const uint32_t cand = lam_mask & ~(rsel(held, kk) >> 16);
            if (!cand) return 0u;
            const int s = rsel(shp, kk);
            const int64_t mr = rsel(mrem, kk);
            int64_t e1 = -1, e2 = -1;
            int e1j = -1;
            while (el) {
                const int j2 = __ffs(el) - 1;
                el &= el - 1;
                const int64_t u2 = tUnit(s, j2);
                if (u2 > e1) {
                    e2 = e1;
                    e1 = u2;
                    e1j = j2;
                } else if (u2 > e2) {
                    e2 = u2;
                }
            }
            const uint64_t T1 = static_cast<uint64_t>(mr) + static_cast<uint64_t>(e1 > 0 ? e1 : 0);
            int lo = 0, hi = tOlen(s);
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (static_cast<uint64_t>(tUnit(s, tOrder(s, mid))) <= T1) lo = mid + 1;
                else hi = mid;
            }
            uint32_t f = lo ? (static_cast<uint32_t>(tPmask(s, lo - 1)) & cand) : 0u;
            if (e1j >= 0 && ((f >> e1j) & 1u)) {
                const uint64_t T2 = static_cast<uint64_t>(mr) + static_cast<uint64_t>(e2 > 0 ? e2 : 0);
                if (static_cast<uint64_t>(tUnit(s, e1j)) > T2) f &= ~(1u << e1j);
            }
            return f;
        };
        uint32_t F[KPL], E[KPL];
#pragma unroll
        for (int kk = 0; kk < KPL; ++kk) F[kk] = E[kk] = 0u;
OSERVE_K1_XUNROLL
        for (int kk = 0; kk < KPL; ++kk) {
            const uint32_t e = g.gl + G * kk < R ? eligible_held(rsel(held, kk), kk) : 0u;
            rput(E, kk, e);
            rput(F, kk, feasible_row(kk, e));
        }
        for (;;) {
            uint32_t anyF = 0;
#pragma unroll
            for (int kk = 0; kk < KPL; ++kk) anyF |= F[kk];
            anyF = g.or_all(anyF);
            if (!anyF) break;
            const int jf = __ffs(anyF) - 1;
            int kf = -1;
#pragma unroll
            for (int kk = KPL - 1; kk >= 0; --kk) {
                const uint32_t b = g.ballot((F[kk] >> jf) & 1u);
                if (b) kf = __ffs(b) - 1 + G * kk;
            }
            // the move at (jf, kf): direct when mrem >= unit, else the first
            // held class j2 asc of kf (j2 != jf, mrem + unit[j2] >= unit[jf])
            // whose A set minus kf is non-empty, and its first replica k2 —
            // class-parallel (lane = j2), kf's state broadcast by its owner
            const int ogl = kf & (G - 1), okk = kf / G;
            const int64_t mr_f = g.bcast(rsel(mrem, okk), ogl);
            const uint32_t hb_f = g.bcast(rsel(held, okk), ogl) & 0xffffu & ~(1u << jf);
            const int s_f = shpS[kf];
            const int64_t u_f = tUnit(s_f, jf);
            int j2 = -1, k2 = -1;
            if (mr_f < u_f && hb_f) {
                int kc = -1;
                if (((hb_f >> g.gl) & 1u) && mr_f + tUnit(s_f, g.gl) >= u_f) {
#pragma unroll
                    for (int k3 = KPL - 1; k3 >= 0; --k3) {
                        uint32_t w = Am[g.gl * KPL + k3];
                        if (k3 == okk) w &= ~(1u << ogl);
                        if (w) kc = __ffs(w) - 1 + G * k3;
                    }
                }
                const uint32_t cb = g.ballot(kc >= 0);
                if (cb) {
                    j2 = __ffs(cb) - 1;
                    k2 = g.bcast(kc, j2);
                }
            }
            // apply the move (logged while a snapshot is live)
            const bool lg = nlog >= 0 && nlog + 3 <= kUndo;
#pragma unroll
            for (int kk = 0; kk < KPL; ++kk) {
                const int k = g.gl + G * kk;
                const int s = shp[kk];
                if (k == kf) {
                    const int32_t xv = xs[jf * RMAX + kf] + 1;
                    xs[jf * RMAX + kf] = xv;
                    mrem[kk] -= tUnit(s, jf);
                    held[kk] |= (1u << jf) | (xv >= tCap(s, jf) ? 1u << (jf + 16) : 0u);
                    if (j2 >= 0) {
                        const int32_t nv = xs[j2 * RMAX + kf] - 1;
                        xs[j2 * RMAX + kf] = nv;
                        mrem[kk] += tUnit(s, j2);
                        held[kk] &= ~(1u << (j2 + 16));  // now below cap
                        if (nv == 0) held[kk] &= ~(1u << j2);
                    }
                    if (lg) {
                        ulog[nlog] = (static_cast<uint32_t>(jf * RMAX + kf) << 1) | 1u;
                        ulog[nlog + 1] = j2 >= 0 ? static_cast<uint32_t>(j2 * RMAX + kf) << 1 : 0xffffffffu;
                        if (j2 < 0) ulog[nlog + 2] = 0xffffffffu;
                    }
                }
                if (j2 >= 0 && k == k2) {
                    const int32_t xv = xs[j2 * RMAX + k2] + 1;
                    xs[j2 * RMAX + k2] = xv;
                    mrem[kk] -= tUnit(s, j2);
                    held[kk] |= (1u << j2) | (xv >= tCap(s, j2) ? 1u << (j2 + 16) : 0u);
                    if (lg) ulog[nlog + 2] = (static_cast<uint32_t>(j2 * RMAX + k2) << 1) | 1u;
                }
            }
            if (lg) nlog += 3;
            else nlog = -1;
#ifdef OSERVE_K1_STATS
            ++st_moves;
#endif
            if (g.gl == jf) lamr -= 1;
            lam_mask = g.ballot(g.gl < J && lamr > 0);
            g.sync();
            // refresh the A bits of rows kf and k2 (lane j = class j)
            uint32_t dirty = 0;
            // apply row r's new direct-take bit p for class j (lane j)
            auto a_apply = [&](int j, int r, bool p) {
                const int rgl = r & (G - 1), rkk = r / G;
                const uint32_t bit = 1u << rgl;
                const uint32_t old = Am[j * KPL + rkk];
                if (p != ((old & bit) != 0)) {
                    int pc = 0;
#pragma unroll
                    for (int k3 = 0; k3 < KPL; ++k3) pc += __popc(Am[j * KPL + k3]);
                    Am[j * KPL + rkk] = p ? (old | bit) : (old & ~bit);
                    const int pn = pc + (p ? 1 : -1);
                    if (pc < 2 || pn < 2) dirty |= 1u << j;
                }
            };
            if constexpr (G == 32) {
                // J <= 16: half h evaluates row (kf, k2)[h]; lane j of the low
                // half applies both in order (they may share an A word)
                const int h = g.gl >> 4, j = g.gl & 15;
                const int r = (h && j2 >= 0) ? k2 : kf;
                const int rgl = r & (G - 1), rkk = r / G;
                int64_t mr = 0;
#pragma unroll
                for (int kk = 0; kk < KPL; ++kk) {
                    const int64_t v = __shfl_sync(0xffffffffu, mrem[kk], rgl);
                    if (kk == rkk) mr = v;
                }
                bool p = false;
                if (j < J) {
                    const int sr = shpS[r];
                    const int64_t u = tUnit(sr, j);
                    p = u > 0 && xs[j * RMAX + r] < tCap(sr, j) && mr >= u;
                }
                const bool p_hi = __shfl_down_sync(0xffffffffu, p, 16) != 0;
                if (h == 0 && j < J) {
                    a_apply(j, kf, p);
                    if (j2 >= 0) a_apply(j, k2, p_hi);
                }
            } else {
                for (int q = 0; q < (j2 >= 0 ? 2 : 1); ++q) {
                    const int r = q == 0 ? kf : k2;
                    const int rgl = r & (G - 1), rkk = r / G;
                    int64_t mr = 0;
#pragma unroll
                    for (int kk = 0; kk < KPL; ++kk)
                        if (kk == rkk) mr = mrem[kk];
                    mr = g.bcast(mr, rgl);
                    if (g.gl < J) {
                        const int j = g.gl;
                        const int sr = shpS[r];
                        const int64_t u = tUnit(sr, j);
                        a_apply(j, r, u > 0 && xs[j * RMAX + r] < tCap(sr, j) && mr >= u);
                    }
                }
            }
            dirty = g.or_all(dirty);
            g.sync();
            if (dirty) {  // an A set crossed size 1 or 2: refresh M1 / M2
                int pc = 0;
                if (g.gl < J) {
#pragma unroll
                    for (int k3 = 0; k3 < KPL; ++k3) pc += __popc(Am[g.gl * KPL + k3]);
                }
                M2 = g.ballot(g.gl < J && pc >= 2);
                M1 = g.ballot(g.gl < J && pc == 1);
            }
            // rows whose feasible set must be rebuilt: kf, k2, and rows whose
            // eligible-held set changed (only possible through dirty classes)
            uint32_t redo = 0;  // bit kk: owned row kk must be rebuilt
OSERVE_K1_XUNROLL
            for (int kk = 0; kk < KPL; ++kk) {
                const int k = g.gl + G * kk;
                if (k >= R) continue;
                const uint32_t hk = rsel(held, kk);
                if (k == kf || k == k2) redo |= 1u << kk;
                else if ((hk & dirty) && eligible_held(hk, kk) != rsel(E, kk)) redo |= 1u << kk;
                else rput(F, kk, rsel(F, kk) & lam_mask);
            }
            // many rows: every lane rebuilds its own rows (in parallel);
            // few rows: class-parallel rebuild, one row at a time
            int nredo = 0;
#pragma unroll
            for (int kk = 0; kk < KPL; ++kk) nredo += __popc(g.ballot((redo >> kk) & 1u));
            if (nredo > 4) {
OSERVE_K1_XUNROLL
                for (int kk = 0; kk < KPL; ++kk)
                    if ((redo >> kk) & 1u) {
                        const uint32_t e = eligible_held(rsel(held, kk), kk);
                        rput(E, kk, e);
                        rput(F, kk, feasible_row(kk, e));
                    }
                redo = 0;
            }
            if constexpr (G == 32) {
                // J <= 16: two rows per step, half h (lanes 16h..16h+15,
                // lane = class) rebuilds the h-th row of the pair
                // rows to rebuild, one 32-bit word per slot (bit = owner lane)
                uint32_t r0 = g.ballot(redo & 1u), r1 = 0, r2 = 0, r3 = 0;
                if (KPL > 1) r1 = g.ballot((redo >> 1) & 1u);
                if (KPL > 2) {
                    r2 = g.ballot((redo >> 2) & 1u);
                    r3 = g.ballot((redo >> 3) & 1u);
                }
                const int h = g.gl >> 4, j = g.gl & 15;
                const uint32_t hm = h ? 0xffff0000u : 0x0000ffffu;
                auto pop1 = [](uint32_t &w, int base) -> int {
                    const int r = __ffs(w) - 1 + base;
                    w &= w - 1;
                    return r;
                };
                auto pop = [&]() -> int {  // next row index, ascending; -1 when none
                    if (r0) return pop1(r0, 0);
                    if (KPL > 1 && r1) return pop1(r1, 32);
                    if (KPL > 2 && r2) return pop1(r2, 64);
                    if (KPL > 2 && r3) return pop1(r3, 96);
                    return -1;
                };
                for (;;) {
                    const int ra = pop();
                    if (ra < 0) break;
                    const int rb = pop();
                    const int r = (h && rb >= 0) ? rb : ra;  // an idle high half mirrors row a
                    const int rgl = r & (G - 1), kk = r / G;
                    int64_t mr = 0;
                    uint32_t hr = 0;
#pragma unroll
                    for (int q = 0; q < KPL; ++q) {
                        const int64_t v = __shfl_sync(0xffffffffu, mrem[q], rgl);
                        const uint32_t w = __shfl_sync(0xffffffffu, held[q], rgl);
                        if (q == kk) {
                            mr = v;
                            hr = w;
                        }
                    }
                    const int sr = shpS[r];
                    bool el = false;
                    if (j < J && ((hr >> j) & 1u))
                        el = ((M2 >> j) & 1u) || (((M1 >> j) & 1u) && !((Am[j * KPL + kk] >> rgl) & 1u));
                    const uint32_t Eb = __ballot_sync(0xffffffffu, el);
                    const uint32_t rk1 = el ? static_cast<uint32_t>(tRank(sr, j)) + 1u : 0u;
                    const uint32_t t1 = __reduce_max_sync(hm, rk1);
                    const uint32_t t2 = __reduce_max_sync(hm, rk1 == t1 ? 0u : rk1);
                    int64_t e1 = -1, e2 = -1;
                    int e1j = -1;
                    if (t1) {
                        e1j = tOrder(sr, t1 - 1);
                        e1 = tUnit(sr, e1j);
                    }
                    if (t2) e2 = tUnit(sr, tOrder(sr, t2 - 1));
                    bool f = false;  // x < cap: not full; u > 0: in the shape's order
                    if (j < J && ((lam_mask >> j) & 1u) && !((hr >> (16 + j)) & 1u) &&
                        tRank(sr, j) != 0xff) {
                        const int64_t u = tUnit(sr, j);
                        f = mr >= u || (e1j == j ? e2 : e1) >= u - mr;
                    }
                    const uint32_t Fb = __ballot_sync(0xffffffffu, f);
                    if (g.gl == (ra & (G - 1))) {
                        rput(E, ra / G, Eb & 0xffffu);
                        rput(F, ra / G, Fb & 0xffffu);
                    }
                    if (rb >= 0 && g.gl == (rb & (G - 1))) {
                        rput(E, rb / G, Eb >> 16);
                        rput(F, rb / G, Fb >> 16);
                    }
                }
            } else
#pragma unroll 1
            for (int kk = 0; kk < KPL; ++kk) {
                uint32_t rows = g.ballot((redo >> kk) & 1u);
                while (rows) {  // class-parallel rebuild, one row at a time
                    const int rgl = __ffs(rows) - 1;
                    rows &= rows - 1;
                    const int r = rgl + G * kk;
                    const int sr = shpS[r];
                    const int64_t mr = g.bcast(rsel(mrem, kk), rgl);
                    const uint32_t hr = g.bcast(rsel(held, kk), rgl);
                    const int j = g.gl;
                    bool el = false;
                    if (j < J && ((hr >> j) & 1u))
                        el = ((M2 >> j) & 1u) || (((M1 >> j) & 1u) && !((Am[j * KPL + kk] >> rgl) & 1u));
                    const uint32_t Er = g.ballot(el);
                    // top-2 eligible unit: order positions ascend with unit
                    const uint32_t rk1 = el ? static_cast<uint32_t>(tRank(sr, j)) + 1u : 0u;
                    const uint32_t t1 = __reduce_max_sync(g.mask, rk1);
                    const uint32_t t2 = __reduce_max_sync(g.mask, rk1 == t1 ? 0u : rk1);
                    int64_t e1 = -1, e2 = -1;
                    int e1j = -1;
                    if (t1) {
                        e1j = tOrder(sr, t1 - 1);
                        e1 = tUnit(sr, e1j);
                    }
                    if (t2) e2 = tUnit(sr, tOrder(sr, t2 - 1));
                    bool f = false;
                    if (j < J && ((lam_mask >> j) & 1u)) {
                        const int64_t u = tUnit(sr, j);
                        if (u > 0 && xs[j * RMAX + r] < tCap(sr, j))
                            f = mr >= u || (e1j == j ? e2 : e1) >= u - mr;
                    }
                    const uint32_t Fr = g.ballot(f);
                    if (g.gl == rgl) {
                        rput(E, kk, Er);
                        rput(F, kk, Fr);
                    }
                }
            }
        }

        // ---- objective, sum_pp, key / outputs ----
        uint32_t served = g.gl < J ? static_cast<uint32_t>(lam_src[g.gl] - lamr) : 0u;
        uint32_t spp = 0;
#pragma unroll
        for (int kk = 0; kk < KPL; ++kk)
            if (g.gl + G * kk < R) spp += tPP(shp[kk]);
        served = g.sum(served);
        spp = g.sum(spp);
        if (kGeneral && out.objective && g.gl == 0) out.objective[i] = served;
        if (kGeneral && out.sum_pp && g.gl == 0) out.sum_pp[i] = static_cast<int32_t>(spp);
        if (kGeneral && out.x) {
#pragma unroll
            for (int kk = 0; kk < KPL; ++kk) {
                const int k = g.gl + G * kk;
                if (k < R) {
                    for (int j = 0; j < J; ++j)
                        out.x[(i * out.rmax + k) * J + j] = xs[j * RMAX + k];
                    if (out.used) out.used[i * out.rmax + k] = tM(shp[kk]) - mrem[kk];
                }
            }
        }
        if (out.best_key) {
            const uint64_t kv = ((key.obj_max - served) << key.sh_obj) |
                                (static_cast<uint64_t>(part) << key.sh_part) |
                                (static_cast<uint64_t>(spp) << key.sh_spp) | local;
            if (g.gl == 0 && kv < cy->best) cy->best = kv;
            if (kLists && out.topk) {
                // per-group top-kTopK list, kTopK/G entries per lane (shared memory)
                const uint64_t tk_max = cy->tk_max;
                if (kv < tk_max) {
                    if (g.gl == 0) {
                        if (tk_max != kNoKey) cy->lossy = 1;  // evicts the current worst
                        tks[cy->tk_idx] = kv;
                    }
                    g.sync();
                    uint64_t lm = tks[g.gl * TKE];
                    int ls = 0;
#pragma unroll
                    for (int e = 1; e < TKE; ++e) {
                        const uint64_t v = tks[g.gl * TKE + e];
                        if (v > lm) {
                            lm = v;
                            ls = e;
                        }
                    }
                    uint64_t gm = lm;
#pragma unroll
                    for (int d = G / 2; d > 0; d >>= 1) {
                        const uint64_t o = __shfl_xor_sync(g.mask, gm, d, G);
                        gm = o > gm ? o : gm;
                    }
                    const int ml = __ffs(g.ballot(lm == gm)) - 1;
                    const int ti = ml * TKE + g.bcast(ls, ml);
                    if (g.gl == 0) {
                        cy->tk_idx = ti;
                        cy->tk_max = gm;
                    }
                } else if (g.gl == 0) {
                    cy->lossy = 1;
                }
            }
            if (kLists && out.collect && kv <= out.collect_thr && g.gl == 0) {
                const unsigned slot = atomicAdd(out.collect_n, 1u);
                if (slot < out.collect_cap) out.collect[slot] = kv;
            }
        }
        g.sync();
    }
    }
    if (kLists && out.topk) {
        const uint64_t gid = static_cast<uint64_t>(blockIdx.x) * GPB + gib;
        g.sync();
        for (int e = 0; e < TKE; ++e) out.topk[gid * kTopK + g.gl * TKE + e] = tks[g.gl * TKE + e];
        if (g.gl == 0) out.topk_meta[gid] = cy->lossy ? cy->tk_max : kNoKey;
    }

#ifdef OSERVE_K1_STATS
    if (g.gl == 0) {
        atomicAdd(&g_k1_stats[0], st_plans);
        atomicAdd(&g_k1_stats[1], st_reuse);
        atomicAdd(&g_k1_stats[2], st_steps);
        atomicAdd(&g_k1_stats[3], st_moves);
    }
#endif
    // ---- CTA argmin -> global atomicMin ----
    if (out.best_key) {
        if (g.gl == 0) blk_best[gib] = cy->best;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long b = blk_best[0];
            for (int q = 1; q < GPB; ++q) b = blk_best[q] < b ? blk_best[q] : b;
            if (b != kNoKey) atomicMin(reinterpret_cast<unsigned long long *>(out.best_key), b);
        }
    }
}

template <int G, int KPL>
size_t plan_eval_smem(int S, int J, bool stage) {
    constexpr int GPB = 256 / G;
    const size_t shapes = stage ? (size_t)S * sizeof(ShapeRow) : 0;
    return ((group_scratch_bytes<G, KPL>(J) * GPB + GPB * 8 + 15) & ~size_t(15)) + shapes;
}

// Launch geometry of K1 (also used to size the top-K lists).
template <int G, int KPL, int V = kK1Round>
int plan_eval_geometry(const ShapeTables &t, int J, int sm_count, uint64_t count, size_t *smem_out, bool *stage_out,
                       uint64_t *grid_out) {
    const bool stage = plan_eval_smem<G, KPL>(t.num_shapes, J, true) <= 160 * 1024;
    const size_t smem = plan_eval_smem<G, KPL>(t.num_shapes, J, stage);
    auto kern = stage ? k_plan_eval<G, KPL, true, V> : k_plan_eval<G, KPL, false, V>;
    // occupancy per (device, kernel, smem), computed once: the attribute and
    // occupancy queries are host API calls that a per-partition caller (search
    // -> best_strategies) would otherwise pay on every launch
    static std::mutex mu;
    static std::map<std::tuple<int, const void *, size_t>, int> occ;
    int dev = 0;
    if (cudaError_t e = cudaGetDevice(&dev)) return static_cast<int>(e);
    int per_sm = 0;
    {
        std::lock_guard<std::mutex> lk(mu);
        const auto key = std::make_tuple(dev, reinterpret_cast<const void *>(kern), smem);
        auto it = occ.find(key);
        if (it != occ.end()) {
            per_sm = it->second;
        } else {
            // the dynamic shared-memory limit only ever rises, once per
            // (device, kernel), to the device's opt-in maximum: a lowered
            // limit would invalidate launches cached at larger sizes
            static std::map<std::pair<int, const void *>, bool> raised;
            const auto rk = std::make_pair(dev, reinterpret_cast<const void *>(kern));
            if (smem > 48 * 1024 && !raised[rk]) {
                int optin = 0;
                cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
                if (e != cudaSuccess) return static_cast<int>(e);
                e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
                if (e != cudaSuccess) return static_cast<int>(e);
                raised[rk] = true;
            }
            if (smem > 48 * 1024) {
                int optin = 0;
                cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
                if (smem > static_cast<size_t>(optin)) return static_cast<int>(cudaErrorInvalidValue);
            }
            cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem);
            if (e != cudaSuccess) return static_cast<int>(e);
            occ.emplace(key, per_sm);
        }
    }
    if (per_sm < 1) return static_cast<int>(cudaErrorInvalidConfiguration);
    constexpr int GPB = 256 / G;
    uint64_t need = (count + GPB - 1) / GPB;
    uint64_t grid = static_cast<uint64_t>(per_sm) * sm_count;
    if (need < grid) grid = need;
    *smem_out = smem;
    *stage_out = stage;
    *grid_out = grid;
    return 0;
}

// K1's dynamic chunk counter: one zeroed 128-byte line per launch, taken
// from the calling context's ring (WorkRing, owned per context and device;
// memset on the launch stream, so launches in flight on other streams or
// from other contexts never share one).
unsigned long long *work_counter(WorkRing *ring, cudaStream_t stream) {
    if (!ring || !ring->base || ring->slots <= 0) return nullptr;
    unsigned long long *c = ring->base + (ring->next++ % static_cast<unsigned>(ring->slots)) * 16;
    if (cudaMemsetAsync(c, 0, sizeof(unsigned long long), stream) != cudaSuccess) return nullptr;
    return c;
}

template <int G, int KPL, int V>
int run_plan_eval_v(const ShapeTables &t, const SpaceTables &sp, const KeyLayout &key, const PlanSource &src,
                  const PlanOutputs &out, const SolveParams &prm, int sm_count, int skip_exact,
                  WorkRing *ring, cudaStream_t stream, uint64_t *launches) {
    cudaGetLastError();  // clear any stale (non-sticky) error before launching
    size_t smem = 0;
    bool stage = false;
    uint64_t grid = 0;
    if (int e = plan_eval_geometry<G, KPL, V>(t, prm.J, sm_count, src.count, &smem, &stage, &grid)) return e;
    auto kern = stage ? k_plan_eval<G, KPL, true, V> : k_plan_eval<G, KPL, false, V>;
    if (grid == 0) return 0;
    // contiguous plans per group (greedy-prefix reuse), >= 4 chunks per group
    constexpr int GPB = 256 / G;
    const uint64_t groups = grid * GPB;
    uint64_t gch = src.count / (groups ? groups * 4 : 1);
    gch = gch < 1 ? 1 : (gch > kGroupChunk ? kGroupChunk : gch);
    unsigned long long *work = work_counter(ring, stream);
    if (!work) return static_cast<int>(cudaErrorMemoryAllocation);
    kern<<<static_cast<unsigned>(grid), 256, smem, stream>>>(t, sp, key, src, out, prm, skip_exact,
                                                               static_cast<int>(gch), work);
    if (launches) ++*launches;
    return check(cudaGetLastError());
}

// The variant a launch needs: per-plan outputs or explicit lists -> general;
// key lists -> top-K; otherwise the round kernel.
template <int G, int KPL>
int run_plan_eval(const ShapeTables &t, const SpaceTables &sp, const KeyLayout &key, const PlanSource &src,
                  const PlanOutputs &out, const SolveParams &prm, int sm_count, int skip_exact, WorkRing *ring,
                  cudaStream_t stream, uint64_t *launches) {
    if (src.mode == 2 || out.objective || out.sum_pp || out.x || out.used)
        return run_plan_eval_v<G, KPL, kK1General>(t, sp, key, src, out, prm, sm_count, skip_exact, ring, stream,
                                                   launches);
    if (out.topk || out.collect)
        return run_plan_eval_v<G, KPL, kK1TopK>(t, sp, key, src, out, prm, sm_count, skip_exact, ring, stream,
                                                launches);
    return run_plan_eval_v<G, KPL, kK1Round>(t, sp, key, src, out, prm, sm_count, skip_exact, ring, stream, launches);
}

// ------------------------------------------------------------------- K4 ---
// Exact branch-and-bound, thread per plan (flowassign.cpp:296-369).  State
// in local memory (R*J <= kMaxExactCells); node counting and first-found-best
// semantics identical to the recursive reference.
struct ExactState {
    int R, J;
    int shp[kMaxExactCells];
    int32_t x[kMaxExactCells];
    int32_t bx[kMaxExactCells];
    int64_t lam[kMaxJ];
    int64_t mrem[kMaxExactCells];
};

__device__ int64_t suffix_bound(const ShapeTables &t, const ExactState &st, int k, int pos, const int64_t *lam,
                                int64_t mr) {
    // greedy_suffix (flowassign.cpp:298-311).  The reference takes lam by
    // value; each class occurs once in a replica's order, so reading it in
    // place gives the same takes without the copy.
    const int s = st.shp[k];
    const int ol = t.olen[s];
    int64_t cnt = 0;
    for (int i = pos; i < ol; ++i) {
        const int j = t.order[s * kMaxJ + i];
        const int64_t u = t.unit[s * st.J + j];
        int64_t tk = t.cap[s * st.J + j];
        if (lam[j] < tk) tk = lam[j];
        if (tk * u > mr) tk = quot_small(mr, u, t.inv_unit[s * st.J + j]);
        if (tk > 0) {
            cnt += tk;
            mr -= tk * u;
        }
    }
    return cnt;
}

// The pruning test of ExactSolver::dfs (flowassign.cpp:351-354): count +
// min(lam_total, bound) <= best, bound = greedy_suffix of replica k from pos
// plus greedy_suffix of every later replica from 0.  lam_total is passed in
// (count + lam_total is the same at every node: each branch moves v from lam
// to count), and since the bound's terms are non-negative the sum stops as
// soon as it clears best - count.
__device__ __forceinline__ bool exact_pruned(const ShapeTables &t, const ExactState &st, int k, int pos,
                                             int64_t count, int64_t lam_total, int64_t best) {
    if (count + lam_total <= best) return true;
    const int64_t need = best - count;  // pruned iff bound <= need
    if (need < 0) return false;
    int64_t acc = 0;
    for (int kk = k; kk < st.R; ++kk) {
        const int s = st.shp[kk];
        const int ol = t.olen[s];
        int64_t mr = kk == k ? st.mrem[k] : t.M[s];
        for (int i = kk == k ? pos : 0; i < ol; ++i) {
            const int j = t.order[s * kMaxJ + i];
            const int64_t u = t.unit[s * st.J + j];
            int64_t tk = t.cap[s * st.J + j];
            if (st.lam[j] < tk) tk = st.lam[j];
            if (tk * u > mr) tk = quot_small(mr, u, t.inv_unit[s * st.J + j]);
            if (tk > 0) {
                acc += tk;
                if (acc > need) return false;
                mr -= tk * u;
            }
        }
    }
    return true;
}

// Resolve plan i of a source into an ExactState; false if it does not take
// the exact path.
__device__ __forceinline__ bool exact_setup(const ShapeTables &t, const SpaceTables &sp, const PlanSource &src,
                                            const SolveParams &prm, uint64_t i, ExactState &st, int64_t &part,
                                            uint64_t &local, uint64_t &gr, const int64_t *&lam_src) {
    const int J = prm.J;
    st.J = J;
    part = 0;
    local = 0;
    lam_src = prm.lambda;
    if (src.mode == 2) {
        const uint64_t li = src.first + i;
        st.R = src.list_R[li];
        if (st.R * J > kMaxExactCells) return false;
        const int32_t *ls = src.list_shapes + src.list_off[li];
        for (int k = 0; k < st.R; ++k) st.shp[k] = ls[k];
        if (src.list_lambda) lam_src = src.list_lambda + li * J;
        int64_t tot = 0;
        for (int j = 0; j < J; ++j) tot += lam_src[j];
        if (!(tot <= prm.exact_demand_limit && st.R * J <= prm.exact_cell_limit)) return false;
        gr = li;
    } else {
        gr = source_rank(src, src.first + i);
        part = find_partition(sp, gr);
        if (!sp.exact[part]) return false;
        local = gr - sp.prefix[part];
        st.R = sp.R[part];
        const int ro = sp.rep_off[part], runo = sp.run_off[part], nr = sp.nruns[part];
        uint8_t pick[kMaxExactCells];
        for (int ri = 0; ri < nr; ++ri) {
            const uint64_t w = sp.run_weight[runo + ri], c = sp.run_count[runo + ri];
            const uint64_t rr = (local / w) % c;
            unrank_run(rr, sp.run_len[runo + ri], sp.run_q[runo + ri], pick + sp.run_start[runo + ri]);
        }
        for (int k = 0; k < st.R; ++k) st.shp[k] = sp.cl_shape[sp.rep_list[ro + k] * kMaxCand + pick[k]];
    }
    for (int j = 0; j < J; ++j) st.lam[j] = lam_src[j];
    for (int k = 0; k < st.R; ++k) st.mrem[k] = t.M[st.shp[k]];
    for (int c = 0; c < st.R * J; ++c) {
        st.x[c] = 0;
        st.bx[c] = 0;
    }
    return true;
}

// Write the final outputs of an exact-path plan.
__device__ __forceinline__ void exact_emit(const ShapeTables &t, const KeyLayout &key, const PlanOutputs &out,
                                           uint64_t i, const ExactState &st, const int32_t *bx, int64_t bestc,
                                           int64_t part, uint64_t local) {
    const int R = st.R, J = st.J;
    int spp = 0;
    for (int kk = 0; kk < R; ++kk) spp += t.pp[st.shp[kk]];
    if (out.objective) out.objective[i] = bestc;
    if (out.sum_pp) out.sum_pp[i] = spp;
    if (out.x) {
        for (int kk = 0; kk < R; ++kk) {
            int64_t used = 0;
            for (int j = 0; j < J; ++j) {
                out.x[(i * out.rmax + kk) * J + j] = bx[kk * J + j];
                used += static_cast<int64_t>(bx[kk * J + j]) * t.unit[st.shp[kk] * J + j];
            }
            if (out.used) out.used[i * out.rmax + kk] = used;
        }
    }
    if (out.best_key) {
        const uint64_t kv = ((key.obj_max - static_cast<uint64_t>(bestc)) << key.sh_obj) |
                            (static_cast<uint64_t>(part) << key.sh_part) |
                            (static_cast<uint64_t>(spp) << key.sh_spp) | local;
        atomicMin(reinterpret_cast<unsigned long long *>(out.best_key), kv);
    }
}

// The plan's decisions flattened: position p is the p-th (replica, order
// slot) pair in DFS order, so a DFS frame is just its position and the
// stack is x[p].  meta[p] = class | replica << 8 | first-of-replica << 16 |
// adv << 24, adv = the nodes entered from the decision before p to p itself:
// the reference's pass-through dfs(k + 1, 0) calls at replica ends (one per
// replica end crossed, empty replicas included) plus p's own node; meta[D]
// holds the leaf's adv.  T is int32_t when every value fits (each cap * unit
// <= M < 2^30 and count + lam_total < 2^20), else int64_t.
template <typename T>
struct ExactFlat {
    using Inv = typename std::conditional<sizeof(T) == 4, float, double>::type;
    int D;
    // per position, slot D included so a pair of positions can be read
    // ahead of the q + 1 < D test
    uint32_t meta[kMaxExactCells + 1];
    T u[kMaxExactCells + 1], cap[kMaxExactCells + 1], mres[kMaxExactCells + 1];  // mres: M if first of replica, else -1
    Inv inv[kMaxExactCells + 1];
    T x[kMaxExactCells], mr_at[kMaxExactCells];
    T lam[kMaxJ];
    T M[kMaxExactCells];  // per replica
};

// floor(m / u) for the take of a position (m < take * u, so the quotient is
// below the take): FP32 reciprocal and a remainder correction on the 32-bit
// table (quotients < 2^20 there: at most 2 off), quot_small on the 64-bit one.
__device__ __forceinline__ int32_t flat_quot(int32_t m, int32_t u, float inv) {
    int32_t q = __float2int_rz(__int2float_rn(m) * inv);
    int64_t r = static_cast<int64_t>(m) - static_cast<int64_t>(q) * u;  // 64-bit: q * u may pass 2^31
    while (r < 0) {
        --q;
        r += u;
    }
    while (r >= u) {
        ++q;
        r -= u;
    }
    return q;
}
__device__ __forceinline__ int64_t flat_quot(int64_t m, int64_t u, double inv) { return quot_small(m, u, inv); }

// The plan's flat decision table and the restored path; false if T cannot
// hold the plan's values.
template <typename T>
__device__ __forceinline__ bool exact_flatten(const ShapeTables &t, const ExactState &st, int64_t conserved,
                                              ExactFlat<T> &f) {
    const int R = st.R, J = st.J;
    if (sizeof(T) == 4 && conserved >= (int64_t{1} << 20)) return false;
    int p = 0, kprev = 0;
    for (int k = 0; k < R; ++k) {
        const int s = st.shp[k];
        const int64_t Mk = t.M[s];
        if (sizeof(T) == 4 && Mk >= (int64_t{1} << 30)) return false;
        f.M[k] = static_cast<T>(Mk);
        for (int i = 0; i < t.olen[s]; ++i, ++p) {
            const int j = t.order[s * kMaxJ + i];
            const int64_t u = t.unit[s * J + j], cp = t.cap[s * J + j];
            if (sizeof(T) == 4 && cp * u > Mk) return false;
            const uint32_t adv = 1u + static_cast<uint32_t>(k - kprev);
            f.meta[p] = static_cast<uint32_t>(j) | (static_cast<uint32_t>(k) << 8) | ((i == 0 ? 1u : 0u) << 16) |
                        (adv << 24);
            kprev = k;
            f.u[p] = static_cast<T>(u);
            f.cap[p] = static_cast<T>(cp);
            f.mres[p] = i == 0 ? static_cast<T>(Mk) : T(-1);
            f.inv[p] = static_cast<typename ExactFlat<T>::Inv>(t.inv_unit[s * J + j]);
            f.x[p] = static_cast<T>(st.x[k * J + j]);
        }
    }
    f.D = p;
    f.meta[p] = (1u + static_cast<uint32_t>(R - kprev)) << 24;
    f.u[p] = 1;
    f.cap[p] = 0;
    f.mres[p] = -1;
    f.inv[p] = 1;
    for (int j = 0; j < J; ++j) f.lam[j] = static_cast<T>(st.lam[j]);
    return true;
}

// The pruning test on the flat table (exact_pruned's rule): prune iff
// count + min(lam_total, bound) <= best, the bound summed from position p
// with the current replica's budget mr.  Two positions per step, their
// table entries loaded together.
template <typename T>
__device__ __forceinline__ bool flat_pruned(const ExactFlat<T> &f, int p, T mr, T count, T conserved, T best) {
    if (conserved <= best) return true;
    const T need = best - count;
    if (need < 0) return false;
    T acc = 0, m = mr;
    for (int q = p; q < f.D; q += 2) {
        const uint32_t ma = f.meta[q], mb = f.meta[q + 1];
        const T ua = f.u[q], ub = f.u[q + 1], ca = f.cap[q], cb = f.cap[q + 1];
        const T ra = f.mres[q], rb = f.mres[q + 1];
        const T la = f.lam[ma & 0xff], lb = f.lam[mb & 0xff];
        if (q > p && ra >= 0) m = ra;
        T tk = la < ca ? la : ca;
        if (tk * ua > m) tk = flat_quot(m, ua, f.inv[q]);
        if (tk > 0) {
            acc += tk;
            if (acc > need) return false;
            m -= tk * ua;
        }
        if (q + 1 >= f.D) break;
        if (rb >= 0) m = rb;
        tk = lb < cb ? lb : cb;
        if (tk * ub > m) tk = flat_quot(m, ub, f.inv[q + 1]);
        if (tk > 0) {
            acc += tk;
            if (acc > need) return false;
            m -= tk * ub;
        }
    }
    return true;
}

// The DFS from position p (entered with e nodes: the task root and its
// pass-through chain).
template <bool TRACK, typename T>
__device__ void exact_dfs_flat(ExactFlat<T> &f, const ExactState &st, int p, int64_t e, int64_t count64,
                               int64_t &best64, int64_t cap, int64_t &nodes, bool &capped, int32_t *bx,
                               unsigned long long *ctr, int64_t ctr_limit, int64_t conserved64) {
    const int R = st.R, J = st.J, D = f.D;
    const int p0 = p;
    T count = static_cast<T>(count64), best = static_cast<T>(best64);
    const T conserved = static_cast<T>(conserved64);
    T mr = p < D ? static_cast<T>(st.mrem[(f.meta[p] >> 8) & 0xff]) : T(0);
    capped = false;
    int64_t flushed = 0, next_flush = 256;
    bool calling = true;
    nodes += e;
    for (;;) {
        if (calling) {
            if (nodes > cap) {
                capped = true;
                break;
            }
            if (ctr && nodes >= next_flush) {  // shared node total (phase B): stop once it passes the limit
                const unsigned long long tot =
                    atomicAdd(ctr, static_cast<unsigned long long>(nodes - flushed)) + (nodes - flushed);
                flushed = nodes;
                next_flush = nodes + 256;
                if (tot > static_cast<unsigned long long>(ctr_limit)) {
                    capped = true;
                    break;
                }
            }
            if (p == D) {  // leaf
                if (count > best) {
                    best = count;
                    if (TRACK) {
                        for (int c = 0; c < R * J; ++c) bx[c] = 0;
                        for (int q = 0; q < D; ++q) {
                            const uint32_t mt = f.meta[q];
                            bx[((mt >> 8) & 0xff) * J + (mt & 0xff)] = static_cast<int32_t>(f.x[q]);
                        }
                    }
                }
                calling = false;
                continue;
            }
            if (flat_pruned(f, p, mr, count, conserved, best)) {
                calling = false;
                continue;
            }
            const uint32_t mt = f.meta[p];
            const int j = mt & 0xff;
            const T u = f.u[p];
            T hi = f.cap[p];
            if (f.lam[j] < hi) hi = f.lam[j];
            if (hi * u > mr) hi = flat_quot(mr, u, f.inv[p]);
            f.mr_at[p] = mr;
            f.x[p] = hi;
            f.lam[j] -= hi;
            mr -= hi * u;
            count += hi;
            ++p;
            const uint32_t mn = f.meta[p];
            if (f.mres[p] >= 0) mr = f.mres[p];
            nodes += mn >> 24;
            continue;
        }
        // return into the frame of position p - 1
        if (p == p0) break;
        const int q = p - 1;
        T v = f.x[q];
        if (v == 0) {
            p = q;
            continue;
        }
        --v;
        f.x[q] = v;
        const uint32_t mt = f.meta[q];
        f.lam[mt & 0xff] += 1;
        count -= 1;
        mr = f.mr_at[q] - v * f.u[q];
        p = q + 1;
        const uint32_t mn = f.meta[p];
        if (f.mres[p] >= 0) mr = f.mres[p];
        nodes += mn >> 24;
        calling = true;
    }
    if (ctr && nodes != flushed) atomicAdd(ctr, static_cast<unsigned long long>(nodes - flushed));
    best64 = best;
}

// Subtree DFS of the reference's ExactSolver::dfs (flowassign.cpp:330-369)
// from the node (k, pos) with `count` assigned above it and incumbent `best`:
// the same node counting, bound, descending branch order and strictly-better
// leaf rule.  Stops (capped) once past `cap` nodes.  TRACK copies improving
// leaves into bx.  Runs on the flat decision table in 32-bit arithmetic when
// the plan's values allow it.
template <bool TRACK>
__device__ void exact_dfs(const ShapeTables &t, ExactState &st, int k, int pos, int64_t count, int64_t &best,
                          int64_t cap, int64_t &nodes, bool &capped, int32_t *bx, unsigned long long *ctr = nullptr,
                          int64_t ctr_limit = 0) {
    int64_t conserved = count;  // count + lam_total, the same at every node
    for (int j = 0; j < st.J; ++j) conserved += st.lam[j];
    // the task root (k, pos) and its pass-through chain: e nodes up to the
    // first decision (position p) or the leaf (p = D)
    int64_t e = 1;
    while (k < st.R && pos == t.olen[st.shp[k]]) {
        ++k;
        pos = 0;
        ++e;
    }
    int p = pos;
    for (int kk = 0; kk < k && kk < st.R; ++kk) p += t.olen[st.shp[kk]];
    {
        ExactFlat<int32_t> f;
        if (exact_flatten(t, st, conserved, f)) {
            exact_dfs_flat<TRACK>(f, st, p, e, count, best, cap, nodes, capped, bx, ctr, ctr_limit, conserved);
            return;
        }
    }
    ExactFlat<int64_t> f;
    exact_flatten(t, st, conserved, f);
    exact_dfs_flat<TRACK>(f, st, p, e, count, best, cap, nodes, capped, bx, ctr, ctr_limit, conserved);
}

// Warp-cooperative exact_dfs: all 32 lanes carry the identical DFS state and
// control flow; the bound's per-replica greedy_suffix terms (the dominant
// per-node cost, R*J dependent loads on one thread) are evaluated one replica
// per lane and summed by a warp reduction.  `ctr` (optional) is a node total
// shared with other warps: every 256 nodes the warp adds its progress and
// stops (capped) once the total passes `ctr_limit`.
template <bool TRACK>
__device__ void exact_dfs_warp(const ShapeTables &t, ExactState &st, int k, int pos, int64_t count, int64_t &best,
                               int64_t cap, int64_t &nodes, bool &capped, int32_t *bx, unsigned long long *ctr,
                               int64_t ctr_limit) {
    const int lane = threadIdx.x & 31;
    const int R = st.R, J = st.J;
    int fk[kMaxExactCells + 1], fpos[kMaxExactCells + 1], fj[kMaxExactCells + 1];
    int64_t fv[kMaxExactCells + 1];
    int depth = 0;
    bool calling = true;
    int64_t flushed = 0;
    capped = false;
    auto flush = [&]() -> bool {  // true: the shared total passed the limit
        unsigned long long tot = 0;
        if (lane == 0) tot = atomicAdd(ctr, static_cast<unsigned long long>(nodes - flushed)) + (nodes - flushed);
        flushed = nodes;
        tot = __shfl_sync(0xffffffffu, tot, 0);
        return tot > static_cast<unsigned long long>(ctr_limit);
    };
    while (true) {
        if (calling) {
            if (++nodes > cap) {
                capped = true;
                break;
            }
            if (ctr && (nodes & 255) == 0 && flush()) {
                capped = true;
                break;
            }
            if (k == R) {
                if (count > best) {
                    best = count;
                    if (TRACK)  // every lane: bx may be lane-local (identical copies)
                        for (int c = 0; c < R * J; ++c) bx[c] = st.x[c];
                }
                calling = false;
                continue;
            }
            const int s = st.shp[k];
            if (pos == t.olen[s]) {
                ++k;
                pos = 0;
                continue;  // tail call dfs(k+1, 0)
            }
            int64_t lam_total = 0;
            for (int j = 0; j < J; ++j) lam_total += st.lam[j];
            int64_t bound = 0;
            for (int kk = lane; kk < R; kk += 32) {
                if (kk == k) bound += suffix_bound(t, st, k, pos, st.lam, st.mrem[k]);
                else if (kk > k) bound += suffix_bound(t, st, kk, 0, st.lam, t.M[st.shp[kk]]);
            }
            for (int d = 16; d > 0; d >>= 1) bound += __shfl_xor_sync(0xffffffffu, bound, d);
            if (count + (lam_total < bound ? lam_total : bound) <= best) {
                calling = false;
                continue;
            }
            const int j = t.order[s * kMaxJ + pos];
            const int64_t u = t.unit[s * J + j];
            int64_t hi = t.cap[s * J + j];
            if (st.lam[j] < hi) hi = st.lam[j];
            if (hi * u > st.mrem[k]) hi = quot_small(st.mrem[k], u, t.inv_unit[s * J + j]);
            fk[depth] = k;
            fpos[depth] = pos;
            fj[depth] = j;
            fv[depth] = hi;
            ++depth;
            st.x[k * J + j] = static_cast<int32_t>(hi);
            st.lam[j] -= hi;
            st.mrem[k] -= hi * u;
            count += hi;
            pos = pos + 1;
            continue;
        }
        if (depth == 0) break;
        const int d = depth - 1;
        const int kk = fk[d], j = fj[d];
        const int64_t u = t.unit[st.shp[kk] * J + j];
        int64_t v = fv[d];
        count -= v;
        st.mrem[kk] += v * u;
        st.lam[j] += v;
        st.x[kk * J + j] = 0;
        if (v == 0) {
            --depth;
            continue;
        }
        v -= 1;
        fv[d] = v;
        st.x[kk * J + j] = static_cast<int32_t>(v);
        st.lam[j] -= v;
        st.mrem[kk] -= v * u;
        count += v;
        k = kk;
        pos = fpos[d] + 1;
        calling = true;
    }
    if (ctr && nodes != flushed) flush();
}

// Warp per plan: the reference's DFS verbatim (sequential fallback).
__global__ void __launch_bounds__(128) k_plan_exact(ShapeTables t, SpaceTables sp, KeyLayout key, PlanSource src,
                                                    PlanOutputs out, SolveParams prm) {
    const int lane = threadIdx.x & 31;
    const uint64_t w0 = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t i = w0; i < src.count; i += nw) {
        ExactState st;
        int64_t part;
        uint64_t local, gr;
        const int64_t *lam_src;
        if (!exact_setup(t, sp, src, prm, i, st, part, local, gr, lam_src)) continue;
        int64_t best = -1, nodes = 0;
        bool aborted;
        exact_dfs_warp<true>(t, st, 0, 0, 0, best, prm.node_budget, nodes, aborted, st.bx, nullptr, 0);
        __syncwarp();
        if (lane != 0) continue;
        if (aborted) {
            if (out.aborted) {
                const unsigned slot2 = atomicAdd(out.aborted_n, 1u);
                out.aborted[slot2] = gr;
            }
            continue;
        }
        exact_emit(t, key, out, i, st, st.bx, best, part, local);
    }
}

// One thread per plan, alone in its warp (one warp per CTA, so plans spread
// over the SMs): the same sequential DFS on the flat decision table.  The
// per-node latency of one thread is far below a warp-cooperative node's, and
// plans sharing a warp would serialise on their diverging searches.
__global__ void __launch_bounds__(32) k_plan_exact_thr(ShapeTables t, SpaceTables sp, KeyLayout key, PlanSource src,
                                                       PlanOutputs out, SolveParams prm) {
    if (threadIdx.x != 0) return;
    for (uint64_t i = blockIdx.x; i < src.count; i += gridDim.x) {
        ExactState st;
        int64_t part;
        uint64_t local, gr;
        const int64_t *lam_src;
        if (!exact_setup(t, sp, src, prm, i, st, part, local, gr, lam_src)) continue;
        int64_t best = -1, nodes = 0;
        bool aborted;
        exact_dfs<true>(t, st, 0, 0, 0, best, prm.node_budget, nodes, aborted, st.bx);
        if (aborted) {
            if (out.aborted) {
                const unsigned slot2 = atomicAdd(out.aborted_n, 1u);
                out.aborted[slot2] = gr;
            }
            continue;
        }
        exact_emit(t, key, out, i, st, st.bx, best, part, local);
    }
}

// ---- frontier-parallel exact path -------------------------------------------
// The sequential DFS's result is decided by two facts (flowassign.cpp:330-369):
//  * the incumbent when a node is checked equals the best leaf among ALL
//    leaves before it in preorder (a pruned leaf is <= the incumbent that
//    pruned it), so a node is visited iff every ancestor passes its bound
//    check against that prefix maximum;
//  * the answer is the first optimal leaf in preorder (pruning is <=, the
//    leaf update strictly >), and the run aborts iff the visited-node count
//    exceeds the budget.
// So the tree is cut after `depth` branching decisions; each frontier node is
// a task.  Phase A (task pass 0) gets each task's best leaf m (seeded with a
// lower bound lb of its entering incumbent: the prefix max of cheap greedy
// dives of earlier tasks, so m = max(best leaf, lb) — exactly what the
// prefix maximum needs).  Pass 2 walks the top of the tree once, in preorder,
// with the exact prefix-maximum incumbent: visited flags, the entering
// incumbent of each task and the top-node count.  Phase B (task pass 1)
// replays every visited task from its exact incumbent — now identical to the
// sequential DFS inside it — and counts its nodes.  The first optimal leaf is
// in the task where the prefix maximum last rose.

// Task root state from its decision path; `leaf` follows the pass-through
// chain to the leaf (a task created by reaching k == R above the cut).
__device__ __forceinline__ void exact_restore(const ShapeTables &t, ExactState &st, const int32_t *path, int nd,
                                              bool leaf, int &k, int &pos, int64_t &count) {
    const int R = st.R, J = st.J;
    k = 0;
    pos = 0;
    count = 0;
    int a = 0;
    while (k < R) {
        const int s = st.shp[k];
        if (a == nd && !leaf) break;
        if (pos == t.olen[s]) {
            ++k;
            pos = 0;
            continue;
        }
        if (a == nd) break;
        const int j = t.order[s * kMaxJ + pos];
        const int64_t u = t.unit[s * J + j];
        const int64_t v = path[a++];
        st.x[k * J + j] = static_cast<int32_t>(v);
        st.lam[j] -= v;
        st.mrem[k] -= v * u;
        count += v;
        ++pos;
    }
}

// Count of the greedy dive (every branch at its largest value) from (k, pos):
// a leaf of the subtree, so a lower bound of its best leaf.
__device__ __forceinline__ int64_t exact_dive(const ShapeTables &t, const ExactState &st, int k, int pos,
                                              int64_t count) {
    const int R = st.R, J = st.J;
    int64_t lam[kMaxJ];
    for (int j = 0; j < J; ++j) lam[j] = st.lam[j];
    for (; k < R; ++k, pos = 0) {
        const int s = st.shp[k];
        int64_t mr = st.mrem[k];  // replicas after k are untouched (mrem = M)
        for (int i = pos; i < t.olen[s]; ++i) {
            const int j = t.order[s * kMaxJ + i];
            const int64_t u = t.unit[s * J + j];
            int64_t hi = t.cap[s * J + j];
            if (lam[j] < hi) hi = lam[j];
            if (hi * u > mr) hi = quot_small(mr, u, t.inv_unit[s * J + j]);
            lam[j] -= hi;
            mr -= hi * u;
            count += hi;
        }
    }
    return count;
}

// Parallel replay of the top of the tree (round 1 walked it on one thread
// per plan, in preorder).  With the exact prefix-maximum incumbents inc[q] of
// the tasks (plan pass 6: the exclusive prefix max of m, the optimum and the
// task holding the first optimal leaf), an internal top node is checked with
// the incumbent of the first task below it, so it is alive iff count +
// min(lam_total, bound) > inc[first task].  Task q enters (first) the nodes
// at depths c+1 .. d-1 of its path (c: decisions shared with task q-1); pass
// 6 writes their alive bits and c, a scan combines (keep the previous task's
// bits 0..c, add the new ones) into each task's ancestor-alive mask, and pass
// 7 marks the visited tasks (every ancestor alive), adds each visited new
// node's calls (the node and its pass-through dfs(k+1, 0) calls) to the
// plan's top-node count and the visited tasks' phase-A counts to its upper
// bound.
__device__ __forceinline__ int exact_shared_prefix(const ExactTasks &et, uint64_t q, uint64_t i, int d) {
    if (q <= et.toff[i]) return -1;
    const int32_t *path = et.path + q * kTaskDepthMax;
    const int32_t *pp = et.path + (q - 1) * kTaskDepthMax;
    const int dp = et.tdepth[q - 1] & 0x7f;
    int c = 0;
    while (c < d && c < dp && pp[c] == path[c]) ++c;
    return c;
}

__device__ void exact_replay_task(int pass, const ShapeTables &t, ExactState &st, const ExactTasks &et, uint64_t q,
                                  uint64_t i) {
    const int R = st.R, J = st.J;
    const int32_t *path = et.path + q * kTaskDepthMax;
    const int d = et.tdepth[q] & 0x7f;
    const int c = exact_shared_prefix(et, q, i, d);
    const int64_t inc = et.inc[q];
    const uint32_t anc = pass == 7 ? et.amask[q] : 0u;
    uint32_t own = 0;
    int64_t top = 0;
    int k = 0, pos = 0;
    int64_t count = 0;
    for (int e = 0; e < d; ++e) {
        int64_t calls = 1;
        while (k < R && pos == t.olen[st.shp[k]]) {
            ++k;
            pos = 0;
            ++calls;
        }
        if (k >= R) break;
        if (e > c) {
            if (pass == 6) {
                int64_t lt = 0;
                for (int j = 0; j < J; ++j) lt += st.lam[j];
                if (!exact_pruned(t, st, k, pos, count, lt, inc)) own |= 1u << e;
            } else {
                const uint32_t need = e ? ((2u << (e - 1)) - 1u) : 0u;  // ancestors 0..e-1
                if ((anc & need) == need) top += calls;
            }
        }
        const int s = st.shp[k];
        const int j = t.order[s * kMaxJ + pos];
        const int64_t u = t.unit[s * J + j];
        const int64_t v = path[e];
        st.x[k * J + j] = static_cast<int32_t>(v);
        st.lam[j] -= v;
        st.mrem[k] -= v * u;
        count += v;
        ++pos;
    }
    if (pass == 6) {
        et.aL[q] = c;
        et.amask[q] = own;
        return;
    }
    const uint32_t need = d ? ((2u << (d - 1)) - 1u) : 0u;
    const bool vis = (anc & need) == need;
    et.vis[q] = vis ? 1 : 0;
    if (top) atomicAdd(et.topn + i, static_cast<unsigned long long>(top));
    if (vis) {
        atomicAdd(et.ubn + i, static_cast<unsigned long long>(et.nodes[q]));
        // entered with the exact incumbent: phase A ran the sequential search itself
        if (et.lbran[q] == inc) atomicAdd(et.lbn + i, static_cast<unsigned long long>(et.nodes[q]));
    }
    if (et.capped[q]) et.anycap[i] = 1;
}

// Per-plan passes: 10 one root task per exact-path plan, 8 certify after the
// replay (or count exactly in phase B), 3 finish (abort decision or outputs).
// The per-plan prefix maxima over the tasks are segmented scans
// (launch_exact_prefix).
__global__ void __launch_bounds__(128) k_exact_plan(int pass, ShapeTables t, SpaceTables sp, KeyLayout key,
                                                    PlanSource src, PlanOutputs out, SolveParams prm, ExactTasks et) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < src.count;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        ExactState st;
        int64_t part;
        uint64_t local, gr;
        const int64_t *lam_src;
        const bool ex = exact_setup(t, sp, src, prm, i, st, part, local, gr, lam_src);
        if (pass == 10) {  // device-built frontier: one root task per exact-path plan
            et.depth[i] = ex ? 0 : -1;
            et.ntask[i] = ex ? 1 : 0;
            et.state[i] = ex ? 1 : 0;
            continue;
        }
        if (!ex || et.state[i] == 0) continue;
        if (pass == 8) {  // after the replay: certify (upper bound) or count exactly in phase B
            if (et.state[i] != 1) continue;
            if (et.anycap[i]) {  // phase A hit the budget somewhere: sequential DFS
                et.state[i] = 2;
                continue;
            }
            const unsigned long long tn = et.topn[i];
            et.top_nodes[i] = static_cast<int64_t>(tn);
            et.running[i] = tn;
            if (tn + et.lbn[i] > static_cast<unsigned long long>(prm.node_budget)) {
                // exact counts of a subset of the visited nodes already pass the
                // budget: the sequential search aborts, no phase-B recount
                et.running[i] = tn + et.lbn[i];
                et.state[i] = 4;
            } else if (tn + et.ubn[i] > static_cast<unsigned long long>(prm.node_budget)) {
                et.state[i] = 3;
            }
            continue;
        }
        // pass 3: finish
        const uint8_t ps = et.state[i];
        if (ps != 1 && ps != 3 && ps != 4) continue;
        if (ps == 4 || (ps == 3 && et.running[i] > static_cast<unsigned long long>(prm.node_budget))) {
            if (out.aborted) {
                const unsigned slot2 = atomicAdd(out.aborted_n, 1u);
                out.aborted[slot2] = gr;
            }
            continue;
        }
        exact_emit(t, key, out, i, st, et.bx + i * kMaxExactCells, et.opt[i], part, local);
    }
}

// Where a task splits: from its root (k, pos), decisions with a single
// branch (hi = 0: v = 0 forced, no state change) are walked down to the first
// decision with hi >= 1; its hi + 1 branches become the children (paths: the
// task's path, nz zeros, then v).  1 (no split) when a leaf comes first or the
// children would pass depth `room`.
__device__ __forceinline__ uint32_t exact_branches(const ShapeTables &t, const ExactState &st, int k, int pos,
                                                   int room, uint8_t &nz) {
    int z = 0;
    for (;;) {
        while (k < st.R && pos == t.olen[st.shp[k]]) {
            ++k;
            pos = 0;
        }
        if (k >= st.R || z >= room) break;
        const int s = st.shp[k];
        const int j = t.order[s * kMaxJ + pos];
        const int64_t u = t.unit[s * st.J + j];
        int64_t hi = t.cap[s * st.J + j];
        if (st.lam[j] < hi) hi = st.lam[j];
        if (hi * u > st.mrem[k]) hi = quot_small(st.mrem[k], u, t.inv_unit[s * st.J + j]);
        if (hi >= 1) {
            nz = static_cast<uint8_t>(z);
            return static_cast<uint32_t>(hi + 1);
        }
        ++z;
        ++pos;
    }
    nz = 0;
    return 1u;
}

// Per-task passes, a thread per task (tasks fetched one at a time from a
// counter, so a long task does not hold up a warp's others; the exact path's
// instances are small — R*J <= exact_cell_limit, 20 by default — where a
// warp-cooperative bound leaves most lanes idle): 0 phase A (best leaf seeded
// with lb, node count, capped at phase_cap), 1 phase B (exact replay from the
// entering incumbent: the first optimal leaf of the istar task; node counts
// into the plan's running total for uncertified plans), 2 greedy dive,
// 3 children of capped tasks, 6 / 7 top replay, 9 frontier children.
__global__ void __launch_bounds__(128) k_exact_task_thr(int pass, ShapeTables t, SpaceTables sp, PlanSource src,
                                                        SolveParams prm, ExactTasks et, uint64_t total,
                                                        unsigned long long *fetch) {
    for (;;) {
        const uint64_t q = atomicAdd(fetch, 1ull);
        if (q >= total) break;
        const uint64_t i = et.plan[q];
        const uint8_t ps = et.state[i];
        if (pass == 3) {  // children count for the next round: capped tasks only
            const uint8_t td3 = et.tdepth[q];
            if (ps != 1 || !et.capped[q] || et.phase_cap >= prm.node_budget || (td3 & 0x7f) >= kTaskDepthMax - 1) {
                et.nchild[q] = 1;
                et.nzero[q] = 0;
                continue;
            }
        }
        if ((pass == 0 || pass == 2) && (ps != 1 || et.done[q])) continue;
        if (pass == 1) {
            if (ps == 1 && static_cast<int64_t>(q) != et.istar[i]) continue;
            if (ps != 1 && (ps != 3 || !et.vis[q])) continue;
        }
        if (pass == 9 && ps != 1) {
            et.nchild[q] = 1;
            et.nzero[q] = 0;
            continue;
        }
        if ((pass == 6 || pass == 7) && ps != 1) {
            if (pass == 6) {  // not a frontier plan's task: neutral scan element
                et.aL[q] = -1;
                et.amask[q] = 0;
            }
            continue;
        }
        ExactState st;
        int64_t part;
        uint64_t local, gr;
        const int64_t *lam_src;
        exact_setup(t, sp, src, prm, i, st, part, local, gr, lam_src);
        const uint8_t td = et.tdepth[q];
        if (pass == 6 || pass == 7) {
            exact_replay_task(pass, t, st, et, q, i);
            continue;
        }
        if (pass == 9) {  // frontier expansion: the root's first decision's branches, growing plans only
            uint32_t nc = 1;
            uint8_t nz = 0;
            const int dq = td & 0x7f;
            if (et.grow[i] && dq < kTaskDepthMax - 1) {
                int k, pos;
                int64_t count;
                exact_restore(t, st, et.path + q * kTaskDepthMax, dq, false, k, pos, count);
                nc = exact_branches(t, st, k, pos, kTaskDepthMax - 2 - dq, nz);
            }
            et.nchild[q] = nc;
            et.nzero[q] = nz;
            atomicAdd(et.plan_sum + i, nc);
            continue;
        }
        int k, pos;
        int64_t count;
        exact_restore(t, st, et.path + q * kTaskDepthMax, td & 0x7f, (td & 0x80) != 0, k, pos, count);
        int64_t nodes = 0;
        bool capped;
        if (pass == 2) {  // greedy dive of the task: a leaf, so a lower bound of its best
            et.g[q] = exact_dive(t, st, k, pos, count);
            continue;
        }
        if (pass == 3) {
            uint8_t nz = 0;
            et.nchild[q] = exact_branches(t, st, k, pos, kTaskDepthMax - 2 - (td & 0x7f), nz);
            et.nzero[q] = nz;
            continue;
        }
        if (pass == 0) {
            int64_t best = et.lb[q];
            et.lbran[q] = best;
            // the plan's phase-A nodes over all rounds are bounded: past
            // work_limit its tasks stop and k_exact_retire hands the plan to
            // the sequential fallback (trees far past the node budget)
            exact_dfs<false>(t, st, k, pos, count, best, et.phase_cap, nodes, capped, nullptr, et.work + i,
                             et.work_limit);
            et.m[q] = best;
            et.nodes[q] = nodes;
            et.capped[q] = capped ? 1 : 0;
            et.done[q] = capped ? 0 : 1;
        } else {
            int64_t best = et.inc[q];
            unsigned long long *ctr = ps == 3 ? et.running + i : nullptr;
            if (static_cast<int64_t>(q) == et.istar[i])
                exact_dfs<true>(t, st, k, pos, count, best, prm.node_budget + 1, nodes, capped,
                                et.bx + i * kMaxExactCells, ctr, prm.node_budget);
            else
                exact_dfs<false>(t, st, k, pos, count, best, prm.node_budget + 1, nodes, capped, nullptr, ctr,
                                 prm.node_budget);
        }
    }
}

// Per-plan prefix maxima of the exact path as segmented scans over the task
// list (tasks of a plan are contiguous; the key is the plan index):
//  lower bounds: lb[q] = exclusive max over the plan's earlier tasks of
//    max(dive g, best leaf m of a task that ran); finished tasks m = max(m, lb)
//  exact incumbents: inc[q] = exclusive max of m; opt = the plan's max; istar
//    = the first task reaching it (the only one with m > inc and m == opt).
struct MaxI64 {
    __device__ __forceinline__ int64_t operator()(int64_t a, int64_t b) const { return a > b ? a : b; }
};

__global__ void k_exact_lb_vals(ExactTasks et, uint64_t total, int64_t *v) {
    for (uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < total;
         q += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const int64_t g = et.g[q];
        const int64_t m = (et.done[q] || et.capped[q]) ? et.m[q] : -1;
        v[q] = g > m ? g : m;
    }
}

__global__ void k_exact_lb_apply(ExactTasks et, uint64_t total) {
    for (uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < total;
         q += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        if (et.done[q] && et.m[q] < et.lb[q]) et.m[q] = et.lb[q];
}

// Plans whose phase-A nodes passed work_limit leave the frontier (state 2:
// the sequential DFS, at most node_budget nodes, decides them).
__global__ void k_exact_retire(ExactTasks et, uint64_t plans) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < plans;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        if (et.state[i] == 1 && et.work[i] > static_cast<unsigned long long>(et.work_limit)) et.state[i] = 2;
}

__global__ void k_exact_inc_reset(ExactTasks et, uint64_t plans) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < plans;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (et.state[i] != 1) continue;
        et.opt[i] = -1;
        et.istar[i] = -1;
        et.topn[i] = 0;
        et.ubn[i] = 0;
        et.lbn[i] = 0;
        et.anycap[i] = 0;
    }
}

__global__ void k_exact_opt(ExactTasks et, uint64_t total) {
    for (uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < total;
         q += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t i = et.plan[q];
        if (et.state[i] != 1) continue;
        if (q + 1 == total || et.plan[q + 1] != i) {
            const int64_t a = et.inc[q], b = et.m[q];
            et.opt[i] = a > b ? a : b;
        }
    }
}

__global__ void k_exact_istar(ExactTasks et, uint64_t total) {
    for (uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < total;
         q += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t i = et.plan[q];
        if (et.state[i] != 1) continue;
        const int64_t m = et.m[q];
        if (m > et.inc[q] && m == et.opt[i]) et.istar[i] = static_cast<int64_t>(q);
    }
}

// ------------------------------------------------------------------- K2 ---
constexpr int kSwMaxDev = 256;   // device slots per deployment pair
constexpr int kSwMaxCuts = 1024; // 2 * (src + dst ranges), padded to pow2

__device__ __forceinline__ double link_bw(const SwitchDeps &d, int s, int t) {
    return d.machine[s] >= 0 && d.machine[s] == d.machine[t] ? d.intra_bw : d.inter_bw;
}

// Cut points, per-target greedy holder choice and the link-time maximum for
// one (source, destination) pair whose layouts are in sB[0]/sE[0] (source)
// and sB[1]/sE[1] (destination).
__device__ __forceinline__ void switch_core(const SwitchDeps &d, const SwitchOut &o, int pair, uint64_t (*sB)[kSwMaxDev],
                                            uint64_t (*sE)[kSwMaxDev], uint64_t *cuts, int &ncuts_s, double *wmax,
                                            unsigned long long *wbytes, int *wstatus) {
    const int ND = d.num_devices;
    // ---- cut points (:70-85): sorted unique begin/end of non-empty ranges ----
    int P2 = 1;
    while (P2 < 4 * ND) P2 <<= 1;
    for (int i = threadIdx.x; i < P2; i += blockDim.x) {
        uint64_t v = ~0ull;
        if (i < 4 * ND) {
            const int w = (i / ND) >> 1, slot = i % ND, be = (i / ND) & 1;
            if (sE[w][slot] > sB[w][slot]) v = be ? sE[w][slot] : sB[w][slot];
        }
        cuts[i] = v;
    }
    __syncthreads();
    for (int kz = 2; kz <= P2; kz <<= 1) {
        for (int jz = kz >> 1; jz > 0; jz >>= 1) {
            for (int i = threadIdx.x; i < P2; i += blockDim.x) {
                const int ixj = i ^ jz;
                if (ixj > i) {
                    const bool up = (i & kz) == 0;
                    const uint64_t a = cuts[i], b = cuts[ixj];
                    if ((a > b) == up) {
                        cuts[i] = b;
                        cuts[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
    if (threadIdx.x == 0) {
        int m = 0;
        for (int i = 0; i < P2 && cuts[i] != ~0ull; ++i)
            if (m == 0 || cuts[i] != cuts[m - 1]) cuts[m++] = cuts[i];
        ncuts_s = m;
        if (o.detail_cuts) {
            for (int i = 0; i < m && i <= o.max_frags; ++i) o.detail_cuts[i] = cuts[i];
            *o.detail_ncuts = m;
        }
    }
    __syncthreads();
    const int ncuts = ncuts_s;
    // ---- greedy_plan (:86-128): warp per target, lane per source replica ----
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    const int sr0 = d.dep_rep_off[0], nsr = d.dep_rep_off[1] - sr0;
    double est = 0.0;
    unsigned long long maxb = 0;
    int status = 0;
    for (int ts = warp; ts < ND; ts += nwarps) {
        const uint64_t ta = sB[1][ts], tz = sE[1][ts];
        if (tz <= ta) continue;  // target holds nothing in the new layout
        const bool self_has = sE[0][ts] > sB[0][ts];
        const uint64_t ha = sB[0][ts], hz = sE[0][ts];
        // first fragment starting at ta
        int f = 0;
        {
            int lo = 0, hi = ncuts - 1;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (cuts[mid] < ta) lo = mid + 1;
                else hi = mid;
            }
            f = lo;
        }
        // per-lane source replicas: lane owns replicas r = lane + 32*q
        constexpr int QR = 4;  // up to 128 source replicas
        int cur[QR], slot[QR];
        uint64_t cend[QR], cbeg[QR], load[QR];
#pragma unroll
        for (int q = 0; q < QR; ++q) {
            cur[q] = -1;
            slot[q] = -1;
            cend[q] = 0;
            cbeg[q] = 0;
            load[q] = 0;
        }
        for (; f + 1 < ncuts && cuts[f + 1] <= tz; ++f) {
            const uint64_t fb = cuts[f], fe = cuts[f + 1];
            if (self_has && ha <= fb && fe <= hz) continue;  // already held
            unsigned long long bestkey = ~0ull;
#pragma unroll
            for (int q = 0; q < QR; ++q) {
                const int r = lane + 32 * q;
                if (r >= nsr) continue;
                const int rep = sr0 + r;
                const uint64_t tp = d.rep_tp[rep], pp = d.rep_pp[rep];
                const int dev0 = d.rep_dev_off[rep];
                const int nd = static_cast<int>(tp * pp);
                // advance to the slice covering fb (slices ascend within a replica)
                while (cur[q] + 1 < nd && (cend[q] <= fb || cend[q] == cbeg[q] || cur[q] < 0)) {
                    // finalize the previous holder's link load toward this target
                    if (load[q] > 0) {
                        const double v = static_cast<double>(load[q]) / link_bw(d, slot[q], ts);
                        est = v > est ? v : est;
                        maxb = load[q] > maxb ? load[q] : maxb;
                        load[q] = 0;
                    }
                    ++cur[q];
                    const uint64_t s = cur[q] / tp, i = cur[q] % tp;
                    const uint64_t sb = d.P * s / pp, se = d.P * (s + 1) / pp, len = se - sb;
                    cbeg[q] = sb + len * i / tp;
                    cend[q] = sb + len * (i + 1) / tp;
                    slot[q] = d.rep_devs[dev0 + cur[q]];
                }
                if (cbeg[q] <= fb && fe <= cend[q] && cend[q] > cbeg[q]) {
                    const bool intra = d.machine[slot[q]] >= 0 && d.machine[slot[q]] == d.machine[ts];
                    const unsigned long long kv = (static_cast<unsigned long long>(!intra) << 63) |
                                                  (static_cast<unsigned long long>(load[q]) << 16) |
                                                  static_cast<unsigned long long>(slot[q]);
                    bestkey = kv < bestkey ? kv : bestkey;
                }
            }
#pragma unroll
            for (int sft = 16; sft > 0; sft >>= 1) {
                const unsigned long long other = __shfl_xor_sync(0xffffffffu, bestkey, sft);
                bestkey = other < bestkey ? other : bestkey;
            }
            if (bestkey == ~0ull) {
                status = 1;  // UnsourcedFragment (:99-103)
                continue;
            }
            const int win = static_cast<int>(bestkey & 0xffff);
#pragma unroll
            for (int q = 0; q < QR; ++q)
                if (lane + 32 * q < nsr && slot[q] == win && cbeg[q] <= fb && fe <= cend[q]) load[q] += fe - fb;
            if (o.detail_src && lane == 0 && f < o.max_frags) o.detail_src[ts * o.max_frags + f] = win;
        }
#pragma unroll
        for (int q = 0; q < QR; ++q) {
            if (load[q] > 0) {
                const double v = static_cast<double>(load[q]) / link_bw(d, slot[q], ts);
                est = v > est ? v : est;
                maxb = load[q] > maxb ? load[q] : maxb;
            }
        }
    }
    // estimate_time (:133-140): max over links
#pragma unroll
    for (int sft = 16; sft > 0; sft >>= 1) {
        const double oe = __shfl_xor_sync(0xffffffffu, est, sft);
        est = oe > est ? oe : est;
        const unsigned long long ob = __shfl_xor_sync(0xffffffffu, maxb, sft);
        maxb = ob > maxb ? ob : maxb;
        status |= __shfl_xor_sync(0xffffffffu, status, sft);
    }
    if (lane == 0) {
        wmax[warp] = est;
        wbytes[warp] = maxb;
        wstatus[warp] = status;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double e = 0.0;
        unsigned long long b = 0;
        int st = 0;
        for (int w = 0; w < nwarps; ++w) {
            e = wmax[w] > e ? wmax[w] : e;
            b = wbytes[w] > b ? wbytes[w] : b;
            st |= wstatus[w];
        }
        o.est[pair] = ncuts < 2 ? 0.0 : e;
        o.max_bytes[pair] = b;
        o.status[pair] = st;
    }
}

__global__ void __launch_bounds__(256) k_switch_cost(SwitchDeps d, SwitchOut o) {
    __shared__ uint64_t sB[2][kSwMaxDev], sE[2][kSwMaxDev];
    __shared__ uint64_t cuts[kSwMaxCuts];
    __shared__ int ncuts_s;
    __shared__ double wmax[8];
    __shared__ unsigned long long wbytes[8];
    __shared__ int wstatus[8];
    const int pair = blockIdx.x;
    const int deps[2] = {0, pair + 1};
    // ---- layouts (switchplan.cpp:40-63): one slice per device slot ----
    for (int i = threadIdx.x; i < 2 * kSwMaxDev; i += blockDim.x) {
        sB[i / kSwMaxDev][i % kSwMaxDev] = 0;
        sE[i / kSwMaxDev][i % kSwMaxDev] = 0;
    }
    __syncthreads();
    for (int w = 0; w < 2; ++w) {
        const int r0 = d.dep_rep_off[deps[w]], r1 = d.dep_rep_off[deps[w] + 1];
        for (int r = r0; r < r1; ++r) {
            const uint64_t tp = d.rep_tp[r], pp = d.rep_pp[r];
            const int dev0 = d.rep_dev_off[r];
            const int nd = d.rep_dev_off[r + 1] - dev0;
            for (int q = threadIdx.x; q < nd; q += blockDim.x) {
                const uint64_t s = q / tp, i = q % tp;
                if (s >= pp) continue;
                const uint64_t sb = d.P * s / pp, se = d.P * (s + 1) / pp, len = se - sb;
                const int slot = d.rep_devs[dev0 + q];
                sB[w][slot] = sb + len * i / tp;
                sE[w][slot] = sb + len * (i + 1) / tp;
            }
        }
    }
    __syncthreads();
    switch_core(d, o, pair, sB, sE, cuts, ncuts_s, wmax, wbytes, wstatus);
}

// K2 over candidates given as packed round keys: the destination deployment
// is unranked on the device (canonical blocks: replica r owns device slots
// [off_r, off_r + d_r) of the cluster's sorted devices).
__global__ void __launch_bounds__(256) k_switch_cost_keys(SwitchDeps d, SpaceTables sp, KeyLayout key,
                                                          ShapeTables t, const uint64_t *keys, SwitchOut o) {
    __shared__ uint64_t sB[2][kSwMaxDev], sE[2][kSwMaxDev];
    __shared__ uint64_t cuts[kSwMaxCuts];
    __shared__ int ncuts_s;
    __shared__ double wmax[8];
    __shared__ unsigned long long wbytes[8];
    __shared__ int wstatus[8];
    __shared__ uint8_t pick[OSERVE_MAX_REPLICAS_DEV];
    __shared__ int rtp[OSERVE_MAX_REPLICAS_DEV], rpp[OSERVE_MAX_REPLICAS_DEV], roff[OSERVE_MAX_REPLICAS_DEV + 1];
    __shared__ int nrep;
    const int pair = blockIdx.x;
    const uint64_t kv = keys[pair];
    for (int i = threadIdx.x; i < 2 * kSwMaxDev; i += blockDim.x) {
        sB[i / kSwMaxDev][i % kSwMaxDev] = 0;
        sE[i / kSwMaxDev][i % kSwMaxDev] = 0;
    }
    if (threadIdx.x == 0) {
        const uint64_t local = kv & ((uint64_t{1} << key.sh_spp) - 1);
        const int64_t part = static_cast<int64_t>((kv >> key.sh_part) & ((uint64_t{1} << (key.sh_obj - key.sh_part)) - 1));
        const int R = sp.R[part];
        const int ro = sp.rep_off[part], runo = sp.run_off[part], nr = sp.nruns[part];
        for (int ri = 0; ri < nr; ++ri) {
            const uint64_t w = sp.run_weight[runo + ri], c = sp.run_count[runo + ri];
            const uint64_t rr = (local / w) % c;
            unrank_run(rr, sp.run_len[runo + ri], sp.run_q[runo + ri], pick + sp.run_start[runo + ri]);
        }
        int off = 0;
        for (int r = 0; r < R; ++r) {
            const int shape = sp.cl_shape[sp.rep_list[ro + r] * kMaxCand + pick[r]];
            rtp[r] = t.param[shape].tp;
            rpp[r] = t.param[shape].pp;
            roff[r] = off;
            off += rtp[r] * rpp[r];
        }
        roff[R] = off;
        nrep = R;
    }
    __syncthreads();
    // ---- layouts (switchplan.cpp:40-63) ----
    {
        const int r0 = d.dep_rep_off[0], r1 = d.dep_rep_off[1];
        for (int r = r0; r < r1; ++r) {
            const uint64_t tp = d.rep_tp[r], pp = d.rep_pp[r];
            const int dev0 = d.rep_dev_off[r];
            const int nd = d.rep_dev_off[r + 1] - dev0;
            for (int q = threadIdx.x; q < nd; q += blockDim.x) {
                const uint64_t s2 = q / tp, i = q % tp;
                if (s2 >= pp) continue;
                const uint64_t sb = d.P * s2 / pp, se = d.P * (s2 + 1) / pp, len = se - sb;
                const int slot = d.rep_devs[dev0 + q];
                sB[0][slot] = sb + len * i / tp;
                sE[0][slot] = sb + len * (i + 1) / tp;
            }
        }
        for (int r = 0; r < nrep; ++r) {
            const uint64_t tp = rtp[r], pp = rpp[r];
            const int nd = roff[r + 1] - roff[r];
            for (int q = threadIdx.x; q < nd; q += blockDim.x) {
                const uint64_t s2 = q / tp, i = q % tp;
                const uint64_t sb = d.P * s2 / pp, se = d.P * (s2 + 1) / pp, len = se - sb;
                const int slot = roff[r] + q;
                sB[1][slot] = sb + len * i / tp;
                sE[1][slot] = sb + len * (i + 1) / tp;
            }
        }
    }
    __syncthreads();
    switch_core(d, o, pair, sB, sE, cuts, ncuts_s, wmax, wbytes, wstatus);
}

// ------------------------------------------------------------------- K5 ---
// kv_plan (switchplan.cpp:142-207): requests in order (the link/inbound loads
// carry over), lanes evaluate the candidate devices of each choice and a
// shuffle reduction takes the lexicographic minimum.
struct KvPick {
    unsigned long long v;  // load (with the !intra flag ahead of it for sources)
    int cls;               // 0 intra / 1 not (sources); 0 for targets
    int slot;              // slot order == device id order
};

__device__ __forceinline__ bool kv_less(const KvPick &a, const KvPick &b) {
    if (a.cls != b.cls) return a.cls < b.cls;
    if (a.v != b.v) return a.v < b.v;
    return a.slot < b.slot;
}

__device__ __forceinline__ KvPick kv_warp_min(KvPick p) {
    for (int d = 16; d > 0; d >>= 1) {
        KvPick o;
        o.v = __shfl_xor_sync(0xffffffffu, p.v, d);
        o.cls = __shfl_xor_sync(0xffffffffu, p.cls, d);
        o.slot = __shfl_xor_sync(0xffffffffu, p.slot, d);
        if (kv_less(o, p)) p = o;
    }
    return p;
}

// One warp.  The slot tables (inbound loads, the link-load matrix, machines,
// replica device lists) are staged in shared memory when they fit (the
// common case: <= ~150 device slots), so each request's selections are
// shared-memory reductions; request fields are prefetched 32 at a time, one
// per lane, and broadcast by shuffles; results are written back coalesced
// by the owning lane.
__global__ void __launch_bounds__(32) k_kv_plan(KvPlanIn in, int use_smem) {
    extern __shared__ __align__(16) unsigned char kv_smem[];
    const int lane = threadIdx.x;
    constexpr int kNone = 0x7fffffff;
    const int NS = in.num_slots;
    const int nsd = in.n_src_devs, ndd = in.n_dst_devs;
    uint64_t *inbound = in.inbound, *load = in.load;
    const int32_t *machine = in.machine, *src_off = in.src_off, *src_devs = in.src_devs, *dst_off = in.dst_off,
                  *dst_devs = in.dst_devs;
    if (use_smem) {
        uint64_t *sl = reinterpret_cast<uint64_t *>(kv_smem);
        uint64_t *si = sl + static_cast<size_t>(NS) * NS;
        int32_t *sm = reinterpret_cast<int32_t *>(si + NS);
        int32_t *so = sm + NS, *sd = so + in.src_reps + 1, *to = sd + nsd, *td = to + in.dst_reps + 1;
        for (int i = lane; i < NS * NS; i += 32) sl[i] = in.load[i];
        for (int i = lane; i < NS; i += 32) {
            si[i] = 0;
            sm[i] = in.machine[i];
        }
        for (int i = lane; i <= in.src_reps; i += 32) so[i] = in.src_off[i];
        for (int i = lane; i < nsd; i += 32) sd[i] = in.src_devs[i];
        for (int i = lane; i <= in.dst_reps; i += 32) to[i] = in.dst_off[i];
        for (int i = lane; i < ndd; i += 32) td[i] = in.dst_devs[i];
        __syncwarp();
        load = sl;
        inbound = si;
        machine = sm;
        src_off = so;
        src_devs = sd;
        dst_off = to;
        dst_devs = td;
    }
    int trep = 0;
    for (int base = 0; base < in.n; base += 32) {
        const int q = base + lane;
        const bool has = q < in.n;
        const int64_t my_gen = has ? in.gen[q] : 0;
        const uint64_t my_kv = has ? in.kv[q] : 0;
        const int my_sr = has ? in.srcrep[q] : 0;
        int my_kind = 0, my_src = 0, my_dst = 0;
        const int cnt = in.n - base < 32 ? in.n - base : 32;
        for (int b = 0; b < cnt; ++b) {
            const int64_t gq = __shfl_sync(0xffffffffu, my_gen, b);
            if (gq <= in.threshold || in.dst_reps == 0) continue;  // drained
            const uint64_t kvq = __shfl_sync(0xffffffffu, my_kv, b);
            const int srq = __shfl_sync(0xffffffffu, my_sr, b);
            // target: least inbound-loaded device of the target replica, lowest id on ties
            KvPick t{~0ull, 2, kNone};
            for (int p = dst_off[trep] + lane; p < dst_off[trep + 1]; p += 32) {
                const KvPick c{inbound[dst_devs[p]], 0, dst_devs[p]};
                if (kv_less(c, t)) t = c;
            }
            t = kv_warp_min(t);
            trep = trep + 1 == in.dst_reps ? 0 : trep + 1;
            const int target = t.slot == kNone ? in.none_slot : t.slot;
            // source: intra-machine first, then least load toward target, then lowest id
            KvPick bsel{~0ull, 2, kNone};
            const int mt = machine[target];
            for (int p = src_off[srq] + lane; p < src_off[srq + 1]; p += 32) {
                const int slot = src_devs[p];
                const bool intra = machine[slot] >= 0 && machine[slot] == mt;
                const KvPick c{load[static_cast<size_t>(slot) * NS + target], intra ? 0 : 1, slot};
                if (kv_less(c, bsel)) bsel = c;
            }
            bsel = kv_warp_min(bsel);
            const int best = bsel.slot == kNone ? in.none_slot : bsel.slot;
            if (lane == 0) {
                load[static_cast<size_t>(best) * NS + target] += kvq;
                inbound[target] += kvq;
            }
            if (lane == b) {
                my_kind = 1;
                my_src = best;
                my_dst = target;
            }
            __syncwarp();
        }
        if (has) {
            in.kind[q] = my_kind;
            in.mig_src[q] = my_kind ? in.dev_id[my_src] : 0;
            in.mig_dst[q] = my_kind ? in.dev_id[my_dst] : 0;
        }
    }
}

// Parallel kv_plan: requests migrating to different target replicas touch
// disjoint state (the target's devices' inbound loads and the link-load
// columns of those devices; replicas own disjoint devices), so one warp per
// target replica walks that replica's requests in order — the same
// sequence of picks as the sequential fold.  The host falls back to
// k_kv_plan when a target replica is empty (its pick, device -1, would be
// shared).  State lives in global memory (volatile: columns of different
// warps share cache lines).
__device__ __forceinline__ KvPick kv_min_width(KvPick p, int width) {
    for (int d = width >> 1; d > 0; d >>= 1) {
        KvPick o;
        o.v = __shfl_xor_sync(0xffffffffu, p.v, d);
        o.cls = __shfl_xor_sync(0xffffffffu, p.cls, d);
        o.slot = __shfl_xor_sync(0xffffffffu, p.slot, d);
        if (kv_less(o, p)) p = o;
    }
    return p;
}

__global__ void __launch_bounds__(128) k_kv_plan_par(KvPlanIn in) {
    const int lane = threadIdx.x & 31;
    const int r = blockIdx.x * 4 + (threadIdx.x >> 5);
    if (r >= in.dst_reps) return;
    constexpr int kNone = 0x7fffffff;
    const int NS = in.num_slots;
    volatile uint64_t *load = in.load;
    volatile uint64_t *inbound = in.inbound;
    const int d0 = in.dst_off[r], d1 = in.dst_off[r + 1];
    const int nd = d1 - d0;
    int wt = 1;
    while (wt < nd && wt < 32) wt <<= 1;
    const int g0 = in.grp_off[r], g1 = in.grp_off[r + 1];
    for (int base = g0; base < g1; base += 32) {
        const int idx = base + lane;
        const uint64_t my_kv = idx < g1 ? in.grp_kv[idx] : 0;
        const int my_sr = idx < g1 ? in.grp_sr[idx] : 0;
        int my_src = 0, my_dst = 0;
        const int cnt = g1 - base < 32 ? g1 - base : 32;
        for (int b = 0; b < cnt; ++b) {
            const uint64_t kvq = __shfl_sync(0xffffffffu, my_kv, b);
            const int srq = __shfl_sync(0xffffffffu, my_sr, b);
            KvPick t{~0ull, 2, kNone};
            for (int p = d0 + lane; p < d1; p += 32) {
                const int slot = in.dst_devs[p];
                const KvPick c{inbound[slot], 0, slot};
                if (kv_less(c, t)) t = c;
            }
            t = kv_min_width(t, nd > 32 ? 32 : wt);
            const int target = __shfl_sync(0xffffffffu, t.slot, 0);  // lanes < width hold the minimum; nd >= 1
            const int s0 = in.src_off[srq], s1 = in.src_off[srq + 1];
            const int ns = s1 - s0;
            int ws = 1;
            while (ws < ns && ws < 32) ws <<= 1;
            KvPick bsel{~0ull, 2, kNone};
            const int mt = in.machine[target];
            for (int p = s0 + lane; p < s1; p += 32) {
                const int slot = in.src_devs[p];
                const bool intra = in.machine[slot] >= 0 && in.machine[slot] == mt;
                const KvPick c{load[static_cast<size_t>(slot) * NS + target], intra ? 0 : 1, slot};
                if (kv_less(c, bsel)) bsel = c;
            }
            bsel = kv_min_width(bsel, ns > 32 ? 32 : ws);
            const int bslot = __shfl_sync(0xffffffffu, bsel.slot, 0);
            const int best = bslot == kNone ? in.none_slot : bslot;
            if (lane == 0) {
                load[static_cast<size_t>(best) * NS + target] += kvq;
                inbound[target] += kvq;
            }
            if (lane == b) {
                my_src = best;
                my_dst = target;
            }
            __syncwarp();
        }
        if (idx < g1) {
            in.grp_src[idx] = in.dev_id[my_src];
            in.grp_dst[idx] = in.dev_id[my_dst];
        }
    }
}

// The lexicographic minimum (cls, v, slot) of the warp's candidates by four
// 32-bit warp reductions (cls, v's high word, low word, slot) instead of a
// shuffle tree; returns the winning slot (0x7fffffff when no lane has one).
__device__ __forceinline__ int kv_pick_redux(const KvPick &p) {
    const bool valid = p.slot != 0x7fffffff;
    const unsigned c = valid ? static_cast<unsigned>(p.cls) : 0xffffffffu;
    const unsigned cm = __reduce_min_sync(0xffffffffu, c);
    bool in = valid && c == cm;
    const unsigned hi = in ? static_cast<unsigned>(p.v >> 32) : 0xffffffffu;
    const unsigned hm = __reduce_min_sync(0xffffffffu, hi);
    in = in && hi == hm;
    const unsigned lo = in ? static_cast<unsigned>(p.v) : 0xffffffffu;
    const unsigned lm = __reduce_min_sync(0xffffffffu, lo);
    in = in && lo == lm;
    const unsigned sl = in ? static_cast<unsigned>(p.slot) : 0x7fffffffu;
    return static_cast<int>(__reduce_min_sync(0xffffffffu, sl));
}

// k_kv_plan_par with the replica's state in shared memory: a warp (one CTA)
// per target replica of <= 32 devices holds the inbound loads of those
// devices and their link-load columns (every source slot -> each of them):
// the only state its picks read or write, so the request walk never leaves
// shared memory.  Columns start from the carried plan's loads.
__global__ void __launch_bounds__(32) k_kv_plan_par_smem(KvPlanIn in, int ndmax) {
    extern __shared__ __align__(16) unsigned char kv_smem[];
    const int lane = threadIdx.x, r = blockIdx.x;
    constexpr int kNone = 0x7fffffff;
    const int NS = in.num_slots;
    const int d0 = in.dst_off[r], nd = in.dst_off[r + 1] - d0;
    uint64_t *inb = reinterpret_cast<uint64_t *>(kv_smem);         // [nd]
    uint64_t *col = inb + ndmax;                                     // [NS][nd]
    for (int i = lane; i < nd; i += 32) inb[i] = in.inbound[in.dst_devs[d0 + i]];
    for (int i = lane; i < NS * nd; i += 32) {
        const int sl = i / nd, tl = i - sl * nd;
        col[i] = in.load[static_cast<size_t>(sl) * NS + in.dst_devs[d0 + tl]];
    }
    __syncwarp();
    const int my_tslot = lane < nd ? in.dst_devs[d0 + lane] : kNone;
    const int g0 = in.grp_off[r], g1 = in.grp_off[r + 1];
    for (int base = g0; base < g1; base += 32) {
        const int idx = base + lane;
        const uint64_t my_kv = idx < g1 ? in.grp_kv[idx] : 0;
        const int my_sr = idx < g1 ? in.grp_sr[idx] : 0;
        int my_src = 0, my_dst = 0;
        const int cnt = g1 - base < 32 ? g1 - base : 32;
        for (int b = 0; b < cnt; ++b) {
            const uint64_t kvq = __shfl_sync(0xffffffffu, my_kv, b);
            const int srq = __shfl_sync(0xffffffffu, my_sr, b);
            KvPick t{~0ull, 2, kNone};
            if (lane < nd) t = KvPick{inb[lane], 0, my_tslot};
            const int target = kv_pick_redux(t);
            const int tl = __ffs(__ballot_sync(0xffffffffu, my_tslot == target)) - 1;
            const int s0 = in.src_off[srq], s1 = in.src_off[srq + 1];
            KvPick bsel{~0ull, 2, kNone};
            const int mt = __ldg(in.machine + target);
            for (int p = s0 + lane; p < s1; p += 32) {
                const int slot = __ldg(in.src_devs + p);
                const int ms = __ldg(in.machine + slot);
                const KvPick c{col[slot * nd + tl], (ms >= 0 && ms == mt) ? 0 : 1, slot};
                if (kv_less(c, bsel)) bsel = c;
            }
            const int bslot = kv_pick_redux(bsel);
            const int best = bslot == kNone ? in.none_slot : bslot;
            __syncwarp();
            if (lane == 0) {
                col[best * nd + tl] += kvq;
                inb[tl] += kvq;
            }
            if (lane == b) {
                my_src = best;
                my_dst = target;
            }
            __syncwarp();
        }
        if (idx < g1) {
            in.grp_src[idx] = in.dev_id[my_src];
            in.grp_dst[idx] = in.dev_id[my_dst];
        }
    }
}

__global__ void k_topk_check(const uint64_t *meta, int groups, const uint64_t *kth, unsigned int *bad) {
    const uint64_t kk = *kth;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < groups; i += gridDim.x * blockDim.x)
        if (meta[i] < kk) atomicAdd(bad, 1u);
}

}  // namespace

// ------------------------------------------------------------- launchers ---
// c_binom is a __constant__ symbol: one copy per device (per loaded module),
// so readiness is tracked per device, under a lock (contexts on several
// devices may be driven from several host threads).
static int ensure_binom() {
    constexpr int kDevMax = 64;
    static std::mutex mu;
    static bool ready[kDevMax] = {};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return static_cast<int>(e);
    if (dev < 0 || dev >= kDevMax) return static_cast<int>(cudaErrorInvalidDevice);
    std::lock_guard<std::mutex> lk(mu);
    if (ready[dev]) return 0;
    static uint64_t h[kBinomN][kBinomK];
    static bool filled = false;
    if (!filled) {
        for (int n = 0; n < kBinomN; ++n)
            for (int k = 0; k < kBinomK; ++k) {
                unsigned __int128 r = 1;
                if (k > n) {
                    r = 0;
                } else {
                    for (int i = 1; i <= k; ++i) r = r * static_cast<unsigned>(n - k + i) / static_cast<unsigned>(i);
                }
                h[n][k] = r > ~0ull ? ~0ull : static_cast<uint64_t>(r);
            }
        filled = true;
    }
    e = cudaMemcpyToSymbol(c_binom, h, sizeof(h));  // synchronous: visible to every later launch
    if (e != cudaSuccess) return static_cast<int>(e);
    ready[dev] = true;
    return 0;
}

int launch_cost_tables(const ShapeTables &t, const double *cin, const double *cout, uint32_t num_layers,
                       uint64_t kvb, double pc, double dc, double ppc, double slope, double span_s, void *stream) {
    cudaGetLastError();
    const int cells = t.num_shapes * t.J;
    if (cells == 0) return 0;
    const int block = 128, grid = (cells + block - 1) / block;
    k_cost_cells<<<grid, block, 0, static_cast<cudaStream_t>(stream)>>>(t, cin, cout, num_layers, kvb, pc, dc, ppc,
                                                                        slope, span_s);
    return check(cudaGetLastError());
}

int launch_normalize_rows(const ShapeTables &t, void *stream) {
    cudaGetLastError();
    if (t.num_shapes == 0) return 0;
    const int block = 128, grid = (t.num_shapes + block - 1) / block;
    k_normalize_rows<<<grid, block, 0, static_cast<cudaStream_t>(stream)>>>(t);
    return check(cudaGetLastError());
}

int launch_plan_eval(const ShapeTables &t, const SpaceTables &sp, const KeyLayout &key, const PlanSource &src,
                     const PlanOutputs &out, const SolveParams &prm, int rmax, int sm_count, int skip_exact,
                     WorkRing *ring, void *stream, uint64_t *launches) {
    if (int e = ensure_binom()) return e;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (src.count == 0) return 0;
    // lanes double as class positions in the greedy scan: G >= J.  Plans with
    // more than 16 replicas use warp-wide groups (measured: two 16-lane plans
    // per warp diverge on exchange length and lose 12%); OSERVE_K1_G=16 opts
    // into 16-lane groups owning up to 4 replicas each.
    const int need = rmax > prm.J ? rmax : prm.J;
    static const int opt16 = [] {
        const char *e = getenv("OSERVE_K1_G");
        return e && atoi(e) == 16;
    }();
    if (need <= 8) return run_plan_eval<8, 1>(t, sp, key, src, out, prm, sm_count, skip_exact, ring, s, launches);
    if (need <= 16) return run_plan_eval<16, 1>(t, sp, key, src, out, prm, sm_count, skip_exact, ring, s, launches);
    if (prm.J <= 16 && opt16) {
        if (rmax <= 32) return run_plan_eval<16, 2>(t, sp, key, src, out, prm, sm_count, skip_exact, ring, s, launches);
        if (rmax <= 64) return run_plan_eval<16, 4>(t, sp, key, src, out, prm, sm_count, skip_exact, ring, s, launches);
    }
    if (rmax <= 32) return run_plan_eval<32, 1>(t, sp, key, src, out, prm, sm_count, skip_exact, ring, s, launches);
    if (rmax <= 64) return run_plan_eval<32, 2>(t, sp, key, src, out, prm, sm_count, skip_exact, ring, s, launches);
    if (rmax <= 128) return run_plan_eval<32, 4>(t, sp, key, src, out, prm, sm_count, skip_exact, ring, s, launches);
    return static_cast<int>(cudaErrorInvalidValue);
}

// Thread per task: copy it to the new list, or write its children (the
// branches v = hi .. 0 of its first decision node, in preorder).
__global__ void __launch_bounds__(128) k_exact_split(ExactTasks et, ExactTasks nt, const uint32_t *newoff,
                                                     uint64_t total) {
    for (uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < total;
         q += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t o = newoff[q];
        const uint32_t nc = et.nchild[q];
        const uint8_t td = et.tdepth[q];
        const int dep = td & 0x7f;
        const int nz = nc > 1 ? et.nzero[q] : 0;
        for (uint32_t c = 0; c < nc; ++c) {
            const uint64_t r = o + c;
            nt.plan[r] = et.plan[q];
            for (int a = 0; a < dep; ++a) nt.path[r * kTaskDepthMax + a] = et.path[q * kTaskDepthMax + a];
            if (nc == 1) {  // unchanged task
                nt.tdepth[r] = td;
                nt.g[r] = et.g[q];
                nt.m[r] = et.m[q];
                nt.nodes[r] = et.nodes[q];
                nt.lbran[r] = et.lbran[q];
                nt.capped[r] = et.capped[q];
                nt.done[r] = et.done[q];
            } else {  // path + nz forced zeros + v
                for (int a = 0; a < nz; ++a) nt.path[r * kTaskDepthMax + dep + a] = 0;
                nt.tdepth[r] = static_cast<uint8_t>(dep + nz + 1);
                nt.path[r * kTaskDepthMax + dep + nz] = static_cast<int32_t>(nc - 1 - c);  // v = hi - c
                nt.capped[r] = 0;
                nt.done[r] = 0;
            }
        }
    }
}

__global__ void k_exact_ranges(ExactTasks et, const uint32_t *newoff, uint64_t plans) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < plans;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (et.state[i] != 1) continue;  // only frontier plans hold tasks
        const uint64_t a = newoff[et.toff[i]], b = newoff[et.toff[i] + et.ntask[i]];
        et.toff[i] = a;
        et.ntask[i] = b - a;
    }
}

// newoff[0..n] = exclusive prefix sum of nchild[0..n) (nchild[n] must be 0),
// then the per-plan task ranges of the new list.
int launch_exact_rescan(const ExactTasks &et, uint64_t n, uint32_t *newoff, uint64_t plans, void **temp,
                        size_t *temp_bytes, void *stream, uint64_t *launches) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    size_t need = 0;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, need, et.nchild, newoff, static_cast<int>(n + 1), s);
    if (e != cudaSuccess) return static_cast<int>(e);
    if (need > *temp_bytes) {
        if (*temp) cudaFree(*temp);
        e = cudaMalloc(temp, need);
        if (e != cudaSuccess) return static_cast<int>(e);
        *temp_bytes = need;
    }
    e = cub::DeviceScan::ExclusiveSum(*temp, need, et.nchild, newoff, static_cast<int>(n + 1), s);
    if (e != cudaSuccess) return static_cast<int>(e);
    if (launches) ++*launches;
    return 0;
}

int launch_exact_ranges(const ExactTasks &et, const uint32_t *newoff, uint64_t plans, void *stream,
                        uint64_t *launches) {
    if (plans == 0) return 0;
    k_exact_ranges<<<static_cast<unsigned>((plans + 127) / 128), 128, 0, static_cast<cudaStream_t>(stream)>>>(
        et, newoff, plans);
    if (launches) ++*launches;
    return check(cudaGetLastError());
}

int launch_exact_split(const ShapeTables &t, const SpaceTables &sp, const PlanSource &src, const SolveParams &prm,
                       const ExactTasks &et, const ExactTasks &nt, const uint32_t *newoff, uint64_t total_tasks,
                       int sm_count, void *stream, uint64_t *launches) {
    (void)t;
    (void)sp;
    (void)src;
    (void)prm;
    cudaGetLastError();
    if (total_tasks == 0) return 0;
    const int block = 128;
    const uint64_t cap = static_cast<uint64_t>(sm_count) * 16;
    uint64_t grid = (total_tasks + block - 1) / block;
    if (grid > cap) grid = cap;
    k_exact_split<<<static_cast<unsigned>(grid), block, 0, static_cast<cudaStream_t>(stream)>>>(et, nt, newoff,
                                                                                                total_tasks);
    if (launches) ++*launches;
    return check(cudaGetLastError());
}

int launch_plan_exact(const ShapeTables &t, const SpaceTables &sp, const KeyLayout &key, const PlanSource &src,
                      const PlanOutputs &out, const SolveParams &prm, int sm_count, void *stream,
                      uint64_t *launches) {
    cudaGetLastError();
    if (int e = ensure_binom()) return e;
    if (src.count == 0) return 0;
    static const bool warp = [] {
        const char *e = getenv("OSERVE_EXACT_SEQ");
        return e && std::strcmp(e, "warp") == 0;
    }();
    const int block = warp ? 128 : 32;
    const uint64_t cap = static_cast<uint64_t>(sm_count) * (warp ? 16 : 64);
    uint64_t grid = warp ? (src.count * 32 + block - 1) / block : src.count;
    if (grid > cap) grid = cap;
    if (warp)  // 4 warps, warp per plan
        k_plan_exact<<<static_cast<unsigned>(grid), block, 0, static_cast<cudaStream_t>(stream)>>>(t, sp, key, src,
                                                                                                   out, prm);
    else  // a thread (a warp) per plan
        k_plan_exact_thr<<<static_cast<unsigned>(grid), block, 0, static_cast<cudaStream_t>(stream)>>>(t, sp, key, src,
                                                                                                       out, prm);
    if (launches) ++*launches;
    return check(cudaGetLastError());
}

// (L, own) scan of the replay: keep the previous task's alive bits 0..L,
// add the task's own bits (associative: see exact_replay_task)
struct AliveOp {
    __device__ __forceinline__ uint64_t operator()(uint64_t a, uint64_t b) const {
        const int la = static_cast<int>(static_cast<int32_t>(a >> 32)), lb = static_cast<int>(static_cast<int32_t>(b >> 32));
        const uint32_t keep = lb >= 0 ? ((2u << lb) - 1u) : 0u;
        const uint32_t own = (static_cast<uint32_t>(a) & keep) | static_cast<uint32_t>(b);
        const int l = la < lb ? la : lb;
        return (static_cast<uint64_t>(static_cast<uint32_t>(l)) << 32) | own;
    }
};

__global__ void k_alive_pack(const int32_t *L, const uint32_t *own, uint64_t *packed, uint64_t n) {
    for (uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < n;
         q += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        packed[q] = (static_cast<uint64_t>(static_cast<uint32_t>(L[q])) << 32) | own[q];
}
__global__ void k_alive_unpack(const uint64_t *packed, uint32_t *mask, uint64_t n) {
    for (uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < n;
         q += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        mask[q] = static_cast<uint32_t>(packed[q]);
}

// Ancestor-alive masks of all tasks (inclusive scan of the packed (L, own)).
int launch_alive_scan(const ExactTasks &et, uint64_t total, uint64_t *tmp, void **temp, size_t *temp_bytes,
                      int sm_count, void *stream, uint64_t *launches) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (total == 0) return 0;
    const uint64_t grid = std::min<uint64_t>((total + 255) / 256, static_cast<uint64_t>(sm_count) * 8);
    uint64_t *out = tmp + total;  // tmp holds 2 * total
    k_alive_pack<<<static_cast<unsigned>(grid), 256, 0, s>>>(et.aL, et.amask, tmp, total);
    size_t need = 0;
    cudaError_t e = cub::DeviceScan::InclusiveScan(nullptr, need, tmp, out, AliveOp(), static_cast<int>(total), s);
    if (e != cudaSuccess) return static_cast<int>(e);
    if (need > *temp_bytes) {
        if (*temp) cudaFree(*temp);
        e = cudaMalloc(temp, need);
        if (e != cudaSuccess) return static_cast<int>(e);
        *temp_bytes = need;
    }
    e = cub::DeviceScan::InclusiveScan(*temp, need, tmp, out, AliveOp(), static_cast<int>(total), s);
    if (e != cudaSuccess) return static_cast<int>(e);
    k_alive_unpack<<<static_cast<unsigned>(grid), 256, 0, s>>>(out, et.amask, total);
    if (launches) *launches += 3;
    return check(cudaGetLastError());
}

int launch_exact_plan_pass(int pass, const ShapeTables &t, const SpaceTables &sp, const KeyLayout &key,
                           const PlanSource &src, const PlanOutputs &out, const SolveParams &prm,
                           const ExactTasks &et, int sm_count, void *stream, uint64_t *launches) {
    cudaGetLastError();
    if (int e = ensure_binom()) return e;
    if (src.count == 0) return 0;
    const int block = 64;
    const uint64_t cap = static_cast<uint64_t>(sm_count) * 32;
    uint64_t grid = (src.count + block - 1) / block;
    if (grid > cap) grid = cap;
    k_exact_plan<<<static_cast<unsigned>(grid), block, 0, static_cast<cudaStream_t>(stream)>>>(pass, t, sp, key, src,
                                                                                               out, prm, et);
    if (launches) ++*launches;
    return check(cudaGetLastError());
}

int launch_exact_task_pass(int pass, const ShapeTables &t, const SpaceTables &sp, const PlanSource &src,
                           const SolveParams &prm, const ExactTasks &et, uint64_t total_tasks, int sm_count,
                           void *stream, uint64_t *launches) {
    cudaGetLastError();
    if (total_tasks == 0) return 0;
    // thread per task, dynamic fetch (counter zeroed on the stream)
    if (cudaError_t e = cudaMemsetAsync(et.fetch, 0, sizeof(unsigned long long), static_cast<cudaStream_t>(stream)))
        return static_cast<int>(e);
    const int block = 128;
    uint64_t grid = (total_tasks + block - 1) / block;
    const uint64_t cap = static_cast<uint64_t>(sm_count) * 16;
    if (grid > cap) grid = cap;
    k_exact_task_thr<<<static_cast<unsigned>(grid), block, 0, static_cast<cudaStream_t>(stream)>>>(
        pass, t, sp, src, prm, et, total_tasks, et.fetch);
    if (launches) ++*launches;
    return check(cudaGetLastError());
}

int launch_exact_prefix(int which, const ExactTasks &et, uint64_t total, uint64_t plans, int64_t *tmp, void **temp,
                        size_t *temp_bytes, int sm_count, void *stream, uint64_t *launches) {
    cudaGetLastError();
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const unsigned gt = static_cast<unsigned>(std::min<uint64_t>((total + 255) / 256, static_cast<uint64_t>(sm_count) * 8));
    const unsigned gp = static_cast<unsigned>(std::min<uint64_t>((plans + 255) / 256, static_cast<uint64_t>(sm_count) * 8));
    if (which == 6 && plans) k_exact_inc_reset<<<gp, 256, 0, s>>>(et, plans);
    if (total == 0) return check(cudaGetLastError());
    const int64_t *in = et.m;
    int64_t *out = et.inc;
    if (which == 4) {
        k_exact_lb_vals<<<gt, 256, 0, s>>>(et, total, tmp);
        in = tmp;
        out = et.lb;
    }
    size_t need = 0;
    const uint32_t n = static_cast<uint32_t>(total);
    cudaError_t e = cub::DeviceScan::ExclusiveScanByKey(nullptr, need, et.plan, in, out, MaxI64(), int64_t{-1}, n,
                                                        ::cuda::std::equal_to<>(), s);
    if (e != cudaSuccess) return static_cast<int>(e);
    if (need > *temp_bytes) {
        if (*temp) cudaFree(*temp);
        e = cudaMalloc(temp, need);
        if (e != cudaSuccess) return static_cast<int>(e);
        *temp_bytes = need;
    }
    e = cub::DeviceScan::ExclusiveScanByKey(*temp, need, et.plan, in, out, MaxI64(), int64_t{-1}, n,
                                            ::cuda::std::equal_to<>(), s);
    if (e != cudaSuccess) return static_cast<int>(e);
    if (which == 4) {
        k_exact_lb_apply<<<gt, 256, 0, s>>>(et, total);
    } else {
        k_exact_opt<<<gt, 256, 0, s>>>(et, total);
        k_exact_istar<<<gt, 256, 0, s>>>(et, total);
    }
    if (launches) *launches += 4;
    return check(cudaGetLastError());
}

int launch_exact_retire(const ExactTasks &et, uint64_t plans, int sm_count, void *stream, uint64_t *launches) {
    cudaGetLastError();
    if (plans == 0) return 0;
    const unsigned gp = static_cast<unsigned>(std::min<uint64_t>((plans + 255) / 256, static_cast<uint64_t>(sm_count) * 8));
    k_exact_retire<<<gp, 256, 0, static_cast<cudaStream_t>(stream)>>>(et, plans);
    if (launches) ++*launches;
    return check(cudaGetLastError());
}

int launch_switch_cost(const SwitchDeps &d, const SwitchOut &o, void *stream, uint64_t *launches) {
    cudaGetLastError();
    if (d.count == 0) return 0;
    if (d.num_devices > kSwMaxDev) return static_cast<int>(cudaErrorInvalidValue);
    k_switch_cost<<<d.count, 256, 0, static_cast<cudaStream_t>(stream)>>>(d, o);
    if (launches) ++*launches;
    return check(cudaGetLastError());
}

int k1_groups(int rmax, int J, int sm_count, const ShapeTables &t, uint64_t count) {
    size_t smem = 0;
    bool stage = false;
    uint64_t grid = 0;
    const int need = rmax > J ? rmax : J;
    const char *env = getenv("OSERVE_K1_G");
    const bool opt16 = env && atoi(env) == 16;
    int e = 0, gpb = 0;
    // (sizes the top-K lists: the top-K variant's geometry)
    constexpr int V = kK1TopK;
    if (need <= 8) e = plan_eval_geometry<8, 1, V>(t, J, sm_count, count, &smem, &stage, &grid), gpb = 32;
    else if (need <= 16) e = plan_eval_geometry<16, 1, V>(t, J, sm_count, count, &smem, &stage, &grid), gpb = 16;
    else if (J <= 16 && opt16 && rmax <= 32) e = plan_eval_geometry<16, 2, V>(t, J, sm_count, count, &smem, &stage, &grid), gpb = 16;
    else if (J <= 16 && opt16 && rmax <= 64) e = plan_eval_geometry<16, 4, V>(t, J, sm_count, count, &smem, &stage, &grid), gpb = 16;
    else if (rmax <= 32) e = plan_eval_geometry<32, 1, V>(t, J, sm_count, count, &smem, &stage, &grid), gpb = 8;
    else if (rmax <= 64) e = plan_eval_geometry<32, 2, V>(t, J, sm_count, count, &smem, &stage, &grid), gpb = 8;
    else e = plan_eval_geometry<32, 4, V>(t, J, sm_count, count, &smem, &stage, &grid), gpb = 8;
    if (e) return -1;
    return static_cast<int>(grid) * gpb;
}

int launch_switch_cost_keys(const SwitchDeps &src, const SpaceTables &sp, const KeyLayout &key, const ShapeTables &t,
                            const uint64_t *keys, int count, const int32_t *, const SwitchOut &o, void *stream,
                            uint64_t *launches) {
    cudaGetLastError();
    if (count == 0) return 0;
    if (src.num_devices > kSwMaxDev) return static_cast<int>(cudaErrorInvalidValue);
    k_switch_cost_keys<<<count, 256, 0, static_cast<cudaStream_t>(stream)>>>(src, sp, key, t, keys, o);
    if (launches) ++*launches;
    return check(cudaGetLastError());
}

int sort_keys(uint64_t *keys, uint64_t *tmp_keys, int n, void **temp, size_t *temp_bytes, void *stream) {
    size_t need = 0;
    cudaError_t e = cub::DeviceRadixSort::SortKeys(nullptr, need, keys, tmp_keys, n, 0, 64,
                                                   static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return static_cast<int>(e);
    if (need > *temp_bytes) {
        if (*temp) cudaFree(*temp);
        e = cudaMalloc(temp, need);
        if (e != cudaSuccess) return static_cast<int>(e);
        *temp_bytes = need;
    }
    e = cub::DeviceRadixSort::SortKeys(*temp, need, keys, tmp_keys, n, 0, 64, static_cast<cudaStream_t>(stream));
    return static_cast<int>(e);
}

int launch_kv_plan(const KvPlanIn &in, void *stream, uint64_t *launches) {
    cudaGetLastError();
    if (in.n == 0) return 0;
    if (in.grp_off) {  // target-replica parallel path (group-ordered arrays)
        int ndmax = 0;
        for (int r = 0; r < in.dst_reps; ++r) ndmax = std::max(ndmax, in.h_dst_off[r + 1] - in.h_dst_off[r]);
        const size_t smem = sizeof(uint64_t) * (static_cast<size_t>(ndmax) + static_cast<size_t>(in.num_slots) * ndmax);
        bool use = ndmax <= 32 && smem <= 96 * 1024;
        if (use && smem > 48 * 1024 &&
            cudaFuncSetAttribute(k_kv_plan_par_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024) !=
                cudaSuccess) {
            cudaGetLastError();
            use = false;
        }
        if (use)
            k_kv_plan_par_smem<<<in.dst_reps, 32, smem, static_cast<cudaStream_t>(stream)>>>(in, ndmax);
        else
            k_kv_plan_par<<<(in.dst_reps + 3) / 4, 128, 0, static_cast<cudaStream_t>(stream)>>>(in);
        if (launches) ++*launches;
        return check(cudaGetLastError());
    }
    const size_t NS = static_cast<size_t>(in.num_slots);
    const size_t smem = sizeof(uint64_t) * (NS * NS + NS) +
                        sizeof(int32_t) * (NS + in.src_reps + 1 + in.dst_reps + 1 + in.n_src_devs + in.n_dst_devs);
    int use = smem <= 200 * 1024;
    if (use && smem > 48 * 1024) {
        if (cudaFuncSetAttribute(k_kv_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) != cudaSuccess) {
            cudaGetLastError();
            use = 0;
        }
    }
    k_kv_plan<<<1, 32, use ? smem : 0, static_cast<cudaStream_t>(stream)>>>(in, use);
    if (launches) ++*launches;
    return check(cudaGetLastError());
}

int launch_topk_check(const uint64_t *meta, int groups, const uint64_t *kth, unsigned int *bad, void *stream) {
    cudaGetLastError();
    if (groups <= 0) return 0;
    k_topk_check<<<(groups + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(meta, groups, kth, bad);
    return check(cudaGetLastError());
}

}  // namespace oserve_gpu
