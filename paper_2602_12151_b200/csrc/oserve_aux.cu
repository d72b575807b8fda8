// oserve_aux.cu — sm_100a kernels behind the remaining reference signatures
// of the C++ shim (include/oserve_gpu.hpp):
//
//   k_layout         switchplan::layout (switchplan.cpp:40-63): thread per
//                    (replica, stage, slice) shard
//   k_switch_held    switchplan::greedy_plan over two arbitrary ShardLayouts
//                    (switchplan.cpp:65-131): per-device held-range lists,
//                    warp per target device, lane per source device
//   k_link_time      switchplan::estimate_time (switchplan.cpp:133-140):
//                    thread per link, max-reduction
//   k_check          flow::check_constraints (flowassign.cpp:529-551): thread
//                    per instance, first violation in the reference's order
//
// (flow::normalize / normalize_or_scale run on K0b, k_normalize_rows.)
#include <cuda_runtime.h>

#include <cstdint>

#include "oserve_internal.h"

namespace oserve_gpu {

namespace {

inline int check(cudaError_t e) { return e == cudaSuccess ? 0 : static_cast<int>(e); }

// ---------------------------------------------------------------- layout ---
__global__ void k_layout(LayoutIn in) {
    const int total = in.total;
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < total; g += gridDim.x * blockDim.x) {
        int lo = 0, hi = in.R - 1;  // replica of shard g
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (in.rep_off[mid] <= g) lo = mid;
            else hi = mid - 1;
        }
        const int r = lo, q = g - in.rep_off[r];
        const uint64_t tp = static_cast<uint64_t>(in.tp[r]), pp = static_cast<uint64_t>(in.pp[r]);
        const uint64_t s = static_cast<uint64_t>(q) / tp, i = static_cast<uint64_t>(q) % tp;
        // u64 arithmetic exactly as the reference (P * s may wrap identically)
        const uint64_t sb = in.P * s / pp, se = in.P * (s + 1) / pp, len = se - sb;
        in.begin[g] = sb + len * i / tp;
        in.end[g] = sb + len * (i + 1) / tp;
        in.holder[g] = in.devs_sorted[in.dev_off[r] + q];
    }
}

// ------------------------------------------------------- greedy (layouts) ---
__device__ __forceinline__ bool covers(const uint64_t *b, const uint64_t *e, int lo, int hi, uint64_t fb, uint64_t fe) {
    for (int q = lo; q < hi; ++q)
        if (b[q] <= fb && fe <= e[q]) return true;
    return false;
}

constexpr int kHeldQ = 8;  // source slots per lane (<= 256 device slots)

__global__ void __launch_bounds__(256) k_switch_held(HeldIn in, HeldOut o) {
    extern __shared__ uint64_t cuts[];  // [P2] every range boundary of both layouts
    __shared__ double wmax[8];
    __shared__ unsigned long long wbytes[8];
    __shared__ int nc_s;
    const int ND = in.num_devices;
    // fragment boundaries (:70-85): the sorted set of all begins / ends
    int P2 = 1;
    while (P2 < in.nbounds) P2 <<= 1;
    for (int i = threadIdx.x; i < P2; i += blockDim.x) cuts[i] = i < in.nbounds ? in.bounds[i] : ~0ull;
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
        for (int i = 0; i < in.nbounds; ++i)
            if (m == 0 || cuts[i] != cuts[m - 1]) cuts[m++] = cuts[i];
        nc_s = m;
        *o.ncuts = m;
        for (int i = 0; i < m; ++i) o.cuts[i] = cuts[i];
    }
    __syncthreads();
    const int NC = nc_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    double est = 0.0;
    unsigned long long maxb = 0;
    for (int t = warp; t < ND; t += nwarps) {
        const int t0 = in.dst_off[t], t1 = in.dst_off[t + 1];
        if (t0 == t1) continue;
        unsigned long long load[kHeldQ];
#pragma unroll
        for (int q = 0; q < kHeldQ; ++q) load[q] = 0;
        for (int f = 0; f + 1 < NC; ++f) {
            const uint64_t fb = cuts[f], fe = cuts[f + 1];
            if (!covers(in.dst_b, in.dst_e, t0, t1, fb, fe)) continue;
            // no transfer when the target already holds these bytes (:95-96)
            if (covers(in.src_b, in.src_e, in.src_off[t], in.src_off[t + 1], fb, fe)) continue;
            // holders in ascending id: (intra first, least load toward t, lowest id)
            unsigned long long best = ~0ull;
#pragma unroll
            for (int q = 0; q < kHeldQ; ++q) {
                const int s = lane + 32 * q;
                if (s >= ND) continue;
                if (!covers(in.src_b, in.src_e, in.src_off[s], in.src_off[s + 1], fb, fe)) continue;
                const bool intra = in.machine[s] >= 0 && in.machine[s] == in.machine[t];
                const unsigned long long kv = (static_cast<unsigned long long>(!intra) << 63) |
                                              (static_cast<unsigned long long>(load[q]) << 8) |
                                              static_cast<unsigned long long>(s);
                best = kv < best ? kv : best;
            }
#pragma unroll
            for (int sft = 16; sft > 0; sft >>= 1) {
                const unsigned long long v = __shfl_xor_sync(0xffffffffu, best, sft);
                best = v < best ? v : best;
            }
            if (best == ~0ull) {  // UnsourcedFragment (:99-103)
                if (lane == 0) o.detail[static_cast<int64_t>(t) * o.max_frags + f] = -2;
                continue;
            }
            const int win = static_cast<int>(best & 0xff);
            if ((win & 31) == lane) {
#pragma unroll
                for (int q = 0; q < kHeldQ; ++q)
                    if (lane + 32 * q == win) load[q] += fe - fb;
            }
            if (lane == 0) o.detail[static_cast<int64_t>(t) * o.max_frags + f] = win;
        }
#pragma unroll
        for (int q = 0; q < kHeldQ; ++q) {
            const int s = lane + 32 * q;
            if (s < ND && load[q] > 0) {
                const bool intra = in.machine[s] >= 0 && in.machine[s] == in.machine[t];
                const double v = static_cast<double>(load[q]) / (intra ? in.intra_bw : in.inter_bw);
                est = v > est ? v : est;
                maxb = load[q] > maxb ? load[q] : maxb;
            }
        }
    }
#pragma unroll
    for (int sft = 16; sft > 0; sft >>= 1) {
        const double e2 = __shfl_xor_sync(0xffffffffu, est, sft);
        est = e2 > est ? e2 : est;
        const unsigned long long b2 = __shfl_xor_sync(0xffffffffu, maxb, sft);
        maxb = b2 > maxb ? b2 : maxb;
    }
    if (lane == 0) {
        wmax[warp] = est;
        wbytes[warp] = maxb;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double e = 0.0;
        unsigned long long b = 0;
        for (int w = 0; w < nwarps; ++w) {
            e = wmax[w] > e ? wmax[w] : e;
            b = wbytes[w] > b ? wbytes[w] : b;
        }
        *o.est = e;
        *o.max_bytes = b;
    }
}

// ------------------------------------------------------------ link time ---
__global__ void k_link_time(LinkIn in, double *est) {
    __shared__ double wm[32];
    double m = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < in.n; i += gridDim.x * blockDim.x) {
        const int a = in.src_machine[i], b = in.dst_machine[i];
        const double bw = (a >= 0 && a == b) ? in.intra_bw : in.inter_bw;
        const double v = static_cast<double>(in.bytes[i]) / bw;
        m = v > m ? v : m;
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, m, s);
        m = o > m ? o : m;
    }
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double r = 0.0;  // estimate_time starts from 0.0
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) r = wm[w] > r ? wm[w] : r;
        *est = r;
    }
}

// ------------------------------------------------------ check_constraints ---
// First violation in the reference's order: C1 over types, C2 over (k, j),
// then per replica C3's zero-capacity test (inside the j loop) and budget.
__global__ void k_check(CheckIn in) {
    const int R = in.R, J = in.J;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < in.count; i += gridDim.x * blockDim.x) {
        const int64_t *x = in.x + static_cast<int64_t>(i) * R * J;
        const int64_t *e = in.e + static_cast<int64_t>(i) * R * J;
        const int64_t *lam = in.lambda + static_cast<int64_t>(i) * J;
        const int64_t *unit = in.t.unit + static_cast<int64_t>(i) * R * J;
        const int64_t *M = in.t.M + static_cast<int64_t>(i) * R;
        int kind = 0, kk = 0, jj = 0;
        for (int j = 0; j < J && !kind; ++j) {
            int64_t tot = 0;
            for (int k = 0; k < R; ++k) tot += x[k * J + j];
            if (tot > lam[j]) kind = 1, jj = j;
        }
        for (int k = 0; k < R && !kind; ++k)
            for (int j = 0; j < J && !kind; ++j)
                if (x[k * J + j] > e[k * J + j]) kind = 2, kk = k, jj = j;
        for (int k = 0; k < R && !kind; ++k) {
            int64_t used = 0;
            for (int j = 0; j < J && !kind; ++j) {
                if (x[k * J + j] > 0 && unit[k * J + j] == 0) {
                    kind = 3, kk = k, jj = j;
                    break;
                }
                used += x[k * J + j] * unit[k * J + j];
            }
            if (!kind && used > M[k]) kind = 4, kk = k;
        }
        in.kind[i] = kind;
        in.k[i] = kk;
        in.j[i] = jj;
    }
}

}  // namespace

int launch_layout(const LayoutIn &in, void *stream, uint64_t *launches) {
    cudaGetLastError();
    if (in.total <= 0) return 0;
    const int grid = (in.total + 127) / 128;
    k_layout<<<grid < 1024 ? grid : 1024, 128, 0, static_cast<cudaStream_t>(stream)>>>(in);
    if (launches) ++*launches;
    return check(cudaGetLastError());
}

int launch_switch_held(const HeldIn &in, const HeldOut &o, void *stream, uint64_t *launches) {
    cudaGetLastError();
    if (in.num_devices > 32 * kHeldQ) return static_cast<int>(cudaErrorInvalidValue);
    int P2 = 1;
    while (P2 < in.nbounds) P2 <<= 1;
    const size_t smem = sizeof(uint64_t) * static_cast<size_t>(P2);
    if (smem > 200 * 1024) return static_cast<int>(cudaErrorInvalidValue);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_switch_held, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        if (e != cudaSuccess) return static_cast<int>(e);
    }
    k_switch_held<<<1, 256, smem, static_cast<cudaStream_t>(stream)>>>(in, o);
    if (launches) ++*launches;
    return check(cudaGetLastError());
}

int launch_link_time(const LinkIn &in, double *est, void *stream, uint64_t *launches) {
    cudaGetLastError();
    k_link_time<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(in, est);
    if (launches) ++*launches;
    return check(cudaGetLastError());
}

int launch_check(const CheckIn &in, void *stream, uint64_t *launches) {
    cudaGetLastError();
    if (in.count <= 0) return 0;
    const int grid = (in.count + 127) / 128;
    k_check<<<grid < 1024 ? grid : 1024, 128, 0, static_cast<cudaStream_t>(stream)>>>(in);
    if (launches) ++*launches;
    return check(cudaGetLastError());
}

}  // namespace oserve_gpu
