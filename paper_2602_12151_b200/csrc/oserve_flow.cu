// oserve_flow.cu — the flow-network formulation of the lower level on sm_100a
// (SURVEY §8 f4):
//
//   K6a k_max_flow        thread per graph: FIFO push-relabel over arbitrary
//                         graphs (flow::max_flow, flowassign.cpp:67-147)
//   K6b k_flow_assign     thread per instance: build_network (:152-199) ->
//                         max_flow -> extract_assignment (:505-519: chain
//                         flows / unit, clamp, warm greedy + exchange)
//   K7  k_simplex         CTA per instance: the dense Bland's-rule simplex of
//                         solve_fractional (:559-645); the pivot column is a
//                         block min-reduction, the ratio test is evaluated in
//                         parallel and resolved in row order by one thread,
//                         the row operations are element-parallel.
//
// Push-relabel is a sequential discipline whose per-edge result depends on
// the queue order, so each graph runs on one thread (the reference's exact
// order); throughput comes from running one graph per plan across the GPU.
// The batch workspaces are interleaved ([i * B + b]) so neighbouring threads
// touch neighbouring words.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "flow_core.hpp"
#include "oserve_internal.h"

namespace oserve_gpu {

namespace {
inline int check(cudaError_t e) { return e == cudaSuccess ? 0 : static_cast<int>(e); }
}  // namespace

// ------------------------------------------------------------------ K6a ---
// Views of graph edges [e0, ...) in the uploaded oserve_flow_edge array.
__device__ __forceinline__ Strided<const int32_t> mf_from(const MaxFlowBatch &b, int64_t e0) {
    return {b.edges32 + 4 * e0, 4};
}
__device__ __forceinline__ Strided<const int32_t> mf_to(const MaxFlowBatch &b, int64_t e0) {
    return {b.edges32 + 4 * e0 + 1, 4};
}
__device__ __forceinline__ Strided<const int64_t> mf_cap(const MaxFlowBatch &b, int64_t e0) {
    return {reinterpret_cast<const int64_t *>(b.edges32) + 2 * e0 + 1, 2};
}

__global__ void __launch_bounds__(128) k_max_flow(MaxFlowBatch b) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= b.count) return;
    const int n = b.num_nodes[g];
    const int64_t e0 = b.edge_off[g], m = b.edge_off[g + 1] - e0;
    const int64_t n0 = b.node_off[g];
    PrGraph pg;
    pg.n = n;
    pg.m = static_cast<int>(m);
    if (b.interleave) {
        const int64_t G = b.count;
        const auto ef = mf_from(b, e0), et = mf_to(b, e0);
        const auto ec = mf_cap(b, e0);
        for (int64_t i = 0; i < m; ++i) {
            b.il_from[i * G + g] = ef[i];
            b.il_to[i * G + g] = et[i];
            b.il_cap[i * G + g] = ec[i];
        }
        pg.from = {b.il_from + g, G};
        pg.to = {b.il_to + g, G};
        pg.cap = {b.il_cap + g, G};
        pg.res = {b.res + g, G};
        pg.arc_to = {b.arc_to + g, G};
        pg.adj = {b.adj + g, G};
        pg.excess = {b.excess + g, G};
        pg.adj_off = {b.adj_off + g, G};
        pg.height = {b.height + g, G};
        pg.cur = {b.cur + g, G};
        pg.fifo = {b.fifo + g, G};
        pg.active = {b.active + g, G};
        if (!pr_build(pg)) {
            b.status[g] = 1;  // negative capacity
            return;
        }
        b.value[g] = pr_run(pg, b.source[g], b.sink[g]);
        for (int64_t i = 0; i < m; ++i) b.flow[e0 + i] = b.il_cap[i * G + g] - b.res[2 * i * G + g];
        b.status[g] = 0;
        return;
    }
    pg.from = mf_from(b, e0);
    pg.to = mf_to(b, e0);
    pg.cap = mf_cap(b, e0);
    pg.res = {b.res + 2 * e0, 1};
    pg.arc_to = {b.arc_to + 2 * e0, 1};
    pg.adj = {b.adj + 2 * e0, 1};
    pg.excess = {b.excess + n0, 1};
    pg.adj_off = {b.adj_off + n0 + g, 1};
    pg.height = {b.height + n0, 1};
    pg.cur = {b.cur + n0, 1};
    pg.fifo = {b.fifo + n0, 1};
    pg.active = {b.active + n0, 1};
    if (!pr_build(pg)) {
        b.status[g] = 1;  // negative capacity
        return;
    }
    b.value[g] = pr_run(pg, b.source[g], b.sink[g]);
    for (int64_t i = 0; i < m; ++i) b.flow[e0 + i] = pg.cap[i] - pg.res[2 * i];
    b.status[g] = 0;
}

// Shared-memory bytes of one graph's residual workspace (res, excess: 8 B;
// arc_to, adj, adj_off, height, cur, fifo: 4 B; active: 1 B).
__host__ __device__ inline size_t mf_smem_bytes(int n, int m) {
    return (static_cast<size_t>(16) * m + 8 * n + 8 * m + 8 * m + 4 * (n + 1) + 12 * n + n + 15) & ~size_t(15);
}

// K6a with the workspace in shared memory: a warp per graph, lane 0 runs the
// sequential discipline (pr_build / pr_run, stride-1 views into the warp's
// slice), the warp writes the flows.  Every dependent access of the push /
// relabel loop is a shared-memory hit instead of an L2 round trip.
__global__ void __launch_bounds__(256) k_max_flow_smem(MaxFlowBatch b, int per_warp) {
    extern __shared__ __align__(16) unsigned char mf_smem[];
    const int wpb = blockDim.x >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = blockIdx.x * wpb + w;
    if (g >= b.count) return;
    const int n = b.num_nodes[g];
    const int64_t e0 = b.edge_off[g];
    const int m = static_cast<int>(b.edge_off[g + 1] - e0);
    unsigned char *p = mf_smem + static_cast<size_t>(w) * per_warp;
    int64_t *res = reinterpret_cast<int64_t *>(p);
    int64_t *excess = res + 2 * m;
    int32_t *arc_to = reinterpret_cast<int32_t *>(excess + n);
    int32_t *adj = arc_to + 2 * m;
    int32_t *adj_off = adj + 2 * m;
    int32_t *height = adj_off + n + 1;
    int32_t *cur = height + n;
    int32_t *fifo = cur + n;
    uint8_t *active = reinterpret_cast<uint8_t *>(fifo + n);
    int ok = 1;
    if (lane == 0) {
        PrGraph pg;
        pg.n = n;
        pg.m = m;
        pg.from = mf_from(b, e0);
        pg.to = mf_to(b, e0);
        pg.cap = mf_cap(b, e0);
        pg.res = {res, 1};
        pg.excess = {excess, 1};
        pg.arc_to = {arc_to, 1};
        pg.adj = {adj, 1};
        pg.adj_off = {adj_off, 1};
        pg.height = {height, 1};
        pg.cur = {cur, 1};
        pg.fifo = {fifo, 1};
        pg.active = {active, 1};
        ok = pr_build(pg) ? 1 : 0;
        if (ok) b.value[g] = pr_run(pg, b.source[g], b.sink[g]);
        b.status[g] = ok ? 0 : 1;  // 1: negative capacity
    }
    ok = __shfl_sync(0xffffffffu, ok, 0);
    __syncwarp();
    if (ok) {
        const auto ec = mf_cap(b, e0);
        for (int i = lane; i < m; i += 32) b.flow[e0 + i] = ec[i] - res[2 * i];
    }
}

int launch_max_flow(const MaxFlowBatch &b, void *stream, uint64_t *launches) {
    cudaGetLastError();
    if (b.count == 0) return 0;
    const size_t per = mf_smem_bytes(b.n_max, b.m_max);
    if (per <= 48 * 1024) {
        const int wpb = static_cast<int>(std::min<size_t>(8, std::max<size_t>(1, (96 * 1024) / per)));
        const size_t smem = per * wpb;
        if (smem > 48 * 1024 &&  // opt in past the 48 KB default (per device: set on every such launch)
            cudaFuncSetAttribute(k_max_flow_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024) !=
                cudaSuccess)
            return check(cudaGetLastError());
        k_max_flow_smem<<<(b.count + wpb - 1) / wpb, 32 * wpb, smem, static_cast<cudaStream_t>(stream)>>>(
            b, static_cast<int>(per));
    } else {
        k_max_flow<<<(b.count + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(b);
    }
    if (launches) ++*launches;
    return check(cudaGetLastError());
}

// ------------------------------------------------------------------ K6b ---
// One instance: workspace element q at base[q * B] (B = the batch size for
// the interleaved HBM workspace, 1 for a shared-memory slice).
__device__ void flow_assign_one(const ShapeTables &t, const FlowAssignBatch &b, int i, int32_t *ws32, int64_t *ws64,
                                uint8_t *ws8, int64_t B, int64_t *xw = nullptr) {
    const int R = b.R, J = b.J;
    const int n = net_nodes(R, J), m = net_edges(R, J);
    const int64_t row0 = static_cast<int64_t>(i) * R;
    NetInstance in;
    in.R = R;
    in.J = J;
    in.n = {t.n + row0 * J, 1};
    in.e = {t.e + row0 * J, 1};
    in.unit = {t.unit + row0 * J, 1};
    in.M = {t.M + row0, 1};
    in.lambda = {b.lambda + static_cast<int64_t>(i) * J, 1};
    // interleaved workspace: element q of instance i at [q * B + i]
    int32_t *from = ws32;
    int32_t *to = from + static_cast<int64_t>(m) * B;
    int32_t *arc_to = to + static_cast<int64_t>(m) * B;
    int32_t *adj = arc_to + static_cast<int64_t>(2 * m) * B;
    int32_t *adj_off = adj + static_cast<int64_t>(2 * m) * B;
    int32_t *height = adj_off + static_cast<int64_t>(n + 1) * B;
    int32_t *cur = height + static_cast<int64_t>(n) * B;
    int32_t *fifo = cur + static_cast<int64_t>(n) * B;
    int64_t *cap = ws64;
    int64_t *res = cap + static_cast<int64_t>(m) * B;
    int64_t *excess = res + static_cast<int64_t>(2 * m) * B;
    int64_t *mrem = excess + static_cast<int64_t>(n) * B;
    uint8_t *active = ws8;
    int64_t *const xout = b.x + static_cast<int64_t>(i) * R * J;
    int64_t *x = xw ? xw : xout;  // xw: a shared-memory working copy
    if (b.flow_in) {  // extract_assignment of a given flow
        const int64_t *fl = b.flow_in + static_cast<int64_t>(i) * m;
        for (int k = 0; k < R; ++k) {
            for (int j = 0; j < J; ++j) {
                const int64_t u = t.unit[(row0 + k) * J + j];
                const int64_t v = u > 0 ? fl[J + 2 * (k * J + j) + 1] / u : 0;
                const int64_t c = t.cap[(row0 + k) * J + j];
                x[k * J + j] = v < c ? v : c;
            }
        }
    } else {
        net_build(in, {from, B}, {to, B}, {cap, B});
        PrGraph pg;
        pg.n = n;
        pg.m = m;
        pg.from = {from, B};
        pg.to = {to, B};
        pg.cap = {cap, B};
        pg.res = {res, B};
        pg.excess = {excess, B};
        pg.arc_to = {arc_to, B};
        pg.adj_off = {adj_off, B};
        pg.adj = {adj, B};
        pg.height = {height, B};
        pg.cur = {cur, B};
        pg.fifo = {fifo, B};
        pg.active = {active, B};
        if (!pr_build(pg)) {
            b.status[i] = 1;
            return;
        }
        b.value[i] = pr_run(pg, 0, n - 1);
        if (b.edge_flow) {
            for (int q = 0; q < m; ++q) b.edge_flow[static_cast<int64_t>(i) * m + q] = cap[q * B] - res[2 * q * B];
        }
        // extract_assignment: x0 = chain flow / unit, clamped into the instance cap
        for (int k = 0; k < R; ++k) {
            for (int j = 0; j < J; ++j) {
                const int64_t u = t.unit[(row0 + k) * J + j];
                int64_t v = 0;
                if (u > 0) {
                    const int q = J + 2 * (k * J + j) + 1;  // edge_i_c(k, j)
                    v = (cap[static_cast<int64_t>(q) * B] - res[static_cast<int64_t>(2 * q) * B]) / u;
                }
                const int64_t c = t.cap[(row0 + k) * J + j];
                x[k * J + j] = v < c ? v : c;
            }
        }
    }
    WarmInstance w;
    w.R = R;
    w.J = J;
    w.unit = in.unit;
    w.M = in.M;
    w.lambda = in.lambda;
    w.cap = {t.cap + row0 * J, 1};
    w.order = {t.order + row0 * kMaxJ, 1};
    w.olen = {t.olen + row0, 1};
    w.x = {x, 1};
    w.mrem = {mrem, B};
    b.objective[i] = warm_solve(w);
    if (x != xout)
        for (int c = 0; c < R * J; ++c) xout[c] = x[c];
    b.status[i] = 0;
}

__global__ void __launch_bounds__(128) k_flow_assign(ShapeTables t, FlowAssignBatch b) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= b.count) return;
    flow_assign_one(t, b, i, b.ws_i32 + i, b.ws_i64 + i, b.ws_u8 + i, b.count);
}

// Workspace bytes of one instance in shared memory (i64 block first).
__host__ __device__ inline size_t fa_smem_bytes(int R, int J) {
    size_t i32, i64, u8;
    const int64_t n = net_nodes(R, J), m = net_edges(R, J);
    i32 = static_cast<size_t>(6 * m + (n + 1) + 3 * n);
    i64 = static_cast<size_t>(3 * m + n + R + R * J);  // + the x working copy
    u8 = static_cast<size_t>(n);
    return (8 * i64 + 4 * i32 + u8 + 15) & ~size_t(15);
}

// K6b with the instance's workspace in shared memory: a warp per instance,
// lane 0 runs it (the dependent loads of push-relabel and the warm start hit
// shared memory instead of L2).
__global__ void __launch_bounds__(256) k_flow_assign_smem(ShapeTables t, FlowAssignBatch b, int per_warp) {
    extern __shared__ __align__(16) unsigned char fa_smem[];
    const int wpb = blockDim.x >> 5, w = threadIdx.x >> 5;
    const int i = blockIdx.x * wpb + w;
    if (i >= b.count || (threadIdx.x & 31) != 0) return;
    const int64_t n = net_nodes(b.R, b.J), m = net_edges(b.R, b.J);
    unsigned char *p = fa_smem + static_cast<size_t>(w) * per_warp;
    int64_t *ws64 = reinterpret_cast<int64_t *>(p);
    int64_t *xw = ws64 + (3 * m + n + b.R);
    int32_t *ws32 = reinterpret_cast<int32_t *>(xw + b.R * b.J);
    uint8_t *ws8 = reinterpret_cast<uint8_t *>(ws32 + (6 * m + (n + 1) + 3 * n));
    flow_assign_one(t, b, i, ws32, ws64, ws8, 1, xw);
}

int launch_flow_assign(const ShapeTables &t, const FlowAssignBatch &b, void *stream, uint64_t *launches) {
    cudaGetLastError();
    if (b.count == 0) return 0;
    const size_t per = fa_smem_bytes(b.R, b.J);
    if (per <= 48 * 1024) {
        const int wpb = static_cast<int>(std::min<size_t>(8, std::max<size_t>(1, (96 * 1024) / per)));
        const size_t smem = per * wpb;
        if (smem > 48 * 1024 &&
            cudaFuncSetAttribute(k_flow_assign_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024) !=
                cudaSuccess)
            return check(cudaGetLastError());
        k_flow_assign_smem<<<(b.count + wpb - 1) / wpb, 32 * wpb, smem, static_cast<cudaStream_t>(stream)>>>(
            t, b, static_cast<int>(per));
    } else {
        k_flow_assign<<<(b.count + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(t, b);
    }
    if (launches) ++*launches;
    return check(cudaGetLastError());
}

void flow_assign_workspace(int R, int J, int64_t count, size_t *i32, size_t *i64, size_t *u8) {
    const int64_t n = net_nodes(R, J), m = net_edges(R, J);
    *i32 = static_cast<size_t>((2 * m + 2 * m + 2 * m + (n + 1) + 3 * n) * count);
    *i64 = static_cast<size_t>((m + 2 * m + n + R) * count);
    *u8 = static_cast<size_t>(n * count);
}

// ------------------------------------------------------------------- K7 ---
// Tableau row r, column c of instance i at tab[i * rows * cols + r * cols + c].
// SMEM: the whole tableau lives in shared memory (small instances; else in
// the instance's HBM slab).
template <bool SMEM>
__global__ void __launch_bounds__(512) k_simplex(LpBatch b) {
    extern __shared__ double sm[];
    const int i = blockIdx.x;
    const int R = b.R, J = b.J;
    const int nvars = R * J, nrows = nvars + J + R, ncols = nvars + nrows + 1;
    const double eps = 1e-9;
    double *t = SMEM ? sm + 2 * nrows + 1 : b.tab + static_cast<int64_t>(i) * (nrows + 1) * ncols;
    double *fcol = sm;                                           // [nrows + 1]
    double *ratio = fcol + (nrows + 1);                          // [nrows]
    int *basis = reinterpret_cast<int *>(SMEM ? t + static_cast<int64_t>(nrows + 1) * ncols : ratio + nrows);  // [nrows]
    int *misc = basis + nrows;                                   // [4]
    const int64_t *n = b.n + static_cast<int64_t>(i) * nvars;
    const int64_t *e = b.e + static_cast<int64_t>(i) * nvars;
    const int64_t *lam = b.lambda + static_cast<int64_t>(i) * J;
    const int64_t total = static_cast<int64_t>(nrows + 1) * ncols;
    for (int64_t q = threadIdx.x; q < total; q += blockDim.x) t[q] = 0.0;
    __syncthreads();
    // rows: C2 bounds (R*J), C1 (J), C3 (R); slack identity; objective -1
    for (int r = threadIdx.x; r < nrows; r += blockDim.x) {
        double *row = t + static_cast<int64_t>(r) * ncols;
        if (r < nvars) {
            row[r] = 1.0;
            const int64_t ev = e[r] > 0 ? e[r] : 0;
            row[ncols - 1] = n[r] <= 0 ? 0.0 : static_cast<double>(ev);
        } else if (r < nvars + J) {
            const int j = r - nvars;
            for (int k = 0; k < R; ++k) row[k * J + j] = 1.0;
            row[ncols - 1] = static_cast<double>(lam[j]);
        } else {
            const int k = r - nvars - J;
            for (int j = 0; j < J; ++j)
                if (n[k * J + j] > 0) row[k * J + j] = 1.0 / static_cast<double>(n[k * J + j]);
            row[ncols - 1] = 1.0;
        }
        row[nvars + r] = 1.0;
        basis[r] = nvars + r;
    }
    for (int v = threadIdx.x; v < nvars; v += blockDim.x) t[static_cast<int64_t>(nrows) * ncols + v] = -1.0;
    __syncthreads();
    const double *obj = t + static_cast<int64_t>(nrows) * ncols;
    int status = 0;
    for (int iter = 0; iter < 100000; ++iter) {
        // Bland: the first column with a negative reduced cost
        if (threadIdx.x == 0) misc[0] = 0x7fffffff;
        __syncthreads();
        for (int c = threadIdx.x; c < ncols - 1; c += blockDim.x) {
            if (obj[c] < -eps) {
                atomicMin(&misc[0], c);
                break;
            }
        }
        __syncthreads();
        const int pc = misc[0];
        if (pc == 0x7fffffff) break;
        // ratio test: candidates in parallel, the tie rule in row order
        for (int r = threadIdx.x; r < nrows; r += blockDim.x) {
            const double a = t[static_cast<int64_t>(r) * ncols + pc];
            ratio[r] = a > eps ? __ddiv_rn(t[static_cast<int64_t>(r) * ncols + ncols - 1], a) : -1.0;
            fcol[r] = a;
        }
        if (threadIdx.x == 0) fcol[nrows] = obj[pc];
        __syncthreads();
        if (threadIdx.x == 0) {
            int pr = -1;
            double best = 0.0;
            for (int r = 0; r < nrows; ++r) {
                if (!(fcol[r] > eps)) continue;
                const double q = ratio[r];
                if (pr < 0 || q < best - eps || (q < best + eps && basis[r] < basis[pr])) {
                    pr = r;
                    best = q;
                }
            }
            misc[1] = pr;
        }
        __syncthreads();
        const int pr = misc[1];
        if (pr < 0) {
            status = 1;  // unbounded (malformed instance)
            break;
        }
        double *prow = t + static_cast<int64_t>(pr) * ncols;
        const double p = fcol[pr];
        for (int c = threadIdx.x; c < ncols; c += blockDim.x) prow[c] = __ddiv_rn(prow[c], p);
        __syncthreads();
        // eliminate: t[r][c] -= f_r * t[pr][c], f_r read before the row changes
        // (warp per row, lanes over the columns)
        {
            const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
            for (int r = warp; r <= nrows; r += nw) {
                if (r == pr) continue;
                const double f = fcol[r];
                if (fabs(f) < eps) continue;
                double *row = t + static_cast<int64_t>(r) * ncols;
                for (int c = lane; c < ncols; c += 32) row[c] = __dsub_rn(row[c], __dmul_rn(f, prow[c]));
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) basis[pr] = pc;
        __syncthreads();
    }
    double *f = b.f + static_cast<int64_t>(i) * nvars;
    for (int v = threadIdx.x; v < nvars; v += blockDim.x) f[v] = 0.0;
    __syncthreads();
    for (int r = threadIdx.x; r < nrows; r += blockDim.x) {
        if (basis[r] < nvars) {
            const double v = t[static_cast<int64_t>(r) * ncols + ncols - 1];
            f[basis[r]] = v > 0.0 ? v : 0.0;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int v = 0; v < nvars; ++v) s = __dadd_rn(s, f[v]);
        b.objective[i] = s;
        b.status[i] = status;
    }
}

size_t simplex_tableau_doubles(int R, int J) {
    const size_t nvars = static_cast<size_t>(R) * J, nrows = nvars + J + R, ncols = nvars + nrows + 1;
    return (nrows + 1) * ncols;
}

int launch_simplex(const LpBatch &b, void *stream, uint64_t *launches) {
    cudaGetLastError();
    if (b.count == 0) return 0;
    const int nvars = b.R * b.J, nrows = nvars + b.J + b.R, ncols = nvars + nrows + 1;
    const size_t small = sizeof(double) * (2 * nrows + 1) + sizeof(int) * (nrows + 4);
    const size_t whole = sizeof(double) * (2 * nrows + 1 + static_cast<size_t>(nrows + 1) * ncols) +
                         sizeof(int) * (nrows + 4);
    const bool in_smem = whole <= 96 * 1024;  // two instances per SM at least
    const size_t smem = in_smem ? whole : small;
    auto kern = in_smem ? k_simplex<true> : k_simplex<false>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return check(e);
    }
    kern<<<b.count, in_smem ? 256 : 512, smem, static_cast<cudaStream_t>(stream)>>>(b);
    if (launches) ++*launches;
    return check(cudaGetLastError());
}

}  // namespace oserve_gpu
