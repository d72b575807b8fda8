// flow_core.hpp — per-instance sequential cores of the flow-network path
// (flowassign.cpp:67-245, 377-448, 505-519), run one GPU thread per graph by
// K6 (oserve_flow.cu).  Every array is addressed through a stride so a batch
// of equal-shape instances can be laid out interleaved ([i * B + b]: the B
// threads of a launch touch consecutive words) while ragged batches use
// per-graph packed storage (stride 1).
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define OSERVE_HD __host__ __device__ __forceinline__
#else
#define OSERVE_HD inline
#endif

namespace oserve_gpu {

template <class T>
struct Strided {
    T *p;
    int64_t s;
    OSERVE_HD T &operator[](int64_t i) const { return p[i * s]; }
};

// Residual graph workspace of one max-flow instance.  Arc 2i is edge i
// forward, arc 2i+1 its reverse (flowassign.cpp:75-88).
struct PrGraph {
    int n, m;
    Strided<const int32_t> from, to;
    Strided<const int64_t> cap;
    Strided<int64_t> res, excess;
    Strided<int32_t> arc_to, adj_off, adj, height, cur, fifo;
    Strided<uint8_t> active;
};

// Adjacency in the reference's push_back order: node u lists its arcs by
// ascending arc id (edge i contributes 2i to `from`, then 2i+1 to `to`).
// Returns false on a negative capacity (max_flow throws invalid_argument).
OSERVE_HD bool pr_build(const PrGraph &g) {
    for (int u = 0; u <= g.n; ++u) g.adj_off[u] = 0;
    for (int i = 0; i < g.m; ++i) {
        if (g.cap[i] < 0) return false;
        g.adj_off[g.from[i] + 1] += 1;
        g.adj_off[g.to[i] + 1] += 1;
    }
    for (int u = 0; u < g.n; ++u) g.adj_off[u + 1] += g.adj_off[u];
    for (int u = 0; u < g.n; ++u) g.cur[u] = g.adj_off[u];
    for (int i = 0; i < g.m; ++i) {
        const int a = g.from[i], b = g.to[i];
        g.adj[g.cur[a]] = 2 * i;
        g.cur[a] += 1;
        g.adj[g.cur[b]] = 2 * i + 1;
        g.cur[b] += 1;
        g.res[2 * i] = g.cap[i];
        g.res[2 * i + 1] = 0;
        g.arc_to[2 * i] = b;
        g.arc_to[2 * i + 1] = a;
    }
    for (int u = 0; u < g.n; ++u) {
        g.cur[u] = 0;
        g.height[u] = 0;
        g.excess[u] = 0;
        g.active[u] = 0;
    }
    return true;
}

// FIFO push-relabel (flowassign.cpp:67-147): same queue discipline, arc scan
// order and relabel rule, so the per-edge flows — not only the value — are
// the reference's.  Returns the flow value (excess at the sink).
OSERVE_HD int64_t pr_run(const PrGraph &g, int source, int sink) {
    int head = 0, size = 0;
    const int qn = g.n;
    auto enqueue = [&](int u) {
        if (!g.active[u] && g.excess[u] > 0 && u != source && u != sink) {
            g.active[u] = 1;
            int tail = head + size;
            if (tail >= qn) tail -= qn;
            g.fifo[tail] = u;
            ++size;
        }
    };
    g.height[source] = g.n;
    for (int p = g.adj_off[source]; p < g.adj_off[source + 1]; ++p) {
        const int a = g.adj[p];
        if ((a & 1) != 0 || g.res[a] == 0) continue;
        const int64_t d = g.res[a];
        g.res[a] -= d;
        g.res[a ^ 1] += d;
        g.excess[g.arc_to[a]] += d;
        g.excess[source] -= d;
        enqueue(g.arc_to[a]);
    }
    while (size > 0) {
        const int u = g.fifo[head];
        head = head + 1 == qn ? 0 : head + 1;
        --size;
        g.active[u] = 0;
        const int base = g.adj_off[u], deg = g.adj_off[u + 1] - base;
        while (g.excess[u] > 0) {
            int c = g.cur[u];
            if (c == deg) {
                int h = 0x7fffffff;
                for (int p = 0; p < deg; ++p) {
                    const int a = g.adj[base + p];
                    if (g.res[a] > 0) {
                        const int hv = g.height[g.arc_to[a]] + 1;
                        h = hv < h ? hv : h;
                    }
                }
                g.height[u] = h;
                g.cur[u] = 0;
            } else {
                const int a = g.adj[base + c];
                const int v = g.arc_to[a];
                if (g.res[a] > 0 && g.height[u] == g.height[v] + 1) {
                    const int64_t ex = g.excess[u], ra = g.res[a];
                    const int64_t d = ex < ra ? ex : ra;
                    g.res[a] -= d;
                    g.res[a ^ 1] += d;
                    g.excess[u] -= d;
                    g.excess[v] += d;
                    enqueue(v);
                } else {
                    g.cur[u] = c + 1;
                }
            }
        }
    }
    return g.excess[sink];
}

// The four-edge-class network (flowassign.cpp:152-199) of one normalised
// instance: S->w_j (lambda), w_j->i_kj and i_kj->c_k^in (e*unit, or M when
// it would exceed M), c_k^in->c_k^out (M), c_k^out->T (M*J, saturating).
// Node and edge numbering are FlowNetwork's (flowassign.hpp:52-79).
struct NetInstance {
    int R, J;
    Strided<const int64_t> n, e, unit;  // [k*J + j]
    Strided<const int64_t> M;           // [k]
    Strided<const int64_t> lambda;      // [j]
};

OSERVE_HD int net_nodes(int R, int J) { return 2 + J + R * J + 2 * R; }
OSERVE_HD int net_edges(int R, int J) { return J + 2 * R * J + 2 * R; }

OSERVE_HD void net_build(const NetInstance &in, Strided<int32_t> from, Strided<int32_t> to, Strided<int64_t> cap) {
    const int R = in.R, J = in.J;
    const int S = 0, T = 1 + J + R * J + 2 * R;
    int ei = 0;
    for (int j = 0; j < J; ++j, ++ei) {
        from[ei] = S;
        to[ei] = 1 + j;
        cap[ei] = in.lambda[j];
    }
    for (int k = 0; k < R; ++k) {
        for (int j = 0; j < J; ++j) {
            int64_t c = 0;
            const int64_t u = in.unit[k * J + j];
            if (u > 0) {
                const int64_t ekj = in.e[k * J + j] < in.n[k * J + j] ? in.e[k * J + j] : in.n[k * J + j];
                c = ekj > in.M[k] / u ? in.M[k] : ekj * u;
            }
            const int node_i = 1 + J + k * J + j;
            from[ei] = 1 + j;
            to[ei] = node_i;
            cap[ei] = c;
            ++ei;
            from[ei] = node_i;
            to[ei] = 1 + J + R * J + k;
            cap[ei] = c;
            ++ei;
        }
    }
    for (int k = 0; k < R; ++k, ++ei) {
        from[ei] = 1 + J + R * J + k;
        to[ei] = 1 + J + R * J + R + k;
        cap[ei] = in.M[k];
    }
    for (int k = 0; k < R; ++k, ++ei) {
        int64_t c = in.M[k];
        const int64_t jj = J > 1 ? J : 1;
        c = c > INT64_MAX / jj ? INT64_MAX : c * jj;
        from[ei] = 1 + J + R * J + R + k;
        to[ei] = T;
        cap[ei] = c;
    }
}

// from_matrix + greedy_fill + exchange_improve (flowassign.cpp:377-448)
// from a warm start x (in/out), over the instance of make_instance
// (:267-294): cap [k*J+j], order/olen per replica.  Returns the count.
struct WarmInstance {
    int R, J;
    Strided<const int64_t> unit, M, lambda;
    Strided<const int32_t> cap;    // make_instance cap (ShapeTables::cap)
    Strided<const uint8_t> order;  // [k*16 + i]
    Strided<const uint8_t> olen;   // [k]
    Strided<int64_t> x;            // [k*J + j]
    Strided<int64_t> mrem;         // [k] scratch
};

OSERVE_HD int64_t warm_solve(const WarmInstance &w) {
    const int R = w.R, J = w.J;
    int64_t lam[16];
    int64_t count = 0;
    for (int j = 0; j < J; ++j) lam[j] = w.lambda[j];
    for (int k = 0; k < R; ++k) {
        int64_t mr = w.M[k];
        for (int j = 0; j < J; ++j) {
            const int64_t v = w.x[k * J + j];
            lam[j] -= v;
            mr -= v * w.unit[k * J + j];
            count += v;
        }
        w.mrem[k] = mr;
    }
    for (int k = 0; k < R; ++k) {  // greedy_fill
        const int ol = w.olen[k];
        for (int i = 0; i < ol; ++i) {
            const int j = w.order[k * 16 + i];
            const int64_t u = w.unit[k * J + j];
            int64_t take = w.cap[k * J + j] - w.x[k * J + j];
            if (lam[j] < take) take = lam[j];
            const int64_t q = w.mrem[k] / u;
            if (q < take) take = q;
            if (take > 0) {
                w.x[k * J + j] += take;
                lam[j] -= take;
                w.mrem[k] -= take * u;
                count += take;
            }
        }
    }
    bool improved = true;  // exchange_improve: first improving move, restart
    while (improved) {
        improved = false;
        for (int j = 0; j < J && !improved; ++j) {
            if (lam[j] <= 0) continue;
            for (int k = 0; k < R && !improved; ++k) {
                const int64_t ukj = w.unit[k * J + j];
                if (ukj <= 0 || w.x[k * J + j] >= w.cap[k * J + j]) continue;
                if (w.mrem[k] >= ukj) {
                    w.x[k * J + j] += 1;
                    lam[j] -= 1;
                    w.mrem[k] -= ukj;
                    count += 1;
                    improved = true;
                    break;
                }
                for (int j2 = 0; j2 < J && !improved; ++j2) {
                    if (j2 == j || w.x[k * J + j2] <= 0) continue;
                    const int64_t ukj2 = w.unit[k * J + j2];
                    if (w.mrem[k] + ukj2 < ukj) continue;
                    for (int k2 = 0; k2 < R && !improved; ++k2) {
                        const int64_t u2 = w.unit[k2 * J + j2];
                        if (k2 == k || u2 <= 0) continue;
                        if (w.x[k2 * J + j2] >= w.cap[k2 * J + j2]) continue;
                        if (w.mrem[k2] < u2) continue;
                        w.x[k * J + j2] -= 1;
                        w.mrem[k] += ukj2;
                        w.x[k2 * J + j2] += 1;
                        w.mrem[k2] -= u2;
                        w.x[k * J + j] += 1;
                        w.mrem[k] -= ukj;
                        lam[j] -= 1;
                        count += 1;
                        improved = true;
                    }
                }
            }
        }
    }
    return count;
}

}  // namespace oserve_gpu
