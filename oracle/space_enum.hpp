// space_enum.hpp — TEST INFRASTRUCTURE ONLY (shared by the two CPU oracles).
//
// Enumeration of the scheduling round's plan space in the reference's order:
//  * partitions: restates partitions_desc (deploysearch.cpp:421-432) — parts
//    non-increasing, >= g_min, largest first; optionally restricted to an
//    allowed size set (canonical space);
//  * blocks: canonical_blocks (deploysearch.cpp:89-103) — sorted device ids
//    handed out in replica order;
//  * combos: best_strategies' mixed radix (deploysearch.cpp:167-174), replica
//    R-1 least significant, candidates tp-descending (:105-118).
//    Canonical mode keeps only combos whose picks are non-decreasing inside
//    runs of consecutive replicas with equal size and identical candidate
//    lists, ranked in the same (lexicographic) order.
// The candidate function is injected so the reference harness can use the
// reference's own strategy_candidates and the restatement its own.
#pragma once

#include <algorithm>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <utility>
#include <vector>

namespace oracle_space {

using Cands = std::vector<std::pair<int, int>>;  // (tp, pp), tp descending

struct Run {
    int start = 0;
    int len = 0;
    int q = 0;           // candidates per replica in the run
    uint64_t count = 0;  // C(len + q - 1, q - 1)
};

struct Partition {
    std::vector<int> sizes;         // non-increasing
    std::vector<int> offsets;       // first sorted-device index per replica
    std::vector<Cands> cands;       // per replica
    std::vector<Run> runs;
    uint64_t count = 0;             // 0 => infeasible (some block has no candidate)
};

struct Space {
    std::vector<Partition> parts;
    std::vector<uint64_t> prefix;   // prefix[i] = plans before partition i
    uint64_t total = 0;
};

inline uint64_t binom(int n, int k) {
    if (k < 0 || k > n) return 0;
    unsigned __int128 r = 1;
    for (int i = 1; i <= k; ++i) {
        r = r * static_cast<unsigned>(n - k + i) / static_cast<unsigned>(i);
        if (r > (static_cast<unsigned __int128>(1) << 63)) throw std::overflow_error("binomial overflow");
    }
    return static_cast<uint64_t>(r);
}

inline void partitions_desc(int remaining, int max_part, int min_part, const std::vector<char> &allowed,
                            std::vector<int> &cur,
                            const std::function<void(const std::vector<int> &)> &emit) {
    if (remaining == 0) {
        emit(cur);
        return;
    }
    for (int p = std::min(remaining, max_part); p >= min_part; --p) {
        if (!allowed.empty() && !allowed[p]) continue;
        cur.push_back(p);
        partitions_desc(remaining - p, p, min_part, allowed, cur, emit);
        cur.pop_back();
    }
}

// candidates(offset, size) -> tp-descending feasible (tp, pp) list.
inline Space build(int D, int g_min, bool canonical, const std::vector<int> &sizes_allowed,
                   const std::function<Cands(int, int)> &candidates) {
    std::vector<char> allowed;
    if (!sizes_allowed.empty()) {
        allowed.assign(D + 1, 0);
        for (int s : sizes_allowed)
            if (s >= 1 && s <= D) allowed[s] = 1;
    }
    Space sp;
    std::vector<int> cur;
    partitions_desc(D, D, g_min, allowed, cur, [&](const std::vector<int> &sizes) {
        Partition part;
        part.sizes = sizes;
        int off = 0;
        bool feasible = true;
        for (int s : sizes) {
            part.offsets.push_back(off);
            part.cands.push_back(candidates(off, s));
            if (part.cands.back().empty()) feasible = false;
            off += s;
        }
        if (feasible) {
            const int R = static_cast<int>(sizes.size());
            for (int r = 0; r < R;) {
                int e = r + 1;
                if (canonical) {
                    while (e < R && sizes[e] == sizes[r] && part.cands[e] == part.cands[r]) ++e;
                }
                Run run;
                run.start = r;
                run.len = e - r;
                run.q = static_cast<int>(part.cands[r].size());
                run.count = binom(run.len + run.q - 1, run.q - 1);
                part.runs.push_back(run);
                r = e;
            }
            unsigned __int128 c = 1;
            for (const auto &run : part.runs) {
                c *= run.count;
                if (c > (static_cast<unsigned __int128>(1) << 62)) throw std::overflow_error("plan count overflow");
            }
            part.count = static_cast<uint64_t>(c);
        }
        sp.prefix.push_back(sp.total);
        sp.total += part.count;
        sp.parts.push_back(std::move(part));
    });
    return sp;
}

// Unrank a non-decreasing sequence of length len over [0, q) in lex order.
inline void unrank_run(uint64_t r, int len, int q, int *out) {
    int prev = 0;
    for (int pos = 0; pos < len; ++pos) {
        for (int v = prev; v < q; ++v) {
            uint64_t c = binom((len - pos - 1) + (q - v) - 1, (q - v) - 1);
            if (r < c) {
                out[pos] = v;
                prev = v;
                break;
            }
            r -= c;
        }
    }
}

// Global rank -> (partition index, local rank, picks).
inline void unrank(const Space &sp, uint64_t rank, int64_t &p_idx, uint64_t &local, std::vector<int> &picks) {
    auto it = std::upper_bound(sp.prefix.begin(), sp.prefix.end(), rank);
    int64_t p = static_cast<int64_t>(it - sp.prefix.begin()) - 1;
    // Skip empty partitions that share the same prefix value.
    while (sp.parts[p].count == 0 || rank - sp.prefix[p] >= sp.parts[p].count) ++p;
    p_idx = p;
    local = rank - sp.prefix[p];
    const Partition &part = sp.parts[p];
    picks.assign(part.sizes.size(), 0);
    uint64_t r = local;
    for (int i = static_cast<int>(part.runs.size()) - 1; i >= 0; --i) {
        const Run &run = part.runs[i];
        uint64_t rr = r % run.count;
        r /= run.count;
        unrank_run(rr, run.len, run.q, picks.data() + run.start);
    }
}

// Inverse of unrank for a pick vector (used to recover the key of a
// deployment returned by the reference's best_strategies).
inline uint64_t rank_of(const Partition &part, const std::vector<int> &picks) {
    uint64_t r = 0;
    for (const auto &run : part.runs) {
        uint64_t rr = 0;
        int prev = 0;
        for (int pos = 0; pos < run.len; ++pos) {
            int v = picks[run.start + pos];
            for (int u = prev; u < v; ++u) rr += binom((run.len - pos - 1) + (run.q - u) - 1, (run.q - u) - 1);
            prev = v;
        }
        r = r * run.count + rr;
    }
    return r;
}

// Selection key order: objective desc, partition asc, sum_pp asc, rank asc.
struct Best {
    int64_t obj = -1;
    int64_t part = 0;
    int sum_pp = 0;
    uint64_t local = 0;
    bool valid = false;
    bool better(int64_t o, int64_t p, int s, uint64_t l) const {
        if (!valid) return true;
        if (o != obj) return o > obj;
        if (p != part) return p < part;
        if (s != sum_pp) return s < sum_pp;
        return l < local;
    }
    void offer(int64_t o, int64_t p, int s, uint64_t l) {
        if (better(o, p, s, l)) {
            obj = o;
            part = p;
            sum_pp = s;
            local = l;
            valid = true;
        }
    }
};

}  // namespace oracle_space
