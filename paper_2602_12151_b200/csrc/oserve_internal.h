// oserve_internal.h — device-side table layouts shared by the host runtime
// (oserve_host.cpp) and the sm_100a kernels (oserve_kernels.cu).
//
// HBM layout (all SoA, one copy per context):
//   shape tables   one "shape" = a replica cost row keyed by (tp, pp, sum of
//                  device memory); K0 fills n/e/latency per (shape, class),
//                  then the LCM normalisation M, unit, cap and the
//                  ascending-unit class order per shape.
//   space tables   partitions (plan-count prefix, R, replica/run offsets),
//                  per-replica candidate-list ids, per-run (start, len, q,
//                  count, radix weight), candidate lists of shape ids.
// K1 stages the shape tables into shared memory once per CTA.
#pragma once

#include <cstdint>

namespace oserve_gpu {

constexpr int kMaxJ = 16;       // classes (OSERVE_MAX_CLASSES)
constexpr int kMaxCand = 8;     // (tp, pp) candidates per replica block
constexpr int kMaxExactCells = 64;
constexpr uint64_t kNoKey = ~0ull;
constexpr int kTopK = 64;  // per-group candidate list of the top-K round

// Per-shape inputs of the cost kernel (K0).
struct ShapeParam {
    int tp;
    int pp;
    uint64_t kv_budget;  // sum(device_mem) - param_bytes, clamped at 0 (costmodel.cpp:64-68)
    double speedup;      // tp * eff^log2(tp) (costmodel.cpp:22-24), host libm
};

// Device views of the shape tables.  Row s, class j at [s * J + j].
struct ShapeTables {
    int num_shapes;
    int J;
    const ShapeParam *param;
    int64_t *n;
    int64_t *e;
    double *latency;
    int64_t *M;       // [S]
    int64_t *unit;    // [S*J]
    double *inv_unit; // [S*J] 1/unit (division-free quotient estimate, corrected exactly)
    int32_t *cap;     // [S*J] min(e, n, M/unit), clamped to INT32_MAX (exact while lambda < 2^31)
    uint8_t *order;   // [S*kMaxJ] classes with cap > 0, stable-sorted by unit
    uint8_t *rank;    // [S*kMaxJ] position of class j in order (0xff: not in order)
    uint16_t *pmask;  // [S*kMaxJ] class mask of order positions 0..p (units ascend along the order)
    uint8_t *olen;    // [S]
    uint8_t *pp;      // [S]
    uint8_t *scaled;  // [S] LCM fallback used
};

// Device views of a prepared plan space.
struct SpaceTables {
    int64_t num_parts;
    const uint64_t *prefix;    // [P+1] plans before partition p
    const int32_t *R;          // [P]
    const int32_t *rep_off;    // [P] into rep_list
    const int32_t *run_off;    // [P] into run arrays
    const int32_t *nruns;      // [P]
    const uint8_t *exact;      // [P] plans of this partition take the exact (B&B) path
    const int32_t *rep_list;   // [sum R] candidate-list id per replica
    const int32_t *run_start;  // [sum runs]
    const int32_t *run_len;
    const int32_t *run_q;
    const uint64_t *run_count;
    const uint64_t *run_weight;  // product of later runs' counts (mixed radix)
    const uint8_t *cl_n;         // [L] candidates per list
    const uint16_t *cl_shape;    // [L*kMaxCand] shape ids, tp-descending
};

// Packed selection key: (OBJMAX - obj, partition, sum_pp, local rank).
struct KeyLayout {
    int sh_obj, sh_part, sh_spp;
    uint64_t obj_max;
};

// Which plans a K1/K4 launch evaluates.
struct PlanSource {
    int mode;  // 0: space ranks of this shard; 1: explicit rank list; 2: explicit shape lists
    // mode 0: local index i -> global rank via interleaved chunks
    uint64_t count;       // plans in this launch
    uint64_t first;       // first local index (mode 0) / first list entry
    int rank, world;      // shard
    uint64_t chunk;       // shard interleave chunk
    const uint64_t *ranks;  // mode 1
    // mode 2: plan i has R = list_R[i] shapes at list_shapes[list_off[i] ...]
    const int32_t *list_R;
    const int32_t *list_off;
    const int32_t *list_shapes;
    const int64_t *list_lambda;  // optional per-plan lambda [count*J] (solve_batch)
    // mode 3: bucket of rank ranges; bucket index b -> global rank
    //   range r = last with range_prefix[r] <= b, rank = range_start[r] + (b - range_prefix[r])
    const uint64_t *range_start;
    const uint64_t *range_prefix;
    int num_ranges;
};

// Optional per-plan outputs.
struct PlanOutputs {
    int64_t *objective;   // [count] or null
    int32_t *sum_pp;      // [count] or null
    int64_t *x;           // [count * rmax * J] (mode 2 detail) or null
    int64_t *used;        // [count * rmax] or null
    int rmax;             // row stride for x/used
    uint64_t *best_key;   // argmin target (atomicMin) or null
    uint64_t *aborted;    // [count] ranks whose B&B blew the budget (K4) or null
    unsigned int *aborted_n;
    // top-K round: per-group best-kTopK key lists + the worst kept key of
    // groups that dropped any key (kNoKey otherwise)
    uint64_t *topk;       // [groups * kTopK] or null
    uint64_t *topk_meta;  // [groups]
    // threshold collect (exact fallback): every key <= collect_thr appended
    uint64_t *collect;
    unsigned int *collect_n;
    unsigned int collect_cap;
    uint64_t collect_thr;
};

// Frontier-parallel exact path (see k_exact_plan in oserve_kernels.cu).  The
// B&B tree of each plan is cut after its first `depth` branching decisions;
// every frontier node is a task.
constexpr int kTaskDepthMax = 24;  // initial cut <= 6; phase-A splitting goes deeper
struct ExactTasks {
    // per plan (src index)
    int32_t *depth;       // chosen cut depth; -1: not an exact-path plan
    uint64_t *ntask;      // tasks of the plan (pass 0)
    uint64_t *toff;       // first task of the plan (host exclusive scan)
    int64_t *top_nodes;   // visited nodes above the cut (pass 2)
    int64_t *opt;         // optimum (pass 2)
    int64_t *istar;       // task holding the first optimal leaf (pass 2)
    uint8_t *state;       // 0 not exact, 1 frontier, 2 sequential fallback, 3 frontier + phase-B counts,
                          // 4 abort proven by exact phase-A counts
    unsigned long long *work;  // phase-A nodes run so far, all rounds (pass 0 adds to it)
    int64_t work_limit;   // a plan past it leaves the frontier for the sequential fallback
    unsigned long long *running;  // phase-B running node total (top + finished task nodes)
    int32_t *bx;          // [plans][kMaxExactCells] first optimal leaf
    int64_t phase_cap;    // phase-A node cap of this round (tasks above it are split)
    // per task (preorder within each plan; plans contiguous)
    uint32_t *plan;
    uint8_t *tdepth;      // decisions on the path; bit 7: root is a leaf reached above the cut
    int32_t *path;        // [tasks][kTaskDepthMax]
    int64_t *g;           // greedy-dive leaf count of the task
    int64_t *lb;          // lower bound of the incumbent entering the task (prefix max of g)
    int64_t *lbran;       // the lower bound phase A actually ran the task with
    int64_t *m;           // max(best leaf in the subtree, lb)  (phase A)
    int64_t *inc;         // exact incumbent entering the task (pass 2)
    uint8_t *vis;         // task root visited by the sequential DFS (pass 2)
    int64_t *nodes;       // phase A node count (an upper bound of the sequential count below the task)
    uint8_t *capped;      // phase A exceeded its cap
    uint8_t *done;        // phase A finished (m, nodes valid)
    uint32_t *nchild;     // tasks this one becomes in the next round
    uint8_t *nzero;       // single-branch decisions (v = 0 forced) between the root and the split point
    uint64_t target;      // desired tasks per plan
    uint64_t max_tasks;   // cap per plan
    unsigned long long *fetch;  // task counter of the thread-per-task passes
    // parallel top replay: per task the shared-prefix length and own / ancestor
    // alive bits; per plan the top-node count, phase-A upper bound, capped flag
    int32_t *aL;
    uint32_t *amask;
    unsigned long long *topn, *ubn;
    unsigned long long *lbn;  // per plan: exact counts of visited tasks whose phase-A bound was the exact incumbent
    uint8_t *anycap;
    // device-built frontier: per plan, grow this level / children summed
    uint8_t *grow;
    uint32_t *plan_sum;
};
// Exclusive scan of the tasks' child counts (nchild[n] = 0) and the per-plan
// ranges of the list it describes.
int launch_exact_rescan(const ExactTasks &et, uint64_t n, uint32_t *newoff, uint64_t plans, void **temp,
                        size_t *temp_bytes, void *stream, uint64_t *launches);
int launch_exact_ranges(const ExactTasks &et, const uint32_t *newoff, uint64_t plans, void *stream,
                        uint64_t *launches);
// Ancestor-alive masks of the replay (inclusive scan over the tasks).
int launch_alive_scan(const ExactTasks &et, uint64_t total, uint64_t *tmp, void **temp, size_t *temp_bytes,
                      int sm_count, void *stream, uint64_t *launches);

struct SolveParams {
    int J;
    int64_t lambda[kMaxJ];
    int64_t exact_demand_limit;
    int exact_cell_limit;
    int64_t node_budget;
};

// K1 dynamic-chunk counters: `slots` 128-byte lines of device memory owned by
// one context (one line per launch, round robin, zeroed on the launch stream).
struct WorkRing {
    unsigned long long *base;
    int slots;
    unsigned next;
};

// ---- launchers (oserve_kernels.cu) -----------------------------------------
int launch_cost_tables(const ShapeTables &t, const double *cin, const double *cout, uint32_t num_layers,
                       uint64_t bytes_per_token_kv, double prefill_coeff, double decode_coeff,
                       double pp_comm_cost, double mem_bw_penalty, double span_s, void *stream);
int launch_normalize_rows(const ShapeTables &t, void *stream);
// Greedy + exchange (heuristic path) over a plan source; returns CUDA status.
int launch_plan_eval(const ShapeTables &t, const SpaceTables &sp, const KeyLayout &key, const PlanSource &src,
                     const PlanOutputs &out, const SolveParams &sp_params, int rmax, int sm_count,
                     int skip_exact, WorkRing *ring, void *stream, uint64_t *launches);
// Exact branch-and-bound path (thread per plan).
int launch_plan_exact(const ShapeTables &t, const SpaceTables &sp, const KeyLayout &key, const PlanSource &src,
                      const PlanOutputs &out, const SolveParams &sp_params, int sm_count, void *stream,
                      uint64_t *launches);
// Frontier-parallel exact path: per-plan passes (10 root tasks, 8 certify,
// 3 finish/emit) and per-task passes (9 frontier children, 2 greedy dives,
// 0 phase A subtree maxima, 3 split counts, 6/7 top replay, 1 phase B node
// counts + first optimal leaf).
int launch_exact_plan_pass(int pass, const ShapeTables &t, const SpaceTables &sp, const KeyLayout &key,
                           const PlanSource &src, const PlanOutputs &out, const SolveParams &prm,
                           const ExactTasks &et, int sm_count, void *stream, uint64_t *launches);
int launch_exact_task_pass(int pass, const ShapeTables &t, const SpaceTables &sp, const PlanSource &src,
                           const SolveParams &prm, const ExactTasks &et, uint64_t total_tasks, int sm_count,
                           void *stream, uint64_t *launches);
// Per-plan prefix maxima over the task list as segmented scans: which = 4
// lower bounds (lb, and m of finished tasks), 6 exact incumbents (inc, opt,
// istar; resets the replay's per-plan counters).  tmp: [total] int64.
// Plans whose phase-A node total passed et.work_limit -> state 2 (sequential).
int launch_exact_retire(const ExactTasks &et, uint64_t plans, int sm_count, void *stream, uint64_t *launches);
int launch_exact_prefix(int which, const ExactTasks &et, uint64_t total, uint64_t plans, int64_t *tmp, void **temp,
                        size_t *temp_bytes, int sm_count, void *stream, uint64_t *launches);

// Split capped tasks into their children: `nt` receives the new list at the
// exclusive-scan offsets `newoff` of et.nchild.
int launch_exact_split(const ShapeTables &t, const SpaceTables &sp, const PlanSource &src, const SolveParams &prm,
                       const ExactTasks &et, const ExactTasks &nt, const uint32_t *newoff, uint64_t total_tasks,
                       int sm_count, void *stream, uint64_t *launches);

// Switching cost (K2).
struct SwitchDeps {
    int count;                 // candidate deployments
    int num_devices;           // distinct device slots (cluster size)
    const int32_t *machine;    // [num_devices] machine index per device slot
    const int32_t *dev_id;     // [num_devices] device id per slot (ascending)
    // deployments: dep 0 = source, 1..count = candidates
    const int32_t *dep_rep_off;  // [count+2] replica offset per deployment
    const int32_t *rep_tp;
    const int32_t *rep_pp;
    const int32_t *rep_dev_off;  // [total reps + 1] offset into rep_devs
    const int32_t *rep_devs;     // device slots, ascending per replica
    uint64_t P;
    double intra_bw, inter_bw;
};
struct SwitchOut {
    double *est;            // [count]
    uint64_t *max_bytes;    // [count]
    int32_t *status;        // [count] 0 ok, 1 unsourced fragment
    // detail (count == 1): per (target slot, fragment) chosen source slot or -1
    int32_t *detail_src;    // [num_devices * max_frags] or null
    uint64_t *detail_cuts;  // [max_frags + 1]
    int32_t *detail_ncuts;  // [1]
    int max_frags;
};
int launch_switch_cost(const SwitchDeps &d, const SwitchOut &o, void *stream, uint64_t *launches);
// K2 with candidates decoded on the device from packed keys (canonical blocks
// of a prepared space): est[i] = switching cost src -> plan(keys[i]).
int launch_switch_cost_keys(const SwitchDeps &src, const SpaceTables &sp, const KeyLayout &key, const ShapeTables &t,
                            const uint64_t *keys, int count, const int32_t *part_off, const SwitchOut &o,
                            void *stream, uint64_t *launches);
// kv_plan (K5): one warp, requests in order.
struct KvPlanIn {
    int n;                       // inflight requests
    const int64_t *gen;          // generated tokens
    const uint64_t *kv;          // kv bytes
    const int32_t *srcrep;       // source replica
    int64_t threshold;
    int num_slots;
    int none_slot;               // slot of device id -1 (an empty replica's pick), or -1
    const int32_t *machine;      // [slots]
    const int32_t *dev_id;       // [slots]
    int src_reps, dst_reps;
    int n_src_devs, n_dst_devs;  // lengths of src_devs / dst_devs
    const int32_t *src_off;      // [src_reps+1] into src_devs
    const int32_t *src_devs;     // device slots
    const int32_t *dst_off;
    const int32_t *dst_devs;
    uint64_t *load;              // [slots*slots] link loads (pre-filled with carry)
    uint64_t *inbound;           // [slots] zero
    // outputs
    int32_t *kind;               // [n] 0 drained, 1 migrated
    int32_t *mig_src, *mig_dst;  // [n] device ids
    // target-replica partition (parallel path): the migrated requests of
    // target replica r, in order, are entries grp_off[r] .. grp_off[r+1] of
    // the group-ordered arrays (kv bytes, source replica in; picked source
    // and target device ids out); kind / mig_* / gen are unused then
    const int32_t *grp_off;      // [dst_reps+1] or null (sequential kernel)
    const uint64_t *grp_kv;
    const int32_t *grp_sr;
    int32_t *grp_src, *grp_dst;
    const int32_t *h_dst_off;    // host copy of dst_off (launch geometry)
};
int launch_kv_plan(const KvPlanIn &in, void *stream, uint64_t *launches);

// K6a: max_flow over a ragged batch of graphs (packed per graph).
struct MaxFlowBatch {
    int count;
    const int32_t *num_nodes;  // [count]
    const int64_t *edge_off;   // [count+1]
    const int64_t *node_off;   // [count+1] (adj_off uses node_off[g] + g)
    const int32_t *edges32;    // the caller's oserve_flow_edge array as is (from, to, cap: 4 words per edge)
    const int32_t *source, *sink;
    int64_t *res, *excess;
    int32_t *arc_to, *adj, *adj_off, *height, *cur, *fifo;
    uint8_t *active;
    int64_t *flow, *value;
    int32_t *status;
    // interleaved workspace (graphs of similar size): element q of graph g
    // at [q * count + g], sized for the largest graph (n_max, m_max); the
    // edge lists are copied in (il_from / il_to / il_cap) so every access of
    // a warp's 32 graphs is one coalesced line
    int interleave, n_max, m_max;
    int32_t *il_from, *il_to;
    int64_t *il_cap;
};
int launch_max_flow(const MaxFlowBatch &b, void *stream, uint64_t *launches);

// K6b: build_network + max_flow + extract_assignment over equal-shape
// instances whose rows are already normalised in a ShapeTables (rows i*R+k).
struct FlowAssignBatch {
    int count, R, J;
    const int64_t *lambda;  // [count][J]
    int32_t *ws_i32;
    int64_t *ws_i64;
    uint8_t *ws_u8;
    int64_t *x;             // [count][R][J]
    int64_t *objective, *value;
    int64_t *edge_flow;     // [count][edges] or null
    const int64_t *flow_in; // [count][edges]: given flows (extract_assignment only), or null
    int32_t *status;
};
struct ShapeTables;
int launch_flow_assign(const ShapeTables &t, const FlowAssignBatch &b, void *stream, uint64_t *launches);
void flow_assign_workspace(int R, int J, int64_t count, size_t *i32, size_t *i64, size_t *u8);

// K7: solve_fractional's dense simplex, CTA per instance.
struct LpBatch {
    int count, R, J;
    const int64_t *n, *e, *lambda;
    double *tab;  // [count][(nrows+1)*ncols]
    double *f, *objective;
    int32_t *status;
};
int launch_simplex(const LpBatch &b, void *stream, uint64_t *launches);
size_t simplex_tableau_doubles(int R, int J);

// Reference-signature helpers of the C++ shim (oserve_aux.cu).
// switchplan::layout: shard g of replica r (g - rep_off[r] = stage * tp + slice).
struct LayoutIn {
    int R, total;                 // replicas, shards (sum of tp * pp)
    const int32_t *rep_off;       // [R+1] first shard of each replica
    const int32_t *dev_off;       // [R] first device of each replica in devs_sorted
    const int32_t *tp, *pp;
    const int32_t *devs_sorted;   // device ids, ascending within each replica
    uint64_t P;
    uint64_t *begin, *end;        // [total]
    int32_t *holder;              // [total]
};
int launch_layout(const LayoutIn &in, void *stream, uint64_t *launches);
// switchplan::greedy_plan over two ShardLayouts: per device slot (ascending
// id) its held ranges, CSR.
struct HeldIn {
    int num_devices;
    const int32_t *machine;               // [slots] machine index or -1
    const int32_t *src_off, *dst_off;     // [slots+1]
    const uint64_t *src_b, *src_e, *dst_b, *dst_e;
    int nbounds;                          // every begin/end of both layouts (unsorted)
    const uint64_t *bounds;
    double intra_bw, inter_bw;
};
struct HeldOut {
    int32_t *detail;                  // [slots * max_frags] source slot per (target, fragment); -1 none, -2 unsourced
    int max_frags;
    uint64_t *cuts;                   // [nbounds] sorted unique boundaries
    int32_t *ncuts;
    double *est;
    unsigned long long *max_bytes;
};
int launch_switch_held(const HeldIn &in, const HeldOut &o, void *stream, uint64_t *launches);
// switchplan::estimate_time over link loads.
struct LinkIn {
    int n;
    const int32_t *src_machine, *dst_machine;
    const uint64_t *bytes;
    double intra_bw, inter_bw;
};
int launch_link_time(const LinkIn &in, double *est, void *stream, uint64_t *launches);
// flow::check_constraints over `count` instances (normalised rows in t).
struct CheckIn {
    int count, R, J;
    const int64_t *x, *e, *lambda;
    ShapeTables t;
    int32_t *kind, *k, *j;  // 0 ok, 1 C1 (j), 2 C2 (k, j), 3 C3 zero-capacity (k, j), 4 C3 (k)
};
int launch_check(const CheckIn &in, void *stream, uint64_t *launches);

// Sort n u64 keys ascending on the device (CUB radix sort); temp is reused.
int sort_keys(uint64_t *keys, uint64_t *tmp_keys, int n, void **temp, size_t *temp_bytes, void *stream);
// Groups whose list dropped a key better than `kth` (0 => the lists are exact).
int launch_topk_check(const uint64_t *meta, int groups, const uint64_t *kth, unsigned int *bad, void *stream);
int k1_groups(int rmax, int J, int sm_count, const ShapeTables &t, uint64_t count);

}  // namespace oserve_gpu
