/*
 * oserve_gpu.h — C-ABI of the B200-native OServe scheduling round.
 *
 * This is the drop-in boundary between the reference's C++ scheduler
 * (/root/reference/proj, namespace oserve::) and the sm_100a kernels in
 * paper_2602_12151_b200/csrc.  Plain C: POD structs, pointers + sizes,
 * int status codes; no C++ or torch types cross it.
 *
 * Each entry point names the reference interface it replaces.  Results are
 * bit-identical to the reference on the same inputs.
 *
 * Threading: one oserve_gpu_ctx is used by one host thread at a time
 * (the reference functions are reentrant; contexts are independent).
 * All calls are synchronous with respect to the host unless named
 * "_async"; asynchronous calls run on the context's stream.
 */
#ifndef OSERVE_GPU_H
#define OSERVE_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OSERVE_MAX_REPLICAS 128
#define OSERVE_MAX_CLASSES 16
#define OSERVE_MAX_DEVICES 1024

/* Status codes.  Each maps to the exception the reference throws
 * (proj/include/oserve/errors.hpp:9-82, std::invalid_argument, std::logic_error). */
typedef enum {
    OSERVE_OK = 0,
    OSERVE_ERR_INVALID_ARGUMENT = 1,   /* std::invalid_argument                 */
    OSERVE_ERR_INFEASIBLE_REPLICA = 2, /* oserve::InfeasibleReplica  errors.hpp:15 */
    OSERVE_ERR_MODEL_TOO_LARGE = 3,    /* oserve::ModelTooLarge      errors.hpp:21 */
    OSERVE_ERR_TOO_LARGE = 4,          /* oserve::TooLarge           errors.hpp:27 */
    OSERVE_ERR_EMPTY_DEPLOYMENT = 5,   /* oserve::EmptyDeployment    errors.hpp:32 */
    OSERVE_ERR_UNSOURCED_FRAGMENT = 6, /* oserve::UnsourcedFragment  errors.hpp:51 */
    OSERVE_ERR_LOGIC = 7,              /* std::logic_error (check_constraints)    */
    OSERVE_ERR_UNSUPPORTED = 8,        /* input outside the GPU path's limits     */
    OSERVE_ERR_CUDA = 9,
    OSERVE_ERR_NO_DEVICE = 10,
    OSERVE_ERR_NCCL = 11,              /* communicator / collective failure        */
    OSERVE_ERR_LCM_OVERFLOW = 12       /* oserve::LcmOverflow        errors.hpp:39 */
} oserve_status;

/* ---- L0 types (proj/include/oserve/core.hpp:11-95) -------------------- */

/* ClusterSpec (core.hpp:21-34): machines with device ids and per-device
 * memory; two link classes. */
typedef struct {
    int num_machines;
    const int *machine_num_devices; /* [num_machines]                       */
    const int *device_ids;          /* concatenated per machine             */
    const uint64_t *device_mem;     /* [num_machines] bytes per device      */
    double intra_bw;                /* bytes/s within a machine             */
    double inter_bw;                /* bytes/s across machines              */
} oserve_cluster_desc;

/* ModelSpec (core.hpp:36-45). */
typedef struct {
    uint64_t param_bytes;
    uint32_t num_layers;
    uint64_t bytes_per_token_kv;
    uint64_t flops_per_token_prefill;
    uint64_t min_mem_bytes;
} oserve_model_desc;

/* cost::ProfileParams (costmodel.hpp:14-22). */
typedef struct {
    double prefill_coeff;
    double decode_coeff;
    double tp_efficiency;
    double pp_comm_cost;
    double mem_bw_penalty;
} oserve_profile;

/* WorkloadType (core.hpp:73-79). */
typedef struct {
    int type_id;
    double centroid_in;
    double centroid_out;
} oserve_class;

/* flow::SolveOptions (flowassign.hpp:97-101). */
typedef struct {
    int64_t exact_demand_limit; /* default 400       */
    int exact_cell_limit;       /* default 20        */
    int64_t node_budget;        /* default 8'000'000 */
} oserve_solve_options;

/* Deployment (core.hpp:63-70) as flat arrays: replica r owns
 * device_ids[off_r, off_r + replica_num_devices[r]) with its (tp, pp). */
typedef struct {
    int num_replicas;
    const int *replica_num_devices; /* [R] */
    const int *device_ids;          /* concatenated per replica */
    const int *tp;                  /* [R] */
    const int *pp;                  /* [R] */
} oserve_deployment;

/* A deployment returned by the GPU path (fixed-capacity, caller-owned). */
typedef struct {
    int num_replicas;
    int num_devices;
    int replica_num_devices[OSERVE_MAX_REPLICAS];
    int tp[OSERVE_MAX_REPLICAS];
    int pp[OSERVE_MAX_REPLICAS];
    int device_ids[OSERVE_MAX_DEVICES]; /* concatenated per replica */
} oserve_plan;

/* Plan spaces enumerated by a scheduling round.
 *  ORDERED   — the reference's own space: every partition of D into parts
 *              >= g_min in partitions_desc order (deploysearch.cpp:421-432),
 *              every ordered strategy combo of best_strategies
 *              (deploysearch.cpp:153-229).
 *  CANONICAL — symmetry-reduced space: parts restricted to
 *              `sizes`, strategy picks non-decreasing within runs of equal
 *              replicas.  Same order/tie-break restricted to that subset. */
typedef enum { OSERVE_SPACE_ORDERED = 0, OSERVE_SPACE_CANONICAL = 1 } oserve_space_mode;

typedef struct {
    int mode;         /* oserve_space_mode                                   */
    int num_sizes;    /* allowed part sizes (0 => every size >= g_min)       */
    const int *sizes;
    int max_devices;  /* >0: TooLarge when D > max_devices (exhaustive guard) */
} oserve_space_desc;

/* Result of a scheduling round (search::SearchState, deploysearch.hpp:86-92,
 * plus the selection key). */
typedef struct {
    int64_t objective;       /* SearchState::throughput                        */
    uint64_t key;            /* packed (obj desc, partition, sum_pp, rank) key */
    int64_t partitions;      /* SearchState::iterations (partitions visited)   */
    uint64_t plans;          /* plans in the space (evaluated by the kernel)   */
    int64_t partition_index; /* winner's partition in enumeration order        */
    uint64_t local_rank;     /* winner's rank inside its partition             */
    int sum_pp;
    oserve_plan plan;        /* SearchState::deployment                        */
} oserve_round_result;

/* switchplan::Transfer (switchplan.hpp:36-42). */
typedef struct {
    uint64_t begin;
    uint64_t end;
    int src;
    int dst;
} oserve_transfer;

typedef struct oserve_gpu_ctx oserve_gpu_ctx;

/* ---- context ---------------------------------------------------------- */

/* Replaces the EvalContext construction (deploysearch.hpp:45-54): copies the
 * cluster/model/profile (never retains caller pointers) and binds a CUDA
 * device.  Validates like core.cpp:67-96 / costmodel.cpp:13-19. */
int oserve_gpu_create(int cuda_device, const oserve_cluster_desc *cluster,
                      const oserve_model_desc *model, const oserve_profile *profile,
                      oserve_gpu_ctx **out);
int oserve_gpu_destroy(oserve_gpu_ctx *ctx);

/* ---- multi-GPU: the plan space sharded over GPUs ---------- */

/* One context over several local devices (one process): each device
 * evaluates interleaved chunks of the plan order (OSERVE_SHARD_CHUNK) and an
 * NCCL communicator over the devices (ncclCommInitAll) carries the one
 * exchange of the round.  oserve_gpu_round / _exhaustive / _best_strategies /
 * _launch_round_async then all-reduce(MIN) the packed key and
 * oserve_gpu_round_topk all-gathers the per-device top-K lists; spaces of
 * fewer than 65,536 plans (OSERVE_SHARD_MIN) and exact-path spaces run whole
 * on cuda_devices[0].  Every other entry point runs on cuda_devices[0]. */
int oserve_gpu_create_multi(const int *cuda_devices, int ndev, const oserve_cluster_desc *cluster,
                            const oserve_model_desc *model, const oserve_profile *profile, oserve_gpu_ctx **out);
/* One process per GPU: rank 0 makes an id (128 bytes, ncclGetUniqueId) and
 * shares it out of band; every rank joins its single-device context to the
 * world (ncclCommInitRank).  The same entry points then shard over the world
 * and return the global result on every rank. */
int oserve_nccl_unique_id(void *id_128_bytes);
int oserve_gpu_join(oserve_gpu_ctx *ctx, const void *id_128_bytes, int rank, int world);
/* Global rank of the context's first device, world size, local devices. */
int oserve_gpu_world(const oserve_gpu_ctx *ctx, int *rank, int *world, int *local_devices);
const char *oserve_gpu_last_error(const oserve_gpu_ctx *ctx);
const char *oserve_gpu_status_name(int status);

/* Workload of one span: classes (the WorkloadType centroids), per-class
 * demand lambda (TraceSpan::counts) and span length.  Runs the cost-table
 * kernel (K0) on the device. */
int oserve_gpu_set_workload(oserve_gpu_ctx *ctx, int num_classes, const oserve_class *classes,
                            const int64_t *lambda, double span_seconds);
int oserve_gpu_set_solve_options(oserve_gpu_ctx *ctx, const oserve_solve_options *opts);
/* Multi-GPU: this context evaluates only the plans of shard `rank` of
 * `world` (interleaved chunks of the global plan order). */
int oserve_gpu_set_shard(oserve_gpu_ctx *ctx, int rank, int world);
/* Launch stream (cudaStream_t as void*), used exactly (NULL = the legacy
 * default stream).  Until called, the context uses a stream of its own. */
int oserve_gpu_set_stream(oserve_gpu_ctx *ctx, void *stream);
/* search::min_feasible_group (deploysearch.cpp:77-87). */
int oserve_gpu_min_feasible_group(oserve_gpu_ctx *ctx, int *g_min);

/* ---- scheduling round (enumerate -> cost -> assign -> argmin) --------- */

/* Enumerate the space on the host and upload its tables. */
int oserve_gpu_prepare_space(oserve_gpu_ctx *ctx, const oserve_space_desc *space,
                             int64_t *partitions, uint64_t *plans);
/* Asynchronously evaluate this shard's plans of the prepared space and write
 * the shard-best packed key to device memory `d_key` (uint64, caller-owned;
 * may be fed straight into an all-reduce(min)). */
int oserve_gpu_launch_round_async(oserve_gpu_ctx *ctx, uint64_t *d_key);
/* Decode a (global) key into the winning plan. */
int oserve_gpu_decode_key(oserve_gpu_ctx *ctx, uint64_t key, oserve_round_result *out);
/* Synchronous round over a space (single GPU or this shard). */
int oserve_gpu_round(oserve_gpu_ctx *ctx, const oserve_space_desc *space,
                     oserve_round_result *out);

/* Top-K round: the K best plans (packed keys ascending = best first) of this
 * shard of the prepared space, written to device memory d_keys[K] (unused
 * slots UINT64_MAX).  Exact: per-group candidate lists are verified on the
 * device and an exact threshold pass runs if a list could have dropped one of
 * the K best.  Synchronous.  Also writes the single best key to d_best (may
 * be NULL).  Multi-GPU: all-gather the per-rank lists and keep the K smallest. */
int oserve_gpu_round_topk(oserve_gpu_ctx *ctx, int K, uint64_t *d_keys, uint64_t *d_best);
/* Switching cost (layout + greedy_plan + estimate_time, switchplan.cpp:40-140)
 * from `current` to the deployments of `count` packed keys of the prepared
 * space (device memory), decoded on the device: one CTA per pair.  Outputs
 * are host arrays (max_link_bytes may be NULL). */
int oserve_gpu_switch_cost_keys(oserve_gpu_ctx *ctx, const oserve_deployment *current, int count,
                                const uint64_t *d_keys, double *est_seconds, uint64_t *max_link_bytes);

/* Asynchronous variant on the context's stream: est_seconds written to
 * device memory d_est[count] (no host synchronisation), e.g. right after the
 * all-reduce of the round key. */
int oserve_gpu_switch_cost_keys_async(oserve_gpu_ctx *ctx, const oserve_deployment *current, int count,
                                      const uint64_t *d_keys, double *d_est);

/* Drop-in for search::exhaustive (deploysearch.cpp:436-466): ordered space,
 * D <= 16 guard, ModelTooLarge when nothing is feasible. */
int oserve_gpu_exhaustive(oserve_gpu_ctx *ctx, oserve_round_result *out);
/* Drop-in for search::best_strategies (deploysearch.cpp:153-229).  An
 * infeasible partition returns OK with objective 0 and num_replicas 0. */
int oserve_gpu_best_strategies(oserve_gpu_ctx *ctx, int num_replicas, const int *sizes,
                               oserve_round_result *out);

/* ---- flow-guided heuristic search (deploysearch.cpp:341-417) ----------- */

/* search::SearchOptions (deploysearch.hpp:76-84). */
typedef struct {
    uint64_t seed;                        /* default 0   */
    int max_iters;                        /* default 500 */
    int stale_limit;                      /* default 20  */
    int mutation_retries;                 /* default 8   */
    const oserve_deployment *warm_start;  /* NULL: init_uniform */
} oserve_search_options;

/* search::SearchLogRow (deploysearch.hpp:68-74). */
typedef struct {
    int iteration;
    int accepted;
    int64_t throughput;
    int devices;
    char op[120];
} oserve_search_log_row;

/* search::SearchState (deploysearch.hpp:86-92). */
typedef struct {
    int64_t throughput;
    uint64_t rng_seed;
    int stale_iters;
    int iterations;
    int log_count;         /* rows written to the caller's log buffer */
    oserve_plan deployment;
} oserve_search_result;

/* Drop-in for search::search: the reference's mutate / enumerate / revert
 * loop on the host (same mt19937_64 stream, mutate_sizes, classify,
 * absorb_leftovers), every best_strategies and the per-iteration
 * capacity-table + assignment on the GPU.  Uses the context's workload. */
int oserve_gpu_search(oserve_gpu_ctx *ctx, const oserve_search_options *opts, oserve_search_result *out,
                      oserve_search_log_row *log, int log_capacity);

/* Per-plan objectives for ranks [first, first+count) of the prepared space
 * (host output arrays; sum_pp may be NULL). */
int oserve_gpu_evaluate_ranks(oserve_gpu_ctx *ctx, uint64_t first, uint64_t count,
                              int64_t *objective, int32_t *sum_pp);
/* search::evaluate_deployment (deploysearch.cpp:138-151) for a batch of
 * explicit deployments.  Throws-equivalent InfeasibleReplica. */
int oserve_gpu_evaluate_deployments(oserve_gpu_ctx *ctx, int count, const oserve_deployment *deps,
                                    int64_t *objective);

/* cost::build_capacity_table (costmodel.cpp:94-116) + flow::solve_assignment
 * (flowassign.cpp:481-503) for one deployment: all outputs [R*J] row-major
 * except M/used [R].  Any output pointer may be NULL. */
int oserve_gpu_plan_detail(oserve_gpu_ctx *ctx, const oserve_deployment *dep, int64_t *n,
                           int64_t *e, double *latency, int64_t *x, int64_t *M, int64_t *unit,
                           int64_t *used, int64_t *objective);

/* flow::solve_assignment over raw capacity tables (test_flowassign.cpp
 * style): `count` independent instances, each R x J with its own lambda.
 * n, e, x, unit: [count][R][J]; lambda: [count][J]; M, used: [count][R]. */
int oserve_gpu_solve_batch(oserve_gpu_ctx *ctx, int count, int R, int J, const int64_t *n,
                           const int64_t *e, const int64_t *lambda, int64_t *x, int64_t *objective,
                           int64_t *M, int64_t *unit, int64_t *used);

/* ---- workload-adaptive switching (switchplan.cpp:40-140) -------------- */

/* est_seconds of layout()+greedy_plan()+estimate_time() from `src` to each of
 * `count` candidate deployments (one CUDA block per pair).  max_link_bytes
 * may be NULL. */
int oserve_gpu_switch_cost_batch(oserve_gpu_ctx *ctx, const oserve_deployment *src, int count,
                                 const oserve_deployment *dsts, double *est_seconds,
                                 uint64_t *max_link_bytes);
/* Full greedy_plan() for one pair: transfers in the reference's order
 * (fragment-major, destination ascending).  `*num_transfers` returns the
 * count (OSERVE_ERR_INVALID_ARGUMENT with the count set if > capacity). */
int oserve_gpu_switch_plan(oserve_gpu_ctx *ctx, const oserve_deployment *src,
                           const oserve_deployment *dst, int capacity, oserve_transfer *transfers,
                           int *num_transfers, double *est_seconds);

/* ---- reference-signature pieces of switching (switchplan.hpp:34, 57, 61) -- */

/* switchplan::ShardLayout::Shard (switchplan.hpp:24-28). */
typedef struct {
    int shard_id;
    uint64_t begin;
    uint64_t end;
    int holder;
} oserve_shard;

/* One entry of ShardLayout::held (device -> sorted ranges), map order. */
typedef struct {
    int device;
    uint64_t begin;
    uint64_t end;
} oserve_held_range;

/* One entry of SwitchPlan::link_load (switchplan.hpp:44). */
typedef struct {
    int src;
    int dst;
    uint64_t bytes;
} oserve_link_load;

/* Drop-in for switchplan::layout (switchplan.cpp:40-63): the shards of one
 * deployment for a model of param_bytes (replica-major, stage, slice), one
 * device thread per shard.  *n_shards = sum tp*pp; OSERVE_ERR_INVALID_ARGUMENT
 * (count set) when capacity is smaller.  The caller coalesces `held`. */
int oserve_gpu_layout(oserve_gpu_ctx *ctx, const oserve_deployment *dep, uint64_t param_bytes, int capacity,
                      oserve_shard *shards, int *n_shards);
/* Drop-in for switchplan::greedy_plan(const ShardLayout&, const ShardLayout&,
 * const ClusterSpec&) (switchplan.cpp:65-131) over arbitrary layouts given
 * as their `held` maps (device ascending, ranges sorted): fragments sorted on
 * the device, warp per target device, lane per source device.  Transfers in
 * the reference's order; est_seconds = estimate_time of the plan.  A needed
 * fragment without holder: OSERVE_ERR_UNSOURCED_FRAGMENT. */
int oserve_gpu_greedy_plan_layouts(oserve_gpu_ctx *ctx, int n_src, const oserve_held_range *src, int n_dst,
                                   const oserve_held_range *dst, int capacity, oserve_transfer *transfers,
                                   int *n_transfers, double *est_seconds);
/* Drop-in for switchplan::estimate_time (switchplan.cpp:133-140): the
 * slowest link's bytes / bandwidth over the cluster's link classes. */
int oserve_gpu_estimate_time(oserve_gpu_ctx *ctx, int n_links, const oserve_link_load *links, double *est_seconds);

/* ---- reference-signature pieces of the assignment (flowassign.hpp:24-28, 122) */

/* flow::normalize (strict != 0; OSERVE_ERR_LCM_OVERFLOW when the LCM exceeds
 * 2^62) or flow::normalize_or_scale (strict == 0) of `count` rows of J
 * capacities (flowassign.cpp:22-62), on the device (K0b).  M [count],
 * units [count][J], scaled [count] (may be NULL). */
int oserve_gpu_normalize_batch(oserve_gpu_ctx *ctx, int count, int J, const int64_t *n, int strict, int64_t *M,
                               int64_t *units, int *scaled);
/* flow::check_constraints (flowassign.cpp:529-551) on `count` instances
 * [count][R][J]: OSERVE_ERR_LOGIC with the reference's message for the first
 * violating instance.  Optional per-instance outputs (may be NULL): kind
 * (0 ok, 1 C1, 2 C2, 3 C3 zero-capacity type, 4 C3 budget), replica, type. */
int oserve_gpu_check_constraints_batch(oserve_gpu_ctx *ctx, int count, int R, int J, const int64_t *x,
                                       const int64_t *n, const int64_t *e, const int64_t *lambda, int *kind,
                                       int *replica, int *type);

/* ---- device-free helpers (host protocol of the multi-GPU round) ------- */

/* Plans of shard `rank` of `world` when the global plan order is dealt out
 * in interleaved chunks of `chunk` plans. */
uint64_t oserve_shard_count(uint64_t total, uint64_t chunk, int rank, int world);
/* Global plan rank of this shard's local index. */
uint64_t oserve_shard_global_rank(uint64_t local, uint64_t chunk, int rank, int world);
/* Bit layout of the packed selection key for a space: key =
 * ((obj_max - objective) << sh_obj) | (partition << sh_part) |
 * (sum_pp << sh_spp) | local_rank.  OSERVE_ERR_TOO_LARGE if > 63 bits. */
int oserve_key_layout(int64_t total_demand, int64_t partitions, int devices, uint64_t max_plans_per_partition,
                      int *sh_obj, int *sh_part, int *sh_spp, uint64_t *obj_max);
/* Default interleave chunk of oserve_gpu_set_shard. */
#define OSERVE_SHARD_CHUNK 4096

/* ---- KV-cache migration plan (switchplan.cpp:142-207) ------------------ */

/* switchplan::InflightRequest (switchplan.hpp:63-68). */
typedef struct {
    int64_t request_id;
    int64_t generated_tokens;
    uint64_t kv_bytes;
    int source_replica;
} oserve_inflight;

/* switchplan::KvTransfer (switchplan.hpp:70-77). */
typedef struct {
    int64_t request_id;
    uint64_t kv_bytes;
    int src;
    int dst;
} oserve_kv_transfer;

/* Drop-in for switchplan::kv_plan: short requests (generated <= threshold)
 * drain on the source; the rest migrate round-robin over the destination
 * replicas to the least inbound-loaded device, from the (intra-first,
 * least-loaded, lowest-id) source device; link loads start from `carry`
 * (the parameter switch plan's transfers; may be NULL).  Runs as one warp on
 * the device (requests in order, lane-parallel selections).  Outputs are
 * host arrays sized n_inflight. */
int oserve_gpu_kv_plan(oserve_gpu_ctx *ctx, int n_inflight, const oserve_inflight *inflight,
                       int64_t threshold_tokens, const oserve_deployment *src, const oserve_deployment *dst,
                       double headroom, int n_carry, const oserve_transfer *carry, int64_t *drained,
                       int *n_drained, oserve_kv_transfer *migrated, int *n_migrated, uint64_t *buffer_bytes);

/* orch::forecast_series (orchestrate.cpp:75-92) with HoltForecaster
 * (workload.cpp:204-222): counts [T][J] of actual arrivals -> per-span
 * demand [T][J]; span 0 uses its own counts, later spans the Holt forecast
 * over the trailing `window` spans, llround, clamped at 0.  Host-side. */
int oserve_forecast_series(int J, int T, const int64_t *counts, int window, double alpha, double beta,
                           int64_t *lambda_out);

/* ---- flow-network formulation (flowassign.cpp:67-245, 505-519, 559-645) -- */

/* flow::Graph::Edge (flowassign.hpp:32-36). */
typedef struct {
    int from;
    int to;
    int64_t cap;
} oserve_flow_edge;

/* Drop-in for flow::max_flow (FIFO push-relabel, flowassign.cpp:67-147) over
 * `count` independent graphs, each run by one device lane (its workspace in
 * shared memory when it fits): graph g has
 * num_nodes[g] nodes and edges[edge_offset[g] .. edge_offset[g+1]).  Writes
 * per-edge flows (parallel to `edges`) and the value per graph — the
 * reference's exact flows, not just an equal value.  Bad source/sink or a
 * negative capacity: OSERVE_ERR_INVALID_ARGUMENT. */
int oserve_gpu_max_flow_batch(oserve_gpu_ctx *ctx, int count, const int *num_nodes, const int64_t *edge_offset,
                              const oserve_flow_edge *edges, const int *source, const int *sink, int64_t *flow,
                              int64_t *value);

/* flow::build_network + max_flow + extract_assignment (flowassign.cpp:152-199,
 * 505-519) for `count` instances of one shape [R][J] (raw n/e rows as in
 * oserve_gpu_solve_batch).  Outputs x [count][R][J], objective and flow
 * value [count], optionally the per-edge flows [count][J+2RJ+2R] in
 * FlowNetwork edge order (edge_flow may be NULL).  Instances that qualify
 * for the exact path (Σλ <= exact_demand_limit, R*J <= exact_cell_limit)
 * take the branch-and-bound result unless its node budget is exceeded, as
 * solve_instance does. */
int oserve_gpu_flow_assign_batch(oserve_gpu_ctx *ctx, int count, int R, int J, const int64_t *n, const int64_t *e,
                                 const int64_t *lambda, int64_t *x, int64_t *objective, int64_t *flow_value,
                                 int64_t *edge_flow);

/* flow::extract_assignment (flowassign.cpp:505-519) of GIVEN per-edge flows
 * [count][J+2RJ+2R] (FlowNetwork edge order) on instances as above. */
int oserve_gpu_extract_assignment_batch(oserve_gpu_ctx *ctx, int count, int R, int J, const int64_t *n,
                                        const int64_t *e, const int64_t *lambda, const int64_t *edge_flow,
                                        int64_t *x, int64_t *objective);

/* flow::solve_fractional (dense Bland's-rule simplex, flowassign.cpp:559-645)
 * for `count` instances of one shape; f [count][R][J], objective [count].
 * Bit-identical FP64 pivots.  An unbounded tableau: OSERVE_ERR_LOGIC. */
int oserve_gpu_solve_fractional_batch(oserve_gpu_ctx *ctx, int count, int R, int J, const int64_t *n,
                                      const int64_t *e, const int64_t *lambda, double *f, double *objective);

/* Kernel launches issued by this context since creation (evidence counter). */
uint64_t oserve_gpu_launch_count(const oserve_gpu_ctx *ctx);
/* Host->device / device->host bytes copied by this context since creation
 * (explicit copies plus the demand vector passed as kernel parameters). */
int oserve_gpu_copy_bytes(const oserve_gpu_ctx *ctx, uint64_t *h2d_bytes, uint64_t *d2h_bytes);

#ifdef __cplusplus
}
#endif

#endif /* OSERVE_GPU_H */
