/*
 * oracle_api.h — TEST INFRASTRUCTURE ONLY.
 *
 * The C-ABI exported by the two CPU oracles:
 *   oracle/_ref/libref_oserve.so   the reference itself (/root/reference/proj/src,
 *                                  compiled unmodified) behind ref_harness.cpp
 *   oracle/liboserve_port.so       oserve_port.cpp, a CPU restatement of the
 *                                  reference algorithm (each function cites
 *                                  the reference file:line it follows)
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
 * load these.  The product path (paper_2602_12151_b200) never does.
 */
#ifndef OSERVE_ORACLE_API_H
#define OSERVE_ORACLE_API_H

#include "../include/oserve_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    oserve_cluster_desc cluster;
    oserve_model_desc model;
    oserve_profile profile;
    int num_classes;
    const oserve_class *classes;
    const int64_t *lambda;
    double span_seconds;
} oracle_problem;

const char *oracle_last_error(void);
/* 1 for the reference build, 0 for the restatement. */
int oracle_is_reference(void);

int oracle_min_feasible_group(const oracle_problem *p, int *g_min);
int oracle_capacity_table(const oracle_problem *p, const oserve_deployment *dep, int64_t *n,
                          int64_t *e, double *latency);
int oracle_normalize(int J, const int64_t *n_row, int strict, int64_t *M, int64_t *units,
                     int *scaled);
/* Default SolveOptions unless opts != NULL.  work (may be NULL) = greedy
 * visits + exchange probes (port only; the reference returns 0). */
int oracle_solve_assignment(int R, int J, const int64_t *n, const int64_t *e, const int64_t *lambda,
                            const oserve_solve_options *opts, int64_t *x, int64_t *objective,
                            int64_t *M, int64_t *unit, int64_t *used, uint64_t *work);
int oracle_check_constraints(int R, int J, const int64_t *x, const int64_t *n, const int64_t *e,
                             const int64_t *lambda);
int oracle_evaluate_deployment(const oracle_problem *p, const oserve_deployment *dep,
                               int64_t *objective);
int oracle_best_strategies(const oracle_problem *p, int R, const int *sizes, int parallel,
                           oserve_round_result *out);
int oracle_exhaustive(const oracle_problem *p, int parallel, oserve_round_result *out);

/* Plan spaces (same definition and order as the GPU path). */
int oracle_space_info(const oracle_problem *p, const oserve_space_desc *s, int64_t *partitions,
                      uint64_t *plans);
int oracle_space_plan(const oracle_problem *p, const oserve_space_desc *s, uint64_t rank,
                      oserve_plan *plan, int64_t *partition_index, uint64_t *local_rank);
int oracle_evaluate_ranks(const oracle_problem *p, const oserve_space_desc *s, int64_t count,
                          const uint64_t *ranks, int64_t *objective, int32_t *sum_pp,
                          uint64_t *work, int threads);
/* Full round: argmin over the space by (obj desc, partition asc, sum_pp asc,
 * rank asc).  threads <= 1 => serial. */
int oracle_round(const oracle_problem *p, const oserve_space_desc *s, int threads,
                 oserve_round_result *out);

int oracle_switch_plan(const oserve_cluster_desc *c, uint64_t param_bytes,
                       const oserve_deployment *src, const oserve_deployment *dst, int capacity,
                       oserve_transfer *transfers, int *num_transfers, double *est_seconds,
                       uint64_t *max_link_bytes);

/* search::search (deploysearch.cpp:341-417) with its log (reference only). */
int oracle_search(const oracle_problem *p, const oserve_search_options *opts, oserve_search_result *out,
                  oserve_search_log_row *log, int log_capacity);

/* orch::build_adaptive_timeline (orchestrate.cpp:94-154) over T spans of
 * actual per-class counts [T][J] (reference only).  Per entry e (< capacity):
 * span_index[e], plans[e], x[e][k][j] (R <= 128, J classes, row stride 128*J),
 * switch_seconds[e], transfers[e]; returns the entry count. */
int oracle_adaptive_timeline(const oracle_problem *p, int T, const int64_t *counts, uint64_t seed, int max_iters,
                             double min_gain, int capacity, int64_t *span_index, oserve_plan *plans, int64_t *x,
                             double *switch_seconds, int *transfers, int *count);

/* Reference-only helpers used to generate the synthetic workloads. */
int oracle_fit_types(int64_t n, const uint32_t *input_len, const uint32_t *output_len, int k,
                     uint64_t seed, double *centroid_in, double *centroid_out);
int oracle_holt_forecast(int J, int T, const int64_t *counts, int window, int64_t *lambda_out);

/* switchplan::kv_plan (reference only); carry = a switch plan's transfers. */
int oracle_kv_plan(const oserve_cluster_desc *c, int n_inflight, const oserve_inflight *inflight,
                   int64_t threshold_tokens, const oserve_deployment *src, const oserve_deployment *dst,
                   double headroom, int n_carry, const oserve_transfer *carry, int64_t *drained, int *n_drained,
                   oserve_kv_transfer *migrated, int *n_migrated, uint64_t *buffer_bytes);

/* io::save_timeline of orch::build_adaptive_timeline (reference only). */
int oracle_adaptive_timeline_json(const oracle_problem *p, int T, const int64_t *counts, uint64_t seed,
                                  int max_iters, double min_gain, const char *path);

/* io::load_timeline(in) then io::save_timeline(out); io::load_deployment /
 * save_deployment likewise (reference only) — schema checks. */
/* flow::max_flow / build_network+max_flow+extract_assignment /
 * solve_fractional / to_dot (reference only; flowassign.cpp:67-245,
 * 505-519, 559-645). */
int oracle_max_flow(int num_nodes, int num_edges, const oserve_flow_edge *edges, int source, int sink,
                    int64_t *flow, int64_t *value);
int oracle_flow_assign(int R, int J, const int64_t *n, const int64_t *e, const int64_t *lambda,
                       const oserve_solve_options *opts, int64_t *x, int64_t *objective, int64_t *flow_value,
                       int64_t *edge_flow);
int oracle_solve_fractional(int R, int J, const int64_t *n, const int64_t *e, const int64_t *lambda, double *f,
                            double *objective);
int oracle_to_dot(int R, int J, const int64_t *n, const int64_t *e, const int64_t *lambda, int with_flow,
                  char *buf, int cap, int *len);

int oracle_timeline_resave(const char *in_path, const char *out_path, int *entries);
int oracle_deployment_resave(const char *in_path, const char *out_path, int *replicas);

#ifdef __cplusplus
}
#endif

#endif
