/*
 * fbsim_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-threaded-per-instance restatement of the reference fbsim
 * hot path (/root/reference/proj), used as the parity checker for the CUDA
 * path.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
 * may load it; the product library never links or calls it.
 *
 * Parity of this restatement is pinned against (a) the reference library
 * itself, compiled unmodified from /root/reference into oracle/_ref by
 * oracle/Makefile, and (b) the reference's own known-answer tests restated in
 * tests/test_oracle_golden.py and the fixtures under tests/golden/.
 *
 * Signatures mirror include/fbgpu.h (prefix orc_ instead of fb_).
 */
#ifndef FBSIM_ORACLE_H_
#define FBSIM_ORACLE_H_

#include "../include/fbgpu.h"

#ifdef __cplusplus
extern "C" {
#endif

int orc_generate_bursty(const fb_burst_profile* profile, int64_t horizon_us,
                        int64_t cap, int64_t* arrival_us, int32_t* prompt_len,
                        int32_t* output_len, int64_t* ttft_us, int64_t* tpot_us,
                        int64_t* n_out);
int orc_scale_trace(int64_t* arrival_us, int64_t n, double factor);
double orc_keyed_uniform(uint64_t seed, uint64_t ordinal);

/* Pure scheduler, one task set. */
int orc_init_time_budget(const fb_task_view* tasks, int64_t n,
                         int64_t* budget_out);
int orc_form_batch(const fb_task_view* tasks, int64_t n,
                   const fb_scheduler_config* cfg, fb_plan_entry_id* entries,
                   fb_batch_plan* plan);
int orc_pab(const fb_task_view* tasks, int64_t n, const fb_cost_model* model,
            int64_t ttft_us, int64_t tpot_us, int64_t* pab_out);

/* run_node for every instance.  Logs (optional, may be NULL) are laid out per
 * instance i at steps + i*log->step_cap etc.  nthreads <= 1 runs serially. */
int orc_run_instances(const fb_trace* rows, const fb_instance* instances,
                      int64_t n_instances, const fb_log_opts* log,
                      fb_instance_result* results, fb_record* records,
                      fb_log_counts* counts, fb_step_log* steps,
                      fb_plan_entry* entries, fb_reject_log* rejects,
                      int nthreads);

/* run_cluster over the whole trace (row index = request id). */
int orc_run_cluster(const fb_trace* rows, const fb_engine_config* cfgs, int32_t n_nodes,
                    const fb_lb_config* lb, int64_t horizon, fb_instance_result* node_results,
                    fb_record* records, int32_t* route_node, int32_t* incomplete_out);

/* run_cluster's epoch decomposition for one rank of a node partition; the
 * caller exchanges fb_node_reports between advance and route_begin. */
typedef struct orc_cluster_shard orc_cluster_shard;
int orc_cluster_partition(int32_t n_nodes, int32_t n_ranks, int32_t rank, int32_t* node_lo,
                          int32_t* n_local);
int orc_cluster_shard_create(const fb_trace* rows, const fb_engine_config* cfgs, int32_t n_nodes,
                             const fb_lb_config* lb, int64_t horizon, int32_t rank,
                             int32_t n_ranks, orc_cluster_shard** out);
int64_t orc_cluster_shard_epochs(const orc_cluster_shard* s);
int orc_cluster_shard_advance(orc_cluster_shard* s, int64_t epoch, fb_node_report* local);
int orc_cluster_shard_route_begin(orc_cluster_shard* s, int64_t epoch, const fb_node_report* all,
                                  int32_t* stopped);
int orc_cluster_shard_fetch(orc_cluster_shard* s, fb_instance_result* local_results,
                            fb_record* records, int32_t* route_node, int64_t* n_routed,
                            int32_t* incomplete);
void orc_cluster_shard_destroy(orc_cluster_shard* s);

#ifdef __cplusplus
}
#endif

#endif
