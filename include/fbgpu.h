/*
 * fbgpu.h -- C ABI of the B200-native FairBatching per-iteration scheduling
 * hot path (drop-in for the fbsim reference, /root/reference/proj).
 *
 * Plain C: pointers, sizes and POD structs only.  No torch types, no C++
 * exceptions cross this boundary; every entry point returns an FB_* status and
 * fb_last_error() holds a message for the calling thread.
 *
 * Reference interfaces replaced (paths relative to /root/reference/proj):
 *   - Pure scheduler surface  sched.h:81-115
 *       init_time_budget / form_batch / pab           -> fb_init_time_budget,
 *                                                        fb_form_batch, fb_pab
 *   - Stateful step machine   engine.h:111-176  (class Node)
 *       Node::enqueue / begin_step / complete_step     -> fb_arena_* (batched
 *       over thousands of independent Node instances resident in HBM)
 *   - Drivers                 engine.h:180  run_node
 *                             cluster.h:107-109 run_cluster
 *                                                      -> fb_arena_run,
 *                                                         fb_run_batch,
 *                                                         fb_cluster_*
 *   - Per-request records     metrics.h:29-49 RequestReport (built online)
 *   - Host trace generation   workload.h:88-94 generate_bursty / scale_trace /
 *                             truncate_trace      -> fb_generate_bursty, ...
 *
 * Time is int64 microseconds (time.h:23-34); cost arithmetic is fp64 in the
 * reference's operation order (sched.cpp:129-166), so batch decisions are
 * bit-identical to the CPU reference.
 */
#ifndef FBGPU_H_
#define FBGPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FBGPU_ABI_VERSION 1

/* Status codes; the host C++ wrapper maps them onto the fbsim exception
 * taxonomy (errors.h:24-53) and the CLI exit codes (commands.h:30-33). */
enum {
  FB_OK = 0,
  FB_ERR_VALIDATION = 1, /* ValidationError: domain invariant violated   */
  FB_ERR_USAGE = 2,      /* UsageError: API misuse / precondition       */
  FB_ERR_CONFIG = 3,     /* ConfigError: bad scenario or command config */
  FB_ERR_PARSE = 4,      /* ParseError                                  */
  FB_ERR_CUDA = 5,       /* device missing / CUDA runtime failure       */
  FB_ERR_CAPACITY = 6,   /* caller buffer too small; *_needed reported  */
  FB_ERR_TIMEOUT = 7     /* a peer rank never reached the epoch exchange */
};

/* Scheduling policies, sched.h:60 (same numbering as the enum order). */
enum {
  FB_POLICY_PREFILL_FIRST = 0,
  FB_POLICY_SARATHI = 1,
  FB_POLICY_FAIRBATCH = 2,
  FB_POLICY_FAIRBATCH_PAB = 3
};

/* Task phase, sched.h:28. */
enum { FB_PHASE_PREFILL = 0, FB_PHASE_DECODE = 1 };

/* Cluster load-balancer policies, cluster.h:31. */
enum { FB_LB_COUNT = 0, FB_LB_PAB = 1 };

/* Linear step-time model a + b*new + c*context (costmodel.h:29-33). */
typedef struct fb_cost_model {
  double a_ms;
  double b_ms;
  double c_ms;
} fb_cost_model;

/* SchedulerConfig, sched.h:65-74. */
typedef struct fb_scheduler_config {
  int32_t policy;       /* FB_POLICY_* */
  int32_t max_chunk;    /* per-chunk ceiling */
  int64_t token_budget; /* per-step token ceiling */
  fb_cost_model model;  /* the scheduler's own estimator */
} fb_scheduler_config;

/* EngineConfig, engine.h:76-82 (NoiseSpec costmodel.h:62-65 inlined,
 * global SloTargets slo.h:34-37 inlined). */
typedef struct fb_engine_config {
  fb_scheduler_config scheduler;
  fb_cost_model truth_model;
  double noise_amplitude; /* multiplicative truth noise, factor 1 + amp*u */
  uint64_t noise_seed;    /* keyed per (seed, step ordinal), rng.h:88-94  */
  int64_t global_ttft_us; /* global SLOs used by PAB admission            */
  int64_t global_tpot_us;
  int32_t max_active; /* 0 = unbounded (engine.h:81)                  */
  int32_t reserved;
} fb_engine_config;

/* Trace rows, structure of arrays (Request, workload.h:28-35).  Rows of one
 * instance are contiguous and sorted by arrival (workload.h:40-43).  The row
 * index inside an instance is the request's id for every output below. */
typedef struct fb_trace {
  const int64_t* arrival_us;
  const int32_t* prompt_len;
  const int32_t* output_len;
  const int64_t* ttft_us;
  const int64_t* tpot_us;
  int64_t n_rows;
} fb_trace;

/* One simulated node (one independent run_node) inside an arena. */
typedef struct fb_instance {
  fb_engine_config cfg;
  int64_t trace_off;  /* first row of this instance's trace               */
  int64_t n_req;      /* rows; several instances may share the same rows  */
  int64_t horizon_us; /* run_node horizon (engine.h:180)                  */
} fb_instance;

/* Per-request outcome, RequestReport (metrics.h:29-49) computed online. */
typedef struct fb_record {
  int64_t first_emit_us;  /* absolute time of token 0; -1 when none       */
  double max_tpot_ms;     /* metrics.cpp:42-49 (0 for < 2 tokens)         */
  double max_tpot_alt_ms; /* metrics.cpp:53-60 (denominator j-1)          */
  int32_t tokens_emitted;
  uint32_t flags; /* FB_REC_* */
} fb_record;

enum {
  FB_REC_ARRIVED = 1u,   /* an arrival event was logged (report exists)    */
  FB_REC_REJECTED = 2u,  /* PAB admission reject and never served          */
  FB_REC_FINISHED = 4u,  /* request_done                                   */
  FB_REC_MET_TTFT = 8u,  /* emits[0] <= ttft_slo (metrics.cpp:105)         */
  FB_REC_MET_TPOT = 16u, /* finished and (e_j-e_0) <= tpot*j for all j     */
  FB_REC_ENV_MISS = 32u  /* some token j>=1 past arrival+ttft+tpot*j       */
};

/* Per-instance summary. */
typedef struct fb_instance_result {
  uint64_t steps;       /* begin_step launches incl. spin steps = Node::steps_completed */
  uint64_t plan_digest; /* rolling digest of every plan + reject (fbgpu_digest.h) */
  int64_t end_time_us;  /* clock when the run stopped */
  int64_t n_arrived;    /* requests enqueued (== reports) */
  int64_t n_rejected;   /* PAB admission rejects */
  int64_t sum_visible;  /* sum over steps of visible tasks A */
  int64_t sum_entries;  /* sum over steps of plan entries E */
  int64_t sum_new_tokens;
  int32_t incomplete; /* EventLog::incomplete (engine.cpp:286) */
  int32_t status;     /* FB_OK or an FB_ERR_* for this instance */
} fb_instance_result;

/* Optional per-step plan log (parity tooling), one row per begin_step. */
typedef struct fb_step_log {
  int64_t t_us;         /* batch_start time */
  int64_t duration_us;  /* max(1, llround(actual_ms*1000)) */
  double predicted_ms;  /* BatchPlan::predicted_ms */
  double actual_ms;     /* ground-truth step time */
  int64_t total_new;    /* batch_start.new_tokens */
  int64_t total_ctx;    /* batch_start.context_tokens */
  double init_budget_ms;/* BatchPlan::init_time_budget_ms (fair batching) */
  int32_t entry_off;    /* first entry in the instance's entry log */
  int32_t n_entries;
} fb_step_log;

/* BatchPlanEntry (sched.h:44-47) with the trace row as request id. */
typedef struct fb_plan_entry {
  int32_t req;
  int32_t new_tokens;
} fb_plan_entry;

/* admission_reject event (engine.cpp:134-142). */
typedef struct fb_reject_log {
  int64_t t_us;
  int64_t pab_tokens;
  int32_t req;
  int32_t step; /* steps the node began before this reject (the rejecting
                   begin_step launches step `step`, if any) */
} fb_reject_log;

/* Plan-log capacities per instance; 0 disables logging. */
typedef struct fb_log_opts {
  int32_t step_cap;
  int32_t entry_cap;
  int32_t reject_cap;
  int32_t reserved;
} fb_log_opts;

/* Log occupancy per instance after a run. */
typedef struct fb_log_counts {
  int32_t steps;
  int32_t entries;
  int32_t rejects;
  int32_t truncated;
} fb_log_counts;

/* ---------------------------------------------------------------------- */
/* Library                                                                */
/* ---------------------------------------------------------------------- */

int fb_abi_version(void);
const char* fb_last_error(void);
/* Number of CUDA devices visible (0 on a host without GPU). */
int fb_device_count(int* n_out);

/* ---------------------------------------------------------------------- */
/* Host-side trace generation (stays on the host: libm log/exp/cos/sqrt). */
/* ---------------------------------------------------------------------- */

/* BurstProfile, workload.h:55-66, plus the generation horizon. */
typedef struct fb_burst_profile {
  double base_rate;  /* req/s in idle phases  */
  double burst_rate; /* req/s in burst phases */
  int64_t burst_duration_us;
  int64_t idle_duration_us;
  double prompt_mean, prompt_p90;
  double output_mean, output_p90;
  int64_t ttft_us, tpot_us; /* stamped on every request */
  uint64_t seed;
} fb_burst_profile;

/* generate_bursty (workload.cpp:244-298).  Writes up to `cap` rows; *n_out
 * receives the row count.  FB_ERR_CAPACITY when cap < *n_out (call again).
 * Any output pointer may be NULL when cap == 0. */
int fb_generate_bursty(const fb_burst_profile* profile, int64_t horizon_us,
                       int64_t cap, int64_t* arrival_us, int32_t* prompt_len,
                       int32_t* output_len, int64_t* ttft_us, int64_t* tpot_us,
                       int64_t* n_out);

/* scale_trace (workload.cpp:211-221), in place. */
int fb_scale_trace(int64_t* arrival_us, int64_t n, double factor);

/* offered_rps (workload.cpp:315-321). */
int fb_offered_rps(const int64_t* arrival_us, int64_t n, double* rps_out);

/* ---------------------------------------------------------------------- */
/* Pure scheduler surface (sched.h:81-115), batched over task sets.        */
/* ---------------------------------------------------------------------- */

/* TaskView, sched.h:34-42. */
typedef struct fb_task_view {
  int64_t request_id;
  int64_t slack_us;
  int64_t context;
  int64_t arrival_seq;
  int64_t tpot_us;
  int32_t new_tokens;
  int32_t phase; /* FB_PHASE_* */
} fb_task_view;

/* BatchPlan scalars, sched.h:49-58. */
typedef struct fb_batch_plan {
  double predicted_ms;
  double time_budget_used_ms;
  int64_t token_budget_used;
  double init_time_budget_ms;
  int64_t entry_off; /* into the entries output */
  int64_t n_entries;
} fb_batch_plan;

/* Plan entry keyed by the caller's request_id. */
typedef struct fb_plan_entry_id {
  int64_t request_id;
  int32_t new_tokens;
  int32_t reserved;
} fb_plan_entry_id;

/* form_batch (sched.cpp:234-246) for n_sets independent task sets on the
 * device.  Set s owns tasks[set_off[s] .. set_off[s+1]).  Entries of set s are
 * written at entries[set_off[s] ...] (a plan never has more entries than
 * tasks) and plans[s].entry_off/n_entries describe them.  Empty sets are a
 * UsageError for the fair-batching policies (sched.cpp:91-93).
 * Any task set the reference's form_batch takes gives the same plan,
 * including zero-token tasks (fair batching's `consider`, sched.cpp:141-150,
 * admits them as {id, 0} whenever c*ctx <= time_budget, even once the token
 * budget is spent) and negative contexts.  Stricter than the reference:
 * new_tokens < 0, |slack_us| >= 2^61 and, for the fair-batching policies,
 * b <= 0 (the chunk size divides by b) are ValidationErrors. */
int fb_form_batch(int device, const fb_task_view* tasks, const int64_t* set_off,
                  const fb_scheduler_config* cfgs, int64_t n_sets,
                  fb_plan_entry_id* entries, fb_batch_plan* plans);

/* init_time_budget (sched.cpp:90-106) per set. */
int fb_init_time_budget(int device, const fb_task_view* tasks,
                        const int64_t* set_off, int64_t n_sets,
                        int64_t* budget_us_out);

/* pab (sched.cpp:248-278) per set; models[s], slos (ttft,tpot us) per set. */
int fb_pab(int device, const fb_task_view* tasks, const int64_t* set_off,
           const fb_cost_model* models, const int64_t* ttft_us,
           const int64_t* tpot_us, int64_t n_sets, int64_t* pab_out);

/* ---------------------------------------------------------------------- */
/* Arena: request-state SoA for thousands of Node instances in HBM.        */
/* ---------------------------------------------------------------------- */

typedef struct fb_arena fb_arena;

/* stream: a cudaStream_t to issue all work on, or NULL for a private one. */
int fb_arena_create(int device, void* stream, fb_arena** out);
int fb_arena_destroy(fb_arena* arena);

/* Uploads trace rows and instances (validated as Node/validate_request do,
 * engine.cpp:83-90, workload.cpp:114-124) and allocates all device state.
 * log may be NULL. */
int fb_arena_load(fb_arena* arena, const fb_trace* rows,
                  const fb_instance* instances, int64_t n_instances,
                  const fb_log_opts* log);

/* Rewinds every instance to t = 0 (device-side, no host traffic). */
int fb_arena_reset(fb_arena* arena);

/* Advances every unfinished instance by at most max_events iterations of the
 * run_node event loop (engine.cpp:271-283); max_events <= 0 runs to
 * quiescence.  Asynchronous on the arena stream.  *n_active_out (may be NULL)
 * receives the number of instances still running after the call, which
 * forces a synchronisation. */
int fb_arena_run(fb_arena* arena, int64_t max_events, int64_t* n_active_out);

int fb_arena_synchronize(fb_arena* arena);

/* Device time of the last fb_arena_run (CUDA events on the arena stream). */
int fb_arena_last_run_ms(fb_arena* arena, float* ms_out);
/* The same run split into the warp engine and the grid-wide wide engine
 * (nodes with more than 512 live requests). */
int fb_arena_last_run_split_ms(fb_arena* arena, float* warp_ms, float* wide_ms);
/* Phase clock of the last run's grid-wide wide engine (wall time seen by
 * CTA 0, each phase including its closing grid barrier): ms_out[5] =
 * {owner advance, K1 views, K2a histogram, K2b gather, owner finish};
 * *iterations (may be NULL) = lockstep iterations. */
int fb_arena_wide_phases(fb_arena* arena, double* ms_out, int64_t* iterations);
/* Selection path counts of the last run's grid-wide wide engine: node steps
 * whose window K1 gathered itself (fused candidate window) and node steps
 * that took the K2a / K2b passes. */
int fb_arena_wide_selection(fb_arena* arena, int64_t* fused_steps, int64_t* k2_steps);

int fb_arena_fetch_results(fb_arena* arena, fb_instance_result* out);
/* Records for instance rows: out has sum over instances of n_req rows, in
 * instance order. */
int fb_arena_fetch_records(fb_arena* arena, fb_record* out);
int64_t fb_arena_record_rows(const fb_arena* arena);
int fb_arena_fetch_log_counts(fb_arena* arena, fb_log_counts* out);
/* Per instance, which device engine paths ran: FB_PATH_* bits (REPEAT_*:
 * repeated-plan steps -- the previous plan admitted every visible task as a
 * one-token decode and nothing entered or left -- on the register / memory
 * path). */
enum {
  FB_PATH_REGISTER = 1u,
  FB_PATH_MEMORY = 2u,
  FB_PATH_WIDE = 4u,
  FB_PATH_REPEAT_REGISTER = 8u,
  FB_PATH_REPEAT_MEMORY = 16u
};
int fb_arena_fetch_paths(fb_arena* arena, uint32_t* out);
/* Copies instance i's logs; buffers sized by the log caps (NULL skips). */
int fb_arena_fetch_log(fb_arena* arena, int64_t instance, fb_step_log* steps,
                       fb_plan_entry* entries, fb_reject_log* rejects);

/* Per-instance ScenarioReport aggregates computed on the device
 * (scenario_report, metrics.cpp:171-205; nearest-rank percentiles,
 * metrics.cpp:118-135) over the requests that arrived.  offered_rps,
 * slo_violation_rate = 1 - good/total and effective_rps = offered * good/total
 * are host arithmetic on these counts. */
typedef struct fb_percentiles {
  double p50, p95, p99;
  int64_t count;
} fb_percentiles;
typedef struct fb_summary {
  int64_t total_requests, rejected, finished, good;
  int64_t ttft_violations;  /* no first token or emits[0] > ttft (acceptance.cpp:105) */
  int64_t envelope_misses;  /* some token j>=1 past its envelope (acceptance.cpp:106-111) */
  fb_percentiles ttft_ms, max_tpot_ms, max_tpot_alt_ms;
} fb_summary;
int fb_arena_fetch_summaries(fb_arena* arena, fb_summary* out);

/* Envelope-lead series (envelope_lead_series, metrics.cpp:137-169) per
 * instance.  fb_arena_set_lead enables the run-time accounting for the next
 * load/reset (bucket_us > 0; at most cap series points per instance; 0
 * disables).  fb_arena_fetch_lead fills out[instance * cap + k] = lead tokens
 * at t = k * bucket_us and n_out[instance] = points (-1 when cap was too
 * small).  Single nodes only (not cluster shards). */
int fb_arena_set_lead(fb_arena* arena, int64_t bucket_us, int32_t cap);
int fb_arena_fetch_lead(fb_arena* arena, int64_t* out, int32_t* n_out);

/* Page-locked host buffers.  Trace rows, instances and record outputs that
 * live in memory from fb_host_alloc move by direct DMA; any other host
 * pointer is staged through the arena's own pinned chunks.  Not a reference
 * interface: the reference keeps everything in host memory. */
int fb_host_alloc(size_t bytes, void** out);
int fb_host_free(void* p);

/* One-shot end-to-end run from host buffers: upload, run to quiescence,
 * download results and records (records may be NULL).  elapsed_ms_out (may be
 * NULL) receives the host wall time of the whole call.  Reuses one cached
 * arena per device (serialised by a lock), so repeated calls pay no device
 * allocation. */
int fb_run_batch(int device, const fb_trace* rows, const fb_instance* instances,
                 int64_t n_instances, fb_instance_result* results,
                 fb_record* records, double* elapsed_ms_out);

/* ---------------------------------------------------------------------- */
/* Cluster: run_cluster (cluster.h:107-109) on the device.                 */
/* ---------------------------------------------------------------------- */

/* One routing decision (RoutingLogEntry, cluster.h:86-91; its view snapshot
 * is a separate row of n_nodes doubles). */
typedef struct fb_route_log {
  int64_t t_us;  /* decision time */
  int32_t req;   /* trace row */
  int32_t node;  /* target */
  int32_t rej_before;   /* the target's admission rejects so far (-1: not recorded) */
  int32_t steps_before; /* the target's steps begun so far (-1: not recorded) */
} fb_route_log;

/* LbConfig, cluster.h:36-47. */
typedef struct fb_lb_config {
  int32_t policy;                /* FB_LB_COUNT / FB_LB_PAB */
  int32_t report_interval_steps; /* reports every k completed steps (0 = none) */
  int64_t report_latency_us;     /* delivery delay of a report */
  double w_waiting;              /* count_lb weights */
  double w_running;
  int32_t retry_reroute; /* route a PAB-rejected request once more (one rank only) */
  int32_t report_cap;    /* per-node in-flight report capacity (0 = default 4096) */
} fb_lb_config;

/* Simulates one data-parallel cluster: the trace rows (sorted by arrival,
 * row index = request id) are routed on arrival to n_nodes nodes with
 * node_cfgs[i] by the load balancer, exactly as run_cluster
 * (cluster.cpp:134-251).  Outputs: per-node results (plan digest, steps,
 * routed/rejected counts), per-request records (global order; a request
 * never routed has flags == 0), route_node[i] = node of request i or -1,
 * *incomplete_out = ClusterResult::incomplete.  Any output may be NULL. */
int fb_run_cluster(int device, const fb_trace* rows, const fb_engine_config* node_cfgs,
                   int32_t n_nodes, const fb_lb_config* lb, int64_t horizon_us,
                   fb_instance_result* node_results, fb_record* records,
                   int32_t* route_node, int32_t* incomplete_out, double* device_ms_out);

/* fb_run_cluster plus the logs ClusterResult carries (cluster.h:93-98): each
 * node's plan log (steps / entries / rejects at node i * cap, counts per
 * node; the node's EventLog is rebuilt from it and the routing log) and the
 * routing log -- one fb_route_log per route_request call (reroutes
 * included) and, in `snapshots`, n_nodes doubles per entry: the balancer's
 * per-node score after the decision (RoutingLogEntry::view_snapshot).
 * *n_routes_out receives the entry count; FB_ERR_CAPACITY when it exceeds
 * route_cap (n_rows suffices without retry_reroute, 2 * n_rows with it). */
int fb_run_cluster_logged(int device, const fb_trace* rows, const fb_engine_config* node_cfgs,
                          int32_t n_nodes, const fb_lb_config* lb, int64_t horizon_us,
                          const fb_log_opts* log, fb_instance_result* node_results,
                          fb_record* records, int32_t* route_node, int32_t* incomplete_out,
                          fb_log_counts* node_counts, fb_step_log* steps, fb_plan_entry* entries,
                          fb_reject_log* rejects, fb_route_log* routes, double* snapshots,
                          int64_t route_cap, int64_t* n_routes_out);

/* ---------------------------------------------------------------------------
 * Multi-GPU cluster: the nodes are partitioned over n_ranks processes (one
 * GPU each, contiguous node ranges, fb_cluster_partition).  Every rank runs
 * one persistent kernel over its nodes; per dispatch epoch (distinct arrival
 * time) each node publishes an fb_node_report into every rank's exchange
 * buffer (NVLink peer memory opened with CUDA IPC), the ranks meet at a
 * device-side barrier, and each rank runs the same deterministic router
 * (route, cluster.cpp:75-112) -- run_cluster's event order.
 * Sequence on every rank:
 *   create -> exchange_handle -> (allgather handles) -> connect -> reset ->
 *   (host barrier across ranks) -> launch -> wait -> fetch -> destroy.
 * Ranks of one process on one device may use exchange_ptr / connect_ptrs.
 * The merged outputs equal fb_run_cluster's: route_node is identical on all
 * ranks; rank r fills node_results of its own nodes and the records of the
 * requests routed to them (the others stay "never routed"). */
#define FB_CLUSTER_MAX_RANKS 8
#define FB_IPC_HANDLE_BYTES 64

typedef struct fb_node_report {
  int64_t emitted_at; /* newest report delivered by the epoch time, -1 none */
  int64_t pab_tokens;
  int32_t waiting;
  int32_t running;
  int32_t fresh; /* delivered since the previous epoch */
  int32_t busy;  /* node busy when the clock reaches the epoch time */
} fb_node_report;

typedef struct fb_cluster_shard fb_cluster_shard;

/* Node range [*node_lo, *node_lo + *n_local) of `rank`. */
int fb_cluster_partition(int32_t n_nodes, int32_t n_ranks, int32_t rank, int32_t* node_lo,
                         int32_t* n_local);
int fb_cluster_shard_create(int device, const fb_trace* rows, const fb_engine_config* node_cfgs,
                            int32_t n_nodes, const fb_lb_config* lb, int64_t horizon_us,
                            int32_t rank, int32_t n_ranks, fb_cluster_shard** out);
int fb_cluster_shard_exchange_handle(fb_cluster_shard* s, void* handle_out);
int fb_cluster_shard_exchange_ptr(fb_cluster_shard* s, void** dev_ptr_out);
/* handles: n_ranks * FB_IPC_HANDLE_BYTES (this rank's entry is ignored). */
int fb_cluster_shard_connect(fb_cluster_shard* s, const void* handles);
int fb_cluster_shard_connect_ptrs(fb_cluster_shard* s, void* const* dev_ptrs);
/* Zeroes this rank's exchange counter; all ranks must finish reset before
 * any rank launches. */
int fb_cluster_shard_reset(fb_cluster_shard* s);
/* A one-rank shard of at most 8 CTAs runs as one thread-block cluster
 * (hardware cluster barrier, reports through distributed shared memory):
 * allow = 1 (default) one CTA per SM, 2 two CTAs per SM (for many shards side
 * by side: each runs slower, twice as many fit), 0 the cooperative grid --
 * e.g. when more shards run side by side than fit the device at once. */
int fb_cluster_shard_allow_hw_cluster(fb_cluster_shard* s, int32_t allow);
/* How many one-cluster grids of n_nodes fit the device at once (one CTA per
 * SM); fb_cluster_fit: the same for ctas_per_sm = 1 or 2. */
int fb_cluster_max_hw_clusters(int device, int32_t n_nodes, int32_t* out);
int fb_cluster_fit(int device, int32_t n_nodes, int32_t ctas_per_sm, int32_t* out);
int fb_cluster_shard_launch(fb_cluster_shard* s);
int fb_cluster_shard_wait(fb_cluster_shard* s, double* device_ms_out);
/* local_results: n_local entries (incomplete = this rank's view);
 * records / route_node: n_rows; *n_routed = requests routed before the loop
 * stopped; *incomplete = this rank's ClusterResult::incomplete share. */
int fb_cluster_shard_fetch(fb_cluster_shard* s, fb_instance_result* local_results,
                           fb_record* records, int32_t* route_node, int64_t* n_routed,
                           int32_t* incomplete);
void fb_cluster_shard_destroy(fb_cluster_shard* s);

/* ---------------------------------------------------------------------- */
/* Interactive node set: the Node surface (engine.h:111-176) of n nodes,   */
/* batched, for an external dispatcher (the upper-level load balancer).    */
/* ---------------------------------------------------------------------- */
/* Every call acts on all nodes at once (one warp per node); node state stays
 * in HBM between calls.  Requests are the rows of the trace given at
 * creation (request_id = row); a dispatcher routes rows to nodes with
 * fb_nodes_enqueue.  Driving the calls in run_cluster's order
 * (cluster.cpp:134-251) reproduces run_cluster exactly
 * (cluster.py run_cluster_host, tests/test_gpu_parity.py). */

typedef struct fb_nodes fb_nodes;

/* Node queries (engine.h:119-139). */
typedef struct fb_node_state {
  int64_t step_end;        /* Node::step_end (valid when busy) */
  int64_t waiting;         /* Node::waiting_count */
  int64_t running;         /* Node::running_count */
  int64_t steps_completed; /* Node::steps_completed */
  int32_t busy;            /* Node::busy */
  int32_t has_live;        /* Node::has_live_requests */
} fb_node_state;

/* Node(i, cfgs[i]) for i < n_nodes (engine.cpp:83-90 validation), over the
 * trace `rows`; the nodes begin no step at or after horizon_us.  reports:
 * NULL, or the metric-report hook of run_cluster -- an initial report at 0
 * and make_report (cluster.cpp:50-58: waiting, running, and current_pab when
 * policy == FB_LB_PAB) after every report_interval_steps-th complete_step,
 * delivered report_latency_us later (fb_nodes_advance). */
int fb_nodes_create(int device, const fb_trace* rows, const fb_engine_config* node_cfgs,
                    int32_t n_nodes, int64_t horizon_us, const fb_lb_config* reports,
                    fb_nodes** out);
void fb_nodes_destroy(fb_nodes* h);
int32_t fb_nodes_count(const fb_nodes* h);
/* Step-to-time: every node completes its in-flight steps ending before t and
 * begins its next ones at their end times (no dispatcher input can reach a
 * node between the dispatcher's calls), then completes a step ending at
 * exactly t -- but begins none at t (that waits for fb_nodes_begin, after
 * routing).  delivered[i] (may be NULL): node i's newest report with
 * emitted_at + latency <= t (fresh = 1 when one arrived since the last
 * call), and busy = node busy when the clock reached t. */
int fb_nodes_advance(fb_nodes* h, int64_t t, fb_node_report* delivered);
/* Node::enqueue(rows[row[k]], t) (engine.cpp:92-105) for k < n, in order:
 * visible at the node's next begin_step (at or after t).  t is the
 * dispatcher's current time (the only form run_cluster uses). */
int fb_nodes_enqueue(fb_nodes* h, int64_t t, const int32_t* node, const int64_t* row, int64_t n);
/* Node::begin_step(t) (engine.cpp:153-202) on every idle node of
 * [node_lo, node_hi): PAB admission of its visible arrivals, batch
 * formation, launch.  Rejected rows collect for fb_nodes_drain_rejects. */
int fb_nodes_begin(fb_nodes* h, int64_t t, int32_t node_lo, int32_t node_hi);
/* Node::drain_rejects (engine.h:143-145) of every node, in node order:
 * (node, row) pairs; *n_out = count (FB_ERR_CAPACITY when cap is smaller,
 * nothing drained). */
int fb_nodes_drain_rejects(fb_nodes* h, int32_t* node_out, int64_t* row_out, int64_t cap,
                           int64_t* n_out);
/* Node::current_pab(now) (engine.cpp:123-125) of every node. */
int fb_nodes_current_pab(fb_nodes* h, int64_t now, int64_t* pab_out);
int fb_nodes_state(fb_nodes* h, fb_node_state* out);
/* Per-node results (steps, plan digest, counters; incomplete = any node
 * still live -- OR in the dispatcher's own unrouted arrivals), per-row
 * records of the node each row was last routed to (rejected only if never
 * served, metrics.cpp:96-98) and that node (-1: never routed). */
int fb_nodes_fetch(fb_nodes* h, fb_instance_result* node_results, fb_record* records,
                   int32_t* node_of_row, int32_t* incomplete_out);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* FBGPU_H_ */
