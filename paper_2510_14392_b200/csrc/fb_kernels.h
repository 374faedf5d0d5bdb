// fb_kernels.h -- host-visible launch wrappers for the device kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/fbgpu.h"

namespace fbgpu {

struct DevInst;
struct DevState;

// Buffers of the grid-wide wide engine (fb_wide.cuh), one slot per CTA.
struct WideGridBufs {
  void* slots;               // WideSlot[n_slots]
  int64_t* partial;          // [max_chunks][8] K1 partial reductions
  uint32_t* hist;            // [n_slots][kSelBins]
  uint64_t* ckey;            // [n_slots][kWideWin] gathered window keys
  int32_t* cpos;             // [n_slots][kWideWin] their view positions
  unsigned long long* bar;   // [0] grid barrier counter, [8..12] phase ns, [13] iterations
                             // (zeroed per launch)
};

// Everything the engine kernel touches, as device pointers.
struct EngineParams {
  const DevInst* inst;
  DevState* state;
  int64_t n_inst;
  // trace rows
  const int64_t* arrival;
  const int32_t* prompt;
  const int32_t* output;
  const int64_t* ttft;
  const int64_t* tpot;
  // per-request state (indexed by rec_off + row)
  int32_t* prefilled;
  int32_t* nidx;
  int32_t* seq;
  uint32_t* flags;
  int64_t* first;
  double* maxtp;
  double* maxtp_alt;
  int2* vlist;                   // [rec_off + i] = {row, take}
  unsigned char* gscratch;       // [rec_off * kScratchBytesPerSlot ...]
  // logs (null when off)
  fb_step_log* log_steps;
  fb_plan_entry* log_entries;
  fb_reject_log* log_rejects;
  int32_t log_step_cap, log_entry_cap, log_reject_cap, log_on;
  // persistent work queues: [0] next instance (warp engine), [1] instances
  // still running after the launch, [2] next escalated instance (wide engine),
  // [3] number of escalated instances (list in wide_list)
  unsigned long long* work;
  int64_t* wide_list;
  // Work queues (host-ordered, scheduling only): queue 0 holds the instances
  // whose predicted cost is at least half the largest (any policy), highest
  // first; queues 1..4 hold the rest by policy (fairbatch_pab, fairbatch,
  // sarathi, prefill_first), highest cost first.  Warps drain them in that
  // order, so apart from the long-tail head every SM runs one policy's code
  // at a time -- the engine is instruction-fetch bound and mixing policies
  // on an SM thrashes its instruction cache (C2: 44 -> 37 ms).
  // order[qoff[q] .. qoff[q+1]) is queue q; work[4 + q] its next index.
  const int64_t* order;
  const int64_t* qoff;  // [kQueues + 1]
  // envelope-lead accounting (lead_bucket > 0): per instance, emitted tokens
  // [0, cap) and finished requests' output tokens [cap, 2 cap) per bucket
  // index ceil(t / bucket); latest emission; overflow flag
  int64_t lead_bucket;
  int32_t lead_cap, pad_lead;
  unsigned long long* lead_hist;  // [n_inst][2 cap]
  long long* lead_tmax;           // [n_inst]
  int32_t* lead_flags;            // [n_inst]
  int64_t* lastem;                // [rec_off + row] last token of a finished request (lead on)
  int64_t max_events;  // per instance per launch
  WideGridBufs wg;
};

constexpr int kQueues = 5;  // long-tail head + one per FB_POLICY_*

// Per-launch geometry of the persistent engine kernel.
struct EngineGeometry {
  int blocks;
  int threads;
  size_t smem;
  int wide_blocks;  // grid-wide wide engine: one cooperative CTA (slot) per SM
  int wide_threads;
  size_t wide_smem;
  int sms;
};
// Sizes of the grid-wide wide engine's buffers for a given geometry.
struct WideGridSizes {
  size_t slot_bytes, partial_rows, hist_words, cand_rows;
};
WideGridSizes wide_grid_sizes(const EngineGeometry& g, int64_t n_rec);

EngineGeometry engine_geometry(int device);
size_t scratch_bytes_per_slot();
size_t dev_inst_bytes();
size_t dev_state_bytes();

// Host packing of fb_instance into the device layout (rec_off / log offsets
// assigned by the caller).
void pack_instance(const fb_instance& in, int64_t rec_off, int64_t log_step_off,
                   int64_t log_entry_off, int64_t log_reject_off, int64_t tpot_uniform,
                   bool wide_ok,
                   void* out);
// Host decode of a DevState into fb_instance_result.
void unpack_state(const void* state, fb_instance_result* out);

cudaError_t launch_reset(const EngineParams& p, int64_t n_rec_rows, cudaStream_t st);
// Per-instance ScenarioReport aggregates (fb_summary.cuh); vals holds one
// u64 per request row (value series of large instances).
cudaError_t launch_summaries(const EngineParams& p, fb_summary* out, uint64_t* vals,
                             cudaStream_t st);
// Envelope-lead series per instance (fb_summary.cuh) into out[inst][cap];
// n_out[inst] = points, or -1 when the bucket capacity overflowed.
cudaError_t launch_lead(const EngineParams& p, int64_t* out, int32_t* n_out, cudaStream_t st);
// Records in fb_record layout, indexed by rec_off + row.
cudaError_t launch_pack_records(const EngineParams& p, fb_record* out, cudaStream_t st);

// Cluster (fb_cluster.cuh): mirrors ClusterParams field for field.
constexpr int kClusterHostMaxRanks = 8;
struct ClusterParamsHost {
  int32_t n_nodes, lb_policy, interval, report_cap;
  int64_t latency, horizon, n_rows, n_epochs;
  double w_waiting, w_running;
  const int64_t* epoch_t;
  const int64_t* epoch_lo;
  int32_t* routed;
  int32_t* route_node;
  int64_t* rep;
  int64_t* out;
  int32_t node_lo, n_local;
  int32_t rank, n_ranks;
  int32_t warps_per_cta, total_ctas;
  int64_t timeout_ns;
  unsigned char* xbuf[kClusterHostMaxRanks];
  int64_t route_stride;
  int32_t retry_reroute, fifo_cap;
  int64_t* fifo;
  uint8_t* row_state;
  fb_route_log* rlog;  // routing log (NULL: off), [rlog_cap]
  double* rsnap;       // its view snapshots, [rlog_cap * n_nodes]
  int64_t rlog_cap;
  int32_t hw_cluster, pad_hw;  // set by launch_cluster
};
size_t cluster_param_bytes();
int cluster_max_nodes();
int cluster_max_ranks();
size_t cluster_xchg_bytes(int n_nodes);
// Warps (nodes) per CTA, shared by all ranks, and this rank's CTA count.
int cluster_warps_per_cta(int n_nodes, int n_ranks);
size_t cluster_smem_bytes(int warps_per_cta);
cudaError_t launch_cluster_serial(const EngineParams& p, const ClusterParamsHost& c,
                                  cudaStream_t st);
// hw_mode: a one-rank grid of <= 8 CTAs may run as one thread-block cluster,
// with one (1) or two (2) CTAs per SM; 0 = cooperative grid.
cudaError_t launch_cluster(const EngineParams& p, const ClusterParamsHost& c, int blocks,
                           cudaStream_t st, int hw_mode = 1);
// How many one-cluster grids of an n_nodes cluster fit the device at once.
int cluster_max_hw_clusters(int n_nodes, int ctas_per_sm = 1);
// Interactive node set (fb_nodes_*, fb_cluster.cuh): ops and NodesIo.
constexpr int32_t kNodesInitOp = 0, kNodesAdvanceOp = 1, kNodesBeginOp = 2, kNodesPabOp = 3,
                  kNodesStateOp = 4, kNodesFinishOp = 5;
struct NodesIoHost {
  int32_t op, lo, hi, reports;
  int64_t t;
  int64_t* rep_ht;
  int64_t* rej;
  int64_t* n_rej;
  int64_t rej_cap;
  int64_t* out;
  int32_t* status;
};
cudaError_t launch_nodes(const EngineParams& p, const ClusterParamsHost& c, const NodesIoHost& io,
                         cudaStream_t st);
cudaError_t launch_nodes_enqueue(const EngineParams& p, const ClusterParamsHost& c, int64_t t,
                                 const int32_t* node, const int64_t* row, int64_t n,
                                 int32_t* status, cudaStream_t st);
// Warp engine, then the grid-wide wide engine; `between` (may be null) is
// recorded between the two launches.
cudaError_t launch_engine(const EngineParams& p, const EngineGeometry& g,
                          cudaStream_t st, cudaEvent_t between = nullptr);

// Pure scheduler surface.  `scratch` must hold total_tasks slots.
cudaError_t launch_form_batch(const fb_task_view* tasks, const int64_t* set_off,
                              const fb_scheduler_config* cfgs, int64_t n_sets,
                              fb_plan_entry_id* entries, fb_batch_plan* plans,
                              unsigned char* scratch, int* status, cudaStream_t st);
cudaError_t launch_init_time_budget(const fb_task_view* tasks, const int64_t* set_off,
                                    int64_t n_sets, int64_t* out, int* status,
                                    cudaStream_t st);
cudaError_t launch_pab(const fb_task_view* tasks, const int64_t* set_off,
                       const fb_cost_model* models, const int64_t* ttft,
                       const int64_t* tpot, int64_t n_sets, int64_t* out,
                       unsigned char* scratch, cudaStream_t st);

}  // namespace fbgpu
