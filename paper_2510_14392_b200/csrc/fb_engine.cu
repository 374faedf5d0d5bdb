// fb_engine.cu -- the persistent per-iteration scheduling engine.
//
// One warp simulates one Node instance (engine.h:111-176) end to end: the
// run_node event loop (engine.cpp:266-288) with arrival injection, PAB
// admission, task views, batch formation and step completion, against a
// structure-of-arrays request arena in HBM.  Warps pull instances from a
// device work queue until every instance is quiescent (or the per-launch
// event budget is spent, for the step-wise API).
//
// Kernel map (north_star): K1 views/slack (load_view + the views pass), K2
// segmented slack order and K3 capacity scan (fb_sched.cuh), K4 event advance
// and arrival injection (run_instance, complete_step, pull_*), K5 load
// estimation (pull_pab / pab kernel).
// Lanes per simulated node.  16 (two nodes per warp) is supported and
// bit-exact, but slower on C2 (100 ms vs 37 ms): nodes with 17-32 live
// requests drop to the memory path and the two half-warps rarely share
// instructions.
#ifndef FB_TILE
#define FB_TILE 32
#endif
#include "fb_engine_dev.cuh"
#include "fb_wide.cuh"
#include "fb_summary.cuh"

namespace fbgpu {

size_t scratch_bytes_per_slot() { return kScratchBytesPerSlot; }
size_t dev_inst_bytes() { return sizeof(DevInst); }
size_t dev_state_bytes() { return sizeof(DevState); }

// One tile (kTile lanes) per simulated node; each tile pulls nodes from the
// work queues and runs their event loops.
__global__ void __launch_bounds__(kWarp * kWarpsPerBlock, kEngineBlocksPerSm)
engine_kernel(const __grid_constant__ EngineParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int tile = threadIdx.x / kTile;
  unsigned char* my = smem + static_cast<size_t>(tile) * kSmemSlots * kScratchBytesPerSlot;
  for (;;) {
    unsigned long long i = static_cast<unsigned long long>(P.n_inst);
    if (tile_lane() == 0) {
      for (int q = 0; q < kQueues; ++q) {
        const int64_t len = P.qoff[q + 1] - P.qoff[q];
        if (static_cast<int64_t>(*(volatile unsigned long long*)&P.work[4 + q]) >= len) continue;
        const unsigned long long k = atomicAdd(&P.work[4 + q], 1ull);
        if (static_cast<int64_t>(k) < len) {
          i = static_cast<unsigned long long>(P.order[P.qoff[q] + static_cast<int64_t>(k)]);
          break;
        }
      }
    }
    i = tile_shfl(i, 0);
    if (i >= static_cast<unsigned long long>(P.n_inst)) break;
    Inst w;
    w.id = static_cast<int64_t>(i);
    w.routed = nullptr;
    w.I = P.inst + i;
    w.S = P.state[i];
    if (w.S.done || w.S.escalated) continue;
    w.toff = w.I->trace_off;
    w.roff = w.I->rec_off;
    w.nreq = w.I->n_req;
    w.horizon = w.I->horizon;
    w.policy = w.I->policy;
    w.max_active = w.I->max_active;
    w.vl = P.vlist + w.roff;
    w.smem = my;
    w.sd.clear();
    run_instance(P, w);
    tile_sync();
    if (tile_lane() == 0) {
      P.state[i] = w.S;
      if (!w.S.done && !w.S.escalated) atomicAdd(&P.work[1], 1ull);
    }
  }
}

__global__ void reset_kernel(const __grid_constant__ EngineParams P, int64_t n_rec) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n_rec;
       i += stride) {
    P.prefilled[i] = 0;
    P.nidx[i] = 0;
    P.seq[i] = 0;
    P.flags[i] = 0;
    P.first[i] = -1;
    P.maxtp[i] = 0.0;
    P.maxtp_alt[i] = 0.0;
    P.lastem[i] = -1;
  }
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < P.n_inst;
       i += stride) {
    DevState s = {};
    s.digest = FB_DIGEST_INIT;
    P.state[i] = s;
  }
}

// Per-request records in the ABI's AoS layout (fb_record), one warp per
// instance, so a fetch is a single D2H.  Flag finishing as in
// request_reports (metrics.cpp:60-116): ARRIVED for rows the event loop
// enqueued, REJECTED only for requests that were never served.
__global__ void pack_records_kernel(const __grid_constant__ EngineParams P, fb_record* out) {
  const int64_t wpb = blockDim.x / kWarp;
  for (int64_t i = blockIdx.x * wpb + threadIdx.x / kWarp; i < P.n_inst; i += gridDim.x * wpb) {
    const int64_t b = P.inst[i].rec_off, n = P.inst[i].n_req;
    const int64_t arrived = P.state[i].arr;
    for (int64_t k = lane_id(); k < n; k += kWarp) {
      const int64_t g = b + k;
      const int32_t ni = P.nidx[g];
      uint32_t f = P.flags[g] & ~kTpotViolated;
      if (k < arrived) f |= FB_REC_ARRIVED;
      if ((f & FB_REC_REJECTED) && ni > 0) f &= ~static_cast<uint32_t>(FB_REC_REJECTED);
      fb_record r;
      r.first_emit_us = P.first[g];
      r.max_tpot_ms = P.maxtp[g];
      r.max_tpot_alt_ms = P.maxtp_alt[g];
      r.tokens_emitted = ni;
      r.flags = f;
      out[g] = r;
    }
  }
}

// ------------------------------------------------------------- host side

#ifdef FB_WIDE_PROF
extern "C" int fb_debug_wide_prof(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, g_wide_prof, sizeof(unsigned long long) * 24);
  if (reset) {
    unsigned long long z[24] = {};
    cudaMemcpyToSymbol(g_wide_prof, z, sizeof(z));
  }
  return static_cast<int>(cudaDeviceSynchronize());
}
extern "C" int fb_debug_sub_prof(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, g_sub_prof, sizeof(unsigned long long) * 256 * 8);
  if (reset) {
    static unsigned long long z[256 * 8] = {};
    cudaMemcpyToSymbol(g_sub_prof, z, sizeof(z));
  }
  return static_cast<int>(cudaDeviceSynchronize());
}
extern "C" int fb_debug_cta_prof(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, g_cta_prof, sizeof(unsigned long long) * 256 * 4);
  if (reset) {
    static unsigned long long z[256 * 4] = {};
    cudaMemcpyToSymbol(g_cta_prof, z, sizeof(z));
  }
  return static_cast<int>(cudaDeviceSynchronize());
}
#endif

cudaError_t launch_summaries(const EngineParams& p, fb_summary* out, uint64_t* vals,
                             cudaStream_t st) {
  if (p.n_inst <= 0) return cudaSuccess;
  int64_t blocks = p.n_inst < 148 * 8 ? p.n_inst : 148 * 8;
  summarize_kernel<<<static_cast<int>(blocks), kSumThreads, 0, st>>>(p, out, vals);
  return cudaGetLastError();
}

cudaError_t launch_lead(const EngineParams& p, int64_t* out, int32_t* n_out, cudaStream_t st) {
  if (p.n_inst <= 0 || p.lead_bucket <= 0) return cudaSuccess;
  int64_t blocks = p.n_inst < 148 * 8 ? p.n_inst : 148 * 8;
  lead_kernel<<<static_cast<int>(blocks), kSumThreads, 0, st>>>(p, out, n_out);
  return cudaGetLastError();
}

cudaError_t launch_pack_records(const EngineParams& p, fb_record* out, cudaStream_t st) {
  if (p.n_inst <= 0) return cudaSuccess;
  int64_t blocks = (p.n_inst + 7) / 8;
  if (blocks > 148 * 8) blocks = 148 * 8;
  pack_records_kernel<<<static_cast<int>(blocks), 256, 0, st>>>(p, out);
  return cudaGetLastError();
}

EngineGeometry engine_geometry(int device) {
  EngineGeometry g;
  g.threads = kWarp * kWarpsPerBlock;
  g.smem = static_cast<size_t>(g.threads / kTile) * kSmemSlots * kScratchBytesPerSlot;
  int sms = 148, per_sm = 1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  g.sms = sms;
  cudaFuncSetAttribute(engine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(g.smem));
#ifdef FB_ENGINE_CARVEOUT
  cudaFuncSetAttribute(engine_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                       FB_ENGINE_CARVEOUT);
#endif
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, engine_kernel, g.threads, g.smem);
  if (per_sm < 1) per_sm = 1;
  g.blocks = sms * per_sm;
  g.wide_threads = kWideThreads;
  g.wide_smem = sizeof(WideSmem);
  cudaFuncSetAttribute(wide_grid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(g.wide_smem));
  int wide_per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&wide_per_sm, wide_grid_kernel, g.wide_threads,
                                                g.wide_smem);
  if (wide_per_sm < 1) wide_per_sm = 1;
  g.wide_blocks = sms * wide_per_sm < kWgMaxSlots ? sms * wide_per_sm : kWgMaxSlots;
  return g;
}

WideGridSizes wide_grid_sizes(const EngineGeometry& g, int64_t n_rec) {
  WideGridSizes z;
  z.slot_bytes = sizeof(WideSlot) * static_cast<size_t>(g.wide_blocks);
  // one partial row per (CTA, slot)
  (void)n_rec;
  z.partial_rows = static_cast<size_t>(g.wide_blocks) * g.wide_blocks * kK1Vals;
  z.hist_words = static_cast<size_t>(g.wide_blocks) * kSelBins;
  z.cand_rows = static_cast<size_t>(g.wide_blocks) * kWideWin;
  return z;
}

void pack_instance(const fb_instance& in, int64_t rec_off, int64_t log_step_off,
                   int64_t log_entry_off, int64_t log_reject_off, int64_t tpot_uniform,
                   bool wide_ok, void* out) {
  DevInst d;
  std::memset(&d, 0, sizeof(d));
  const fb_engine_config& c = in.cfg;
  d.sa = c.scheduler.model.a_ms;
  d.sb = c.scheduler.model.b_ms;
  d.sc = c.scheduler.model.c_ms;
  d.ta = c.truth_model.a_ms;
  d.tb = c.truth_model.b_ms;
  d.tc = c.truth_model.c_ms;
  d.noise_amp = c.noise_amplitude;
  d.noise_seed = c.noise_seed;
  d.token_budget = c.scheduler.token_budget;
  d.g_ttft = c.global_ttft_us;
  d.g_tpot = c.global_tpot_us;
  d.horizon = in.horizon_us;
  d.trace_off = in.trace_off;
  d.rec_off = rec_off;
  d.n_req = in.n_req;
  d.log_step_off = log_step_off;
  d.log_entry_off = log_entry_off;
  d.log_reject_off = log_reject_off;
  d.tpot_uniform = tpot_uniform;
  d.policy = c.scheduler.policy;
  d.max_chunk = c.scheduler.max_chunk;
  d.max_active = c.max_active;
  d.wide_ok = wide_ok ? 1 : 0;
  std::memcpy(out, &d, sizeof(d));
}

void unpack_state(const void* state, fb_instance_result* out) {
  DevState s;
  std::memcpy(&s, state, sizeof(s));
  out->steps = s.step_counter;
  out->plan_digest = s.digest;
  out->end_time_us = s.t_last;
  out->n_arrived = s.arr;
  out->n_rejected = s.n_rejected;
  out->sum_visible = s.sum_visible;
  out->sum_entries = s.sum_entries;
  out->sum_new_tokens = s.sum_new;
  out->incomplete = s.incomplete;
  out->status = s.status;
}

cudaError_t launch_reset(const EngineParams& p, int64_t n_rec, cudaStream_t st) {
  int64_t n = n_rec > p.n_inst ? n_rec : p.n_inst;
  int blocks = static_cast<int>((n + 255) / 256);
  if (blocks < 1) blocks = 1;
  if (blocks > 148 * 16) blocks = 148 * 16;
  cudaMemsetAsync(p.work, 0, 4 * sizeof(unsigned long long), st);
  reset_kernel<<<blocks, 256, 0, st>>>(p, n_rec);
  return cudaGetLastError();
}

cudaError_t launch_engine(const EngineParams& p, const EngineGeometry& g, cudaStream_t st,
                          cudaEvent_t between) {
  cudaMemsetAsync(p.work, 0, 3 * sizeof(unsigned long long), st);
  cudaMemsetAsync(p.work + 4, 0, kQueues * sizeof(unsigned long long), st);
  static_assert(4 + kQueues <= 16, "work counters");
  engine_kernel<<<g.blocks, g.threads, g.smem, st>>>(p);
  if (between) cudaEventRecord(between, st);
  // Escalated instances (more than kEscalateLive live requests) continue on
  // the grid-wide wide engine; with none escalated it exits after one barrier.
  cudaMemsetAsync(p.wg.bar, 0, 16 * sizeof(unsigned long long), st);  // barrier + phase clock
  EngineParams pp = p;
  void* args[] = {&pp};
  // cooperative: every CTA must be co-resident for the grid barriers
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(wide_grid_kernel),
                                     dim3(g.wide_blocks), dim3(g.wide_threads), args,
                                     g.wide_smem, st);
}

}  // namespace fbgpu
