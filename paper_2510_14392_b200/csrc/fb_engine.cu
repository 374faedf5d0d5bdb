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
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "fb_kernels.h"
#include "fb_sched.cuh"

namespace fbgpu {

#ifndef FB_WARPS_PER_BLOCK
#define FB_WARPS_PER_BLOCK 8
#endif
constexpr int kWarpsPerBlock = FB_WARPS_PER_BLOCK;
constexpr int kSmemSlots = 64;  // visible tasks held in shared-memory scratch
#ifndef FB_ENGINE_BLOCKS_PER_SM
#define FB_ENGINE_BLOCKS_PER_SM 2
#endif
constexpr int kEngineBlocksPerSm = FB_ENGINE_BLOCKS_PER_SM;  // register cap for occupancy
constexpr int64_t kEscalateLive = 512;  // live requests beyond which a node goes CTA-wide

size_t scratch_bytes_per_slot() { return kScratchBytesPerSlot; }
size_t dev_inst_bytes() { return sizeof(DevInst); }
size_t dev_state_bytes() { return sizeof(DevState); }

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Warp-uniform view of one instance while a warp owns it.
struct Inst {
  int64_t id;
  const int32_t* routed;  // cluster node: pending slot -> trace row (else identity)
  const DevInst* I;
  DevState S;
  int64_t toff, roff, nreq, horizon;
  int32_t policy, max_active;
  int2* vl;
  unsigned char* smem;  // this warp's shared scratch
};

// Trace row of the q-th request that reached this node (run_node: the trace
// itself; cluster nodes: the router's append order).
__device__ __forceinline__ int64_t arrival_row(const Inst& w, int64_t q) {
  return w.routed ? static_cast<int64_t>(w.routed[q]) : q;
}

__device__ __forceinline__ int64_t visible_count(const Inst& w) {
  int64_t nw = w.S.n_live - w.S.n_active;
  if (w.max_active > 0) {
    int64_t slots = static_cast<int64_t>(w.max_active) - w.S.n_active;
    if (slots < 0) slots = 0;
    if (nw > slots) nw = slots;
  }
  return w.S.n_active + nw;
}

__device__ __forceinline__ Scratch scratch_for(const EngineParams& P, const Inst& w,
                                               int64_t A) {
  if (A <= kSmemSlots) return carve_scratch(w.smem, kSmemSlots);
  return carve_scratch(P.gscratch + w.roff * kScratchBytesPerSlot, static_cast<int>(w.nreq));
}

// K1: one task view (build_task_views, engine.cpp:51-81; slack, slo.h:45-61).
struct View {
  int32_t r;
  int32_t nw;  // new tokens | kDecodeBit
  int64_t slack, ctx, tpot, seq;
  bool decode;
};

__device__ __forceinline__ View load_view(const EngineParams& P, const Inst& w,
                                          int64_t p, int64_t now) {
  View v;
  v.r = w.vl[p].x;
  const int64_t g = w.roff + v.r;
  const int64_t row = w.toff + v.r;
  const int32_t prompt = P.prompt[row];
  const int32_t pf = P.prefilled[g];
  const int32_t ni = P.nidx[g];
  v.tpot = P.tpot[row];
  const int64_t ttft_deadline = P.arrival[row] + P.ttft[row];
  v.seq = P.seq[g];
  if (pf < prompt) {
    v.decode = false;
    v.nw = prompt - pf;
    v.ctx = pf;
    v.slack = ttft_deadline + v.tpot * static_cast<int64_t>(ni) - now;
  } else {
    v.decode = true;
    v.nw = 1 | static_cast<int32_t>(kDecodeBit);
    v.ctx = static_cast<int64_t>(prompt) + ni;
    int64_t anchor = ttft_deadline;
    const int64_t f = P.first[g];
    if (f >= 0 && f < anchor) anchor = f;  // min(arrival+ttft, first emit)
    v.slack = anchor + v.tpot * static_cast<int64_t>(ni) - now;
  }
  return v;
}

// Token emission (engine.cpp:211-232) + online RequestReport bookkeeping
// (metrics.cpp:42-60, 196-214).  Returns true when the request finished.
__device__ __forceinline__ bool emit_token(const EngineParams& P, int64_t g, int64_t row,
                                           int64_t t) {
  const int32_t idx = P.nidx[g];
  const int64_t arr = P.arrival[row];
  const int64_t ttft = P.ttft[row];
  const int64_t tpot = P.tpot[row];
  uint32_t fl = P.flags[g];
  if (idx == 0) {
    P.first[g] = t;
    if (t - arr <= ttft) fl |= FB_REC_MET_TTFT;
  } else {
    const int64_t d = t - P.first[g];
    if (d > tpot * static_cast<int64_t>(idx)) fl |= kTpotViolated;
    double m = P.maxtp[g];
    max_ratio(m, d, idx);  // std::max(best, x)
    P.maxtp[g] = m;
    if (idx >= 2) {
      double ma = P.maxtp_alt[g];
      max_ratio(ma, d, idx - 1);
      P.maxtp_alt[g] = ma;
    }
    if (t - arr > ttft + tpot * static_cast<int64_t>(idx)) fl |= FB_REC_ENV_MISS;
  }
  const int32_t ni = idx + 1;
  P.nidx[g] = ni;
  const bool fin = ni >= P.output[row];
  if (fin) {
    fl |= FB_REC_FINISHED;
    if (!(fl & kTpotViolated)) fl |= FB_REC_MET_TPOT;
  }
  P.flags[g] = fl;
  return fin;
}

// Order-preserving removal of finished entries (row < 0) from vlist[0, n_live)
// (active_.erase, engine.cpp:228-229), clearing the in-flight takes.
__device__ __forceinline__ void compact_vlist(Inst& w) {
  const int64_t n = w.S.n_live;
  int64_t out = 0;
  int64_t removed_active = 0;
  for (int64_t b = 0; b < n; b += kWarp) {
    const int64_t p = b + lane_id();
    int2 v = make_int2(-1, 0);
    if (p < n) v = w.vl[p];
    const bool keep = p < n && v.x >= 0;
    const unsigned m = __ballot_sync(kFull, keep);
    const unsigned rm = __ballot_sync(kFull, p < n && !keep && p < w.S.n_active);
    __syncwarp();
    if (keep) w.vl[out + __popc(m & lanemask_lt())] = make_int2(v.x, 0);
    out += __popc(m);
    removed_active += __popc(rm);
    __syncwarp();
  }
  w.S.n_live = out;
  w.S.n_active -= removed_active;
}

// Node::complete_step, engine.cpp:204-254.  In-flight plan entries are the
// active tasks with a nonzero take (plan order only affects the event log).
__device__ __noinline__ void complete_step(const EngineParams& P, Inst& w) {
  const int64_t t = w.S.step_end;
  bool any_fin = false;
  for (int64_t b = 0; b < w.S.n_active; b += kWarp) {
    const int64_t p = b + lane_id();
    bool fin = false;
    if (p < w.S.n_active) {
      const int2 v = w.vl[p];
      if (v.y > 0) {
        const int64_t g = w.roff + v.x;
        const int64_t row = w.toff + v.x;
        const int32_t prompt = P.prompt[row];
        int32_t pf = P.prefilled[g];
        bool emit = true;
        if (pf < prompt) {
          pf += v.y;
          P.prefilled[g] = pf;
          emit = pf >= prompt;  // the completing chunk yields token 0
        }
        if (emit) fin = emit_token(P, g, row, t);
        if (fin) w.vl[p].x = -1;
      }
    }
    any_fin |= __any_sync(kFull, fin);
  }
  __syncwarp();
  if (any_fin) compact_vlist(w);
  w.S.busy = 0;
}

// Node::pull_arrivals without admission control (engine.cpp:127-151).
__device__ __forceinline__ void pull_plain(const EngineParams& P, Inst& w) {
  const int64_t k = w.S.arr - w.S.pulled;
  for (int64_t j = lane_id(); j < k; j += kWarp) {
    const int64_t r = arrival_row(w, w.S.pulled + j);
    P.seq[w.roff + r] = static_cast<int32_t>(w.S.seq_counter + j);
    w.vl[w.S.n_live + j] = make_int2(static_cast<int>(r), 0);
  }
  __syncwarp();
  w.S.seq_counter += k;
  w.S.n_live += k;
  w.S.pulled = w.S.arr;
}

// K5: Node::pull_arrivals with PAB admission (engine.cpp:127-151, pab
// sched.cpp:248-278).  The view fold is computed once in view order; every
// admitted, visible arrival then appends exactly one term, which is the same
// left-to-right fold the reference recomputes per arrival.
__device__ void pull_pab(const EngineParams& P, Inst& w, int64_t now) {
  const DevInst* I = w.I;
  const double Wm = us_to_ms(I->g_ttft), Tm = us_to_ms(I->g_tpot);
  const double a = I->sa, b = I->sb, c = I->sc;
  int64_t A = visible_count(w);
  const Scratch s = scratch_for(P, w, A);
  int64_t lmin = kInf, lpf = 0;
  for (int64_t p = lane_id(); p < A; p += kWarp) {
    const View v = load_view(P, w, p, now);
    s.tcost[p] = pab_term(Wm, Tm, b, c, v.slack, v.ctx);
    lmin = v.slack < lmin ? v.slack : lmin;
    if (!v.decode) lpf += v.nw;
  }
  __syncwarp();
  int64_t min_slack = warp_min_i64(lmin);
  int64_t pf_tok = warp_sum_small(lpf);
  double r_tasks = ordered_fold(s.tcost, static_cast<int>(A));
  for (int64_t q = w.S.pulled; q < w.S.arr; ++q) {
    const int64_t r = arrival_row(w, q);
    const int64_t row = w.toff + r;
    const int64_t prompt = P.prompt[row];
    const int64_t budget = pab_close(Wm, Tm, a, b, c, A > 0, min_slack, r_tasks, pf_tok);
    if (prompt <= budget) {  // admit, sched.h:113-115
      bool vis = true;
      if (w.max_active > 0) {
        int64_t slots = static_cast<int64_t>(w.max_active) - w.S.n_active;
        if (slots < 0) slots = 0;
        vis = (w.S.n_live - w.S.n_active) < slots;
      }
      if (lane_id() == 0) {
        P.seq[w.roff + r] = static_cast<int32_t>(w.S.seq_counter);
        w.vl[w.S.n_live] = make_int2(static_cast<int>(r), 0);
      }
      w.S.seq_counter++;
      w.S.n_live++;
      if (vis) {
        const int64_t slack = P.arrival[row] + P.ttft[row] - now;  // fresh prefill
        r_tasks = dadd(r_tasks, pab_term(Wm, Tm, b, c, slack, 0));
        min_slack = slack < min_slack ? slack : min_slack;
        pf_tok += prompt;
        A++;
      }
    } else {
      if (lane_id() == 0) {
        P.flags[w.roff + r] |= FB_REC_REJECTED;
        if (P.log_on) {
          if (w.S.log_rejects < P.log_reject_cap) {
            fb_reject_log& rl = P.log_rejects[I->log_reject_off + w.S.log_rejects];
            rl.t_us = now;
            rl.pab_tokens = budget;
            rl.req = static_cast<int32_t>(r);
            rl.reserved = 0;
          }
        }
      }
      if (P.log_on) {
        if (w.S.log_rejects < P.log_reject_cap) {
          w.S.log_rejects++;
        } else {
          w.S.log_trunc = 1;
        }
      }
      w.S.digest = fb_digest_reject(w.S.digest, now, static_cast<uint32_t>(r), budget);
      w.S.n_rejected++;
    }
  }
  __syncwarp();
  w.S.pulled = w.S.arr;
}

// Node::begin_step, engine.cpp:153-202.  Returns false when there is nothing
// to schedule (no step launched, no step ordinal consumed).
__device__ __noinline__ bool begin_step(const EngineParams& P, Inst& w, int64_t now) {
  const DevInst* I = w.I;
  if (w.S.pulled < w.S.arr) {
    if (w.policy == FB_POLICY_FAIRBATCH_PAB) {
      pull_pab(P, w, now);
    } else {
      pull_plain(P, w);
    }
  }
  const int64_t A = visible_count(w);
  if (A == 0) return false;
  const Scratch s = scratch_for(P, w, A);

  // K1: views, envelope slack and the init_time_budget reductions.
  ViewAcc acc;
  for (int64_t p = lane_id(); p < A; p += kWarp) {
    const View v = load_view(P, w, p, now);
    s.slack[p] = v.slack;
    s.seq[p] = v.seq;
    s.ctx[p] = v.ctx;
    s.nw[p] = v.nw;
    s.req[p] = v.r;
    acc.add(v.decode, v.slack, v.tpot);
  }
  __syncwarp();
  acc.reduce();

  // K2 + K3
  FormCfg f;
  f.policy = w.policy;
  f.max_chunk = I->max_chunk;
  f.token_budget = I->token_budget;
  f.a = I->sa;
  f.b = I->sb;
  f.c = I->sc;
  const int Ai = static_cast<int>(A);
  const FormOut o = form_batch_warp(s, Ai, acc, f, /*seq_unique=*/true);

  // ground_truth_step_time_ms, costmodel.cpp:138-146
  double actual = predict_ms(I->ta, I->tb, I->tc, o.total_new, o.total_ctx);
  const double amp = I->noise_amp;
  if (amp != 0.0) {
    actual = apply_noise(actual, amp, I->noise_seed, w.S.step_counter);
  }
  int64_t dur = ms_to_us(actual);
  if (dur < 1) dur = 1;  // engine.cpp:196-198

  // Bookkeeping over the plan in admission order: digest, log, and the
  // waiting -> active move (engine.cpp:176-182) as new vlist positions.
  const int64_t n_act = w.S.n_active;
  const bool log_ok = P.log_on && w.S.log_steps < P.log_step_cap &&
                      w.S.log_entries + o.n_entries <= P.log_entry_cap;
  const int64_t entry_base = I->log_entry_off + w.S.log_entries;
  int run_all = 0, run_w = 0;
  uint64_t esum = 0;
  for (int k0 = 0; k0 < Ai; k0 += kWarp) {
    const int k = k0 + lane_id();
    int tk = 0, p = 0;
    if (k < Ai) {
      p = s.order[k];
      tk = s.take[k];
    }
    const bool adm = tk > 0;
    const unsigned m = __ballot_sync(kFull, adm);
    const bool wadm = adm && p >= n_act;
    const unsigned mw = __ballot_sync(kFull, wadm);
    if (adm) {
      const int idx = run_all + __popc(m & lanemask_lt());
      const int r = s.req[p];
      esum ^= fb_digest_entry(static_cast<uint32_t>(idx), static_cast<uint32_t>(r),
                              static_cast<uint32_t>(tk));
      if (log_ok) P.log_entries[entry_base + idx] = fb_plan_entry{r, tk};
    }
    if (k < Ai) {
      const int64_t np = p < n_act ? p : (wadm ? n_act + run_w + __popc(mw & lanemask_lt()) : -1);
      s.slack[p] = (np << 32) | static_cast<uint32_t>(tk);
    }
    run_all += __popc(m);
    run_w += __popc(mw);
  }
  __syncwarp();
  esum = warp_xor_u64(esum);
  // unadmitted visible waiting keep their relative order after the movers
  int run_u = 0;
  const int64_t base_u = n_act + run_w;
  for (int64_t p0 = n_act; p0 < A; p0 += kWarp) {
    const int64_t p = p0 + lane_id();
    bool un = false;
    if (p < A) un = (s.slack[p] >> 32) < 0;
    const unsigned mu = __ballot_sync(kFull, un);
    if (un) s.slack[p] = (static_cast<int64_t>(base_u + run_u + __popc(mu & lanemask_lt())) << 32);
    run_u += __popc(mu);
  }
  __syncwarp();
  for (int64_t p = lane_id(); p < A; p += kWarp) {
    const int64_t pk = s.slack[p];
    w.vl[pk >> 32] = make_int2(s.req[p], static_cast<int32_t>(pk & 0xffffffff));
  }
  __syncwarp();

  if (P.log_on) {
    if (log_ok) {
      if (lane_id() == 0) {
        fb_step_log& sl = P.log_steps[I->log_step_off + w.S.log_steps];
        sl.t_us = now;
        sl.duration_us = dur;
        sl.predicted_ms = o.predicted_ms;
        sl.actual_ms = actual;
        sl.total_new = o.total_new;
        sl.total_ctx = o.total_ctx;
        sl.init_budget_ms = o.init_ms;
        sl.entry_off = w.S.log_entries;
        sl.n_entries = o.n_entries;
      }
      w.S.log_steps++;
      w.S.log_entries += o.n_entries;
    } else {
      w.S.log_trunc = 1;
    }
  }
  w.S.digest = fb_digest_step(w.S.digest, now, static_cast<uint32_t>(o.n_entries), esum,
                              o.predicted_ms, actual);
  w.S.sum_visible += A;
  w.S.sum_entries += o.n_entries;
  w.S.sum_new += o.total_new;
  w.S.n_active = n_act + run_w;
  w.S.busy = 1;
  w.S.step_end = now + dur;
  w.S.step_counter++;
  return true;
}

}  // namespace fbgpu

#include "fb_engine_rr.cuh"
#include "fb_wide.cuh"
#include "fb_cluster.cuh"
#include "fb_summary.cuh"

namespace fbgpu {

// run_node's event loop (engine.cpp:266-288) for up to max_events times t.
// Steps run on the register-resident path while at most 32 requests are live
// and on the memory path otherwise; the switch happens at step boundaries.
__device__ void run_instance(const EngineParams& P, Inst& w) {
  const int64_t* arrival = P.arrival + w.toff;
  const Scratch s = carve_scratch(w.smem, kSmemSlots);
  TaskReg tk = {};
  bool rr = false;
  int64_t next_arr = w.S.arr < w.nreq ? arrival[w.S.arr] : kInf;
  for (int64_t ev = 0; ev < P.max_events; ++ev) {
    if (w.S.busy && next_arr < w.S.step_end) {
      // Arrivals strictly before the in-flight step's end only enqueue
      // (run_node's loop neither completes nor begins a step at those times):
      // consume them 32 at a time.
      for (;;) {
        const int64_t q = w.S.arr + lane_id();
        const bool early = q < w.nreq && arrival[q] < w.S.step_end;
        const int n = __popc(__ballot_sync(kFull, early));
        w.S.arr += n;
        if (n < kWarp) break;
      }
      next_arr = w.S.arr < w.nreq ? arrival[w.S.arr] : kInf;
    }
    const int64_t t_step = w.S.busy ? w.S.step_end : kInf;
    const int64_t t = t_step < next_arr ? t_step : next_arr;
    if (t == kInf || (!w.S.busy && t >= w.horizon)) {
      if (rr) rr_spill(P, w, tk);
      w.S.done = 1;
      w.S.incomplete = (w.S.busy || w.S.pulled < w.S.arr || w.S.n_live > 0 ||
                        w.S.arr < w.nreq) ? 1 : 0;
      return;
    }
    w.S.t_last = t;
    if (w.S.busy && t_step == t) {
      if (rr) {
        complete_rr(P, w, tk);
      } else {
        complete_step(P, w);
      }
    }
    while (next_arr == t) {  // Node::enqueue (visible at its arrival time)
      w.S.arr++;
      next_arr = w.S.arr < w.nreq ? arrival[w.S.arr] : kInf;
    }
    if (!w.S.busy && t < w.horizon) {
      const int64_t upcoming = w.S.n_live + (w.S.arr - w.S.pulled);
      if (upcoming > kEscalateLive) {  // hand over to the CTA-wide engine
        if (rr) rr_spill(P, w, tk);
        w.S.pending_begin = 1;
        w.S.escalated = 1;
        if (lane_id() == 0) {
          const unsigned long long slot = atomicAdd(&P.work[3], 1ull);
          P.wide_list[slot] = w.id;
        }
        return;
      }
      if (rr && upcoming > kWarp) {
        rr_spill(P, w, tk);
        rr = false;
      } else if (!rr && upcoming <= kWarp) {
        rr_load(P, w, tk);
        rr = true;
        w.S.paths |= kPathRegister;
      }
      if (rr) {
        if (begin_rr(P, w, tk, t, s) < 0) {  // keys outside the packed range
          rr_spill(P, w, tk);
          rr = false;
          begin_step(P, w, t);
          w.S.paths |= kPathMemory;
        }
      } else {
        begin_step(P, w, t);
        w.S.paths |= kPathMemory;
      }
    }
  }
  if (rr) rr_spill(P, w, tk);
}

__global__ void __launch_bounds__(kWarp * kWarpsPerBlock, kEngineBlocksPerSm)
engine_kernel(const __grid_constant__ EngineParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x / kWarp;
  unsigned char* my = smem + static_cast<size_t>(warp) * kSmemSlots * kScratchBytesPerSlot;
  for (;;) {
    unsigned long long i = static_cast<unsigned long long>(P.n_inst);
    if (lane_id() == 0) {
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
    i = __shfl_sync(kFull, i, 0);
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
    run_instance(P, w);
    __syncwarp();
    if (lane_id() == 0) {
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
  g.smem = static_cast<size_t>(kWarpsPerBlock) * kSmemSlots * kScratchBytesPerSlot;
  int sms = 148, per_sm = 1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  g.sms = sms;
  cudaFuncSetAttribute(engine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(g.smem));
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
                   void* out) {
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

size_t cluster_param_bytes() { return sizeof(ClusterParams); }
int cluster_max_nodes() { return kClusterMaxNodes; }
int cluster_max_ranks() { return kClusterMaxRanks; }
size_t cluster_xchg_bytes(int n_nodes) {
  return kXchgHeader + 2 * sizeof(NodeReport) * static_cast<size_t>(n_nodes);
}

int cluster_warps_per_cta(int n_nodes, int n_ranks) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms < 1) sms = 148;
  const int max_local = (n_nodes + n_ranks - 1) / n_ranks;
  // Full CTAs of kClusterMaxWarps nodes: the per-epoch exchange barrier
  // then has few participants (C5, 64 nodes: 8 CTAs 208 ms vs 64 CTAs of
  // one node 227 ms); more nodes than SMs x 8 still spread over every SM.
  int w = (max_local + sms - 1) / sms;
  if (w < kClusterMaxWarps) w = max_local < kClusterMaxWarps ? max_local : kClusterMaxWarps;
  if (w > kClusterMaxWarps) w = kClusterMaxWarps;
  (void)sms;
  return w < 1 ? 1 : w;
}

size_t cluster_smem_bytes(int warps_per_cta) {
  return ((sizeof(RouterSmem) + 15) / 16) * 16 +
         static_cast<size_t>(warps_per_cta) * kSmemSlots * kScratchBytesPerSlot;
}

cudaError_t launch_cluster(const EngineParams& p, const ClusterParamsHost& ch, int blocks,
                           cudaStream_t st) {
  static_assert(sizeof(ClusterParamsHost) == sizeof(ClusterParams), "cluster params layout");
  ClusterParams c;
  std::memcpy(&c, &ch, sizeof(c));
  if (c.warps_per_cta < 1 || c.warps_per_cta > kClusterMaxWarps) return cudaErrorInvalidValue;
  const size_t smem = cluster_smem_bytes(c.warps_per_cta);
  cudaError_t e = cudaFuncSetAttribute(cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  EngineParams pp = p;
  void* args[] = {&pp, &c};
  // cooperative: every CTA must be co-resident for the epoch barrier
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(cluster_kernel), dim3(blocks),
                                     dim3(kWarp * c.warps_per_cta), args, smem, st);
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

// ------------------------------------------------- pure scheduler kernels

__device__ __forceinline__ Scratch set_scratch(unsigned char* smem_warp, unsigned char* g,
                                               int64_t off, int64_t n) {
  if (n <= kSmemSlots) return carve_scratch(smem_warp, kSmemSlots);
  return carve_scratch(g + off * kScratchBytesPerSlot, static_cast<int>(n));
}

// form_batch (sched.cpp:234-246) per task set, one warp per set.
__global__ void __launch_bounds__(kWarp * kWarpsPerBlock)
form_batch_kernel(const fb_task_view* __restrict__ tasks, const int64_t* __restrict__ set_off,
                  const fb_scheduler_config* __restrict__ cfgs, int64_t n_sets,
                  fb_plan_entry_id* __restrict__ entries, fb_batch_plan* __restrict__ plans,
                  unsigned char* gscratch, int* status) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x / kWarp;
  unsigned char* my = smem + static_cast<size_t>(warp) * kSmemSlots * kScratchBytesPerSlot;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kWarpsPerBlock;
  for (int64_t set = static_cast<int64_t>(blockIdx.x) * kWarpsPerBlock + warp; set < n_sets;
       set += nwarps) {
    const int64_t off = set_off[set];
    const int64_t n = set_off[set + 1] - off;
    const fb_scheduler_config cfg = cfgs[set];
    const bool fair = cfg.policy == FB_POLICY_FAIRBATCH || cfg.policy == FB_POLICY_FAIRBATCH_PAB;
    if (n == 0) {
      if (lane_id() == 0) {
        if (fair) atomicExch(status, FB_ERR_USAGE);  // init_time_budget on empty
        fb_batch_plan pl = {};
        pl.entry_off = off;
        plans[set] = pl;
      }
      continue;
    }
    const Scratch s = set_scratch(my, gscratch, off, n);
    ViewAcc acc;
    for (int64_t p = lane_id(); p < n; p += kWarp) {
      const fb_task_view t = tasks[off + p];
      const bool decode = t.phase == FB_PHASE_DECODE;
      s.slack[p] = t.slack_us;
      s.seq[p] = t.arrival_seq;
      s.ctx[p] = t.context;
      s.nw[p] = t.new_tokens | (decode ? static_cast<int32_t>(kDecodeBit) : 0);
      s.req[p] = static_cast<int32_t>(p);
      acc.add(decode, t.slack_us, t.tpot_us);
    }
    __syncwarp();
    acc.reduce();
    FormCfg f;
    f.policy = cfg.policy;
    f.max_chunk = cfg.max_chunk;
    f.token_budget = cfg.token_budget;
    f.a = cfg.model.a_ms;
    f.b = cfg.model.b_ms;
    f.c = cfg.model.c_ms;
    const int Ai = static_cast<int>(n);
    const FormOut o = form_batch_warp(s, Ai, acc, f, /*seq_unique=*/false);
    int run = 0;
    for (int k0 = 0; k0 < Ai; k0 += kWarp) {
      const int k = k0 + lane_id();
      int tk = 0, p = 0;
      if (k < Ai) {
        p = s.order[k];
        tk = s.take[k];
      }
      const unsigned m = __ballot_sync(kFull, tk > 0);
      if (tk > 0) {
        fb_plan_entry_id e;
        e.request_id = tasks[off + p].request_id;
        e.new_tokens = tk;
        e.reserved = 0;
        entries[off + run + __popc(m & lanemask_lt())] = e;
      }
      run += __popc(m);
    }
    if (lane_id() == 0) {
      fb_batch_plan pl;
      const bool empty = o.n_entries == 0;
      pl.predicted_ms = o.predicted_ms;
      pl.time_budget_used_ms = empty ? 0.0 : o.predicted_ms;
      pl.token_budget_used = empty ? 0 : o.total_new;
      pl.init_time_budget_ms = o.init_ms;
      pl.entry_off = off;
      pl.n_entries = o.n_entries;
      plans[set] = pl;
    }
    __syncwarp();
  }
}

__global__ void init_time_budget_kernel(const fb_task_view* __restrict__ tasks,
                                        const int64_t* __restrict__ set_off, int64_t n_sets,
                                        int64_t* out, int* status) {
  const int warp = threadIdx.x / kWarp;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x / kWarp);
  for (int64_t set = static_cast<int64_t>(blockIdx.x) * (blockDim.x / kWarp) + warp;
       set < n_sets; set += nwarps) {
    const int64_t off = set_off[set];
    const int64_t n = set_off[set + 1] - off;
    ViewAcc acc;
    for (int64_t p = lane_id(); p < n; p += kWarp) {
      const fb_task_view t = tasks[off + p];
      acc.add(t.phase == FB_PHASE_DECODE, t.slack_us, t.tpot_us);
    }
    acc.reduce();
    if (lane_id() == 0) {
      if (n == 0) {
        atomicExch(status, FB_ERR_USAGE);
        out[set] = 0;
      } else {
        out[set] = acc.n_dec == 0 ? acc.min_tpot
                                  : (acc.min_dec > acc.min_tpot ? acc.min_dec : acc.min_tpot);
      }
    }
  }
}

// K5 standalone: pab (sched.cpp:248-278) per task set.
__global__ void __launch_bounds__(kWarp * kWarpsPerBlock)
pab_kernel(const fb_task_view* __restrict__ tasks, const int64_t* __restrict__ set_off,
           const fb_cost_model* __restrict__ models, const int64_t* __restrict__ ttft,
           const int64_t* __restrict__ tpot, int64_t n_sets, int64_t* out,
           unsigned char* gscratch) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x / kWarp;
  unsigned char* my = smem + static_cast<size_t>(warp) * kSmemSlots * kScratchBytesPerSlot;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kWarpsPerBlock;
  for (int64_t set = static_cast<int64_t>(blockIdx.x) * kWarpsPerBlock + warp; set < n_sets;
       set += nwarps) {
    const int64_t off = set_off[set];
    const int64_t n = set_off[set + 1] - off;
    const fb_cost_model m = models[set];
    const double Wm = us_to_ms(ttft[set]), Tm = us_to_ms(tpot[set]);
    const Scratch s = set_scratch(my, gscratch, off, n);
    int64_t lmin = kInf, lpf = 0;
    for (int64_t p = lane_id(); p < n; p += kWarp) {
      const fb_task_view t = tasks[off + p];
      s.tcost[p] = pab_term(Wm, Tm, m.b_ms, m.c_ms, t.slack_us, t.context);
      lmin = t.slack_us < lmin ? t.slack_us : lmin;
      if (t.phase == FB_PHASE_PREFILL) lpf += t.new_tokens;
    }
    __syncwarp();
    const int64_t min_slack = warp_min(lmin);
    const int64_t pf = warp_sum(lpf);
    const double r_tasks = ordered_fold(s.tcost, static_cast<int>(n));
    if (lane_id() == 0)
      out[set] = pab_close(Wm, Tm, m.a_ms, m.b_ms, m.c_ms, n > 0, min_slack, r_tasks, pf);
    __syncwarp();
  }
}

static int set_blocks(int64_t n_sets) {
  int64_t b = (n_sets + kWarpsPerBlock - 1) / kWarpsPerBlock;
  if (b < 1) b = 1;
  if (b > 148 * 8) b = 148 * 8;
  return static_cast<int>(b);
}

cudaError_t launch_form_batch(const fb_task_view* tasks, const int64_t* set_off,
                              const fb_scheduler_config* cfgs, int64_t n_sets,
                              fb_plan_entry_id* entries, fb_batch_plan* plans,
                              unsigned char* scratch, int* status, cudaStream_t st) {
  const size_t smem = static_cast<size_t>(kWarpsPerBlock) * kSmemSlots * kScratchBytesPerSlot;
  cudaFuncSetAttribute(form_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(smem));
  form_batch_kernel<<<set_blocks(n_sets), kWarp * kWarpsPerBlock, smem, st>>>(
      tasks, set_off, cfgs, n_sets, entries, plans, scratch, status);
  return cudaGetLastError();
}

cudaError_t launch_init_time_budget(const fb_task_view* tasks, const int64_t* set_off,
                                    int64_t n_sets, int64_t* out, int* status,
                                    cudaStream_t st) {
  init_time_budget_kernel<<<set_blocks(n_sets), kWarp * kWarpsPerBlock, 0, st>>>(
      tasks, set_off, n_sets, out, status);
  return cudaGetLastError();
}

cudaError_t launch_pab(const fb_task_view* tasks, const int64_t* set_off,
                       const fb_cost_model* models, const int64_t* ttft, const int64_t* tpot,
                       int64_t n_sets, int64_t* out, unsigned char* scratch, cudaStream_t st) {
  const size_t smem = static_cast<size_t>(kWarpsPerBlock) * kSmemSlots * kScratchBytesPerSlot;
  cudaFuncSetAttribute(pab_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(smem));
  pab_kernel<<<set_blocks(n_sets), kWarp * kWarpsPerBlock, smem, st>>>(
      tasks, set_off, models, ttft, tpot, n_sets, out, scratch);
  return cudaGetLastError();
}

}  // namespace fbgpu
