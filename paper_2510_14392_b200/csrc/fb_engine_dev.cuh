// fb_engine_dev.cuh -- the warp engine's device code: one tile (kTile
// lanes; a full warp by default, FB_TILE = 16 gives two nodes per warp)
// simulates one Node instance (engine.h:111-176): task views, the
// memory-path begin/complete step, the register-resident path
// (fb_engine_rr.cuh) and run_node's event loop.  Included by fb_engine.cu
// and fb_cluster.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "fb_kernels.h"
#include "fb_sched.cuh"

namespace fbgpu {

// One 16-warp block per SM (the same 16 resident warps as two 8-warp blocks,
// at most 128 registers each): C2 15.4 -> 15.25 ms, C3 sample 32.6 -> 31.8 ms
// (profiles/r02u_engine_blocks_ab.txt); 8 or 12 warps per SM with more
// registers are slower (19.1 / 16.5 ms on C2).
#ifndef FB_WARPS_PER_BLOCK
#define FB_WARPS_PER_BLOCK 16
#endif
constexpr int kWarpsPerBlock = FB_WARPS_PER_BLOCK;
#ifndef FB_SMEM_SLOTS
#define FB_SMEM_SLOTS 64
#endif
// visible tasks held in shared-memory scratch (>= 32: the register path's)
constexpr int kSmemSlots = FB_SMEM_SLOTS;
static_assert(kSmemSlots >= 32, "register-path scratch");
#ifndef FB_ENGINE_BLOCKS_PER_SM
#define FB_ENGINE_BLOCKS_PER_SM 1
#endif
constexpr int kEngineBlocksPerSm = FB_ENGINE_BLOCKS_PER_SM;  // register cap for occupancy
constexpr int64_t kEscalateLive = 512;  // live requests beyond which a node goes CTA-wide


__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

#ifndef FB_STEADY
#define FB_STEADY 1
#endif

// Warp-uniform record of the node's last plan, for repeated-plan steps: `ok`
// when that plan admitted every visible task as a one-token decode (E == A ==
// total_new) and nothing has entered or left the node since (no arrival
// pulled, no request finished).  Then the visible set, its sorted order and
// the plan entries repeat exactly -- see steady_fits.
struct Steady {
  bool ok;
  bool sub;         // (register path) the plan was `ok`, then only finished requests left
                    // (order and ranks of the rest intact): the next plan is the same
                    // minus them if it fits -- see sub_rr
  int32_t E;        // plan size == visible count
  uint64_t esum;    // XOR of the entries' digests (idx, request, 1)
  int64_t tctx;     // the plan's total context
  int64_t min_dec;  // the plan's minimum decode slack (fair batching)
  int64_t now;      // the plan's begin time
  __device__ __forceinline__ void clear() {
    ok = false;
    sub = false;
  }
};

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
  Steady sd;            // repeated-plan state (false whenever a warp takes the node)
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

// Envelope-lead bookkeeping (envelope_lead_series, metrics.cpp:137-169),
// called by one lane per step that emitted: n_emit tokens at `now`, of which
// finishing requests' output lengths sum to fin_tokens.
__device__ __forceinline__ void lead_account(const EngineParams& P, int64_t inst, int64_t now,
                                             uint32_t n_emit, int64_t fin_tokens) {
  const int64_t k = (now + P.lead_bucket - 1) / P.lead_bucket;  // first grid point >= now
  if (k >= P.lead_cap) {
    atomicOr(&P.lead_flags[inst], 1);
    return;
  }
  unsigned long long* row = P.lead_hist + inst * 2 * static_cast<int64_t>(P.lead_cap);
  if (n_emit) atomicAdd(&row[k], static_cast<unsigned long long>(n_emit));
  if (fin_tokens) atomicAdd(&row[P.lead_cap + k], static_cast<unsigned long long>(fin_tokens));
  atomicMax(&P.lead_tmax[inst], static_cast<long long>(now));
}

// The tile's emissions of one step into the lead accounting (out of line:
// off the hot loop when the series is disabled).
static __device__ __noinline__ void lead_step(const EngineParams& P, const Inst& w, int64_t now,
                                              bool emit, bool fin, int32_t r, int32_t output) {
  if (fin) P.lastem[w.roff + r] = now;
  const uint32_t ne = __popc(tile_ballot(emit));
  const int64_t nf = tile_sum_small(fin ? output : 0);
  if (tile_lane() == 0 && ne) lead_account(P, w.id, now, ne, nf);
}

// Order-preserving removal of finished entries (row < 0) from vlist[0, n_live)
// (active_.erase, engine.cpp:228-229), clearing the in-flight takes.
__device__ __forceinline__ void compact_vlist(Inst& w) {
  const int64_t n = w.S.n_live;
  int64_t out = 0;
  int64_t removed_active = 0;
  FB_COLD_LOOP
  for (int64_t b = 0; b < n; b += kTile) {
    const int64_t p = b + tile_lane();
    int2 v = make_int2(-1, 0);
    if (p < n) v = w.vl[p];
    const bool keep = p < n && v.x >= 0;
    const unsigned m = tile_ballot(keep);
    const unsigned rm = tile_ballot(p < n && !keep && p < w.S.n_active);
    tile_sync();
    if (keep) w.vl[out + __popc(m & tile_lanemask_lt())] = make_int2(v.x, 0);
    out += __popc(m);
    removed_active += __popc(rm);
    tile_sync();
  }
  w.S.n_live = out;
  w.S.n_active -= removed_active;
}

// Node::complete_step, engine.cpp:204-254.  In-flight plan entries are the
// active tasks with a nonzero take (plan order only affects the event log).
static __device__ __noinline__ void complete_step(const EngineParams& P, Inst& w) {
  const int64_t t = w.S.step_end;
  bool any_fin = false;
  uint32_t lemit = 0;
  int64_t lfin = 0;
  FB_COLD_LOOP
  for (int64_t b = 0; b < w.S.n_active; b += kTile) {
    const int64_t p = b + tile_lane();
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
        if (P.lead_bucket > 0) {
          if (fin) P.lastem[g] = t;
          lemit += emit;
          lfin += fin ? P.output[row] : 0;
        }
      }
    }
    any_fin |= tile_any(fin);
  }
  if (P.lead_bucket > 0) {
    const uint32_t ne = tile_add_u32(lemit);
    const int64_t nf = tile_sum_small(lfin);
    if (tile_lane() == 0 && (ne || nf)) lead_account(P, w.id, t, ne, nf);
  }
  tile_sync();
  if (any_fin) {
    w.sd.clear();
    compact_vlist(w);
  }
  w.S.busy = 0;
}

// Node::pull_arrivals without admission control (engine.cpp:127-151).
__device__ __forceinline__ void pull_plain(const EngineParams& P, Inst& w) {
  const int64_t k = w.S.arr - w.S.pulled;
  FB_COLD_LOOP
  for (int64_t j = tile_lane(); j < k; j += kTile) {
    const int64_t r = arrival_row(w, w.S.pulled + j);
    P.seq[w.roff + r] = static_cast<int32_t>(w.S.seq_counter + j);
    w.vl[w.S.n_live + j] = make_int2(static_cast<int>(r), 0);
  }
  tile_sync();
  w.S.seq_counter += k;
  w.S.n_live += k;
  w.S.pulled = w.S.arr;
}

// K5: Node::pull_arrivals with PAB admission (engine.cpp:127-151, pab
// sched.cpp:248-278).  The view fold is computed once in view order; every
// admitted, visible arrival then appends exactly one term, which is the same
// left-to-right fold the reference recomputes per arrival.
static __device__ void pull_pab(const EngineParams& P, Inst& w, int64_t now) {
  const DevInst* I = w.I;
  const double Wm = us_to_ms(I->g_ttft), Tm = us_to_ms(I->g_tpot);
  const double a = I->sa, b = I->sb, c = I->sc;
  int64_t A = visible_count(w);
  const Scratch s = scratch_for(P, w, A);
  int64_t lmin = kInf, lpf = 0;
  FB_COLD_LOOP
  for (int64_t p = tile_lane(); p < A; p += kTile) {
    const View v = load_view(P, w, p, now);
    s.tcost[p] = pab_term(Wm, Tm, b, c, v.slack, v.ctx);
    lmin = v.slack < lmin ? v.slack : lmin;
    if (!v.decode) lpf += v.nw;
  }
  tile_sync();
  int64_t min_slack = tile_min_i64(lmin);
  int64_t pf_tok = tile_sum_small(lpf);
  double r_tasks = ordered_fold(s.tcost, static_cast<int>(A));
  FB_COLD_LOOP
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
      if (tile_lane() == 0) {
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
      if (tile_lane() == 0) {
        P.flags[w.roff + r] |= FB_REC_REJECTED;
        if (P.log_on) {
          if (w.S.log_rejects < P.log_reject_cap) {
            fb_reject_log& rl = P.log_rejects[I->log_reject_off + w.S.log_rejects];
            rl.t_us = now;
            rl.pab_tokens = budget;
            rl.req = static_cast<int32_t>(r);
            rl.step = static_cast<int32_t>(w.S.step_counter);
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
  tile_sync();
  w.S.pulled = w.S.arr;
}


// The step's begin_step log row and counters (event logs on; out of line,
// off the engines' hot code).
static __device__ __noinline__ void log_step(const EngineParams& P, Inst& w, bool log_ok,
                                             int64_t now, int64_t dur, double predicted,
                                             double actual, int64_t tn, int64_t tctx,
                                             double init_ms, int E) {
  if (log_ok) {
    if (tile_lane() == 0) {
      fb_step_log& sl = P.log_steps[w.I->log_step_off + w.S.log_steps];
      sl.t_us = now;
      sl.duration_us = dur;
      sl.predicted_ms = predicted;
      sl.actual_ms = actual;
      sl.total_new = tn;
      sl.total_ctx = tctx;
      sl.init_budget_ms = init_ms;
      sl.entry_off = w.S.log_entries;
      sl.n_entries = E;
    }
    w.S.log_steps++;
    w.S.log_entries += E;
  } else {
    w.S.log_trunc = 1;
  }
}

__device__ __forceinline__ void steady_record(Steady& sd, const Inst& w, bool all_decode_whole,
                                              int E, uint64_t esum, int64_t tctx,
                                              int64_t min_dec, int64_t now) {
  const bool fair = w.policy == FB_POLICY_FAIRBATCH || w.policy == FB_POLICY_FAIRBATCH_PAB;
  sd.ok = all_decode_whole && (!fair || w.I->tpot_uniform >= 0);
  sd.sub = false;
  sd.E = E;
  sd.esum = esum;
  sd.tctx = tctx;
  sd.min_dec = min_dec;
  sd.now = now;
}

// A repeated-plan step: begin_step at `now` when the previous plan (begun at
// sd.now, ending exactly at now) admitted all A visible tasks as one-token
// decodes and no request has entered or left the node since.  The plan is
// the same one again:
//  * order -- every task is a decode.  Sarathi / prefill-first order by seq
//    alone.  Fair batching orders by (group, slack, seq) with group 0 iff
//    slack < urgency, i.e. by (slack, seq); with one tpot every decode's
//    slack moved by the same tpot - (now - sd.now), so the order is unchanged
//    and the minimum decode slack moved by that amount;
//  * admission -- sarathi admits every decode (sched.cpp:180-183);
//    prefill-first does while A <= token_budget (sched.cpp:214-224); fair
//    batching admits everything whole when the all-fit test of begin_rr holds,
//    here evaluated on an upper bound of the cost sum: with b > 0, c >= 0
//    (validated on input) and one new token per task, sum_i fl(b + fl(c
//    ctx_i)) <= (1 + 2^-53)^2 (A b + c sum ctx) <= RU(RU(RU(A b) + RU(c sum
//    ctx)) (1 + 2^-51)); when the bound fails the caller takes the full path;
//  * totals -- total_new = A, total_ctx = previous + A (every decode's
//    context grew by its one emitted token), the entry digests repeat.
// Returns false (nothing modified) when the full path must decide.
// Does the plan "all A visible decodes, one token each" (total context tctx,
// minimum decode slack min_dec) pass the policy's admission whole?
__device__ __forceinline__ bool plan_fits(const Inst& w, int A, int64_t tctx, int64_t min_dec,
                                          double& init_ms) {
  const DevInst* I = w.I;
  const int policy = w.policy;
  init_ms = 0.0;
  if (policy == FB_POLICY_FAIRBATCH || policy == FB_POLICY_FAIRBATCH_PAB) {
    const int64_t tpot_u = I->tpot_uniform;
    init_ms = us_to_ms(min_dec > tpot_u ? min_dec : tpot_u);
    const double tb0 = dsub(init_ms, I->sa);
    if (!(tb0 >= 0.0 && A <= I->token_budget)) return false;
    const double s_up = __dmul_ru(__dadd_ru(__dmul_ru(static_cast<double>(A), I->sb),
                                            __dmul_ru(I->sc, static_cast<double>(tctx))),
                                  1.0 + 0x1p-51);
    return __dsub_rd(tb0, s_up) >= __dmul_ru(__dmul_ru(static_cast<double>(A), 0x1p-52), tb0);
  }
  return policy != FB_POLICY_PREFILL_FIRST || A <= I->token_budget;
}
__device__ __forceinline__ bool steady_fits(const Inst& w, const Steady& sd, int64_t now, int A,
                                            double& init_ms, int64_t& min_dec) {
  min_dec = sd.min_dec + w.I->tpot_uniform - (now - sd.now);  // used by fair batching only
  return plan_fits(w, A, sd.tctx + A, min_dec, init_ms);
}

// The repeated plan's scalar bookkeeping (finalize_plan, the truth step time,
// step log, digest, counters); the caller has written the entry log.
__device__ __forceinline__ void steady_commit(const EngineParams& P, Inst& w, Steady& sd,
                                              int64_t now, int A, double init_ms,
                                              int64_t min_dec, bool log_ok, int64_t tctx) {
  const DevInst* I = w.I;
  const int64_t tn = A;
  const double predicted = predict_ms(I->sa, I->sb, I->sc, tn, tctx);
  double actual = predict_ms(I->ta, I->tb, I->tc, tn, tctx);
  const double amp = I->noise_amp;
  if (amp != 0.0) actual = apply_noise(actual, amp, I->noise_seed, w.S.step_counter);
  int64_t dur = ms_to_us(actual);
  if (dur < 1) dur = 1;
  if (P.log_on) log_step(P, w, log_ok, now, dur, predicted, actual, tn, tctx, init_ms, A);
  w.S.digest = fb_digest_step(w.S.digest, now, static_cast<uint32_t>(A), sd.esum, predicted,
                              actual);
  w.S.sum_visible += A;
  w.S.sum_entries += A;
  w.S.sum_new += tn;
  w.S.busy = 1;
  w.S.step_end = now + dur;
  w.S.step_counter++;
  sd.tctx = tctx;
  sd.min_dec = min_dec;
  sd.now = now;
}

// A run of repeated-plan steps back to back (run_event's repeated-plan lane,
// without event logs or the envelope-lead series): each iteration is one
// event of run_node's loop -- the in-flight step ends before the next arrival
// with nothing pending: complete_step (`complete(now, steps started)`, true
// when a request finished; it has then done the removal), then begin_step
// repeats the plan
// (steady_fits / steady_commit, same arithmetic; `recommit()` re-arms the
// path's in-flight takes).  The node's hot scalars stay in registers for the
// whole run.  Returns -1 when the run stopped with a step in flight (the next
// event is not a repeated-plan one), else the time t of an event whose step
// completed but whose begin_step the general code still has to decide (a
// request finished, the horizon, or the capacity bound failed).
template <class CompleteFn, class RecommitFn>
__device__ __forceinline__ int64_t steady_run(const EngineParams& P, Inst& w, int64_t& ev,
                                              int64_t next_arr, CompleteFn&& complete,
                                              RecommitFn&& recommit, uint32_t path_bit) {
  const DevInst* I = w.I;
  const bool fair = w.policy == FB_POLICY_FAIRBATCH || w.policy == FB_POLICY_FAIRBATCH_PAB;
  const int A = w.sd.E;
  const int64_t horizon = w.horizon, max_ev = P.max_events;
  const int64_t tpot_u = I->tpot_uniform;
  const double sa = I->sa, sb = I->sb, sc = I->sc, ta = I->ta, tb = I->tb, tc = I->tc;
  const double amp = I->noise_amp;
  // truth model == scheduler model bit for bit (C1-C3): one evaluation per step
  const bool same_model = __double_as_longlong(sa) == __double_as_longlong(ta) &&
                          __double_as_longlong(sb) == __double_as_longlong(tb) &&
                          __double_as_longlong(sc) == __double_as_longlong(tc);
  const uint64_t esum = w.sd.esum;
  const double slack_a = __dmul_ru(static_cast<double>(A), 0x1p-52);
  const double s_b = __dmul_ru(static_cast<double>(A), sb);
  const bool budget_ok = w.policy == FB_POLICY_SARATHI || A <= I->token_budget;
  int64_t step_end = w.S.step_end, tctx = w.sd.tctx, min_dec = w.sd.min_dec, snow = w.sd.now;
  uint64_t digest = w.S.digest, steps = w.S.step_counter;
  int64_t n_steps = 0;
  int64_t owed = -1;
  while (ev < max_ev && next_arr > step_end) {
    const int64_t now = step_end;
    ++ev;
    if (FB_UNLIKELY(complete(now, steps) || now >= horizon || !budget_ok)) {
      owed = now;
      break;
    }
    // begin_step: the same plan again
    double init_ms = 0.0;
    int64_t md = 0;
    if (fair) {
      md = min_dec + tpot_u - (now - snow);
      init_ms = us_to_ms(md > tpot_u ? md : tpot_u);
      const double tb0 = dsub(init_ms, sa);
      const double s_up = __dmul_ru(__dadd_ru(s_b, __dmul_ru(sc, static_cast<double>(tctx + A))),
                                    1.0 + 0x1p-51);
      if (FB_UNLIKELY(!(tb0 >= 0.0 && __dsub_rd(tb0, s_up) >= __dmul_ru(slack_a, tb0)))) {
        owed = now;
        break;
      }
    }
    tctx += A;
    const double predicted = predict_ms(sa, sb, sc, A, tctx);
    double actual = predicted;
    if (!same_model) actual = predict_ms(ta, tb, tc, A, tctx);
    if (FB_UNLIKELY(amp != 0.0)) actual = apply_noise(actual, amp, I->noise_seed, steps);
    int64_t dur = ms_to_us(actual);
    if (dur < 1) dur = 1;
    digest = fb_digest_step(digest, now, static_cast<uint32_t>(A), esum, predicted, actual);
    steps++;
    n_steps++;
    step_end = now + dur;
    min_dec = md;
    snow = now;
    recommit();
  }
  w.S.digest = digest;
  w.S.step_counter = steps;
  w.S.sum_visible += n_steps * A;
  w.S.sum_entries += n_steps * A;
  w.S.sum_new += n_steps * A;
  w.sd.tctx = tctx;
  w.sd.min_dec = min_dec;
  w.sd.now = snow;
  w.S.step_end = step_end;
  if (n_steps > 0) w.S.paths |= path_bit;
  if (owed >= 0) {
    w.S.t_last = owed;
    w.S.busy = 0;
  } else if (n_steps > 0) {
    w.S.t_last = snow;
  }
  return owed;
}

// The memory path's run: every visible task is active with its one-token
// take still in vlist (complete_step never clears takes) and is a decode.
__device__ __forceinline__ int64_t steady_burst_mem(const EngineParams& P, Inst& w,
                                                    int64_t& ev, int64_t next_arr) {
  const int64_t A = w.sd.E;
  return steady_run(
      P, w, ev, next_arr,
      [&](int64_t now, uint64_t) {  // complete_step (engine.cpp:204-254) for decodes
        bool any_fin = false;
        FB_COLD_LOOP
        for (int64_t b = 0; b < A; b += kTile) {
          const int64_t p = b + tile_lane();
          bool fin = false;
          if (p < A) {
            const int32_t r = w.vl[p].x;
            fin = emit_token(P, w.roff + r, w.toff + r, now);
            if (FB_UNLIKELY(fin)) w.vl[p].x = -1;
          }
          any_fin |= tile_any(fin);
        }
        tile_sync();
        if (FB_UNLIKELY(any_fin)) {
          w.sd.clear();
          compact_vlist(w);
        }
        return any_fin;
      },
      [] {}, kPathRepeatMemory);
}

// Node::begin_step, engine.cpp:153-202.  Returns false when there is nothing
// to schedule (no step launched, no step ordinal consumed).
static __device__ __noinline__ bool begin_step(const EngineParams& P, Inst& w, int64_t now) {
  const DevInst* I = w.I;
  Steady& sd = w.sd;
  if (w.S.pulled < w.S.arr) {
    sd.clear();
    if (w.policy == FB_POLICY_FAIRBATCH_PAB) {
      pull_pab(P, w, now);
    } else {
      pull_plain(P, w);
    }
  }
  const int64_t A = visible_count(w);
  if (A == 0) {
    sd.clear();
    return false;
  }
#if FB_STEADY
  // repeated plan: the in-flight takes in vlist are already the plan's
  // (complete_step leaves them; every visible task is active), so only the
  // scalar bookkeeping remains -- without the entry log, which needs the order
  if (sd.ok && A == sd.E && !P.log_on) {
    double init_ms;
    int64_t min_dec;
    if (steady_fits(w, sd, now, static_cast<int>(A), init_ms, min_dec)) {
      steady_commit(P, w, sd, now, static_cast<int>(A), init_ms, min_dec, false, sd.tctx + A);
      w.S.paths |= kPathRepeatMemory;
      return true;
    }
  }
  sd.clear();
#endif
  const Scratch s = scratch_for(P, w, A);

  // K1: views, envelope slack and the init_time_budget reductions.
  ViewAcc acc;
  FB_COLD_LOOP
  for (int64_t p = tile_lane(); p < A; p += kTile) {
    const View v = load_view(P, w, p, now);
    s.slack[p] = v.slack;
    s.seq[p] = v.seq;
    s.ctx[p] = v.ctx;
    s.nw[p] = v.nw;
    s.req[p] = v.r;
    acc.add(v.decode, v.slack, v.tpot);
  }
  tile_sync();
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
  FB_COLD_LOOP
  for (int k0 = 0; k0 < Ai; k0 += kTile) {
    const int k = k0 + tile_lane();
    int tk = 0, p = 0;
    if (k < Ai) {
      p = s.order[k];
      tk = s.take[k];
    }
    const bool adm = tk > 0;
    const unsigned m = tile_ballot(adm);
    const bool wadm = adm && p >= n_act;
    const unsigned mw = tile_ballot(wadm);
    if (adm) {
      const int idx = run_all + __popc(m & tile_lanemask_lt());
      const int r = s.req[p];
      esum ^= fb_digest_entry(static_cast<uint32_t>(idx), static_cast<uint32_t>(r),
                              static_cast<uint32_t>(tk));
      if (log_ok) P.log_entries[entry_base + idx] = fb_plan_entry{r, tk};
    }
    if (k < Ai) {
      const int64_t np = p < n_act ? p : (wadm ? n_act + run_w + __popc(mw & tile_lanemask_lt()) : -1);
      s.slack[p] = (np << 32) | static_cast<uint32_t>(tk);
    }
    run_all += __popc(m);
    run_w += __popc(mw);
  }
  tile_sync();
  esum = tile_xor_u64(esum);
  // unadmitted visible waiting keep their relative order after the movers
  int run_u = 0;
  const int64_t base_u = n_act + run_w;
  FB_COLD_LOOP
  for (int64_t p0 = n_act; p0 < A; p0 += kTile) {
    const int64_t p = p0 + tile_lane();
    bool un = false;
    if (p < A) un = (s.slack[p] >> 32) < 0;
    const unsigned mu = tile_ballot(un);
    if (un) s.slack[p] = (static_cast<int64_t>(base_u + run_u + __popc(mu & tile_lanemask_lt())) << 32);
    run_u += __popc(mu);
  }
  tile_sync();
  FB_COLD_LOOP
  for (int64_t p = tile_lane(); p < A; p += kTile) {
    const int64_t pk = s.slack[p];
    w.vl[pk >> 32] = make_int2(s.req[p], static_cast<int32_t>(pk & 0xffffffff));
  }
  tile_sync();

  if (P.log_on)
    log_step(P, w, log_ok, now, dur, o.predicted_ms, actual, o.total_new, o.total_ctx, o.init_ms,
             o.n_entries);
  w.S.digest = fb_digest_step(w.S.digest, now, static_cast<uint32_t>(o.n_entries), esum,
                              o.predicted_ms, actual);
  w.S.sum_visible += A;
  w.S.sum_entries += o.n_entries;
  w.S.sum_new += o.total_new;
  w.S.n_active = n_act + run_w;
  w.S.busy = 1;
  w.S.step_end = now + dur;
  w.S.step_counter++;
#if FB_STEADY
  steady_record(sd, w, o.n_entries == Ai && o.total_new == A && acc.n_dec == Ai, Ai, esum,
                o.total_ctx, acc.min_dec, now);
#endif
  return true;
}

}  // namespace fbgpu

#include "fb_engine_rr.cuh"

namespace fbgpu {

// run_node's event loop (engine.cpp:266-288) for up to max_events times t.
// Steps run on the register-resident path while at most 32 requests are live
// and on the memory path otherwise; the switch happens at step boundaries.
// Per-instance loop state of run_node's event loop.
struct RunCtx {
  TaskReg tk;
  bool rr;           // live requests held in registers (fb_engine_rr.cuh)
  int64_t next_arr;  // arrival time of the next trace row
  int64_t ev;        // events processed in this launch
};

__device__ __forceinline__ void run_begin(const EngineParams& P, const Inst& w, RunCtx& c) {
  c.tk = TaskReg{};
  c.rr = false;
  c.next_arr = w.S.arr < w.nreq ? P.arrival[w.toff + w.S.arr] : kInf;
  c.ev = 0;
}

// One iteration of run_node's event loop (engine.cpp:266-288).  Returns true
// when the node stops for this launch: quiescent (done), handed to the wide
// engine, or out of its event budget -- its registers are spilled then.
// Steps run on the register-resident path while at most kTile requests are
// live and on the memory path otherwise; the switch happens at step
// boundaries.
__device__ __forceinline__ bool run_event(const EngineParams& P, Inst& w, RunCtx& c,
                                          const Scratch& s) {
  const int64_t* arrival = P.arrival + w.toff;
  if (c.ev >= P.max_events) {
    if (c.rr) rr_spill(P, w, c.tk);
    return true;
  }
  int64_t t;
#ifndef FB_EVENT_LANE
#define FB_EVENT_LANE 0  // per-event repeated-plan lane (logs / lead series on): code size costs C2 3 %
#endif
#if FB_STEADY
  // Repeated-plan lane: the in-flight step of a repeated-plan-eligible node
  // ends before the next arrival with nothing pending -- the event is that
  // step's end: complete it and, when nothing finished, begin the same plan
  // again (the general code below would take the same branches).  Without
  // logs and lead series, a whole run of such events at once.
  const bool lane_ok = c.rr && w.sd.ok && w.S.busy && c.next_arr > w.S.step_end &&
                       w.S.pulled == w.S.arr;
  if (!c.rr && w.sd.ok && w.S.busy && c.next_arr > w.S.step_end && w.S.pulled == w.S.arr &&
      !P.log_on && P.lead_bucket == 0) {
    t = steady_burst_mem(P, w, c.ev, c.next_arr);
    if (t < 0) return false;
  } else if (lane_ok && !P.log_on && P.lead_bucket == 0) {
    t = steady_burst(P, w, c.tk, c.ev, c.next_arr);
    if (t < 0) return false;
#if FB_EVENT_LANE
  } else if (lane_ok) {
    c.ev++;
    t = w.S.step_end;
    w.S.t_last = t;
    complete_rr(P, w, c.tk);
    if (w.sd.ok && t < w.horizon && steady_rr(P, w, c.tk, t, w.sd, w.sd.E)) return false;
#endif
  } else
#endif
  {
  c.ev++;
  if (w.S.busy && c.next_arr < w.S.step_end) {
    // Arrivals strictly before the in-flight step's end only enqueue
    // (run_node's loop neither completes nor begins a step at those times):
    // consume them a tile at a time.
    for (;;) {
      const int64_t q = w.S.arr + tile_lane();
      const bool early = q < w.nreq && arrival[q] < w.S.step_end;
      const int n = __popc(tile_ballot(early));
      w.S.arr += n;
      if (n < kTile) break;
    }
    c.next_arr = w.S.arr < w.nreq ? arrival[w.S.arr] : kInf;
  }
  const int64_t t_step = w.S.busy ? w.S.step_end : kInf;
  t = t_step < c.next_arr ? t_step : c.next_arr;
  if (t == kInf || (!w.S.busy && t >= w.horizon)) {
    if (c.rr) rr_spill(P, w, c.tk);
    w.S.done = 1;
    w.S.incomplete = (w.S.busy || w.S.pulled < w.S.arr || w.S.n_live > 0 ||
                      w.S.arr < w.nreq) ? 1 : 0;
    return true;
  }
  w.S.t_last = t;
  if (w.S.busy && t_step == t) {
    if (c.rr) {
      complete_rr(P, w, c.tk);
    } else {
      complete_step(P, w);
    }
  }
  while (c.next_arr == t) {  // Node::enqueue (visible at its arrival time)
    w.S.arr++;
    c.next_arr = w.S.arr < w.nreq ? arrival[w.S.arr] : kInf;
  }
  }
  if (!w.S.busy && t < w.horizon) {
    const int64_t upcoming = w.S.n_live + (w.S.arr - w.S.pulled);
    if (upcoming > kEscalateLive && w.I->wide_ok) {  // hand over to the wide engine
      if (c.rr) rr_spill(P, w, c.tk);
      w.S.pending_begin = 1;
      w.S.escalated = 1;
      if (tile_lane() == 0) {
        const unsigned long long slot = atomicAdd(&P.work[3], 1ull);
        P.wide_list[slot] = w.id;
      }
      return true;
    }
    if (c.rr && upcoming > kTile) {
      rr_spill(P, w, c.tk);
      w.sd.clear();
      c.rr = false;
    } else if (!c.rr && upcoming <= kTile) {
      rr_load(P, w, c.tk);
      w.sd.clear();
      c.rr = true;
      w.S.paths |= kPathRegister;
    }
    if (c.rr) {
      if (begin_rr(P, w, c.tk, t, s) < 0) {  // keys outside the packed range
        rr_spill(P, w, c.tk);
        c.rr = false;
        begin_step(P, w, t);
        w.S.paths |= kPathMemory;
      }
    } else {
      begin_step(P, w, t);
      w.S.paths |= kPathMemory;
    }
  }
  return false;
}

// run_node's event loop for up to max_events events (one node per tile).
static __device__ void run_instance(const EngineParams& P, Inst& w) {
  RunCtx c;
  run_begin(P, w, c);
  const Scratch s = carve_scratch(w.smem, kSmemSlots);
  while (!run_event(P, w, c, s)) {
  }
}

}  // namespace fbgpu
