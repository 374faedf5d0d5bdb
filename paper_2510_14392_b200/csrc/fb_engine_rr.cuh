// fb_engine_rr.cuh -- register-resident fast path of the warp engine.
//
// While a node has at most 32 live requests (the common case: C1/C2/C3 see
// A <= 32 in ~99% of steps), lane i of the owning warp keeps
// the state of live request i (views order: active in activation order, then
// waiting in admission order) in registers across steps.  A step then costs
// no global traffic except new arrivals and finished-request records, and the
// K1-K5 stages run as register / shuffle / redux code.  Reordering (finished
// requests leaving active_, waiting -> active moves) is a shuffle permutation
// of the per-lane state.  Semantics are identical to the memory path in
// fb_engine.cu (same helpers, same operation order); the engine switches
// between the two at step boundaries (spill / load).
#pragma once

namespace fbgpu {

#ifndef FB_RANK_REUSE
#define FB_RANK_REUSE 1  // C1 77.7 -> 74.9 ms, C2 35.55 -> 35.27 ms (tools/ab_time.py)
#endif
#ifndef FB_RANK_UNROLL
#define FB_RANK_UNROLL 1  // C2: 4 -> 1 20.3 -> 19.2 ms (code size: the pass is instruction-fetch bound)
#endif
constexpr int kRankUnroll = FB_RANK_UNROLL;

// One live request held by one lane.
struct TaskReg {
  int32_t r, seq, prompt, output, prefilled, nidx, take;
  int32_t rk;  // rank in the previous step's slack order, -1 unknown
  uint32_t flags;
  int64_t dl0;  // arrival + ttft_slo (TTFT deadline)
  int64_t tpot;
  int64_t first;  // time of token 0, -1 none
  double maxtp, maxtp_alt;
};

__device__ __forceinline__ void permute_task(TaskReg& t, int src) {
  t.r = tile_shfl(t.r, src);
  t.seq = tile_shfl(t.seq, src);
  t.prompt = tile_shfl(t.prompt, src);
  t.output = tile_shfl(t.output, src);
  t.prefilled = tile_shfl(t.prefilled, src);
  t.nidx = tile_shfl(t.nidx, src);
  t.take = tile_shfl(t.take, src);
  t.rk = tile_shfl(t.rk, src);
  t.flags = tile_shfl(t.flags, src);
  t.dl0 = tile_shfl(t.dl0, src);
  t.tpot = tile_shfl(t.tpot, src);
  t.first = tile_shfl(t.first, src);
  t.maxtp = tile_shfl(t.maxtp, src);
  t.maxtp_alt = tile_shfl(t.maxtp_alt, src);
}

// A request entering the node (Node::pull_arrivals, engine.cpp:146-149).
__device__ __forceinline__ void fresh_task(const EngineParams& P, const Inst& w, int64_t r,
                                           int64_t seq, TaskReg& t) {
  const int64_t row = w.toff + r;
  t.r = static_cast<int32_t>(r);
  t.seq = static_cast<int32_t>(seq);
  t.prompt = P.prompt[row];
  t.output = P.output[row];
  t.dl0 = P.arrival[row] + P.ttft[row];
  t.tpot = P.tpot[row];
  t.prefilled = 0;
  t.nidx = 0;
  t.take = 0;
  t.rk = -1;
  t.flags = 0;
  t.first = -1;
  t.maxtp = 0.0;
  t.maxtp_alt = 0.0;
}

// Writes a request's progress + record back to the arena.
__device__ __forceinline__ void flush_task(const EngineParams& P, const Inst& w,
                                           const TaskReg& t) {
  const int64_t g = w.roff + t.r;
  P.prefilled[g] = t.prefilled;
  P.nidx[g] = t.nidx;
  P.seq[g] = t.seq;
  P.flags[g] = t.flags;
  P.first[g] = t.first;
  P.maxtp[g] = t.maxtp;
  P.maxtp_alt[g] = t.maxtp_alt;
}

__device__ __forceinline__ void load_task(const EngineParams& P, const Inst& w, int p,
                                          TaskReg& t) {
  const int2 v = w.vl[p];
  const int64_t g = w.roff + v.x;
  const int64_t row = w.toff + v.x;
  t.r = v.x;
  t.take = v.y;
  t.rk = -1;
  t.prompt = P.prompt[row];
  t.output = P.output[row];
  t.dl0 = P.arrival[row] + P.ttft[row];
  t.tpot = P.tpot[row];
  t.prefilled = P.prefilled[g];
  t.nidx = P.nidx[g];
  t.seq = P.seq[g];
  t.flags = P.flags[g];
  t.first = P.first[g];
  t.maxtp = P.maxtp[g];
  t.maxtp_alt = P.maxtp_alt[g];
}

// Memory path -> registers (at a step boundary).
__device__ __forceinline__ void rr_load(const EngineParams& P, const Inst& w, TaskReg& t) {
  if (tile_lane() < w.S.n_live) load_task(P, w, tile_lane(), t);
}

// Registers -> memory path / end of launch.
__device__ __forceinline__ void rr_spill(const EngineParams& P, const Inst& w,
                                         const TaskReg& t) {
  if (tile_lane() < w.S.n_live) {
    flush_task(P, w, t);
    w.vl[tile_lane()] = make_int2(t.r, t.take);
  }
  tile_sync();
}

// Token emission on registers (engine.cpp:211-232, metrics.cpp:42-60,196-214).
__device__ __forceinline__ bool emit_reg(TaskReg& t, int64_t now) {
  const int32_t idx = t.nidx;
  if (FB_UNLIKELY(idx == 0)) {
    t.first = now;
    if (now <= t.dl0) t.flags |= FB_REC_MET_TTFT;  // emits[0] <= ttft_slo
  } else {
    const int64_t d = now - t.first;
    if (d > t.tpot * static_cast<int64_t>(idx)) t.flags |= kTpotViolated;
    max_ratio(t.maxtp, d, idx);
    if (idx >= 2) max_ratio(t.maxtp_alt, d, idx - 1);
    if (now > t.dl0 + t.tpot * static_cast<int64_t>(idx)) t.flags |= FB_REC_ENV_MISS;
  }
  t.nidx = idx + 1;
  const bool fin = t.nidx >= t.output;
  if (FB_UNLIKELY(fin)) {
    t.flags |= FB_REC_FINISHED;
    if (!(t.flags & kTpotViolated)) t.flags |= FB_REC_MET_TPOT;
  }
  return fin;
}

// Order-preserving removal of the finished requests from active_
// (engine.cpp:228-229) on registers.
__device__ __forceinline__ void remove_finished_rr(Inst& w, TaskReg& t, bool fin, bool live,
                                                   unsigned finm) {
  const int lane = tile_lane();
  w.sd.sub = w.sd.ok;  // the rest of an all-decode plan keeps its order and dense ranks
  w.sd.ok = false;
#if FB_RANK_REUSE
  // previous-order ranks stay dense over the remaining tasks
  const unsigned gone = tile_or(fin && t.rk >= 0 ? 1u << t.rk : 0u);
  if (t.rk >= 0) t.rk -= __popc(gone & ((1u << t.rk) - 1u));
#endif
  const unsigned keep = tile_ballot(live && !fin);
  const int nk = __popc(keep);
  const int src = lane < nk ? static_cast<int>(__fns(keep, 0, lane + 1)) : lane;
  permute_task(t, src);
  w.S.n_live -= __popc(finm);
  w.S.n_active -= __popc(finm);
}

// Node::complete_step (engine.cpp:204-254) on registers.
__device__ __forceinline__ void complete_rr(const EngineParams& P, Inst& w, TaskReg& t) {
  const int64_t now = w.S.step_end;
  const int lane = tile_lane();
  const bool live = lane < w.S.n_live;
  bool fin = false, emit = false;
  if (live && t.take > 0) {
    emit = true;
    if (t.prefilled < t.prompt) {
      t.prefilled += t.take;
      emit = t.prefilled >= t.prompt;  // the completing chunk yields token 0
    }
    if (emit) fin = emit_reg(t, now);
    if (fin) flush_task(P, w, t);
  }
  t.take = 0;
  if (P.lead_bucket > 0) lead_step(P, w, now, emit, fin, t.r, t.output);
  const unsigned finm = tile_ballot(fin);
  if (finm) remove_finished_rr(w, t, fin, live, finm);
  w.S.busy = 0;
}

// Per-lane K1 view (build_task_views, engine.cpp:51-81).
struct RView {
  bool decode;
  int32_t nw;  // new tokens available
  int64_t ctx, slack;
};

__device__ __forceinline__ RView view_reg(const TaskReg& t, int64_t now) {
  RView v;
  v.decode = t.prefilled >= t.prompt;
  if (!v.decode) {
    v.nw = t.prompt - t.prefilled;
    v.ctx = t.prefilled;
    v.slack = t.dl0 + t.tpot * static_cast<int64_t>(t.nidx) - now;
  } else {
    v.nw = 1;
    v.ctx = static_cast<int64_t>(t.prompt) + t.nidx;
    int64_t anchor = t.dl0;
    if (t.first >= 0 && t.first < anchor) anchor = t.first;
    v.slack = anchor + t.tpot * static_cast<int64_t>(t.nidx) - now;
  }
  return v;
}

// Node::pull_arrivals (engine.cpp:127-151) on registers; the caller
// guarantees n_live + pending <= 32.
__device__ __forceinline__ void pull_rr(const EngineParams& P, Inst& w, TaskReg& t,
                                        int64_t now, const Scratch& s) {
  const int lane = tile_lane();
  if (w.policy != FB_POLICY_FAIRBATCH_PAB) {
    const int64_t k = w.S.arr - w.S.pulled;
    const int j = lane - static_cast<int>(w.S.n_live);
    if (j >= 0 && j < k) fresh_task(P, w, arrival_row(w, w.S.pulled + j), w.S.seq_counter + j, t);
    w.S.seq_counter += k;
    w.S.n_live += k;
    w.S.pulled = w.S.arr;
    return;
  }
  // K5: PAB admission with the view fold in views order (sched.cpp:248-278)
  const DevInst* I = w.I;
  const double Wm = us_to_ms(I->g_ttft), Tm = us_to_ms(I->g_tpot);
  const double a = I->sa, b = I->sb, c = I->sc;
  int64_t A = visible_count(w);
  int64_t lmin = kInf, lpf = 0;
  if (lane < A) {
    const RView v = view_reg(t, now);
    s.tcost[lane] = pab_term(Wm, Tm, b, c, v.slack, v.ctx);
    lmin = v.slack;
    if (!v.decode) lpf = v.nw;
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
    if (prompt <= budget) {
      bool vis = true;
      if (w.max_active > 0) {
        int64_t slots = static_cast<int64_t>(w.max_active) - w.S.n_active;
        if (slots < 0) slots = 0;
        vis = (w.S.n_live - w.S.n_active) < slots;
      }
      if (lane == w.S.n_live) fresh_task(P, w, r, w.S.seq_counter, t);
      w.S.seq_counter++;
      w.S.n_live++;
      if (vis) {
        const int64_t slack = P.arrival[row] + P.ttft[row] - now;
        r_tasks = dadd(r_tasks, pab_term(Wm, Tm, b, c, slack, 0));
        min_slack = slack < min_slack ? slack : min_slack;
        pf_tok += prompt;
        A++;
      }
    } else {
      if (lane == 0) {
        P.flags[w.roff + r] |= FB_REC_REJECTED;
        if (P.log_on && w.S.log_rejects < P.log_reject_cap) {
          fb_reject_log& rl = P.log_rejects[I->log_reject_off + w.S.log_rejects];
          rl.t_us = now;
          rl.pab_tokens = budget;
          rl.req = static_cast<int32_t>(r);
          rl.step = static_cast<int32_t>(w.S.step_counter);
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

#if FB_STEADY
// A repeated-plan step on registers (steady_fits / steady_commit): every
// visible lane's task is admitted again with one token, at its unchanged rank.
__device__ __forceinline__ bool steady_rr(const EngineParams& P, Inst& w, TaskReg& t,
                                          int64_t now, Steady& sd, int A) {
  double init_ms;
  int64_t min_dec;
  if (!steady_fits(w, sd, now, A, init_ms, min_dec)) return false;
  const bool log_ok = P.log_on && w.S.log_steps < P.log_step_cap &&
                      w.S.log_entries + A <= P.log_entry_cap;
  const bool vis = tile_lane() < A;
  if (log_ok && vis)
    P.log_entries[w.I->log_entry_off + w.S.log_entries + t.rk] = fb_plan_entry{t.r, 1};
  t.take = vis ? 1 : 0;
  steady_commit(P, w, sd, now, A, init_ms, min_dec, log_ok, sd.tctx + A);
  w.S.paths |= kPathRepeatRegister;
  return true;
}

#ifndef FB_SUB
#define FB_SUB 0  // C2 +2 % slower (code size), C1 2 % faster: off
#endif
// The plan after requests finished out of an all-decode, all-admitted plan
// (nothing arrived): the A remaining visible tasks are that plan's decodes
// (A == n_active: no waiting task became visible), their order is unchanged
// and their ranks were kept dense by remove_finished_rr -- so the plan is
// again "all A decodes, one token each, in rank order" when it fits.  Only
// the totals are recounted: the context sum, the entry digests (positions
// moved) and the minimum decode slack (the rank-0 task's).
__device__ __forceinline__ bool sub_rr(const EngineParams& P, Inst& w, TaskReg& t, int64_t now,
                                       Steady& sd, int A) {
  const bool vis = tile_lane() < A;
  const int64_t tctx = tile_sum_small(vis ? static_cast<int64_t>(t.prompt) + t.nidx : 0);
  int64_t anchor = t.dl0;
  if (t.first >= 0 && t.first < anchor) anchor = t.first;
  const int l0 = __ffs(tile_ballot(vis && t.rk == 0)) - 1;
  const int64_t min_dec = tile_shfl(anchor + t.tpot * static_cast<int64_t>(t.nidx) - now, l0);
  double init_ms;
  if (!plan_fits(w, A, tctx, min_dec, init_ms)) return false;
  const uint64_t eh = vis ? fb_digest_entry(static_cast<uint32_t>(t.rk),
                                            static_cast<uint32_t>(t.r), 1u)
                          : 0;
  sd.esum = tile_xor_u64(eh);
  sd.E = A;
  const bool log_ok = P.log_on && w.S.log_steps < P.log_step_cap &&
                      w.S.log_entries + A <= P.log_entry_cap;
  if (log_ok && vis)
    P.log_entries[w.I->log_entry_off + w.S.log_entries + t.rk] = fb_plan_entry{t.r, 1};
  t.take = vis ? 1 : 0;
  steady_commit(P, w, sd, now, A, init_ms, min_dec, log_ok, tctx);
  sd.ok = true;
  sd.sub = false;
  w.S.paths |= kPathRepeatRegister;
  return true;
}
#endif


#if FB_STEADY
// A run of repeated-plan steps on registers (steady_run): every visible lane's
// task emits its token, and the plan gives it one token again.
__device__ __forceinline__ int64_t steady_burst(const EngineParams& P, Inst& w, TaskReg& t,
                                                int64_t& ev, int64_t next_arr) {
  const bool vis = tile_lane() < w.sd.E;
  return steady_run(
      P, w, ev, next_arr,
      [&](int64_t now, uint64_t) {  // complete_step
        bool fin = false;
        if (t.take > 0) {
          fin = emit_reg(t, now);
          if (FB_UNLIKELY(fin)) flush_task(P, w, t);
        }
        t.take = 0;
        const unsigned finm = tile_ballot(fin);
        if (FB_UNLIKELY(finm)) remove_finished_rr(w, t, fin, tile_lane() < w.S.n_live, finm);
        return finm != 0;
      },
      [&]() { t.take = vis ? 1 : 0; },
      kPathRepeatRegister);
}
#endif

// Node::begin_step (engine.cpp:153-202) on registers.  Returns 0 when no step
// was launched (nothing visible), 1 when a step was launched, and -1 when the
// keys do not fit the packed form (caller spills and takes the memory path;
// nothing has been modified except the pulled arrivals, which are spilled).
__device__ __forceinline__ int begin_rr(const EngineParams& P, Inst& w, TaskReg& t,
                                        int64_t now, const Scratch& s) {
  const DevInst* I = w.I;
  Steady& sd = w.sd;
  const int lane = tile_lane();
  if (w.S.pulled < w.S.arr) {
    sd.clear();
    pull_rr(P, w, t, now, s);
  }
  const int A = static_cast<int>(visible_count(w));
  if (A == 0) {
    sd.clear();
    return 0;
  }
#if FB_STEADY
  if (sd.ok && A == sd.E && steady_rr(P, w, t, now, sd, A)) return 1;
#if FB_SUB
  if (sd.sub && A == w.S.n_active && sub_rr(P, w, t, now, sd, A)) return 1;
#endif
  sd.clear();
#endif
  const bool vis = lane < A;
  const int policy = w.policy;
  const bool fair = policy == FB_POLICY_FAIRBATCH || policy == FB_POLICY_FAIRBATCH_PAB;

  // K1: views + init_time_budget reductions (sched.cpp:90-106)
  const RView v = view_reg(t, now);
  const int64_t tpot_u = I->tpot_uniform;
  const int64_t min_tpot = tpot_u >= 0 ? tpot_u : tile_min_i64(vis ? t.tpot : kInf);
  const int64_t min_dec = tile_min_i64(vis && v.decode ? v.slack : kInf);
  const int n_dec = __popc(tile_ballot(vis && v.decode));
  double init_ms = 0.0;
  int64_t urgency = 0;
  if (fair) {
    const int64_t init = n_dec == 0 ? min_tpot : (min_dec > min_tpot ? min_dec : min_tpot);
    urgency = init + min_tpot;
    init_ms = us_to_ms(init);
  }

  // K2: packed key (group, slack, seq) and rank by counting
  const bool fits = !vis || (t.seq >= 0 && t.seq < kPackSeq &&
                             (!fair || (v.slack >= -kPackSlack && v.slack < kPackSlack)));
  if (!tile_all(fits)) return -1;
  // Ranks are counted on 32-bit keys whenever that is exact: sarathi /
  // prefill-first keys (group, seq) fit in 32 bits; fair-batching keys use
  // their high half when it is distinct across the visible tasks (the order of
  // distinct high halves is the order of the full keys).
#if FB_RANK_REUSE
  // The previous step's order is usually still sorted (every admitted decode
  // advances by one tpot, every prefill by the same clock): when the visible
  // tasks carry dense previous ranks 0..A-1 and the keys increase along them,
  // those ranks ARE the sort (keys are unique).  Otherwise rank by counting.
  uint64_t key_r;
  if (fair) {
    const uint64_t g = (v.decode && v.slack < urgency) ? 0 : (!v.decode ? 1 : 2);
    key_r = (g << 62) | (static_cast<uint64_t>(v.slack + kPackSlack) << 22) |
            static_cast<uint64_t>(t.seq);
  } else {
    const uint32_t g = policy == FB_POLICY_SARATHI ? (v.decode ? 0u : 1u) : 0u;
    key_r = (static_cast<uint64_t>(g) << 62) | static_cast<uint64_t>(t.seq);
  }
  if (!vis) key_r = ~uint64_t(0);
  const bool rk_ok = !vis || (t.rk >= 0 && t.rk < A);
  const unsigned rk_bits = tile_or(vis && rk_ok ? 1u << t.rk : 0u);
  bool reuse = tile_all(rk_ok) && rk_bits == (A == 32 ? ~0u : (1u << A) - 1u);
  if (reuse) {
    s.order[vis ? t.rk : lane] = lane;
    tile_sync();
    const int nx = vis && t.rk + 1 < A ? s.order[t.rk + 1] : lane;
    const uint64_t kn = tile_shfl(key_r, nx);
    reuse = tile_all(!vis || t.rk + 1 >= A || key_r < kn);
  }
  int rank;
  if (reuse) {
    rank = vis ? t.rk : lane;
  } else {
#endif
  uint64_t key;
    uint32_t k32;
    bool use32;
    if (fair) {
      const uint64_t g = (v.decode && v.slack < urgency) ? 0 : (!v.decode ? 1 : 2);
      key = (g << 62) | (static_cast<uint64_t>(v.slack + kPackSlack) << 22) |
            static_cast<uint64_t>(t.seq);
      k32 = vis ? static_cast<uint32_t>(key >> 32) : 0xffffffffu;  // visible hi <= 0xbfffffff
      const unsigned same = tile_match_any(k32);
      use32 = tile_all(!vis || same == (1u << lane));
    } else {
      const uint32_t g = policy == FB_POLICY_SARATHI ? (v.decode ? 0u : 1u) : 0u;
      key = (static_cast<uint64_t>(g) << 62) | static_cast<uint64_t>(t.seq);
      k32 = vis ? ((g << 30) | static_cast<uint32_t>(t.seq)) : 0xffffffffu;
      use32 = true;
    }
    if (!vis) key = ~uint64_t(0);
#if FB_RANK_REUSE
    rank = 0;
#else
    int rank = 0;
#endif
    if (use32) {
  #pragma unroll kRankUnroll
      for (int q = 0; q < A; ++q) rank += tile_shfl(k32, q) < k32;
    } else {
  #pragma unroll kRankUnroll
      for (int q = 0; q < A; ++q) rank += tile_shfl(key, q) < key;
    }
    if (!vis) rank = lane;
#if FB_RANK_REUSE
    tile_sync();  // the reuse check read s.order
#endif
    s.order[rank] = lane;
    tile_sync();
#if FB_RANK_REUSE
  }
  t.rk = vis ? rank : -1;
#endif
  const int pk = s.order[lane];  // view position at sorted rank `lane` (k < A)

  // K3: sorted costs (sched.cpp:142-144) -> shared scratch -> greedy scan
  const FormCfg f{policy, I->max_chunk, I->token_budget, I->sa, I->sb, I->sc};
  const double cc = dmul(f.c, static_cast<double>(v.ctx));
  const double tc = dadd(dmul(f.b, static_cast<double>(v.nw)), cc);
  const uint32_t nwp = static_cast<uint32_t>(v.nw) | (v.decode ? kDecodeBit : 0u);
  const double tc_s = tile_shfl(tc, pk);
  const double cc_s = tile_shfl(cc, pk);
  const uint32_t nw_s = tile_shfl(nwp, pk);
  const int64_t ctx_s = tile_shfl(v.ctx, pk);
  const int32_t r_s = tile_shfl(t.r, pk);
  // Fair batching, everything fits: the greedy pass admits every task whole
  // iff each prefix fits.  Exact sufficient test without the serial pass:
  // with tb0 = init - a, S = sum of the (already rounded) task costs and
  // N = sum of new tokens, the reference's rounded running budget satisfies
  // tb_k >= tb0 - S_k - k*u*tb0 (u = 2^-53, every intermediate in [0, tb0]),
  // so tb0 - S >= A*2^-52*tb0 (checked with directed rounding on an upper
  // bound of S) and N <= token_budget imply every `consider` admits whole.
  bool all_fit = false;
  if (fair) {
    const double tb0 = dsub(init_ms, f.a);
    const double s_up = tile_sum_ru(vis ? tc : 0.0);
    const int64_t n_new = tile_sum_small(vis ? static_cast<int64_t>(v.nw) : 0);
    all_fit = tb0 >= 0.0 && n_new <= f.token_budget &&
              __dsub_rd(tb0, s_up) >= __dmul_ru(__dmul_ru(static_cast<double>(A), 0x1p-52), tb0);
  }
  int32_t take_s;
  if (all_fit) {
    take_s = vis ? static_cast<int32_t>(nw_s & 0x7fffffffu) : 0;
  } else {
    if (vis) {
      s.tcost[lane] = tc_s;
      s.ccost[lane] = cc_s;
      s.khi[lane] = nw_s;
      s.take[lane] = 0;
    }
    tile_sync();
    if (fair) {
      scan_fairbatch(s, A, init_ms, f);
    } else if (policy == FB_POLICY_SARATHI) {
      scan_sarathi(s, A, n_dec, f);
    } else {
      scan_prefill_first(s, A, f);
    }
    take_s = vis ? s.take[lane] : 0;
  }

  // finalize_plan (sched.cpp:37-48) + digest + log, in admission order
  const unsigned madm = tile_ballot(take_s > 0);
  const int E = __popc(madm);
  const int64_t tn = tile_sum_small(take_s);
  const int64_t tctx = tile_sum_small(take_s > 0 ? ctx_s : 0);
  const double predicted = E == 0 ? 0.0 : predict_ms(f.a, f.b, f.c, tn, tctx);
  const int idx = __popc(madm & tile_lanemask_lt());
  const uint64_t eh = take_s > 0 ? fb_digest_entry(static_cast<uint32_t>(idx),
                                                   static_cast<uint32_t>(r_s),
                                                   static_cast<uint32_t>(take_s))
                                 : 0;
  const uint64_t esum = tile_xor_u64(eh);
  const bool log_ok = P.log_on && w.S.log_steps < P.log_step_cap &&
                      w.S.log_entries + E <= P.log_entry_cap;
  if (log_ok && take_s > 0)
    P.log_entries[I->log_entry_off + w.S.log_entries + idx] = fb_plan_entry{r_s, take_s};

  // ground_truth_step_time_ms, costmodel.cpp:138-146
  double actual = predict_ms(I->ta, I->tb, I->tc, tn, tctx);
  const double amp = I->noise_amp;
  if (amp != 0.0) {
    actual = apply_noise(actual, amp, I->noise_seed, w.S.step_counter);
  }
  int64_t dur = ms_to_us(actual);
  if (dur < 1) dur = 1;

  // takes back to view positions; waiting -> active in plan order
  // (engine.cpp:176-182) as a shuffle permutation
  const int n_act = static_cast<int>(w.S.n_active);
  const int32_t take_v = tile_shfl(take_s, vis ? rank : lane);
  t.take = vis ? take_v : 0;
  const unsigned mw = tile_ballot(take_s > 0 && pk >= n_act);
  const int n_w = __popc(mw);
  if (n_w > 0) {
    const int widx = __popc(mw & tile_lanemask_lt());
    const int widx_v = tile_shfl(widx, vis ? rank : lane);
    const bool un = vis && lane >= n_act && t.take == 0;
    const unsigned mu = tile_ballot(un);
    int dest = lane;
    if (vis && lane >= n_act)
      dest = t.take > 0 ? n_act + widx_v : n_act + n_w + __popc(mu & tile_lanemask_lt());
    tile_sync();
    s.order[dest] = lane;
    tile_sync();
    const int src = s.order[lane];
    permute_task(t, src);
  }

  if (P.log_on) log_step(P, w, log_ok, now, dur, predicted, actual, tn, tctx, init_ms, E);

  w.S.digest = fb_digest_step(w.S.digest, now, static_cast<uint32_t>(E), esum, predicted, actual);
  w.S.sum_visible += A;
  w.S.sum_entries += E;
  w.S.sum_new += tn;
  w.S.n_active = n_act + n_w;
  w.S.busy = 1;
  w.S.step_end = now + dur;
  w.S.step_counter++;
#if FB_STEADY
  // every visible task admitted as a one-token decode: the next step repeats
  // this plan while nothing enters or leaves (fair batching also needs one
  // tpot for the order to stay put)
  steady_record(sd, w, E == A && tn == A && n_dec == A, E, esum, tctx, min_dec, now);
#endif
  return 1;
}

}  // namespace fbgpu
