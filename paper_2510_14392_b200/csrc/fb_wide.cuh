// fb_wide.cuh -- CTA-per-instance engine for nodes with very large live sets
// (BASELINE config 4: 100k+ active requests per instance).
//
// The warp engine escalates an instance to this path when more than
// kEscalateLive requests would be live at a step.  Per step the CTA
//   K1  streams the instance's views (SoA arena, coalesced by view position)
//       once, writing a 64-bit key stem, the context and the new-token count
//       per task and reducing init_time_budget / min context;
//   K2  selects, window by window, the smallest keys of the slack order with
//       an exact MSD radix select (11-bit digits; keys are unique), and
//       bitonic-sorts each window of <= kWideWin keys in shared memory;
//   K3  runs the greedy capacity scan over the sorted windows and stops as
//       soon as no remaining task can be admitted (whole-admission test at
//       (new=1, ctx_min) and chunk test at ctx_min both fail; both tests are
//       monotone under round-to-nearest, SURVEY §7 hard part 2), so only the
//       admitted prefix of the order is ever materialised;
//   K4  moves admitted waiting requests to the active segment in plan order
//       and completes steps with block-wide order-preserving compaction.
// Semantics are those of the warp engine's memory path (same helpers).
#pragma once

namespace fbgpu {

constexpr int kWideThreads = 512;
constexpr int kWideWarps = kWideThreads / kWarp;
constexpr int kWideWin = 2048;
constexpr int kRadixBits = 11;
constexpr int kRadixBins = 1 << kRadixBits;

struct WideSmem {
  uint64_t wkey[kWideWin];
  double wtc[kWideWin];
  double wcc[kWideWin];
  int64_t wcx[kWideWin];
  int32_t wpos[kWideWin];
  uint32_t wnw[kWideWin];
  int32_t wtake[kWideWin];
  uint32_t hist[kRadixBins];
  int64_t red[kWideWarps * 4];
  int64_t bcast[8];
  double dbcast[4];
  int32_t ibcast[8];
};

// Per-instance global scratch (72 bytes per request slot, see Scratch).
struct WideScratch {
  uint64_t* klow;  // [p] decode<<63 | (slack+2^39)<<22 | seq   (stem of the key)
  int64_t* cx;     // [p] context
  int2* vtmp;      // reorder buffer / PAB terms
  uint32_t* nwv;   // [p] new tokens | decode bit
  int32_t* mark;   // [p] admitted-waiting flag
};

__device__ __forceinline__ WideScratch wide_scratch(const EngineParams& P, const Inst& w) {
  WideScratch s;
  unsigned char* base = P.gscratch + w.roff * kScratchBytesPerSlot;
  const size_t n = static_cast<size_t>(w.nreq);
  s.klow = reinterpret_cast<uint64_t*>(base);
  s.cx = reinterpret_cast<int64_t*>(base + 8 * n);
  s.vtmp = reinterpret_cast<int2*>(base + 16 * n);
  s.nwv = reinterpret_cast<uint32_t*>(base + 24 * n);
  s.mark = reinterpret_cast<int32_t*>(base + 28 * n);
  return s;
}

// ------------------------------------------------------ block primitives

__device__ __forceinline__ int wid() { return threadIdx.x / kWarp; }

// Block reductions return the same value in every thread.
__device__ __forceinline__ int64_t block_min(int64_t v, WideSmem& sm) {
  v = warp_min(v);
  if (lane_id() == 0) sm.red[wid()] = v;
  __syncthreads();
  if (wid() == 0) {
    int64_t x = lane_id() < kWideWarps ? sm.red[lane_id()] : kInf;
    x = warp_min(x);
    if (lane_id() == 0) sm.bcast[0] = x;
  }
  __syncthreads();
  const int64_t r = sm.bcast[0];
  __syncthreads();
  return r;
}
__device__ __forceinline__ int64_t block_sum(int64_t v, WideSmem& sm) {
  v = warp_sum(v);
  if (lane_id() == 0) sm.red[wid()] = v;
  __syncthreads();
  if (wid() == 0) {
    int64_t x = lane_id() < kWideWarps ? sm.red[lane_id()] : 0;
    x = warp_sum(x);
    if (lane_id() == 0) sm.bcast[0] = x;
  }
  __syncthreads();
  const int64_t r = sm.bcast[0];
  __syncthreads();
  return r;
}
__device__ __forceinline__ uint64_t block_xor(uint64_t v, WideSmem& sm) {
  v = warp_xor_u64(v);
  if (lane_id() == 0) sm.red[wid()] = static_cast<int64_t>(v);
  __syncthreads();
  if (wid() == 0) {
    uint64_t x = lane_id() < kWideWarps ? static_cast<uint64_t>(sm.red[lane_id()]) : 0;
    x = warp_xor_u64(x);
    if (lane_id() == 0) sm.bcast[0] = static_cast<int64_t>(x);
  }
  __syncthreads();
  const uint64_t r = static_cast<uint64_t>(sm.bcast[0]);
  __syncthreads();
  return r;
}
// Exclusive prefix count of `flag` over the block (thread order) plus the
// block total.
__device__ __forceinline__ int block_excl_count(bool flag, int& total, WideSmem& sm) {
  const unsigned m = __ballot_sync(kFull, flag);
  if (lane_id() == 0) sm.red[wid()] = __popc(m);
  __syncthreads();
  int before = 0, tot = 0;
  for (int i = 0; i < kWideWarps; ++i) {
    const int c = static_cast<int>(sm.red[i]);
    if (i < wid()) before += c;
    tot += c;
  }
  __syncthreads();
  total = tot;
  return before + __popc(m & lanemask_lt());
}

// Exclusive prefix sum of non-negative ints over the block (thread order).
__device__ __forceinline__ int block_excl_sum(int v, int& total, WideSmem& sm) {
  int incl = v;
#pragma unroll
  for (int o = 1; o < kWarp; o <<= 1) {
    const int y = __shfl_up_sync(kFull, incl, o);
    if (lane_id() >= o) incl += y;
  }
  if (lane_id() == kWarp - 1) sm.red[wid()] = incl;
  __syncthreads();
  int before = 0, tot = 0;
  for (int i = 0; i < kWideWarps; ++i) {
    const int c = static_cast<int>(sm.red[i]);
    if (i < wid()) before += c;
    tot += c;
  }
  __syncthreads();
  total = tot;
  return before + incl - v;
}

// Key of a task from its stem (K2a, sched.cpp:110-127): fair batching ranks
// (urgent decode, prefill, relaxed decode) then slack then seq.
__device__ __forceinline__ uint64_t wide_key(uint64_t klow, int policy, int64_t urgency) {
  const bool decode = (klow >> 63) != 0;
  const uint64_t low = klow & ((uint64_t(1) << 62) - 1);
  if (policy == FB_POLICY_FAIRBATCH || policy == FB_POLICY_FAIRBATCH_PAB) {
    const int64_t slack = static_cast<int64_t>(low >> 22) - kPackSlack;
    const uint64_t g = decode ? (slack < urgency ? 0 : 2) : 1;
    return (g << 62) | low;
  }
  const uint64_t seq = low & ((uint64_t(1) << 22) - 1);
  if (policy == FB_POLICY_SARATHI) return ((decode ? uint64_t(0) : uint64_t(1)) << 62) | seq;
  return seq;
}

// K2: the K = min(kWideWin, #{key > lo}) smallest keys above `lo` (all keys
// when !has_lo), sorted ascending into sm.wkey / sm.wpos.  Exact MSD radix
// select on 64-bit unique keys, then a shared-memory bitonic sort.
__device__ int wide_select(const WideScratch& ws, int A, bool has_lo, uint64_t lo, int policy,
                           int64_t urgency, WideSmem& sm) {
  uint64_t prefix = 0, pmask = 0;
  int need = kWideWin;
  bool take_all = false;
  uint64_t hi = ~uint64_t(0);  // inclusive upper bound of the selected set
  for (int pass = 0; pass < 6; ++pass) {
    const int shift = 64 - kRadixBits * (pass + 1) > 0 ? 64 - kRadixBits * (pass + 1) : 0;
    const int bits = pass < 5 ? kRadixBits : 64 - 5 * kRadixBits;  // 11 x5 + 9
    const uint64_t dmask = (uint64_t(1) << bits) - 1;
    for (int i = threadIdx.x; i < kRadixBins; i += kWideThreads) sm.hist[i] = 0;
    __syncthreads();
    for (int b0 = 0; b0 < A; b0 += kWideThreads) {  // warp-aggregated histogram
      const int p = b0 + threadIdx.x;
      int bin = -1;
      if (p < A) {
        const uint64_t key = wide_key(ws.klow[p], policy, urgency);
        if ((!has_lo || key > lo) && (key & pmask) == prefix)
          bin = static_cast<int>((key >> shift) & dmask);
      }
      const unsigned same = __match_any_sync(kFull, bin);
      if (bin >= 0 && lane_id() == __ffs(same) - 1) atomicAdd(&sm.hist[bin], __popc(same));
    }
    __syncthreads();
    {  // locate the bin holding the need-th candidate: block scan over bins
      constexpr int kPer = kRadixBins / kWideThreads;
      const int b0 = threadIdx.x * kPer;
      int loc = 0;
#pragma unroll
      for (int q = 0; q < kPer; ++q) loc += static_cast<int>(sm.hist[b0 + q]);
      int tot;
      const int before = block_excl_sum(loc, tot, sm);
      if (threadIdx.x == 0) sm.ibcast[0] = (pass == 0 && tot <= kWideWin) ? 1 : 0;
      if (before < need && need <= before + loc) {
        int cum = before;
        for (int q = 0; q < kPer; ++q) {
          const int c = static_cast<int>(sm.hist[b0 + q]);
          if (cum + c >= need) {
            sm.ibcast[1] = b0 + q;
            sm.ibcast[2] = need - cum;  // still needed inside the bin
            sm.ibcast[3] = c == need - cum;
            break;
          }
          cum += c;
        }
      }
    }
    __syncthreads();
    if (sm.ibcast[0]) {
      take_all = true;
      break;
    }
    const uint64_t bin = static_cast<uint64_t>(sm.ibcast[1]);
    need = sm.ibcast[2];
    prefix |= bin << shift;
    pmask |= dmask << shift;
    const bool exact = sm.ibcast[3] != 0;
    __syncthreads();
    if (exact || pass == 5) {
      hi = prefix | ((shift > 0) ? ((uint64_t(1) << shift) - 1) : 0);
      break;
    }
  }
  // gather the selected keys
  if (threadIdx.x == 0) sm.ibcast[4] = 0;
  __syncthreads();
  for (int p = threadIdx.x; p < A; p += kWideThreads) {
    const uint64_t key = wide_key(ws.klow[p], policy, urgency);
    if ((!has_lo || key > lo) && (take_all || key <= hi)) {
      const int slot = atomicAdd(&sm.ibcast[4], 1);
      sm.wkey[slot] = key;
      sm.wpos[slot] = p;
    }
  }
  __syncthreads();
  const int K = sm.ibcast[4];
  int n2 = 1;
  while (n2 < K) n2 <<= 1;
  for (int i = K + threadIdx.x; i < n2; i += kWideThreads) {
    sm.wkey[i] = ~uint64_t(0);
    sm.wpos[i] = -1;
  }
  __syncthreads();
  for (int k = 2; k <= n2; k <<= 1) {  // bitonic sort (keys unique)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n2; i += kWideThreads) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const uint64_t a = sm.wkey[i], b = sm.wkey[ixj];
          const bool asc = (i & k) == 0;
          if ((a > b) == asc) {
            sm.wkey[i] = b;
            sm.wkey[ixj] = a;
            const int t = sm.wpos[i];
            sm.wpos[i] = sm.wpos[ixj];
            sm.wpos[ixj] = t;
          }
        }
      }
      __syncthreads();
    }
  }
  __syncthreads();
  return K;
}

// K3 scan state carried across windows (thread 0 owns it).
struct WideScan {
  double tb;
  int64_t tok;      // fair: token budget; sarathi: remaining prefill tokens; pf: budget
  int64_t n_seen;   // tasks already considered (sarathi: decodes come first)
  int32_t E;
  int64_t tn, tctx;
  bool done;
};

// Greedy pass over one sorted window (sched.cpp:129-232), thread 0.
__device__ void wide_scan_window(WideScan& st, int K, int policy, const FormCfg& f, int n_dec,
                                 double tc_min, double cc_min, const WideScratch& ws,
                                 WideSmem& sm) {
  if (threadIdx.x != 0) return;
  const bool fair = policy == FB_POLICY_FAIRBATCH || policy == FB_POLICY_FAIRBATCH_PAB;
  for (int k = 0; k < K && !st.done; ++k) {
    const uint32_t w = sm.wnw[k];
    const int64_t nv = w & 0x7fffffffu;
    int64_t take = 0;
    if (fair) {
      if (st.tok <= 0 || st.tb < 0.0) {
        st.done = true;
        break;
      }
      if (st.tb < tc_min) {  // no task fits whole any more: stop if none can chunk
        const double lim = ddiv(dsub(st.tb, cc_min), f.b);
        const double dt = static_cast<double>(st.tok);
        const double cpr = lim < dt ? lim : dt;
        if (!(cc_min <= st.tb && floor(cpr) >= 1.0)) {
          st.done = true;
          break;
        }
      }
      const double tc = sm.wtc[k], cc = sm.wcc[k];
      if (tc <= st.tb && nv <= st.tok) {
        take = nv;
        st.tb = dsub(st.tb, tc);
        st.tok -= nv;
      } else if (st.tok > 0 && cc <= st.tb) {
        const double lim = ddiv(dsub(st.tb, cc), f.b);
        const double dt = static_cast<double>(st.tok);
        const double cp_real = lim < dt ? lim : dt;
        const int64_t cp = static_cast<int64_t>(floor(cp_real));
        if (cp >= 1) {
          take = cp;
          st.tb = dsub(st.tb, dadd(dmul(f.b, static_cast<double>(cp)), cc));
          st.tok -= cp;
        }
      }
    } else if (policy == FB_POLICY_SARATHI) {
      if (st.n_seen < n_dec) {
        take = 1;
      } else {
        if (st.tok <= 0) {
          st.done = true;
          break;
        }
        int64_t chunk = st.tok;
        if (f.max_chunk < chunk) chunk = f.max_chunk;
        if (nv < chunk) chunk = nv;
        if (chunk >= 1) {
          take = chunk;
          st.tok -= chunk;
        }
      }
    } else {
      if (st.tok <= 0) {
        st.done = true;
        break;
      }
      int64_t t2;
      if (w & kDecodeBit) {
        t2 = 1;
      } else {
        t2 = st.tok;
        if (f.max_chunk < t2) t2 = f.max_chunk;
        if (nv < t2) t2 = nv;
      }
      if (t2 >= 1 && t2 <= st.tok) {
        take = t2;
        st.tok -= t2;
      }
    }
    st.n_seen++;
    sm.wtake[k] = static_cast<int32_t>(take);
    if (take > 0) {
      st.E++;
      st.tn += take;
      st.tctx += sm.wcx[k];
    }
  }
}

// Node::complete_step (engine.cpp:204-254), block-wide.
__device__ void wide_complete(const EngineParams& P, Inst& w, WideSmem& sm) {
  const int64_t t = w.S.step_end;
  int any = 0;
  for (int64_t p = threadIdx.x; p < w.S.n_active; p += kWideThreads) {
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
        emit = pf >= prompt;
      }
      bool fin = false;
      if (emit) fin = emit_token(P, g, row, t);
      w.vl[p] = make_int2(fin ? -1 : v.x, 0);
      any |= fin;
    }
  }
  if (__syncthreads_or(any)) {  // order-preserving removal (engine.cpp:228-229)
    const int64_t n = w.S.n_live;
    int64_t out = 0, removed_active = 0;
    for (int64_t b = 0; b < n; b += kWideThreads) {
      const int64_t p = b + threadIdx.x;
      int2 v = make_int2(-1, 0);
      if (p < n) v = w.vl[p];
      const bool keep = p < n && v.x >= 0;
      int tot;
      const int pos = block_excl_count(keep, tot, sm);
      int rtot;
      block_excl_count(p < n && !keep && p < w.S.n_active, rtot, sm);
      if (keep) w.vl[out + pos] = v;
      __syncthreads();
      out += tot;
      removed_active += rtot;
    }
    w.S.n_live = out;
    w.S.n_active -= removed_active;
  }
  __syncthreads();
  w.S.busy = 0;
}

// Node::pull_arrivals (engine.cpp:127-151), block-wide.
__device__ void wide_pull(const EngineParams& P, Inst& w, int64_t now, const WideScratch& ws,
                          WideSmem& sm) {
  if (w.policy != FB_POLICY_FAIRBATCH_PAB) {
    const int64_t k = w.S.arr - w.S.pulled;
    for (int64_t j = threadIdx.x; j < k; j += kWideThreads) {
      const int64_t r = arrival_row(w, w.S.pulled + j);
      P.seq[w.roff + r] = static_cast<int32_t>(w.S.seq_counter + j);
      w.vl[w.S.n_live + j] = make_int2(static_cast<int>(r), 0);
    }
    __syncthreads();
    w.S.seq_counter += k;
    w.S.n_live += k;
    w.S.pulled = w.S.arr;
    return;
  }
  // K5 with the ordered view fold (sched.cpp:248-278, engine.cpp:128-150)
  const DevInst* I = w.I;
  const double Wm = us_to_ms(I->g_ttft), Tm = us_to_ms(I->g_tpot);
  const double a = I->sa, b = I->sb, c = I->sc;
  int64_t A = visible_count(w);
  double* terms = reinterpret_cast<double*>(ws.vtmp);
  int64_t lmin = kInf, lpf = 0;
  for (int64_t p = threadIdx.x; p < A; p += kWideThreads) {
    const View v = load_view(P, w, p, now);
    terms[p] = pab_term(Wm, Tm, b, c, v.slack, v.ctx);
    lmin = v.slack < lmin ? v.slack : lmin;
    if (!v.decode) lpf += v.nw;
  }
  int64_t min_slack = block_min(lmin, sm);
  int64_t pf_tok = block_sum(lpf, sm);
  if (threadIdx.x == 0) {
    double r_tasks = 0.0;
    for (int64_t p = 0; p < A; ++p) r_tasks = dadd(r_tasks, terms[p]);
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
        P.seq[w.roff + r] = static_cast<int32_t>(w.S.seq_counter);
        w.vl[w.S.n_live] = make_int2(static_cast<int>(r), 0);
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
        P.flags[w.roff + r] |= FB_REC_REJECTED;
        if (P.log_on) {
          if (w.S.log_rejects < P.log_reject_cap) {
            fb_reject_log& rl = P.log_rejects[I->log_reject_off + w.S.log_rejects];
            rl.t_us = now;
            rl.pab_tokens = budget;
            rl.req = static_cast<int32_t>(r);
            rl.reserved = 0;
            w.S.log_rejects++;
          } else {
            w.S.log_trunc = 1;
          }
        }
        w.S.digest = fb_digest_reject(w.S.digest, now, static_cast<uint32_t>(r), budget);
        w.S.n_rejected++;
      }
    }
    w.S.pulled = w.S.arr;
    sm.bcast[1] = w.S.seq_counter;
    sm.bcast[2] = w.S.n_live;
    sm.bcast[3] = w.S.n_rejected;
    sm.bcast[4] = static_cast<int64_t>(w.S.digest);
    sm.ibcast[5] = w.S.log_rejects;
    sm.ibcast[6] = w.S.log_trunc;
  }
  __syncthreads();
  w.S.pulled = w.S.arr;
  w.S.seq_counter = sm.bcast[1];
  w.S.n_live = sm.bcast[2];
  w.S.n_rejected = sm.bcast[3];
  w.S.digest = static_cast<uint64_t>(sm.bcast[4]);
  w.S.log_rejects = sm.ibcast[5];
  w.S.log_trunc = sm.ibcast[6];
  __syncthreads();
}

// Node::begin_step (engine.cpp:153-202), block-wide.
__device__ void wide_begin(const EngineParams& P, Inst& w, int64_t now, WideSmem& sm) {
  const DevInst* I = w.I;
  const WideScratch ws = wide_scratch(P, w);
  w.S.paths |= kPathWide;
  if (w.S.pulled < w.S.arr) wide_pull(P, w, now, ws, sm);
  const int64_t A64 = visible_count(w);
  if (A64 == 0) return;
  const int A = static_cast<int>(A64);
  const int policy = w.policy;
  const bool fair = policy == FB_POLICY_FAIRBATCH || policy == FB_POLICY_FAIRBATCH_PAB;
  const int64_t n_act = w.S.n_active;

  // K1: one streaming pass over the views
  int64_t l_tpot = kInf, l_dec = kInf, l_ctx = kInf, l_ndec = 0, l_bad = 0;
  for (int64_t p = threadIdx.x; p < A; p += kWideThreads) {
    const View v = load_view(P, w, p, now);
    const bool fits = v.seq >= 0 && v.seq < kPackSeq &&
                      (!fair || (v.slack >= -kPackSlack && v.slack < kPackSlack));
    l_bad |= !fits;
    const uint64_t sl = fair ? static_cast<uint64_t>(v.slack + kPackSlack) : 0;
    ws.klow[p] = (v.decode ? (uint64_t(1) << 63) : 0) | (sl << 22) | static_cast<uint64_t>(v.seq);
    ws.cx[p] = v.ctx;
    ws.nwv[p] = static_cast<uint32_t>(v.nw);
    ws.mark[p] = 0;
    if (p < n_act) w.vl[p].y = 0;  // takes are rewritten for admitted tasks below
    l_tpot = v.tpot < l_tpot ? v.tpot : l_tpot;
    l_ctx = v.ctx < l_ctx ? v.ctx : l_ctx;
    if (v.decode) {
      l_ndec++;
      l_dec = v.slack < l_dec ? v.slack : l_dec;
    }
  }
  const int64_t min_tpot = block_min(l_tpot, sm);
  const int64_t min_dec = block_min(l_dec, sm);
  const int64_t ctx_min = block_min(l_ctx, sm);
  const int64_t n_dec = block_sum(l_ndec, sm);
  if (block_sum(l_bad, sm) != 0) {  // keys outside the packed range: not supported here
    w.S.status = FB_ERR_VALIDATION;
    w.S.done = 1;
    return;
  }
  double init_ms = 0.0;
  int64_t urgency = 0;
  if (fair) {
    const int64_t init = n_dec == 0 ? min_tpot : (min_dec > min_tpot ? min_dec : min_tpot);
    urgency = init + min_tpot;
    init_ms = us_to_ms(init);
  }
  const FormCfg f{policy, I->max_chunk, I->token_budget, I->sa, I->sb, I->sc};
  const double cc_min = dmul(f.c, static_cast<double>(ctx_min));
  const double tc_min = dadd(dmul(f.b, 1.0), cc_min);

  // K2 + K3 over sorted windows
  WideScan st;
  st.tb = fair ? dsub(init_ms, f.a) : 0.0;
  st.tok = f.token_budget;
  if (policy == FB_POLICY_SARATHI) {
    st.tok = f.token_budget - n_dec;
    if (st.tok < 0) st.tok = 0;
  }
  st.n_seen = 0;
  st.E = 0;
  st.tn = 0;
  st.tctx = 0;
  st.done = false;
  bool has_lo = false;
  uint64_t lo = 0;
  uint64_t esum = 0;
  int E_before = 0, Ew_before = 0;
  const bool log_on = P.log_on != 0;
  const int64_t entry_base = I->log_entry_off + w.S.log_entries;
  for (;;) {
    const int K = wide_select(ws, A, has_lo, lo, policy, urgency, sm);
    if (K == 0) break;
    for (int k = threadIdx.x; k < K; k += kWideThreads) {
      const int p = sm.wpos[k];
      const uint32_t nwp = ws.nwv[p];
      const int64_t cxp = ws.cx[p];
      const double cc = dmul(f.c, static_cast<double>(cxp));
      sm.wcc[k] = cc;
      sm.wcx[k] = cxp;
      sm.wtc[k] = dadd(dmul(f.b, static_cast<double>(nwp & 0x7fffffffu)), cc);
      sm.wnw[k] = nwp;
      sm.wtake[k] = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      wide_scan_window(st, K, policy, f, static_cast<int>(n_dec), tc_min, cc_min, ws, sm);
      sm.ibcast[7] = st.done ? 1 : 0;
    }
    __syncthreads();
    const bool done = sm.ibcast[7] != 0;
    // plan bookkeeping for this window, in admission order
    for (int k0 = 0; k0 < K; k0 += kWideThreads) {
      const int k = k0 + threadIdx.x;
      int take = 0, p = 0;
      if (k < K) {
        take = sm.wtake[k];
        p = sm.wpos[k];
      }
      int tot, totw;
      const int idx = block_excl_count(take > 0, tot, sm);
      const bool wadm = take > 0 && p >= n_act;
      const int widx = block_excl_count(wadm, totw, sm);
      if (take > 0) {
        const int r = w.vl[p].x;
        esum ^= fb_digest_entry(static_cast<uint32_t>(E_before + idx), static_cast<uint32_t>(r),
                                static_cast<uint32_t>(take));
        if (log_on) {
          const int64_t e = w.S.log_entries + E_before + idx;
          if (e < P.log_entry_cap) P.log_entries[entry_base + E_before + idx] = fb_plan_entry{r, take};
        }
        if (p < n_act) {
          w.vl[p].y = take;
        } else {
          ws.vtmp[Ew_before + widx] = make_int2(r, take);
          ws.mark[p] = 1;
        }
      }
      E_before += tot;
      Ew_before += totw;
    }
    __syncthreads();
    if (done || K < kWideWin) break;
    has_lo = true;
    lo = sm.wkey[K - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    sm.bcast[5] = st.tn;
    sm.bcast[6] = st.tctx;
    sm.ibcast[5] = st.E;
  }
  __syncthreads();
  const int64_t tn = sm.bcast[5];
  const int64_t tctx = sm.bcast[6];
  const int E = sm.ibcast[5];
  esum = block_xor(esum, sm);
  const double predicted = E == 0 ? 0.0 : predict_ms(f.a, f.b, f.c, tn, tctx);

  // waiting -> active in plan order (engine.cpp:176-182): admitted waiting
  // are already in vtmp[0, n_w); the rest of the visible waiting follow in
  // their old order, then everything is copied back.
  const int n_w = Ew_before;
  if (n_w > 0) {
    int64_t run = 0;
    for (int64_t b = n_act; b < A64; b += kWideThreads) {
      const int64_t p = b + threadIdx.x;
      int2 v = make_int2(0, 0);
      bool un = false;
      if (p < A64) {
        v = w.vl[p];
        un = ws.mark[p] == 0;
      }
      int tot;
      const int pos = block_excl_count(un, tot, sm);
      if (un) ws.vtmp[n_w + run + pos] = make_int2(v.x, 0);
      run += tot;
    }
    __syncthreads();
    for (int64_t q = threadIdx.x; q < A64 - n_act; q += kWideThreads) w.vl[n_act + q] = ws.vtmp[q];
    __syncthreads();
  }

  // ground_truth_step_time_ms, costmodel.cpp:138-146
  double actual = predict_ms(I->ta, I->tb, I->tc, tn, tctx);
  const double amp = I->noise_amp;
  if (amp != 0.0) {
    const double u = dsub(dmul(2.0, keyed_uniform(I->noise_seed, w.S.step_counter)), 1.0);
    actual = dmul(actual, dadd(1.0, dmul(amp, u)));
  }
  int64_t dur = ms_to_us(actual);
  if (dur < 1) dur = 1;
  if (log_on) {
    const bool ok = w.S.log_steps < P.log_step_cap && w.S.log_entries + E <= P.log_entry_cap;
    if (ok) {
      if (threadIdx.x == 0) {
        fb_step_log& sl = P.log_steps[I->log_step_off + w.S.log_steps];
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
  w.S.digest = fb_digest_step(w.S.digest, now, static_cast<uint32_t>(E), esum, predicted, actual);
  w.S.sum_visible += A64;
  w.S.sum_entries += E;
  w.S.sum_new += tn;
  w.S.n_active = n_act + n_w;
  w.S.busy = 1;
  w.S.step_end = now + dur;
  w.S.step_counter++;
  __syncthreads();
}

// run_node's loop for an escalated instance; resumes a begin_step that the
// warp engine deferred.
__device__ void wide_run(const EngineParams& P, Inst& w, WideSmem& sm) {
  const int64_t* arrival = P.arrival + w.toff;
  if (w.S.pending_begin) {
    w.S.pending_begin = 0;
    wide_begin(P, w, w.S.t_last, sm);
    if (w.S.done) return;
  }
  for (int64_t ev = 0; ev < P.max_events; ++ev) {
    if (w.S.busy) {
      // Arrivals strictly before the in-flight step's end only enqueue
      // (run_node's loop neither completes nor begins a step at those
      // times), so they are consumed in one block-wide sweep.
      while (w.S.arr < w.nreq) {
        const int64_t q = w.S.arr + threadIdx.x;
        const bool early = q < w.nreq && arrival[q] < w.S.step_end;
        const int n = __syncthreads_count(early);
        w.S.arr += n;
        if (n < kWideThreads) break;
      }
    }
    const int64_t t_step = w.S.busy ? w.S.step_end : kInf;
    const int64_t t_arr = w.S.arr < w.nreq ? arrival[w.S.arr] : kInf;
    const int64_t t = t_step < t_arr ? t_step : t_arr;
    if (t == kInf || (!w.S.busy && t >= w.horizon)) {
      w.S.done = 1;
      w.S.incomplete = (w.S.busy || w.S.pulled < w.S.arr || w.S.n_live > 0 ||
                        w.S.arr < w.nreq) ? 1 : 0;
      return;
    }
    w.S.t_last = t;
    if (w.S.busy && t_step == t) wide_complete(P, w, sm);
    while (w.S.arr < w.nreq && arrival[w.S.arr] == t) w.S.arr++;
    if (!w.S.busy && t < w.horizon) {
      wide_begin(P, w, t, sm);
      if (w.S.done) return;
    }
  }
}

__global__ void __launch_bounds__(kWideThreads, 1)
wide_kernel(const __grid_constant__ EngineParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WideSmem& sm = *reinterpret_cast<WideSmem*>(smem_raw);
  __shared__ unsigned long long s_idx;
  for (;;) {
    if (threadIdx.x == 0) s_idx = atomicAdd(&P.work[2], 1ull);
    __syncthreads();
    const unsigned long long j = s_idx;
    __syncthreads();
    if (j >= P.work[3]) break;
    const int64_t i = P.wide_list[j];
    Inst w;
    w.id = i;
    w.routed = nullptr;
    w.I = P.inst + i;
    w.S = P.state[i];
    if (w.S.done) continue;
    w.toff = w.I->trace_off;
    w.roff = w.I->rec_off;
    w.nreq = w.I->n_req;
    w.horizon = w.I->horizon;
    w.policy = w.I->policy;
    w.max_active = w.I->max_active;
    w.vl = P.vlist + w.roff;
    w.smem = nullptr;
    wide_run(P, w, sm);
    __syncthreads();
    if (threadIdx.x == 0) {
      P.state[i] = w.S;
      if (!w.S.done) atomicAdd(&P.work[1], 1ull);
    }
    __syncthreads();
  }
}

}  // namespace fbgpu
