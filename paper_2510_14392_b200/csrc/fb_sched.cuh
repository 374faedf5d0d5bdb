// fb_sched.cuh -- per-warp batch formation over one task set.
//
//   K1  envelope slack + grouping     (callers fill Scratch [p], see fb_engine.cu)
//   K2  slack-ordered selection       make_keys + rank_order
//   K3  adaptive capacity scan        gather_sorted + scan_* (+ finalize)
//   K5  prefill admission budget      pab_term / pab_close
//
// One warp owns one task set.  Views live in a Scratch (shared memory for
// small sets, the instance's global scratch otherwise).  All lanes execute
// every function (warp-uniform control flow); results are warp-uniform.
#pragma once

#include "fb_device.cuh"

namespace fbgpu {

struct FormCfg {
  int32_t policy;
  int32_t max_chunk;
  int64_t token_budget;
  double a, b, c;  // scheduler model
};

struct FormOut {
  int32_t n_entries;
  int64_t total_new;
  int64_t total_ctx;
  double predicted_ms;
  double init_ms;  // BatchPlan::init_time_budget_ms (0 unless fair batching)
};

// Lane-local accumulators of the K1 reductions (init_time_budget inputs).
struct ViewAcc {
  int64_t min_tpot = kInf;
  int64_t min_dec = kInf;
  int32_t n_dec = 0;
  __device__ __forceinline__ void add(bool decode, int64_t slack, int64_t tpot) {
    min_tpot = tpot < min_tpot ? tpot : min_tpot;
    if (decode) {
      n_dec++;
      min_dec = slack < min_dec ? slack : min_dec;
    }
  }
  __device__ __forceinline__ void reduce() {
    min_tpot = tile_min_i64(min_tpot);
    min_dec = tile_min_i64(min_dec);
    n_dec = static_cast<int32_t>(__reduce_add_sync(tile_mask(), static_cast<uint32_t>(n_dec)));
  }
};

constexpr int64_t kPackSlack = int64_t(1) << 39;  // packed slack range [-2^39, 2^39)
constexpr int64_t kPackSeq = int64_t(1) << 22;    // packed seq range [0, 2^22)

// K2a: sort keys.  Fair batching: (group, slack, seq) with group 0 urgent
// decode / 1 prefill / 2 relaxed decode (sched.cpp:110-127); sarathi:
// (decode first, fifo) (sched.cpp:174-178); prefill-first: fifo
// (sched.cpp:210-211).
//
// With unique seqs inside the packing range (always, for engine nodes) the key
// is ONE u64: (group << 62) | ((slack + 2^39) << 22) | seq.  Otherwise khi
// holds (group << 62) | (slack + 2^61) and seq breaks ties (slack must lie in
// [-2^61, 2^61), validated on input).  Returns the (warp-uniform) packing.
__device__ __forceinline__ bool make_keys(const Scratch& s, int A, int policy,
                                          int64_t urgency, bool seq_unique) {
  const bool fair = policy == FB_POLICY_FAIRBATCH || policy == FB_POLICY_FAIRBATCH_PAB;
  bool ok = seq_unique;
  if (ok) {
    FB_COLD_LOOP
    for (int p = tile_lane(); p < A; p += kTile) {
      const int64_t sq = s.seq[p];
      bool f = sq >= 0 && sq < kPackSeq;
      if (fair) {
        const int64_t slack = s.slack[p];
        f = f && slack >= -kPackSlack && slack < kPackSlack;
      }
      ok = ok && f;
    }
  }
  const bool packed = tile_all(ok);
  FB_COLD_LOOP
  for (int p = tile_lane(); p < A; p += kTile) {
    const bool decode = (static_cast<uint32_t>(s.nw[p]) & kDecodeBit) != 0;
    uint64_t g, sl = 0;
    if (fair) {
      const int64_t slack = s.slack[p];
      g = (decode && slack < urgency) ? 0 : (!decode ? 1 : 2);
      sl = packed ? (static_cast<uint64_t>(slack + kPackSlack) << 22) |
                        static_cast<uint64_t>(s.seq[p])
                  : static_cast<uint64_t>(slack + (int64_t(1) << 61)) &
                        ((uint64_t(1) << 62) - 1);
    } else {
      g = policy == FB_POLICY_SARATHI ? (decode ? 0 : 1) : 0;
      if (packed) sl = static_cast<uint64_t>(s.seq[p]);
    }
    s.khi[p] = (g << 62) | sl;
  }
  tile_sync();
  return packed;
}

// K2b: order[k] = view position of rank k, by counting smaller keys.  Packed
// keys are unique (seq_counter_ only grows, engine.cpp:147), so one u64
// compare per pair suffices; the general form breaks exact ties by view
// position so the result is always a permutation.
__device__ __forceinline__ void rank_order(const Scratch& s, int A, bool packed) {
  if (packed && A <= 2 * kTile) {
    // at most two keys per lane, compared over shuffles (no shared-memory
    // round trip per compare; absent slots hold ~0, above every packed key)
    const int l = tile_lane();
    const uint64_t k0 = l < A ? s.khi[l] : ~uint64_t(0);
    const uint64_t k1 = l + kTile < A ? s.khi[l + kTile] : ~uint64_t(0);
    int r0 = 0, r1 = 0;
    FB_COLD_LOOP
    for (int q = 0; q < kTile; ++q) {
      const uint64_t b0 = tile_shfl(k0, q), b1 = tile_shfl(k1, q);
      r0 += (b0 < k0) + (b1 < k0);
      r1 += (b0 < k1) + (b1 < k1);
    }
    tile_sync();
    if (l < A) s.order[r0] = l;
    if (l + kTile < A) s.order[r1] = l + kTile;
    tile_sync();
    return;
  }
  if (packed) {
    FB_COLD_LOOP
    for (int p0 = 0; p0 < A; p0 += kTile) {
      const int p = p0 + tile_lane();
      const uint64_t kh = p < A ? s.khi[p] : 0;
      int rank = 0;
FB_COLD_LOOP
      for (int q = 0; q < A; ++q) rank += s.khi[q] < kh;
      if (p < A) s.order[rank] = p;
    }
    tile_sync();
    return;
  }
  FB_COLD_LOOP
  for (int p0 = 0; p0 < A; p0 += kTile) {
    const int p = p0 + tile_lane();
    uint64_t kh = 0;
    int64_t ks = 0;
    if (p < A) {
      kh = s.khi[p];
      ks = s.seq[p];
    }
    int rank = 0;
    FB_COLD_LOOP
    for (int q = 0; q < A; ++q) {
      const uint64_t qh = s.khi[q];
      const int64_t qs = s.seq[q];
      rank += (qh < kh) || (qh == kh && (qs < ks || (qs == ks && q < p)));
    }
    if (p < A) s.order[rank] = p;
  }
  tile_sync();
}

// K3a: per sorted position, the state-independent costs (sched.cpp:142-144)
// and the sorted (new|phase) / context, into arrays K2 no longer needs.
__device__ __forceinline__ void gather_sorted(const Scratch& s, int A, double b,
                                              double c) {
  // khi / seq are free after rank_order (which ends in __syncwarp).
  FB_COLD_LOOP
  for (int k = tile_lane(); k < A; k += kTile) {
    {
      const int p = s.order[k];
      const int32_t nwv = s.nw[p];
      const int64_t cx = s.ctx[p];
      const int32_t nv = nwv & 0x7fffffff;
      const double cc = dmul(c, static_cast<double>(cx));
      s.ccost[k] = cc;
      s.tcost[k] = dadd(dmul(b, static_cast<double>(nv)), cc);
      s.khi[k] = static_cast<uint32_t>(nwv);  // sorted new|phase
      s.seq[k] = cx;                          // sorted context
      s.take[k] = 0;
    }
  }
  tile_sync();
}

// K3b: the greedy `consider` pass of form_batch_fairbatching
// (sched.cpp:129-166).  Skipped tasks never mutate the budgets, and the
// budgets only shrink, so the pass stops exactly when neither branch can
// admit anything any more (token_budget <= 0, or time_budget < 0 since
// b > 0 and c*ctx >= 0).  That early exit needs every task to carry
// new >= 1 and c*ctx >= 0 -- always true for the engines' views; the pure
// scheduler (fb_form_batch) passes `exits_ok` = false for sets holding a
// zero-token task (which `consider` admits as {id, 0} whenever
// c*ctx <= time_budget, even at token_budget 0) or a negative context.
__device__ __forceinline__ void scan_fairbatch(const Scratch& s, int A,
                                               double init_ms, const FormCfg& f,
                                               bool exits_ok = true) {
  if (tile_lane() == 0) {
    double tb = dsub(init_ms, f.a);
    int64_t tok = f.token_budget;
    // b_lo = RD(b (1 - 2^-52)): x < b_lo gives fl(x / b) < 1, so a chunk of
    // x = tb - cc budget floors to 0 tokens (no division needed), and with
    // every task's new >= 1 and c*ctx >= 0 (exits_ok) each task costs at
    // least b, so tb < b_lo admits nothing more: the exact stop (it implies
    // the reference's implicit tb < 0 one).
    const bool bpos = f.b > 0.0;
    const double b_lo = bpos ? __dmul_rd(f.b, 1.0 - 0x1p-52) : 0.0;
    FB_COLD_LOOP
    for (int k = 0; k < A; ++k) {
      if (exits_ok && (tok <= 0 || tb < 0.0 || tb < b_lo)) break;
      const double tc = s.tcost[k];
      const double cc = s.ccost[k];
      const int64_t nv = static_cast<int64_t>(static_cast<uint32_t>(s.khi[k]) & 0x7fffffffu);
      if (tc <= tb && nv <= tok) {
        s.take[k] = static_cast<int32_t>(nv);
        tb = dsub(tb, tc);
        tok -= nv;
      } else if (tok > 0 && cc <= tb) {
        const double x = dsub(tb, cc);
        if (bpos && x < b_lo) continue;  // floor(min(tok, x / b)) == 0
        const double lim = ddiv(x, f.b);
        const double dt = static_cast<double>(tok);
        const double cp_real = lim < dt ? lim : dt;  // std::min(dt, lim)
        const int64_t cp = static_cast<int64_t>(floor(cp_real));
        if (cp >= 1) {
          s.take[k] = static_cast<int32_t>(cp);
          tb = dsub(tb, dadd(dmul(f.b, static_cast<double>(cp)), cc));
          tok -= cp;
        }
      }
    }
  }
  tile_sync();
}

// K3b': form_batch_sarathi (sched.cpp:172-206); sorted decodes first.
__device__ __forceinline__ void scan_sarathi(const Scratch& s, int A, int n_dec,
                                             const FormCfg& f) {
  FB_COLD_LOOP
  for (int k = tile_lane(); k < n_dec; k += kTile) s.take[k] = 1;
  if (tile_lane() == 0) {
    int64_t remaining = f.token_budget - n_dec;
    if (remaining < 0) remaining = 0;
    FB_COLD_LOOP
    for (int k = n_dec; k < A; ++k) {
      if (remaining <= 0) break;
      const int64_t nv = static_cast<uint32_t>(s.khi[k]) & 0x7fffffffu;
      int64_t chunk = remaining;
      if (f.max_chunk < chunk) chunk = f.max_chunk;
      if (nv < chunk) chunk = nv;
      if (chunk < 1) continue;
      s.take[k] = static_cast<int32_t>(chunk);
      remaining -= chunk;
    }
  }
  tile_sync();
}

// K3b'': form_batch_prefill_first (sched.cpp:208-232); fifo order.
__device__ __forceinline__ void scan_prefill_first(const Scratch& s, int A,
                                                   const FormCfg& f) {
  if (tile_lane() == 0) {
    int64_t budget = f.token_budget;
    FB_COLD_LOOP
    for (int k = 0; k < A; ++k) {
      if (budget <= 0) break;
      const uint32_t w = static_cast<uint32_t>(s.khi[k]);
      int64_t take;
      if (w & kDecodeBit) {
        take = 1;
      } else {
        take = budget;
        if (f.max_chunk < take) take = f.max_chunk;
        const int64_t nv = w & 0x7fffffffu;
        if (nv < take) take = nv;
      }
      if (take < 1 || take > budget) continue;
      s.take[k] = static_cast<int32_t>(take);
      budget -= take;
    }
  }
  tile_sync();
}

// Whole K2+K3 pipeline after K1 filled s.{slack,seq,ctx,nw} for [0, A) and
// acc holds the reduced K1 accumulators.  Leaves s.order / s.take (sorted) and
// s.seq (sorted context) for the caller's bookkeeping.
//
// Admission marks: on the engine paths every task has new >= 1, so an
// admitted entry has take >= 1 and take == 0 means "not admitted".  The pure
// scheduler (kExact) also takes arbitrary task sets, where fair batching
// admits zero-token entries {id, 0}: there take == -1 means "not admitted"
// and every take >= 0 is a plan entry (`admitted_take`).
template <bool kExact = false>
__device__ __forceinline__ bool admitted_take(int32_t take) {
  return kExact ? take >= 0 : take > 0;
}

template <bool kExact = false>
__device__ __forceinline__ FormOut form_batch_warp(const Scratch& s, int A,
                                                   const ViewAcc& acc,
                                                   const FormCfg& f, bool seq_unique,
                                                   bool exits_ok = true) {
  FormOut out;
  out.init_ms = 0.0;
  const bool fair = f.policy == FB_POLICY_FAIRBATCH || f.policy == FB_POLICY_FAIRBATCH_PAB;
  int64_t urgency = 0;
  if (fair) {
    // init_time_budget, sched.cpp:90-106; urgency bound sched.cpp:111-113
    const int64_t init = acc.n_dec == 0 ? acc.min_tpot
                                        : (acc.min_dec > acc.min_tpot ? acc.min_dec : acc.min_tpot);
    urgency = init + acc.min_tpot;
    out.init_ms = us_to_ms(init);
  }
  const bool packed = make_keys(s, A, f.policy, urgency, seq_unique);
  rank_order(s, A, packed);
  gather_sorted(s, A, f.b, f.c);
  if (kExact) {
    FB_COLD_LOOP
    for (int k = tile_lane(); k < A; k += kTile) s.take[k] = -1;
    tile_sync();
  }
  if (fair) {
    // Everything fits whole (the register path's exact sufficient test, see
    // begin_rr): tb0 - RU(sum of the rounded costs) >= A 2^-52 tb0 and the
    // new tokens within token_budget imply every `consider` admits whole.
    bool all_fit = false;
    if (!kExact && exits_ok) {
      const double tb0 = dsub(out.init_ms, f.a);
      double part = 0.0;
      int64_t nn = 0;
      FB_COLD_LOOP
      for (int k = tile_lane(); k < A; k += kTile) {
        part = __dadd_ru(part, s.tcost[k]);
        nn += static_cast<int64_t>(s.khi[k] & 0x7fffffffu);
      }
      const double s_up = tile_sum_ru(part);
      const int64_t n_new = tile_sum_small(nn);
      all_fit = tb0 >= 0.0 && n_new <= f.token_budget &&
                __dsub_rd(tb0, s_up) >= __dmul_ru(__dmul_ru(static_cast<double>(A), 0x1p-52), tb0);
    }
    if (all_fit) {
      FB_COLD_LOOP
      for (int k = tile_lane(); k < A; k += kTile)
        s.take[k] = static_cast<int32_t>(s.khi[k] & 0x7fffffffu);
      tile_sync();
    } else {
      scan_fairbatch(s, A, out.init_ms, f, exits_ok);
    }
  } else if (f.policy == FB_POLICY_SARATHI) {
    scan_sarathi(s, A, acc.n_dec, f);
  } else {
    scan_prefill_first(s, A, f);
  }
  // finalize_plan, sched.cpp:37-48 (integer sums: any order is exact)
  int32_t e = 0;
  int64_t tn = 0, tc = 0;
  FB_COLD_LOOP
  for (int k = tile_lane(); k < A; k += kTile) {
    const int32_t tk = s.take[k];
    if (admitted_take<kExact>(tk)) {
      e++;
      tn += tk;
      tc += s.seq[k];
    }
  }
  out.n_entries = static_cast<int32_t>(__reduce_add_sync(tile_mask(), static_cast<uint32_t>(e)));
  out.total_new = tile_sum_small(tn);
  if (kExact) {  // arbitrary (possibly negative) contexts: full 64-bit sum
#pragma unroll
    for (int o = kTile / 2; o > 0; o >>= 1) tc += tile_shfl_xor(tc, o);
    out.total_ctx = tc;
  } else {
    out.total_ctx = tile_sum_small(tc);
  }
  out.predicted_ms = out.n_entries == 0 ? 0.0 : predict_ms(f.a, f.b, f.c, out.total_new, out.total_ctx);
  return out;
}

// ------------------------------------------------------------------- K5

// One task's share of pab's r_tasks (sched.cpp:268-271):
//   max(0, (W - slack_ms) / T) * (b + ctx * c)
__device__ __forceinline__ double pab_term(double W, double T, double b, double c,
                                           int64_t slack, int64_t ctx) {
  const double x = ddiv(dsub(W, us_to_ms(slack)), T);
  const double steps = 0.0 < x ? x : 0.0;  // std::max(0.0, x)
  return dmul(steps, dadd(b, dmul(static_cast<double>(ctx), c)));
}

// Closing arithmetic of pab (sched.cpp:257-277) given the view aggregates.
__device__ __forceinline__ int64_t pab_close(double W, double T, double a, double b,
                                             double c, bool any, int64_t min_slack,
                                             double r_tasks, int64_t prefill_tokens) {
  double nb = 1.0;
  if (any) {
    const double ms = us_to_ms(min_slack);
    const double msm = W < ms ? W : ms;  // std::min(ms, W)
    nb = dadd(ddiv(dsub(W, msm), T), 1.0);
  }
  const double r_batches = dmul(nb, a);
  const double r_prefill = dsub(dsub(W, r_batches), r_tasks);
  const double t_prefill = ddiv(r_prefill, dadd(b, c));
  return static_cast<int64_t>(floor(t_prefill)) - prefill_tokens;
}

// Ordered fp64 fold of s.tcost[0..A) in view order (pab's r_tasks is an
// order-dependent sum, SURVEY §7 hard part 3).  Result is warp-uniform.
__device__ __forceinline__ double ordered_fold(const double* v, int A) {
  double r = 0.0;
  if (tile_lane() == 0) {
    // a serial chain: unrolled so the shared-memory loads run ahead of it
    // (the cluster's per-step PAB report sits on the epoch's critical path)
#pragma unroll 4
    for (int p = 0; p < A; ++p) r = dadd(r, v[p]);
  }
  return tile_shfl(r, 0);
}

}  // namespace fbgpu
