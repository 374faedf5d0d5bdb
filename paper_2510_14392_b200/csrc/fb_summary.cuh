// fb_summary.cuh -- per-instance ScenarioReport aggregates on the device
// (scenario_report, metrics.cpp:171-205; nearest-rank percentiles,
// metrics.cpp:118-135), so a sweep of tens of thousands of nodes returns a
// few hundred bytes per node instead of every request's record.
//
// One CTA per instance: one pass over the instance's request state counts
// the outcomes and compacts the three metric series (TTFT ms for requests
// with a first token, max-TPOT ms for >= 2 tokens, alternative max-TPOT for
// >= 3 tokens); each percentile is the rank-th smallest value, found by
// rank-by-count in shared memory (<= kSumCap values) or by an exact MSD radix
// select over the values' bit patterns (all values are >= 0, so the IEEE bit
// order is the numeric order).  Ties are exact: the selected value is the
// one whose [#less, #less + #equal) range holds the rank.
#pragma once

namespace fbgpu {

constexpr int kSumThreads = 256;
constexpr int kSumWarps = kSumThreads / kWarp;
constexpr int kSumCap = 2048;

struct SumSmem {
  uint64_t v[kSumCap];
  uint32_t hist[2048];
  int64_t red[kSumWarps * 8];
  int64_t bcast[4];
};

__device__ __forceinline__ int64_t sum_block_sum(int64_t x, SumSmem& sm) {
  x = warp_sum(x);
  if (lane_id() == 0) sm.red[threadIdx.x / kWarp] = x;
  __syncthreads();
  int64_t t = 0;
  for (int q = 0; q < kSumWarps; ++q) t += sm.red[q];
  __syncthreads();
  return t;
}

// Exclusive prefix count of `flag` (thread order) and the block total.
__device__ __forceinline__ int sum_excl_count(bool flag, int& total, SumSmem& sm) {
  const unsigned m = __ballot_sync(kFull, flag);
  const int w = threadIdx.x / kWarp;
  if (lane_id() == 0) sm.red[w] = __popc(m);
  __syncthreads();
  int before = 0, tot = 0;
  for (int q = 0; q < kSumWarps; ++q) {
    const int c = static_cast<int>(sm.red[q]);
    if (q < w) before += c;
    tot += c;
  }
  __syncthreads();
  total = tot;
  unsigned lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  return before + __popc(m & lt);
}

// The r-th smallest (1-based) of the n values in sm.v (n <= kSumCap).
__device__ __forceinline__ uint64_t sum_rank_smem(int n, int64_t r, SumSmem& sm) {
  for (int i = threadIdx.x; i < n; i += kSumThreads) {
    const uint64_t x = sm.v[i];
    int less = 0, eq = 0;
    for (int j = 0; j < n; ++j) {
      const uint64_t y = sm.v[j];
      less += y < x;
      eq += y == x;
    }
    if (less < r && r <= less + eq) sm.bcast[0] = static_cast<int64_t>(x);
  }
  __syncthreads();
  const uint64_t out = static_cast<uint64_t>(sm.bcast[0]);
  __syncthreads();
  return out;
}

// The r-th smallest (1-based) of the n values at g (global), exact MSD radix
// select with 11-bit digits.
__device__ uint64_t sum_rank_global(const uint64_t* g, int64_t n, int64_t r, SumSmem& sm) {
  uint64_t prefix = 0, pmask = 0;
  int64_t need = r;
  for (int pass = 0; pass < 6; ++pass) {
    const int bits = pass < 5 ? 11 : 9;
    const int shift = 64 - 11 * pass - bits;
    const uint64_t dmask = (uint64_t(1) << bits) - 1;
    for (int i = threadIdx.x; i < 2048; i += kSumThreads) sm.hist[i] = 0;
    __syncthreads();
    for (int64_t i = threadIdx.x; i < n; i += kSumThreads) {
      const uint64_t x = g[i];
      if ((x & pmask) == prefix) atomicAdd(&sm.hist[(x >> shift) & dmask], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t cum = 0;
      int b = 0;
      for (; b < (1 << bits); ++b) {
        if (cum + sm.hist[b] >= need) break;
        cum += sm.hist[b];
      }
      sm.bcast[0] = b;
      sm.bcast[1] = need - cum;
    }
    __syncthreads();
    prefix |= static_cast<uint64_t>(sm.bcast[0]) << shift;
    pmask |= dmask << shift;
    need = sm.bcast[1];
    __syncthreads();
  }
  return prefix;
}

__device__ __forceinline__ int64_t nearest_rank(double p, int64_t n) {
  // metrics.cpp:124-129: ceil(p / 100 * n), clamped to [1, n]
  int64_t r = static_cast<int64_t>(ceil(dmul(ddiv(p, 100.0), static_cast<double>(n))));
  if (r < 1) r = 1;
  if (r > n) r = n;
  return r;
}

__global__ void __launch_bounds__(kSumThreads)
summarize_kernel(const __grid_constant__ EngineParams P, fb_summary* out, uint64_t* vals) {
  __shared__ SumSmem sm;
  for (int64_t i = blockIdx.x; i < P.n_inst; i += gridDim.x) {
    const DevInst* I = P.inst + i;
    const int64_t b = I->rec_off, toff = I->trace_off;
    const int64_t arrived = P.state[i].arr;  // requests [0, arrived) reached the node
    fb_summary s;
    memset(&s, 0, sizeof(s));
    int64_t c_rej = 0, c_fin = 0, c_good = 0, c_tv = 0, c_env = 0;
    for (int64_t k = threadIdx.x; k < arrived; k += kSumThreads) {
      const int32_t ni = P.nidx[b + k];
      uint32_t f = P.flags[b + k] & ~kTpotViolated;
      if ((f & FB_REC_REJECTED) && ni > 0) f &= ~static_cast<uint32_t>(FB_REC_REJECTED);
      const bool rej = (f & FB_REC_REJECTED) != 0, fin = (f & FB_REC_FINISHED) != 0;
      c_rej += rej;
      c_fin += fin;
      c_good += !rej && fin && (f & FB_REC_MET_TTFT) && (f & FB_REC_MET_TPOT);
      c_tv += ni < 1 || !(f & FB_REC_MET_TTFT);
      c_env += (f & FB_REC_ENV_MISS) != 0;
    }
    s.total_requests = arrived;
    s.rejected = sum_block_sum(c_rej, sm);
    s.finished = sum_block_sum(c_fin, sm);
    s.good = sum_block_sum(c_good, sm);
    s.ttft_violations = sum_block_sum(c_tv, sm);
    s.envelope_misses = sum_block_sum(c_env, sm);
    // metric series: 0 TTFT, 1 max-TPOT, 2 alternative max-TPOT
    uint64_t* gv = vals + b;  // this instance's value series (large instances)
    for (int m = 0; m < 3; ++m) {
      const int min_tok = m + 1;
      int64_t n = 0;
      for (int64_t k0 = 0; k0 < arrived; k0 += kSumThreads) {
        const int64_t k = k0 + threadIdx.x;
        bool take = false;
        uint64_t bits = 0;
        if (k < arrived && P.nidx[b + k] >= min_tok) {
          take = true;
          double x;
          if (m == 0) {
            x = us_to_ms(P.first[b + k] - P.arrival[toff + k]);  // RequestReport::ttft_ms
          } else if (m == 1) {
            x = P.maxtp[b + k];
          } else {
            x = P.maxtp_alt[b + k];
          }
          bits = static_cast<uint64_t>(__double_as_longlong(x));
        }
        int tot;
        const int pos = sum_excl_count(take, tot, sm);
        if (take) {
          if (n + pos < kSumCap) sm.v[n + pos] = bits;
          gv[n + pos] = bits;
        }
        n += tot;
      }
      __syncthreads();
      fb_percentiles pr;
      pr.count = n;
      pr.p50 = pr.p95 = pr.p99 = 0.0;
      if (n > 0) {
        const double ps[3] = {50.0, 95.0, 99.0};
        double res[3];
        for (int q = 0; q < 3; ++q) {
          const int64_t r = nearest_rank(ps[q], n);
          const uint64_t v = n <= kSumCap ? sum_rank_smem(static_cast<int>(n), r, sm)
                                          : sum_rank_global(gv, n, r, sm);
          res[q] = __longlong_as_double(static_cast<long long>(v));
        }
        pr.p50 = res[0];
        pr.p95 = res[1];
        pr.p99 = res[2];
      }
      if (m == 0) s.ttft_ms = pr;
      else if (m == 1) s.max_tpot_ms = pr;
      else s.max_tpot_alt_ms = pr;
      __syncthreads();
    }
    if (threadIdx.x == 0) out[i] = s;
    __syncthreads();
  }
}

// Envelope-lead series (envelope_lead_series, metrics.cpp:137-169) of every
// instance at t_k = k * bucket, k = 0 .. floor(t_max / bucket):
//   lead(t) = sum over requests in decode at t of (emitted by t - required by t)
//           = C(t) - F(t) - R(t)
// with C the emissions at or before t (run-time histogram), F the output
// lengths of requests whose last token came at or before t (run-time
// histogram), R the envelope's required tokens of the requests in decode at
// t (first token <= t < last token of a finished request), accumulated here.
__global__ void __launch_bounds__(kSumThreads)
lead_kernel(const __grid_constant__ EngineParams P, int64_t* out, int32_t* n_out) {
  const int64_t B = P.lead_bucket, cap = P.lead_cap;
  for (int64_t i = blockIdx.x; i < P.n_inst; i += gridDim.x) {
    const long long tmax = P.lead_tmax[i];
    const int64_t K = tmax >= 0 ? tmax / B + 1 : 1;
    int64_t* R = out + i * cap;
    if (K > cap || P.lead_flags[i]) {
      if (threadIdx.x == 0) n_out[i] = -1;
      continue;
    }
    for (int64_t k = threadIdx.x; k < K; k += kSumThreads) R[k] = 0;
    __syncthreads();
    const DevInst* I = P.inst + i;
    const int64_t b = I->rec_off, toff = I->trace_off, n = P.state[i].arr;
    for (int64_t r = threadIdx.x; r < n; r += kSumThreads) {
      const int64_t first = P.first[b + r];
      if (first < 0) continue;
      const int64_t row = toff + r;
      const int64_t k0 = (first + B - 1) / B;
      int64_t k1 = K;
      if (P.flags[b + r] & FB_REC_FINISHED) {
        const int64_t kl = (P.lastem[b + r] + B - 1) / B;  // in decode while t < last
        k1 = kl < K ? kl : K;
      }
      const int64_t ddl = P.arrival[row] + P.ttft[row];
      const int64_t tpot = P.tpot[row];
      const int64_t outl = P.output[row];
      for (int64_t k = k0; k < k1; ++k) {
        const int64_t t = k * B;
        if (t < ddl) continue;
        int64_t req = (t - ddl) / tpot + 1;
        if (req > outl) req = outl;
        atomicAdd(reinterpret_cast<unsigned long long*>(R + k), static_cast<unsigned long long>(req));
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned long long* h = P.lead_hist + i * 2 * cap;
      int64_t c = 0, f = 0;
      for (int64_t k = 0; k < K; ++k) {
        c += static_cast<int64_t>(h[k]);
        f += static_cast<int64_t>(h[cap + k]);
        R[k] = c - f - R[k];
      }
      n_out[i] = static_cast<int32_t>(K);
    }
    __syncthreads();
  }
}

}  // namespace fbgpu
