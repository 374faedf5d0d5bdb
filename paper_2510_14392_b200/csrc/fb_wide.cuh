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

// Dev-only phase timers (tools/wide_prof.py builds a variant with
// -DFB_WIDE_PROF): thread 0 accumulates clock64 deltas per phase.
#ifdef FB_WIDE_PROF
__device__ unsigned long long g_wide_prof[24];
__device__ unsigned long long g_cta_prof[256][4];  // per CTA busy clocks: K1, hist, gather, owner
__device__ unsigned long long g_sub_prof[256][8];   // per CTA sub-phase clocks (SPROF)
#define WPROF_START long long wp_t_ = clock64();
#define WPROF(slot)                                                               \
  if (threadIdx.x == 0) {                                                         \
    const long long n_ = clock64();                                               \
    atomicAdd(&g_wide_prof[slot], static_cast<unsigned long long>(n_ - wp_t_));   \
    wp_t_ = n_;                                                                   \
  }
#define WPROF_COUNT(slot, v) \
  if (threadIdx.x == 0) atomicAdd(&g_wide_prof[slot], static_cast<unsigned long long>(v));
#else
#define WPROF_START
#define WPROF(slot)
#define WPROF_COUNT(slot, v)
#endif

constexpr int kWideThreads = 512;
constexpr int kWideWarps = kWideThreads / kWarp;
constexpr int kWideWin = 2048;
constexpr int kRadixBits = 11;
constexpr int kRadixBins = 1 << kRadixBits;
// Range-binned selection (wide_select_binned): 1024 linear bins per key group.
constexpr int kGroupBins = 1024;
constexpr int kSelBins = 4 * kGroupBins;
constexpr int kRed = 8;  // values per warp in block_reduce

struct WideSmem {
  uint64_t wkey[kWideWin];
  double wtc[kWideWin];
  double wcc[kWideWin];
  int64_t wcx[kWideWin];
  int32_t wpos[kWideWin];
  uint32_t wnw[kWideWin];
  int32_t wtake[kWideWin];
  uint32_t hist[kSelBins];
  int64_t red[kWideWarps * kRed];
  int64_t bcast[8];
  double dbcast[4];
  int32_t ibcast[8];
};

// Between K2a and K2b the window arrays (owner-phase only) hold the
// selection bin of each view of the CTA's range, as uint16.
constexpr int64_t kWgBinCap =
    static_cast<int64_t>(offsetof(WideSmem, hist) - offsetof(WideSmem, wkey)) / 2;
static_assert(kSelBins <= 65536, "bins must fit uint16");
__device__ __forceinline__ uint16_t* wg_bins(WideSmem& sm) {
  return reinterpret_cast<uint16_t*>(sm.wkey);
}

// Per-request view record of an escalated node (request index r): the
// K1-relevant progress, mirrored from the SoA arena at escalation and kept
// in step by pull / complete, so K1 reads one 16-byte record per view (one
// vector load) instead of seven gathers.  Everything K1 derives a view from
// (build_task_views, engine.cpp:51-81; slack, slo.h:45-61):
//   anchor  = min(first token, arrival + ttft_slo) once token 0 is out, else
//             arrival + ttft_slo  -- fixed from the first token on
//   slack   = anchor + tpot_slo * next_idx - now   (prefill: next_idx = 0)
//   context = prefilled (prefill) or prompt + next_idx (decode)
// Packing needs anchor < 2^41 and seq < 2^22: DevInst::wide_ok (host-checked
// arrival, ttft_slo < 2^40 and n_req < 2^22; anchor <= arrival + ttft_slo).
struct __align__(16) WRec {
  int64_t anc_seq;  // anchor << 22 | seq
  int32_t ctx;      // context tokens
  int32_t nid;      // next_idx | decode << 31
};
constexpr int64_t kWRecSeqMask = (int64_t(1) << 22) - 1;

__device__ __forceinline__ WRec make_wrec(int64_t dl0, int64_t first, int32_t prompt,
                                          int32_t prefilled, int32_t nidx, int32_t seq) {
  const bool decode = prefilled >= prompt;
  const int64_t anchor = (first >= 0 && first < dl0) ? first : dl0;
  WRec r;
  r.anc_seq = (anchor << 22) | (static_cast<int64_t>(static_cast<uint32_t>(seq)) & kWRecSeqMask);
  r.ctx = decode ? prompt + nidx : prefilled;
  r.nid = static_cast<int32_t>(static_cast<uint32_t>(nidx) | (decode ? 0x80000000u : 0u));
  return r;
}

// Per-instance global scratch (kScratchBytesPerSlot per request slot).

// Per-instance global scratch (kScratchBytesPerSlot per request slot).
struct WideScratch {
  WRec* rec;       // [r] view records (16 of the slot's first 32 bytes)
  uint64_t* klow;  // [p] decode<<63 | (slack+2^39)<<22 | seq   (stem of the key)
  int2* vtmp;      // reorder buffer / PAB terms
  int32_t* mark;   // [p] admitted-waiting flag
};

__device__ __forceinline__ WideScratch wide_scratch(const EngineParams& P, const Inst& w) {
  static_assert(kScratchBytesPerSlot % 16 == 0 && kScratchBytesPerSlot >= 52, "wide scratch");
  WideScratch s;
  unsigned char* base = P.gscratch + w.roff * kScratchBytesPerSlot;
  const size_t n = static_cast<size_t>(w.nreq);
  s.rec = reinterpret_cast<WRec*>(base);
  s.klow = reinterpret_cast<uint64_t*>(base + 32 * n);
  s.vtmp = reinterpret_cast<int2*>(base + 40 * n);
  s.mark = reinterpret_cast<int32_t*>(base + 48 * n);
  return s;
}

// ------------------------------------------------------ L2 residency
//
// One iteration streams every beginning node's views once (K1: row index +
// 32-byte record, ~200 MB at C4) and writes the 8-byte key stems (~40 MB)
// that K2a reads back.  The records and row indices are marked evict_first
// and the stems evict_last, so the stems stay in the 126 MB L2 between K1
// and K2a instead of being written back and re-read from HBM.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ int4 ld_stream_v4(const int4* a, uint64_t pol) {
  int4 r;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(a), "l"(pol));
  return r;
}
__device__ __forceinline__ int32_t ld_stream_s32(const int32_t* a, uint64_t pol) {
  int32_t r;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
               : "=r"(r)
               : "l"(a), "l"(pol));
  return r;
}
__device__ __forceinline__ void st_keep_u64(uint64_t* a, uint64_t v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.b64 [%0], %1, %2;" ::"l"(a), "l"(v), "l"(pol)
               : "memory");
}
__device__ __forceinline__ uint64_t ld_keep_u64(const uint64_t* a, uint64_t pol) {
  uint64_t r;
  asm volatile("ld.global.cg.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(r) : "l"(a), "l"(pol));
  return r;
}
__device__ __forceinline__ void prefetch_l2(const void* a) {
  asm volatile("prefetch.global.L2::evict_normal [%0];" ::"l"(a));
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
// Block-wide minima of N int64 values at once (maxima: pass negations);
// one pair of barriers for all of them.  Results in every thread.
template <int N>
__device__ __forceinline__ void block_min_n(int64_t (&v)[N], WideSmem& sm) {
  static_assert(N <= kRed, "block_min_n");
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = warp_min(v[i]);
  if (lane_id() == 0) {
#pragma unroll
    for (int i = 0; i < N; ++i) sm.red[wid() * kRed + i] = v[i];
  }
  __syncthreads();
  if (wid() == 0) {  // lane q of warp 0 folds warp q's partials
#pragma unroll
    for (int i = 0; i < N; ++i) {
      int64_t x = lane_id() < kWideWarps ? sm.red[lane_id() * kRed + i] : kInf;
      x = warp_min(x);
      if (lane_id() == 0) sm.red[kWideWarps * kRed - kRed + i] = x;  // last row: results
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = sm.red[kWideWarps * kRed - kRed + i];
  __syncthreads();
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

// Branch-free bitonic sort of sm.wkey / sm.wpos [0, K) (keys unique, K <=
// kWideWin; padding keys ~0 sort last), at the smallest size N = 512 * PER
// (PER = 1, 2, 4 elements per thread) that holds K.  Element e = warp *
// 32 * PER + lane * PER + q lives in register q of its lane: compare-
// exchange distances below PER are in-thread, up to a warp's run (32 * PER)
// lane shuffles, longer ones go through shared memory (one barrier per
// distance).  Every exchange is a mask select, never a branch, and every
// stage is unrolled at compile time (the earlier loop-form merge sort
// compiled to divergent branches per element: 15 us for any K; this one
// 9 us at N = 2048, tools/micro/sortbench.cu).
__device__ __forceinline__ uint64_t msel64(uint64_t m, uint64_t x, uint64_t y) {
  return (x & m) | (y & ~m);
}
__device__ __forceinline__ int32_t msel32(uint32_t m, int32_t x, int32_t y) {
  return static_cast<int32_t>((static_cast<uint32_t>(x) & m) | (static_cast<uint32_t>(y) & ~m));
}
// keys unique (padding ~0 only meets padding): b < a <=> !(a < b)
__device__ __forceinline__ void cx_sel(uint64_t& a, int32_t& pa, uint64_t b, int32_t pb,
                                       bool take_min) {
  const uint32_t pick = 0u - static_cast<uint32_t>((b < a) == take_min);
  const uint64_t pick64 = 0ull - static_cast<uint64_t>(pick & 1u);
  a = msel64(pick64, b, a);
  pa = msel32(pick, pb, pa);
}
__device__ __forceinline__ void cx_pair(uint64_t& a, int32_t& pa, uint64_t& b, int32_t& pb,
                                        bool asc) {
  const uint32_t sw = 0u - static_cast<uint32_t>((b < a) == asc);
  const uint64_t sw64 = 0ull - static_cast<uint64_t>(sw & 1u);
  const uint64_t lo = msel64(sw64, b, a), hi = msel64(sw64, a, b);
  const int32_t plo = msel32(sw, pb, pa), phi = msel32(sw, pa, pb);
  a = lo;
  b = hi;
  pa = plo;
  pb = phi;
}
template <int PER, int KK, int J>
__device__ __forceinline__ void bsort_reg_stages(uint64_t (&k)[PER], int32_t (&v)[PER], int e0) {
  if constexpr (J >= PER) {
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int e = e0 + q;
      const uint64_t b = __shfl_xor_sync(kFull, k[q], J / PER);
      const int32_t pb = __shfl_xor_sync(kFull, v[q], J / PER);
      cx_sel(k[q], v[q], b, pb, ((e & J) == 0) == ((e & KK) == 0));
    }
  } else {
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      if ((q & J) != 0) continue;
      cx_pair(k[q], v[q], k[q + J], v[q + J], ((e0 + q) & KK) == 0);
    }
  }
  if constexpr (J > 1) bsort_reg_stages<PER, KK, J / 2>(k, v, e0);
}
template <int PER, int KK, int J>
__device__ __forceinline__ void bsort_smem_stages(uint64_t* key, int32_t* pos) {
#pragma unroll
  for (int h = 0; h < PER / 2 + (PER == 1 ? 1 : 0); ++h) {
    const int pid = threadIdx.x + h * kWideThreads;  // pair index
    if (PER == 1 && pid >= kWideThreads / 2) break;
    const int e = (pid / J) * (2 * J) + (pid % J);
    uint64_t a = key[e], b = key[e + J];
    int32_t pa = pos[e], pb = pos[e + J];
    cx_pair(a, pa, b, pb, (e & KK) == 0);
    key[e] = a;
    pos[e] = pa;
    key[e + J] = b;
    pos[e + J] = pb;
  }
  __syncthreads();
  if constexpr (J / 2 >= kWarp * PER) bsort_smem_stages<PER, KK, J / 2>(key, pos);
}
template <int PER, int KK>
__device__ __forceinline__ void bsort_merge(uint64_t (&k)[PER], int32_t (&v)[PER], int e0,
                                            WideSmem& sm) {
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    sm.wkey[e0 + q] = k[q];
    sm.wpos[e0 + q] = v[q];
  }
  __syncthreads();
  bsort_smem_stages<PER, KK, KK / 2>(sm.wkey, sm.wpos);
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    k[q] = sm.wkey[e0 + q];
    v[q] = sm.wpos[e0 + q];
  }
  bsort_reg_stages<PER, KK, kWarp * PER / 2>(k, v, e0);
  if constexpr (KK < kWideThreads * PER) bsort_merge<PER, KK * 2>(k, v, e0, sm);
}
template <int PER, int KK>
__device__ __forceinline__ void bsort_runs(uint64_t (&k)[PER], int32_t (&v)[PER], int e0) {
  bsort_reg_stages<PER, KK, KK / 2>(k, v, e0);
  if constexpr (KK < kWarp * PER) bsort_runs<PER, KK * 2>(k, v, e0);
}
template <int PER>
__device__ void wide_bitonic_sort_n(int K, WideSmem& sm) {
  static_assert(kWideThreads * PER <= kWideWin, "sort size");
  uint64_t k[PER];
  int32_t v[PER];
  const int e0 = threadIdx.x * PER;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int e = e0 + q;
    k[q] = e < K ? sm.wkey[e] : ~uint64_t(0);
    v[q] = e < K ? sm.wpos[e] : -1;
  }
  __syncthreads();  // every thread read its elements before the first smem stage
  bsort_runs<PER, 2>(k, v, e0);
  bsort_merge<PER, 2 * kWarp * PER>(k, v, e0, sm);
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    if (e0 + q < K) {
      sm.wkey[e0 + q] = k[q];
      sm.wpos[e0 + q] = v[q];
    }
  }
  __syncthreads();
}
__device__ void wide_bitonic_sort(int K, WideSmem& sm) {
  if (K <= kWideThreads) {
    wide_bitonic_sort_n<1>(K, sm);
  } else if (K <= 2 * kWideThreads) {
    wide_bitonic_sort_n<2>(K, sm);
  } else {
    wide_bitonic_sort_n<4>(K, sm);
  }
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
  wide_bitonic_sort(K, sm);
  return K;
}

// Linear key bins per group for the binned selection.  bin(key) is
// nondecreasing in key, so the keys of bins [0, b] are exactly the smallest
// keys.  Fair batching orders (urgent decode, prefill, relaxed decode) by
// (slack, seq) -- the ordinal is the stem's low 62 bits, so equal slacks
// (a prefill batch's decodes share first-token times) still spread over
// bins by seq; sarathi (decode, prefill) and prefill-first order by seq.
struct SelBins {
  int64_t lo[3];
  int32_t sh[3];
  int64_t urg;  // fair batching: urgency bound as an ordinal
};

__device__ __forceinline__ int sel_bin(uint64_t klow, int policy, int64_t urgency,
                                       const SelBins& b) {
  const bool decode = (klow >> 63) != 0;
  const uint64_t low = klow & ((uint64_t(1) << 62) - 1);
  int g;
  int64_t ord;
  if (policy == FB_POLICY_FAIRBATCH || policy == FB_POLICY_FAIRBATCH_PAB) {
    ord = static_cast<int64_t>(low);
    g = decode ? (ord < b.urg ? 0 : 2) : 1;
  } else {
    ord = static_cast<int64_t>(low & ((uint64_t(1) << 22) - 1));
    g = (policy == FB_POLICY_SARATHI && !decode) ? 1 : 0;
  }
  // select, not index: a dynamic index would put the bins in local memory
  const int64_t lo = g == 0 ? b.lo[0] : (g == 1 ? b.lo[1] : b.lo[2]);
  const int sh = g == 0 ? b.sh[0] : (g == 1 ? b.sh[1] : b.sh[2]);
  int64_t d = (ord - lo) >> sh;
  d = d < 0 ? 0 : (d > kGroupBins - 1 ? kGroupBins - 1 : d);
  return g * kGroupBins + static_cast<int>(d);
}

// Bins of group g over ordinals [lo, hi] holding about `count` keys.  The
// bin width is chosen so that, at uniform density, one window (kWideWin
// keys) spans about half the group's bins; ordinals past the last bin are
// clamped into it (any nondecreasing binning is exact -- the width only sets
// how full a window gets).
__device__ __forceinline__ void sel_range(SelBins& b, int g, int64_t lo, int64_t hi,
                                          int64_t count) {
  b.lo[g] = lo;
  int64_t span = hi > lo ? hi - lo : 0;
  if (count > 2 * kWideWin) span = span / (count / (2 * kWideWin));
  // smallest sh with (span >> sh) < kGroupBins
  const int bits = span > 0 ? 64 - __clzll(static_cast<unsigned long long>(span)) : 0;
  b.sh[g] = bits > 10 ? bits - 10 : 0;
  static_assert(kGroupBins == 1024, "sel_range: 10-bit bin index");
}

// K2 (common case): the smallest keys above `lo` that fit one window, in two
// streaming passes over the key stems -- a histogram over the group ranges,
// then a gather of every key in the bins up to the last one whose inclusive
// count still fits -- followed by the shared-memory bitonic sort.  Returns
// the window size, or -1 when the first nonempty bin alone overflows the
// window (the caller falls back to the exact radix select).  sm.ibcast[1]
// tells whether the window holds every remaining key.
__device__ int wide_select_binned(const WideScratch& ws, int A, bool has_lo, uint64_t lo,
                                  int policy, int64_t urgency, const SelBins& sb,
                                  WideSmem& sm) {
  constexpr int U = 8;
  for (int i = threadIdx.x; i < kSelBins; i += kWideThreads) sm.hist[i] = 0;
  if (threadIdx.x == 0) sm.ibcast[4] = 0;
  __syncthreads();
  for (int b0 = 0; b0 < A; b0 += kWideThreads * U) {
    uint64_t k[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int p = b0 + j * kWideThreads + threadIdx.x;
      k[j] = p < A ? ws.klow[p] : 0;
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int p = b0 + j * kWideThreads + threadIdx.x;
      if (p < A && (!has_lo || wide_key(k[j], policy, urgency) > lo))
        atomicAdd(&sm.hist[sel_bin(k[j], policy, urgency, sb)], 1u);
    }
  }
  __syncthreads();
  constexpr int kPer = kSelBins / kWideThreads;
  const int c0 = threadIdx.x * kPer;
  int loc = 0;
#pragma unroll
  for (int q = 0; q < kPer; ++q) loc += static_cast<int>(sm.hist[c0 + q]);
  int tot;
  const int before = block_excl_sum(loc, tot, sm);
  if (threadIdx.x == 0) sm.ibcast[1] = tot <= kWideWin ? 1 : 0;  // window takes all
  if (tot <= kWideWin) {
    if (threadIdx.x == 0) sm.ibcast[0] = kSelBins - 1;
  } else if (before <= kWideWin && before + loc > kWideWin) {
    int cum = before;
    for (int q = 0; q < kPer; ++q) {
      const int c = static_cast<int>(sm.hist[c0 + q]);
      if (cum + c > kWideWin) {
        sm.ibcast[0] = cum == 0 ? -1 : c0 + q - 1;  // last bin that still fits
        break;
      }
      cum += c;
    }
  }
  __syncthreads();
  const int bmax = sm.ibcast[0];
  const int all = sm.ibcast[1];
  if (bmax < 0) return -1;
  for (int b0 = 0; b0 < A; b0 += kWideThreads * U) {
    uint64_t k[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int p = b0 + j * kWideThreads + threadIdx.x;
      k[j] = p < A ? ws.klow[p] : 0;
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int p = b0 + j * kWideThreads + threadIdx.x;
      const uint64_t key = wide_key(k[j], policy, urgency);
      const bool sel = p < A && (!has_lo || key > lo) && sel_bin(k[j], policy, urgency, sb) <= bmax;
      const unsigned m = __ballot_sync(kFull, sel);
      int base = 0;
      if (m && lane_id() == 0) base = atomicAdd(&sm.ibcast[4], __popc(m));
      base = __shfl_sync(kFull, base, 0);
      if (sel) {
        const int slot = base + __popc(m & lanemask_lt());
        sm.wkey[slot] = key;
        sm.wpos[slot] = p;
      }
    }
  }
  __syncthreads();
  const int K = sm.ibcast[4];
  wide_bitonic_sort(K, sm);
  if (threadIdx.x == 0) sm.ibcast[1] = all;
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

// Fair batching, the provably whole-admitted prefix of a sorted window,
// found in parallel.  With tb0 the exact budget before the window and
// S_k an upper bound (every partial rounded up) of the sum of the rounded
// task costs tc_0..tc_k, the reference's running budget before task k is
// t_k >= tb0 - S_{k-1} - k*u*tb0 (u = 2^-53, every intermediate in [0, tb0]),
// so tb0 - S_k >= k*2^-52*tb0 (directed rounding) together with
// N_k = sum of new tokens <= tok0 proves tc_k <= t_k and new_k <= tok_k:
// task k is admitted whole, and the stop test is false before it (tc_k >=
// tc_min).  Both conditions are monotone in k, so the proven tasks form a
// prefix [0, m).  Thread 0 then folds the exact budget over the prefix in
// the reference's order (one dependent subtraction per task) and the
// serial scan resumes at m.  Returns m.
__device__ int wide_admit_prefix(WideScan& st, int K, WideSmem& sm) {
  if (threadIdx.x == 0) {
    sm.dbcast[1] = st.tb;
    sm.bcast[7] = st.done ? 0 : st.tok;
  }
  __syncthreads();
  const double tb0 = sm.dbcast[1];
  const int64_t tok0 = sm.bcast[7];
  __syncthreads();
  if (tok0 <= 0 || !(tb0 >= 0.0)) return 0;
  constexpr int kPer = kWideWin / kWideThreads;
  const int k0 = threadIdx.x * kPer;
  double s_loc[kPer];
  int64_t n_loc[kPer];
  double s = 0.0;
  int64_t n = 0;
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int k = k0 + q;
    if (k < K) {
      s = __dadd_ru(s, sm.wtc[k]);
      n += static_cast<int64_t>(sm.wnw[k] & 0x7fffffffu);
    }
    s_loc[q] = s;
    n_loc[q] = n;
  }
  // block exclusive scan of the thread totals (sums rounded up stay upper bounds)
  double si = s;
  int64_t ni = n;
#pragma unroll
  for (int o = 1; o < kWarp; o <<= 1) {
    const double ys = __shfl_up_sync(kFull, si, o);
    const int64_t yn = __shfl_up_sync(kFull, ni, o);
    if (lane_id() >= o) {
      si = __dadd_ru(ys, si);
      ni += yn;
    }
  }
  double* wsum = reinterpret_cast<double*>(sm.red);   // [kWideWarps]
  int64_t* wtok = sm.red + kWideWarps;               // [kWideWarps]
  if (lane_id() == kWarp - 1) {
    wsum[wid()] = si;
    wtok[wid()] = ni;
  }
  __syncthreads();
  double ex_s = 0.0;
  int64_t ex_n = 0;
  for (int q = 0; q < wid(); ++q) {
    ex_s = __dadd_ru(ex_s, wsum[q]);
    ex_n += wtok[q];
  }
  {
    const double ps = __shfl_up_sync(kFull, si, 1);
    const int64_t pn = __shfl_up_sync(kFull, ni, 1);
    if (lane_id() > 0) {
      ex_s = __dadd_ru(ex_s, ps);
      ex_n += pn;
    }
  }
  __syncthreads();
  int my_ok = 0;
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int k = k0 + q;
    if (k < K) {
      const double S = __dadd_ru(ex_s, s_loc[q]);
      const int64_t N = ex_n + n_loc[q];
      const double slack = __dsub_rd(tb0, S);
      const double need = __dmul_ru(__dmul_ru(static_cast<double>(k), 0x1p-52), tb0);
      if (N <= tok0 && slack >= need) my_ok++;
    }
  }
  const int m = static_cast<int>(block_sum(my_ok, sm));
  if (m == 0) return 0;
  int64_t ctx_part = 0;
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int k = k0 + q;
    if (k < m) {
      sm.wtake[k] = static_cast<int32_t>(sm.wnw[k] & 0x7fffffffu);
      ctx_part += sm.wcx[k];
    }
    if (k == m - 1) sm.bcast[6] = ex_n + n_loc[q];  // tokens of the prefix
  }
  const int64_t ctx_sum = block_sum(ctx_part, sm);  // (barriers publish bcast[6])
  if (threadIdx.x == 0) {
    const int64_t n_m = sm.bcast[6];
    double tb = st.tb;
    int k = 0;
    for (; k + 4 <= m; k += 4) {
      const double a0 = sm.wtc[k], a1 = sm.wtc[k + 1], a2 = sm.wtc[k + 2], a3 = sm.wtc[k + 3];
      tb = dsub(dsub(dsub(dsub(tb, a0), a1), a2), a3);
    }
    for (; k < m; ++k) tb = dsub(tb, sm.wtc[k]);
    st.tb = tb;
    st.tok -= n_m;
    st.E += m;
    st.tn += n_m;
    st.tctx += ctx_sum;
    st.n_seen += m;
  }
  __syncthreads();
  return m;
}

// Greedy pass over one sorted window (sched.cpp:129-232), thread 0.  The
// scan state lives in registers for the loop.
__device__ __forceinline__ void wide_scan_window(WideScan& st_io, int K, int policy,
                                                 const FormCfg& f, int n_dec, double tc_min,
                                                 double cc_min, WideSmem& sm, int k_start = 0) {
  if (threadIdx.x != 0) return;
  WideScan st = st_io;
  const bool fair = policy == FB_POLICY_FAIRBATCH || policy == FB_POLICY_FAIRBATCH_PAB;
  if (fair) {
    // consider (sched.cpp:129-166).  The stop test depends only on the
    // budgets, which change only on an admission, so it is evaluated on entry
    // and after each admission -- the same points at which the reference's
    // per-task test could first fail.
    double tb = st.tb;
    int64_t tok = st.tok;
    auto exhausted = [&]() -> bool {
      if (tok <= 0 || tb < 0.0) return true;
      if (tb < tc_min) {  // no task fits whole any more: stop if none can chunk
        const double lim = ddiv(dsub(tb, cc_min), f.b);
        const double dt = static_cast<double>(tok);
        const double cpr = lim < dt ? lim : dt;
        if (!(cc_min <= tb && floor(cpr) >= 1.0)) return true;
      }
      return false;
    };
    bool done = st.done || exhausted();
    int k = k_start;
    if (!done && k < K) {
      double tc_n = sm.wtc[k], cc_n = sm.wcc[k];
      uint32_t w_n = sm.wnw[k];
      for (; k < K; ++k) {
        const double tc = tc_n, cc = cc_n;
        const int64_t nv = w_n & 0x7fffffffu;
        if (k + 1 < K) {  // software prefetch of the next sorted task
          tc_n = sm.wtc[k + 1];
          cc_n = sm.wcc[k + 1];
          w_n = sm.wnw[k + 1];
        }
        int64_t take = 0;
        if (tc <= tb && nv <= tok) {
          take = nv;
          tb = dsub(tb, tc);
          tok -= nv;
        } else if (tok > 0 && cc <= tb) {
          const double lim = ddiv(dsub(tb, cc), f.b);
          const double dt = static_cast<double>(tok);
          const double cp_real = lim < dt ? lim : dt;
          const int64_t cp = static_cast<int64_t>(floor(cp_real));
          if (cp >= 1) {
            take = cp;
            tb = dsub(tb, dadd(dmul(f.b, static_cast<double>(cp)), cc));
            tok -= cp;
          }
        }
        if (take > 0) {
          sm.wtake[k] = static_cast<int32_t>(take);
          st.E++;
          st.tn += take;
          st.tctx += sm.wcx[k];
          if (exhausted()) {
            ++k;
            done = true;
            break;
          }
        }
      }
    }
    st.n_seen += k - k_start;
    st.tb = tb;
    st.tok = tok;
    st.done = done;
    st_io = st;
    return;
  }
  for (int k = 0; k < K && !st.done; ++k) {
    const uint32_t w = sm.wnw[k];
    const int64_t nv = w & 0x7fffffffu;
    int64_t take = 0;
    if (false) {
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
  st_io = st;
}

// Node::complete_step (engine.cpp:204-254), block-wide.
__device__ void wide_complete(const EngineParams& P, Inst& w, WideSmem& sm) {
  const int64_t t = w.S.step_end;
  const WideScratch ws = wide_scratch(P, w);
  int any = 0;
  int64_t lemit = 0, lfin = 0;
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
      if (P.lead_bucket > 0) {
        if (fin) P.lastem[g] = t;
        lemit += emit;
        lfin += fin ? P.output[row] : 0;
      }
      WRec& rec = ws.rec[v.x];  // keep the view record in step
      rec = make_wrec(P.arrival[row] + P.ttft[row], P.first[g], prompt, pf, P.nidx[g],
                      static_cast<int32_t>(rec.anc_seq & kWRecSeqMask));
      w.vl[p] = make_int2(fin ? -1 : v.x, 0);
      any |= fin;
    }
  }
  if (P.lead_bucket > 0) {
    const int64_t ne = block_sum(lemit, sm);
    const int64_t nf = block_sum(lfin, sm);
    if (threadIdx.x == 0 && ne) lead_account(P, w.id, t, static_cast<uint32_t>(ne), nf);
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
      ws.rec[r].anc_seq = (ws.rec[r].anc_seq & ~kWRecSeqMask) | (w.S.seq_counter + j);
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
        ws.rec[r].anc_seq = (ws.rec[r].anc_seq & ~kWRecSeqMask) | w.S.seq_counter;
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
            rl.step = static_cast<int32_t>(w.S.step_counter);
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

// ------------------------------------------------ begin_step, in pieces
//
// Node::begin_step (engine.cpp:153-202) for an escalated node is split so
// that its streaming stages (K1 views, K2 histogram + gather) can run on the
// whole grid while the owner CTA runs the rest:
//   wide_prepare   pull arrivals (PAB admission), visible count   [owner]
//   wide_k1_views  K1 over a range of view positions               [any CTA]
//   wide_step      init_time_budget / urgency / selection bins     [pure]
//   wide_finish    K2 windows, K3 scan, plan, moves, truth time    [owner]

// K1 partial reductions over a view range: mins of tpot, ctx, decode
// ordinal, -decode ordinal, prefill ordinal, -prefill ordinal (ordinal =
// (slack + 2^39) << 22 | seq for fair batching, seq otherwise), [6] unused,
// and n_dec | (keys outside the packed range << 40) in [7] (summed).
constexpr int kK1Vals = 8;

// Fused candidate window.  K1 can select the window itself: with ordinal
// thresholds (Td, Tp) published by the owner, a view is a candidate iff its
// ordinal is below the threshold of its phase (decode: Td, prefill: Tp), and
// K1 gathers the candidates' positions while it streams the views.  Whatever
// the thresholds, the candidates are exactly the smallest keys -- a window,
// as the K2 passes would select it -- iff every candidate key is below every
// other key.  The thresholds are built per group of the threshold key so
// that this holds by construction except for the one quantity K1 itself
// reduces: the urgency, which splits fair batching's decodes into groups 0
// and 2.  wide_fused_ok checks the decode threshold against the true
// urgency ordinal.  When it fails, or the candidates overflow the window,
// the node takes the K2a / K2b passes as before.  The thresholds are a prediction from the node's
// previous step (WidePred): the boundary key its scan reached plus a margin,
// kept as an absolute deadline so it stays put while `now` advances.
struct WidePred {
  int32_t valid;  // 0: no prediction (first wide step of a node)
  int32_t g;      // group of the threshold key
  int64_t d;      // fair batching: threshold deadline (slack + now); else 0
  int64_t seq;    // threshold seq (fair: tie-break inside the deadline)
  int64_t urgency;  // the step's urgency (fair), predicts the next one
};

// Ordinal thresholds (Td, Tp) for a step at `now` from the prediction.
__device__ __forceinline__ void wide_thresholds(const WidePred& pr, int policy, int64_t now,
                                                int64_t& td, int64_t& tp, bool& on) {
  td = 0;
  tp = 0;
  on = pr.valid != 0;
  if (!on) return;
  const bool fair = policy == FB_POLICY_FAIRBATCH || policy == FB_POLICY_FAIRBATCH_PAB;
  constexpr int64_t kOrdMax = int64_t(1) << 62;
  int64_t ord;
  if (fair) {
    int64_t sl = pr.d - now + kPackSlack;
    if (sl < 0) {  // below every packed key: no candidates
      on = false;
      return;
    }
    ord = sl >= 2 * kPackSlack ? (2 * kPackSlack) << 22 : (sl << 22) | pr.seq;
    const int64_t u = pr.urgency < -kPackSlack
                          ? -kPackSlack
                          : (pr.urgency > kPackSlack ? kPackSlack : pr.urgency);
    const int64_t uord = (u + kPackSlack) << 22;
    if (pr.g == 0) {
      td = ord;
    } else if (pr.g == 1) {
      td = uord;
      tp = ord;
    } else {
      td = ord;
      tp = kOrdMax;
    }
  } else {
    ord = pr.seq;
    if (policy == FB_POLICY_SARATHI) {
      if (pr.g == 0) {
        td = ord;
      } else {
        td = kOrdMax;
        tp = ord;
      }
    } else {
      td = ord;
      tp = ord;
    }
  }
}

struct WideStep {
  int64_t A, n_dec, min_tpot, min_dec, ctx_min, urgency;
  double init_ms;
  bool bad;
  SelBins sb;
};

// Light view context for a K1 range (what load_view needs).
__device__ __forceinline__ Inst wide_view_ctx(const EngineParams& P, int64_t inst) {
  Inst w;
  w.id = inst;
  w.routed = nullptr;
  w.I = P.inst + inst;
  w.toff = w.I->trace_off;
  w.roff = w.I->rec_off;
  w.nreq = w.I->n_req;
  w.horizon = w.I->horizon;
  w.policy = w.I->policy;
  w.max_active = w.I->max_active;
  w.vl = P.vlist + w.roff;
  w.smem = nullptr;
  w.sd.clear();
  return w;
}

// K1 over view positions [p_lo, p_hi) by the calling CTA, U views in flight
// per thread (build_task_views, engine.cpp:51-81; slack, slo.h:45-61).
// Per view it reads the row index, then the request's 32-byte view record
// (TTFT deadline, first-token time, prompt, prefilled, next index, seq), plus
// tpot unless the node's tpot_slo is uniform.  For a
// prefill view next_idx == 0 and first == -1, so one expression gives both
// phases' slack.  Writes the key stem; the reductions stay in every thread's
// r[].
__device__ __forceinline__ void wide_k1_views(const EngineParams& P, const Inst& w, int64_t p_lo,
                                              int64_t p_hi, int64_t now, bool fair,
                                              int64_t (&r)[kK1Vals], WideSmem& sm, bool fused,
                                              int64_t td, int64_t tp, int32_t* ncand,
                                              int32_t* cpos, uint64_t* ckey) {
  const WideScratch ws = wide_scratch(P, w);
  const int64_t tpu = w.I->tpot_uniform;
  const uint64_t pol_stream = l2_evict_first_policy();
  const uint64_t pol_keep = l2_evict_last_policy();
  const int32_t* vrow = reinterpret_cast<const int32_t*>(w.vl);  // .x of {row, take}
  constexpr int U = 4;
  int64_t mn[6] = {kInf, kInf, kInf, kInf, kInf, kInf};
  int64_t l_cnt = 0, l_views = 0;
  // The row indices are loaded two batches ahead and the records of the
  // next batch prefetched into L2 one batch ahead (prefetches hold no
  // registers), so each batch's record loads hit L2 instead of waiting on
  // HBM behind their row index.
  int32_t rn[U], rn2[U];
#pragma unroll
  for (int j = 0; j < U; ++j) {
    const int64_t p = p_lo + j * kWideThreads + threadIdx.x;
    rn[j] = p < p_hi ? ld_stream_s32(vrow + 2 * p, pol_stream) : -1;
    const int64_t p2 = p + U * kWideThreads;
    rn2[j] = p2 < p_hi ? ld_stream_s32(vrow + 2 * p2, pol_stream) : -1;
  }
#pragma unroll
  for (int j = 0; j < U; ++j)
    if (rn[j] >= 0) prefetch_l2(ws.rec + rn[j]);
  for (int64_t b0 = p_lo; b0 < p_hi; b0 += kWideThreads * U) {
    int32_t rr[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      rr[j] = rn[j];
      rn[j] = rn2[j];
      const int64_t p = b0 + (2 * U + j) * kWideThreads + threadIdx.x;
      rn2[j] = p < p_hi ? ld_stream_s32(vrow + 2 * p, pol_stream) : -1;
    }
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (rn[j] >= 0) prefetch_l2(ws.rec + rn[j]);
    int4 rc[U];
    int64_t tpot[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      if (rr[j] < 0) continue;
      rc[j] = ld_stream_v4(reinterpret_cast<const int4*>(ws.rec + rr[j]), pol_stream);
      tpot[j] = tpu >= 0 ? tpu : P.tpot[w.toff + rr[j]];
    }
    int32_t seq[U];
    uint64_t stem[U];
    unsigned cmask = 0;  // candidates of this batch (bit j)
#pragma unroll
    for (int j = 0; j < U; ++j) {
      if (rr[j] < 0) continue;
      const int64_t p = b0 + j * kWideThreads + threadIdx.x;
      ++l_views;
      const int64_t as = (static_cast<int64_t>(static_cast<uint32_t>(rc[j].y)) << 32) |
                         static_cast<uint32_t>(rc[j].x);
      seq[j] = static_cast<int32_t>(as & kWRecSeqMask);
      const bool decode = rc[j].w < 0;
      const int64_t ni = rc[j].w & 0x7fffffff;
      const int64_t slack = (as >> 22) + tpot[j] * ni - now;
      const int64_t ctx = rc[j].z;
      const uint64_t sl = fair ? static_cast<uint64_t>(slack + kPackSlack) : 0;
      stem[j] = (decode ? (uint64_t(1) << 63) : 0) | (sl << 22) | static_cast<uint64_t>(seq[j]);
      // a fused node keeps only its candidates' stems (ckey); the others
      // are written for the K2 passes
      if (!fused) st_keep_u64(ws.klow + p, stem[j], pol_keep);
      if (fair && (slack < -kPackSlack || slack >= kPackSlack)) l_cnt |= int64_t(1) << 40;
      const int64_t ord = fair ? static_cast<int64_t>((sl << 22) | static_cast<uint64_t>(seq[j]))
                               : seq[j];  // selection ordinal
      mn[0] = tpot[j] < mn[0] ? tpot[j] : mn[0];
      mn[1] = ctx < mn[1] ? ctx : mn[1];
      if (ord < (decode ? td : tp)) cmask |= 1u << j;
      if (decode) {
        l_cnt++;
        mn[2] = ord < mn[2] ? ord : mn[2];
        mn[3] = -ord < mn[3] ? -ord : mn[3];
      } else {
        mn[4] = ord < mn[4] ? ord : mn[4];
        mn[5] = -ord < mn[5] ? -ord : mn[5];
      }
    }
    // candidate gather: one slot reservation per warp and batch
    if (fused && __any_sync(kFull, cmask != 0)) {
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const bool cand = (cmask >> j) & 1u;
        const unsigned m = __ballot_sync(kFull, cand);
        if (m) {
          const int leader = __ffs(m) - 1;
          int base = 0;
          if (lane_id() == leader) base = atomicAdd(ncand, __popc(m));
          base = __shfl_sync(kFull, base, leader);
          const int slot = base + __popc(m & lanemask_lt());
          if (cand && slot < kWideWin) {
            cpos[slot] = static_cast<int32_t>(b0 + j * kWideThreads + threadIdx.x);
            ckey[slot] = stem[j];
          }
        }
      }
    }
  }
  // warp-level reductions only: the warps fold into the node's global row
  // with atomics (no CTA barrier per view range)
#pragma unroll
  for (int q = 0; q < 6; ++q) r[q] = warp_min_i64(mn[q]);
  r[6] = warp_sum_small(l_views);
  int64_t c = l_cnt;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
  r[7] = c;
}

// The key stems of view positions [p_lo, p_hi) (K1's view code, stems only):
// a fused node whose candidates were not a window needs them for the K2
// passes or a later window.  Out of line: the rare path.
__device__ __noinline__ void wide_write_stems(const EngineParams& P, const Inst& w, int64_t p_lo,
                                              int64_t p_hi, int64_t now, bool fair, WideSmem& sm) {
  int64_t r[kK1Vals];
  wide_k1_views(P, w, p_lo, p_hi, now, fair, r, sm, false, 0, 0, nullptr, nullptr, nullptr);
  __syncthreads();
}

// init_time_budget (sched.cpp:90-106), urgency bound (sched.cpp:111-113) and
// the selection bins from the reduced K1 values.
__device__ __forceinline__ WideStep wide_step(const int64_t (&mn)[kK1Vals], int64_t A,
                                              int policy) {
  WideStep s;
  const bool fair = policy == FB_POLICY_FAIRBATCH || policy == FB_POLICY_FAIRBATCH_PAB;
  const int64_t dlo = mn[2], dhi = -mn[3], plo = mn[4], phi = -mn[5];
  s.A = A;
  s.min_tpot = mn[0];
  s.ctx_min = mn[1];
  s.n_dec = mn[7] & ((int64_t(1) << 40) - 1);
  // fair batching: the decode ordinal's high part is the slack
  s.min_dec = s.n_dec > 0 ? (dlo >> 22) - kPackSlack : kInf;
  // packed keys need seq < 2^22 and (fair) slack in [-2^39, 2^39)
  s.bad = (mn[7] >> 40) != 0;
  s.init_ms = 0.0;
  s.urgency = 0;
  if (fair) {
    const int64_t init =
        s.n_dec == 0 ? s.min_tpot : (s.min_dec > s.min_tpot ? s.min_dec : s.min_tpot);
    s.urgency = init + s.min_tpot;
    s.init_ms = us_to_ms(init);
  }
  const int64_t n_pf = A - s.n_dec;
  s.sb.urg = 0;
  if (fair) {
    // decodes with slack < urgency <=> ordinal < (urgency + 2^39) << 22
    const int64_t u = s.urgency < -kPackSlack ? -kPackSlack
                                              : (s.urgency > kPackSlack ? kPackSlack : s.urgency);
    const int64_t urg = (u + kPackSlack) << 22;
    s.sb.urg = urg;
    // UD and ND share the decode count (the urgency split is not counted)
    sel_range(s.sb, 0, dlo, dhi < urg - 1 ? dhi : urg - 1, s.n_dec);
    sel_range(s.sb, 1, plo, phi, n_pf);
    sel_range(s.sb, 2, dlo > urg ? dlo : urg, dhi, s.n_dec);
  } else if (policy == FB_POLICY_SARATHI) {
    sel_range(s.sb, 0, dlo, dhi, s.n_dec);
    sel_range(s.sb, 1, plo, phi, n_pf);
    sel_range(s.sb, 2, 0, 0, 0);
  } else {
    sel_range(s.sb, 0, dlo < plo ? dlo : plo, dhi > phi ? dhi : phi, A);
    sel_range(s.sb, 1, 0, 0, 0);
    sel_range(s.sb, 2, 0, 0, 0);
  }
  return s;
}

// Whether K1's candidates are a window that fits.  Fair batching: group 0
// threshold -> the candidates are the decodes below Td, a prefix of group 0
// iff Td <= the urgency ordinal U; group 1 -> all decodes below Td = the
// predicted U plus the prefills below Tp: groups 0 and a prefix of 1 iff Td
// == U; group 2 -> decodes below Td and every prefill: iff Td >= U.  Sarathi
// and prefill-first thresholds are prefixes by construction (seq order).
__device__ __forceinline__ bool wide_fused_ok(const WideStep& ss, int policy, int g, int64_t td,
                                              int ncand) {
  if (ss.bad || ncand <= 0 || ncand > kWideWin) return false;
  if (policy == FB_POLICY_FAIRBATCH || policy == FB_POLICY_FAIRBATCH_PAB) {
    const int64_t uord = ss.sb.urg;
    return g == 0 ? td <= uord : (g == 1 ? td == uord : td >= uord);
  }
  return true;
}

// Pull (engine.cpp:127-151) and the visible count; 0 means no step.
__device__ int64_t wide_prepare(const EngineParams& P, Inst& w, int64_t now, WideSmem& sm) {
  w.S.paths |= kPathWide;
  if (w.S.pulled < w.S.arr) wide_pull(P, w, now, wide_scratch(P, w), sm);
  return visible_count(w);
}

// The rest of begin_step once K1 ran.  K0 >= 0: the first window (the K0
// smallest keys; all of them when all0) is already sorted in sm.wkey /
// sm.wpos; K0 < 0: select it here.
__device__ void wide_finish(const EngineParams& P, Inst& w, int64_t now, const WideStep& ss,
                            int K0, bool all0, WideSmem& sm, WidePred& pred, bool stems) {
  const DevInst* I = w.I;
  const WideScratch ws = wide_scratch(P, w);
  WPROF_START
  WPROF_COUNT(10, 1)
  if (ss.bad) {  // keys outside the packed range: not supported here
    w.S.status = FB_ERR_VALIDATION;
    w.S.done = 1;
    return;
  }
  const int64_t A64 = ss.A;
  const int A = static_cast<int>(A64);
  const int policy = w.policy;
  const bool fair = policy == FB_POLICY_FAIRBATCH || policy == FB_POLICY_FAIRBATCH_PAB;
  const int64_t n_act = w.S.n_active;
  const int64_t n_dec = ss.n_dec;
  const int64_t ctx_min = ss.ctx_min;
  const int64_t urgency = ss.urgency;
  const double init_ms = ss.init_ms;
  const SelBins& sb = ss.sb;
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
  int64_t seen_before = 0;  // keys of the earlier windows (all considered)
  int64_t l_pmax = -1;  // last view position of an admitted waiting task
  const bool log_on = P.log_on != 0;
  const int64_t entry_base = I->log_entry_off + w.S.log_entries;
  for (;;) {
    WPROF(1)
    int K = K0;
    bool all = all0;
    K0 = -1;
    if (K < 0 && !stems) {  // a later window of a fused node: its stems first
      wide_write_stems(P, w, 0, A64, now, fair, sm);
      stems = true;
    }
    if (K < 0) {
      K = wide_select_binned(ws, A, has_lo, lo, policy, urgency, sb, sm);
      all = sm.ibcast[1] != 0;
      __syncthreads();
    }
    if (K < 0) {
      K = wide_select(ws, A, has_lo, lo, policy, urgency, sm);
      all = K < kWideWin;
    }
    WPROF(2)
    WPROF_COUNT(20, 1)
    if (K == 0) break;
    for (int k = threadIdx.x; k < K; k += kWideThreads) {
      const View v = load_view(P, w, sm.wpos[k], now);
      const uint32_t nwp = static_cast<uint32_t>(v.nw);
      const int64_t cxp = v.ctx;
      const double cc = dmul(f.c, static_cast<double>(cxp));
      sm.wcc[k] = cc;
      sm.wcx[k] = cxp;
      sm.wtc[k] = dadd(dmul(f.b, static_cast<double>(nwp & 0x7fffffffu)), cc);
      sm.wnw[k] = nwp;
      sm.wtake[k] = 0;
    }
    __syncthreads();
    WPROF(3)
    const int m0 = fair ? wide_admit_prefix(st, K, sm) : 0;
    WPROF(11)
    if (threadIdx.x == 0) {
      wide_scan_window(st, K, policy, f, static_cast<int>(n_dec), tc_min, cc_min, sm, m0);
      sm.ibcast[7] = st.done ? 1 : 0;
    }
    __syncthreads();
    const bool done = sm.ibcast[7] != 0;
    WPROF(4)
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
          l_pmax = p > l_pmax ? p : l_pmax;
        }
      }
      E_before += tot;
      Ew_before += totw;
    }
    __syncthreads();
    WPROF(5)
    if (done || all) {
      // the next step's candidate thresholds (WidePred): the boundary key the
      // scan reached plus a margin of 5/4 of the keys of its group it took
      // (+64).  Past the window's end the margin is extrapolated from the
      // deadline (or seq) density of those keys, so the prediction can grow.
      if (threadIdx.x == 0)
        sm.ibcast[2] = done ? static_cast<int>(st.n_seen - seen_before) - 1 : K - 1;
      __syncthreads();
      int kb = sm.ibcast[2];
      kb = kb < 0 ? 0 : (kb > K - 1 ? K - 1 : kb);
      const uint64_t gb = sm.wkey[kb] >> 62;
      int c = 0;
      for (int k = threadIdx.x; k <= kb; k += kWideThreads) c += (sm.wkey[k] >> 62) == gb;
      const int m_gb = static_cast<int>(block_sum(c, sm));
      if (threadIdx.x == 0) {
        constexpr uint64_t kLow = (uint64_t(1) << 62) - 1;
        const int margin = m_gb + m_gb / 4 + 64;
        pred.valid = 1;
        pred.urgency = urgency;
        const int R = kb + margin < K - 1 ? kb + margin : K - 1;
        const uint64_t kr = sm.wkey[R];
        if (kb + margin <= K - 1 || (kr >> 62) != gb) {
          const int64_t ord = static_cast<int64_t>(kr & kLow);
          pred.g = static_cast<int32_t>(kr >> 62);
          pred.seq = ord & kWRecSeqMask;
          pred.d = fair ? (ord >> 22) - kPackSlack + now : 0;
        } else {
          // the window ends inside group gb: extrapolate over [f, kb]
          const int f = kb - m_gb + 1 > 0 ? kb - m_gb + 1 : 0;
          const int n = kb - f;
          const int64_t ob = static_cast<int64_t>(sm.wkey[kb] & kLow);
          const int64_t of = static_cast<int64_t>(sm.wkey[f] & kLow);
          const int64_t sb = ob & kWRecSeqMask, sf = of & kWRecSeqMask;
          pred.g = static_cast<int32_t>(gb);
          const int64_t db = fair ? (ob >> 22) - kPackSlack + now : 0;
          const int64_t df = fair ? (of >> 22) - kPackSlack + now : 0;
          if (fair && n > 0 && db > df) {
            pred.d = db + ((db - df) * margin + n - 1) / n;
            pred.seq = 0;
          } else {
            int64_t sq = n > 0 && sb > sf ? sb + ((sb - sf) * margin + n - 1) / n : sb + margin;
            pred.d = db;
            pred.seq = sq > kWRecSeqMask ? kWRecSeqMask : sq;
          }
        }
      }
      break;
    }
    seen_before += K;
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
  WPROF(5)
  const int n_w = Ew_before;
  if (n_w > 0) {
    // Only [n_act, H) changes, H = one past the last admitted waiting task:
    // [n_act, n_act + n_w) takes the admitted in plan order (already in
    // vtmp), then the unadmitted of the range in their old order.  Marks are
    // cleared on the way (they are all-zero between steps).
    const int64_t nl_pmax = -block_min(-l_pmax, sm);
    const int64_t H = nl_pmax + 1;
    int64_t run = 0;
    for (int64_t b = n_act; b < H; b += kWideThreads) {
      const int64_t p = b + threadIdx.x;
      int2 v = make_int2(0, 0);
      bool un = false;
      if (p < H) {
        v = w.vl[p];
        un = ws.mark[p] == 0;
        if (!un) ws.mark[p] = 0;
      }
      int tot;
      const int pos = block_excl_count(un, tot, sm);
      if (un) ws.vtmp[n_w + run + pos] = make_int2(v.x, 0);
      run += tot;
    }
    __syncthreads();
    for (int64_t q = threadIdx.x; q < H - n_act; q += kWideThreads) w.vl[n_act + q] = ws.vtmp[q];
    __syncthreads();
  }
  WPROF(6)
  // ground_truth_step_time_ms, costmodel.cpp:138-146
  double actual = predict_ms(I->ta, I->tb, I->tc, tn, tctx);
  const double amp = I->noise_amp;
  if (amp != 0.0) {
    actual = apply_noise(actual, amp, I->noise_seed, w.S.step_counter);
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
  WPROF(7)
  __syncthreads();
}

// ------------------------------------------------ grid-wide wide engine
//
// Escalated nodes advance in lockstep iterations of one cooperative
// persistent kernel (one CTA per SM).  CTA b owns slot b: it runs its node's
// run_node event loop (engine.cpp:266-288) up to the next begin_step, then
// every CTA of the grid streams the views of every beginning node:
//
//   owner  events, complete_step, arrivals, pull            | barrier
//   grid   K1 views -> key stems + partial reductions       | barrier
//   grid   K2a histogram of the key bins (bins from the      |
//          combined K1 reductions: urgency, group ranges)    | barrier
//   grid   K2b gather of the keys up to the window's last    |
//          bin (from the node's histogram)                   | barrier
//   owner  sort, K3 scan (proven prefix + serial tail), plan, moves, truth
//
// so the bandwidth-bound K1/K2 passes use all SMs whatever the number of
// escalated nodes.  Each CTA takes an equal share of the iteration's views
// (all beginning nodes' views end to end), so the passes are balanced; the
// per-CTA partial reductions of a node are combined by whoever needs them.

struct WideSlot {
  int64_t inst;  // instance id, -1 = idle
  int64_t A, n_act, now;
  int32_t begin, policy;
  int32_t ncand, pad;  // K2b: gathered window keys
  // per-iteration results, written once by the CTA that completes a phase's
  // last view range of the node (views counted in k1_done / hist_done)
  unsigned long long k1_done, hist_done;
  int64_t red[kK1Vals];  // combined K1 reductions
  int64_t urgency;
  SelBins sb;
  int32_t bmax, all;     // window: last bin, holds every key
  // fused candidate window: thresholds published by the owner, result of K1
  int64_t td, tp;
  int32_t fused, fok, fg, pad2;  // fg: group of the threshold key
};

// What a helper CTA needs of a slot, read from L2 (the slot is written by
// another CTA).
struct WgView {
  int64_t inst, A, now, urgency, td, tp;
  int32_t policy, bmax, fused, fok, fg;
  SelBins sb;
};
__device__ __forceinline__ WgView wg_view(const WideSlot* s) {
  const volatile WideSlot* v = s;
  WgView o;
  o.inst = v->inst;
  o.A = v->A;
  o.now = v->now;
  o.policy = v->policy;
  o.urgency = v->urgency;
  o.bmax = v->bmax;
  o.td = v->td;
  o.tp = v->tp;
  o.fused = v->fused;
  o.fok = v->fok;
  o.fg = v->fg;
#pragma unroll
  for (int g = 0; g < 3; ++g) {
    o.sb.lo[g] = v->sb.lo[g];
    o.sb.sh[g] = v->sb.sh[g];
  }
  o.sb.urg = v->sb.urg;
  return o;
}

__device__ __forceinline__ void wg_barrier(unsigned long long* ctr, uint64_t gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(ctr), "l"(1ull) : "memory");
    const uint64_t target = gen * static_cast<uint64_t>(gridDim.x);
    uint64_t v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
      if (v >= target) break;
      __nanosleep(64);
    }
  }
  // the acquire load invalidates this SM's L1 (CCTL.IVALL), and the CTA
  // barrier orders every thread's later loads after it
  __syncthreads();
}

// Owner: stores the node's state and frees the slot.
__device__ __forceinline__ void wg_release(const EngineParams& P, Inst& w, bool& have) {
  __syncthreads();
  if (threadIdx.x == 0) {
    P.state[w.id] = w.S;
    if (!w.S.done) atomicAdd(&P.work[1], 1ull);
  }
  have = false;
  __syncthreads();
}

// Owner: publishes a beginning node to the grid.
__device__ __forceinline__ void wg_publish(const EngineParams& P, const Inst& w, int64_t A,
                                           int64_t now, WideSlot* my, const WidePred& pred) {
  uint32_t* hist = P.wg.hist + static_cast<size_t>(blockIdx.x) * kSelBins;
  for (int q = threadIdx.x; q < kSelBins; q += kWideThreads) hist[q] = 0;
  if (threadIdx.x == 0) {
    my->inst = w.id;
    my->A = A;
    my->n_act = w.S.n_active;
    my->now = now;
    my->begin = 1;
    my->policy = w.policy;
    my->ncand = 0;
    int64_t* row = P.wg.partial + static_cast<int64_t>(blockIdx.x) * kK1Vals;
#pragma unroll
    for (int k = 0; k < kK1Vals; ++k) row[k] = kInf;
    row[7] = 0;
    int64_t td, tp;
    bool on;
    wide_thresholds(pred, w.policy, now, td, tp, on);
    my->td = td;
    my->tp = tp;
    my->fused = on ? 1 : 0;
    my->fg = pred.g;
    my->fok = 0;
    my->k1_done = 0;
    my->hist_done = 0;
    my->bmax = -2;
  }
}

// Owner: runs the node's event loop until it must form a batch (returns
// true, slot published) or the slot has no node left (returns false).
// Escalation records of every node the warp engine handed over (begin
// pending): admitted-waiting marks all-zero and the 16-byte view record of
// every request, built by the whole grid -- an equal share of all those
// nodes' requests per CTA -- instead of by each node's owner alone (C4: 64
// nodes x 120 k requests, 254 us when the 64 owners built their own).
__device__ void wg_build_records(const EngineParams& P) {
  const int64_t n_list = static_cast<int64_t>(P.work[3]);
  auto pending = [&](int64_t i) { return P.state[i].pending_begin && !P.state[i].done; };
  int64_t tot = 0;
  for (int64_t j = 0; j < n_list; ++j) {
    const int64_t i = P.wide_list[j];
    if (pending(i)) tot += P.inst[i].n_req;
  }
  const int64_t lo = tot * blockIdx.x / gridDim.x, hi = tot * (blockIdx.x + 1) / gridDim.x;
  int64_t base = 0;
  for (int64_t j = 0; j < n_list && base < hi; ++j) {
    const int64_t i = P.wide_list[j];
    if (!pending(i)) continue;
    const int64_t n = P.inst[i].n_req;
    const int64_t a = lo > base ? lo - base : 0;
    const int64_t z = hi - base < n ? hi - base : n;
    if (a < z) {
      const Inst w = wide_view_ctx(P, i);
      const WideScratch ws = wide_scratch(P, w);
      for (int64_t q = a + threadIdx.x; q < z; q += kWideThreads) {
        ws.mark[q] = 0;
        const int64_t g = w.roff + q, row = w.toff + q;
        ws.rec[q] = make_wrec(P.arrival[row] + P.ttft[row], P.first[g], P.prompt[row],
                              P.prefilled[g], P.nidx[g], P.seq[g]);
      }
    }
    base += n;
  }
}

__device__ bool wg_advance(const EngineParams& P, Inst& w, bool& have, int64_t& ev,
                           WideSlot* my, WideSmem& sm, WidePred& pred) {
  for (;;) {
    if (!have) {
      if (threadIdx.x == 0) sm.bcast[0] = static_cast<int64_t>(atomicAdd(&P.work[2], 1ull));
      __syncthreads();
      const int64_t j = sm.bcast[0];
      __syncthreads();
      if (j >= static_cast<int64_t>(P.work[3])) {
        if (threadIdx.x == 0) {
          my->inst = -1;
          my->begin = 0;
        }
        return false;
      }
      const int64_t i = P.wide_list[j];
      w = wide_view_ctx(P, i);
      w.S = P.state[i];
      if (w.S.done) continue;
      have = true;
      ev = 0;
      __syncthreads();
      if (threadIdx.x == 0) pred.valid = 0;  // a new node: no prediction yet
      __syncthreads();
      if (w.S.pending_begin) {
        // escalation (view records and admitted-waiting marks were built by
        // the whole grid at launch, wg_build_records): in-flight takes cleared
        // (the warp engine's memory path leaves consumed takes behind)
        for (int64_t q = threadIdx.x; q < w.S.n_active; q += kWideThreads) w.vl[q].y = 0;
        __syncthreads();
        w.S.pending_begin = 0;
        const int64_t now = w.S.t_last;
        const int64_t A = wide_prepare(P, w, now, sm);
        if (A > 0) {
          wg_publish(P, w, A, now, my, pred);
          return true;
        }
      }
    }
    if (ev >= P.max_events) {
      wg_release(P, w, have);
      continue;
    }
    ev++;
    const int64_t* arrival = P.arrival + w.toff;
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
      wg_release(P, w, have);
      continue;
    }
    w.S.t_last = t;
    if (w.S.busy && t_step == t) {
      WPROF_START
      wide_complete(P, w, sm);
      WPROF(8)
    }
    while (w.S.arr < w.nreq && arrival[w.S.arr] == t) w.S.arr++;
    if (!w.S.busy && t < w.horizon) {
      const int64_t A = wide_prepare(P, w, t, sm);
      if (A > 0) {
        wg_publish(P, w, A, t, my, pred);
        return true;
      }
    }
  }
}

// Block exclusive prefix sum of int64 values (thread order) plus the total.
__device__ __forceinline__ int64_t block_excl_sum64(int64_t v, int64_t& total, WideSmem& sm) {
  int64_t incl = v;
#pragma unroll
  for (int o = 1; o < kWarp; o <<= 1) {
    const int64_t y = __shfl_up_sync(kFull, incl, o);
    if (lane_id() >= o) incl += y;
  }
  if (lane_id() == kWarp - 1) sm.red[wid()] = incl;
  __syncthreads();
  int64_t before = 0, tot = 0;
  for (int q = 0; q < kWideWarps; ++q) {
    const int64_t c = sm.red[q];
    if (q < wid()) before += c;
    tot += c;
  }
  __syncthreads();
  total = tot;
  return before + incl - v;
}

constexpr int kWgMaxSlots = 256;

// Work split of one iteration: the views of all beginning slots, laid end to
// end ([v0[t], v0[t+1]) for slot t), cut into gridDim.x equal ranges.
struct WgSplit {
  const int64_t* v0;   // smem, n_slots + 1 entries
  const int64_t* clo;  // smem, G + 1 entries: first view of CTA b
  int64_t V;
  int G, n_slots;
  __device__ __forceinline__ int64_t lo(int b) const { return clo[b]; }
  // slot holding view x (v0[t] <= x < v0[t+1])
  __device__ __forceinline__ int slot_of(int64_t x) const {
    int a = 0, z = n_slots - 1;
    while (a < z) {
      const int mid = (a + z + 1) >> 1;
      if (v0[mid] <= x) a = mid; else z = mid - 1;
    }
    return a;
  }
  // CTA whose range holds view x
  __device__ __forceinline__ int cta_of(int64_t x) const {
    int b = static_cast<int>((x * G) / V);
    if (b >= G) b = G - 1;
    while (b + 1 < G && lo(b + 1) <= x) ++b;
    while (b > 0 && lo(b) > x) --b;
    return b;
  }
};

// The window of slot t from its global histogram: last bin whose inclusive
// count fits (-1: the first nonempty bin overflows), and whether it holds
// every key.  Results in every thread.
__device__ __forceinline__ void wg_window(const EngineParams& P, int t, int64_t A, int& bmax,
                                          bool& all, WideSmem& sm) {
  const uint32_t* gh = P.wg.hist + static_cast<size_t>(t) * kSelBins;
  constexpr int kPer = kSelBins / kWideThreads;
  const int c0 = threadIdx.x * kPer;
  uint32_t hv[kPer];
  int loc = 0;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    hv[k] = __ldcg(gh + c0 + k);
    loc += static_cast<int>(hv[k]);
  }
  int tot;
  const int before = block_excl_sum(loc, tot, sm);
  if (tot <= kWideWin) {
    if (threadIdx.x == 0) sm.ibcast[0] = kSelBins - 1;
  } else if (before <= kWideWin && before + loc > kWideWin) {
    int cum = before;
    for (int k = 0; k < kPer; ++k) {
      const int cnt = static_cast<int>(hv[k]);
      if (cum + cnt > kWideWin) {
        sm.ibcast[0] = cum == 0 ? -1 : c0 + k - 1;
        break;
      }
      cum += cnt;
    }
  }
  __syncthreads();
  bmax = sm.ibcast[0];
  all = A <= kWideWin;  // first window of the step: every key is above nothing
  __syncthreads();
}

// Owner: the window's K gathered key stems of slot t, sorted into sm.wkey /
// sm.wpos.  The stems arrive in arbitrary order; their bins (nondecreasing
// in key) give a counting sort with the node's histogram as bin offsets, and
// each key's place inside its bin is its rank among the bin's keys (keys are
// unique), counted by the key's thread: sum over bins of count^2 compares.
// When that exceeds kBinRankWork (heavy slack ties crowding a few bins) the
// merge sort is cheaper.
constexpr int64_t kBinRankWork = int64_t(1) << 20;
__device__ void wg_bin_sort(const EngineParams& P, int t, int K, int bmax, int policy,
                            const WideStep& ss, const uint64_t* klow, WideSmem& sm) {
  const uint32_t* gh = P.wg.hist + static_cast<size_t>(t) * kSelBins;
  uint32_t* start = sm.hist;                                // [bin] first slot
  uint32_t* cur = reinterpret_cast<uint32_t*>(sm.wcc);      // [bin] fill cursor
  uint64_t* tkey = reinterpret_cast<uint64_t*>(sm.wtc);     // bin-ordered keys
  int32_t* tpos = sm.wtake;                                 // their positions
  constexpr int kPer = kSelBins / kWideThreads;
  const int c0 = threadIdx.x * kPer;
  uint32_t hv[kPer];
  int loc = 0;
  int64_t sq = 0;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    hv[k] = c0 + k <= bmax ? __ldcg(gh + c0 + k) : 0u;
    loc += static_cast<int>(hv[k]);
    sq += static_cast<int64_t>(hv[k]) * hv[k];
  }
  int tot;
  int run = block_excl_sum(loc, tot, sm);
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    start[c0 + k] = static_cast<uint32_t>(run);
    cur[c0 + k] = static_cast<uint32_t>(run);
    run += static_cast<int>(hv[k]);
  }
  const int64_t rank_work = block_sum(sq, sm);
  WPROF_COUNT(16, rank_work > kBinRankWork ? 1 : 0)
  WPROF_COUNT(17, rank_work)
  WPROF_COUNT(18, K)
  WPROF_COUNT(19, bmax)
  const int32_t* cp = P.wg.cpos + static_cast<size_t>(t) * kWideWin;
  if (rank_work > kBinRankWork) {
    for (int k = threadIdx.x; k < K; k += kWideThreads) {
      sm.wkey[k] = wide_key(__ldcg(klow + __ldcg(cp + k)), policy, ss.urgency);
      sm.wpos[k] = __ldcg(cp + k);
    }
    __syncthreads();
    wide_bitonic_sort(K, sm);
    return;
  }
#pragma unroll
  for (int q = 0; q < kWideWin / kWideThreads; ++q) {
    const int k = threadIdx.x + q * kWideThreads;
    if (k < K) {
      const uint64_t kl = __ldcg(klow + __ldcg(cp + k));
      const int b = sel_bin(kl, policy, ss.urgency, ss.sb);
      const uint32_t dst = atomicAdd(&cur[b], 1u);
      tkey[dst] = wide_key(kl, policy, ss.urgency);
      tpos[dst] = __ldcg(cp + k);
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += kWideThreads) {
    const uint64_t x = tkey[k];
    // bin of slot k: the last bin whose start is <= k (binary search)
    int lo = 0, hi = bmax;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (static_cast<int>(start[mid]) <= k) lo = mid; else hi = mid - 1;
    }
    const int b0 = static_cast<int>(start[lo]), b1 = static_cast<int>(cur[lo]);
    int rank = 0;
    for (int q = b0; q < b1; ++q) rank += tkey[q] < x;
    sm.wkey[b0 + rank] = x;
    sm.wpos[b0 + rank] = tpos[k];
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kWideThreads, 1)
wide_grid_kernel(const __grid_constant__ EngineParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WideSmem& sm = *reinterpret_cast<WideSmem*>(smem_raw);
  __shared__ int64_t s_v0[kWgMaxSlots + 1];
  __shared__ int64_t s_clo[kWgMaxSlots + 1];
  WideSlot* slots = reinterpret_cast<WideSlot*>(P.wg.slots);
  WideSlot* my = slots + blockIdx.x;
  const int n_slots = static_cast<int>(gridDim.x);
  // The owner's node lives in shared memory between owner phases, so it
  // holds no registers while the CTA streams other nodes' views.
  __shared__ __align__(16) unsigned char s_wbuf[sizeof(Inst)];
  Inst& s_w = *reinterpret_cast<Inst*>(s_wbuf);
  __shared__ int s_have;
  __shared__ int64_t s_ev;
  __shared__ WidePred s_pred;  // the owned node's candidate-window prediction
  if (threadIdx.x == 0) {
    s_have = 0;
    s_ev = 0;
    s_pred.valid = 0;
  }
  __syncthreads();
  uint64_t gen = 0;
  // Always-on phase clock (CTA 0, %globaltimer ns) -> wg.bar[8 + phase],
  // wg.bar[13] = iterations; read by fb_arena_wide_phases.
  uint64_t ph_t = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0)
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ph_t));
  auto phase = [&](int k) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      uint64_t n;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(n));
      P.wg.bar[8 + k] += n - ph_t;
      ph_t = n;
    }
  };
#ifdef FB_WIDE_PROF
  long long gp_t = clock64();
#define GPROF(slot)                                                                    \
  if (blockIdx.x == 0 && threadIdx.x == 0) {                                           \
    const long long n_ = clock64();                                                    \
    atomicAdd(&g_wide_prof[slot], static_cast<unsigned long long>(n_ - gp_t));         \
    gp_t = n_;                                                                         \
  }
#define CPROF_START long long cp_t_ = clock64(); long long sp_t_ = cp_t_;
#define SPROF(k)                                                                       \
  if (threadIdx.x == 0) {                                                              \
    const long long n_ = clock64();                                                    \
    g_sub_prof[blockIdx.x][k] += n_ - sp_t_;                                           \
    sp_t_ = n_;                                                                        \
  }
#define CPROF(k)                                                                       \
  if (threadIdx.x == 0) g_cta_prof[blockIdx.x][k] += clock64() - cp_t_;
#else
#define GPROF(slot)
#define CPROF_START
#define CPROF(k)
#define SPROF(k)
#endif
  wg_build_records(P);
  wg_barrier(P.wg.bar, ++gen);
  for (;;) {
    // ---- owner: advance to the next begin_step
    {
      CPROF_START
      Inst w = s_w;
      bool have = s_have != 0;
      int64_t ev = s_ev;
      wg_advance(P, w, have, ev, my, sm, s_pred);
      __syncthreads();
      if (threadIdx.x == 0) {
        s_w = w;
        s_have = have ? 1 : 0;
        s_ev = ev;
      }
      CPROF(3)
    }
    wg_barrier(P.wg.bar, ++gen);
#ifdef FB_WIDE_PROF
    if (blockIdx.x == 0 && threadIdx.x == 0 && g_wide_prof[23] == 0)
      g_wide_prof[23] = static_cast<unsigned long long>(clock64() - gp_t);  // first advance
#endif
    GPROF(12)
    phase(0);
    // ---- work split (every CTA, from the published slots)
    WgSplit sp;
    {
      int64_t a = 0;
      if (threadIdx.x < n_slots) {
        const volatile WideSlot* sl = slots + threadIdx.x;
        if (sl->inst >= 0 && sl->begin) a = sl->A;
      }
      int64_t tot;
      const int64_t before = block_excl_sum64(a, tot, sm);
      if (threadIdx.x < n_slots) s_v0[threadIdx.x] = before;
      if (threadIdx.x == 0) s_v0[n_slots] = tot;
      for (int b = threadIdx.x; b <= static_cast<int>(gridDim.x); b += kWideThreads)
        s_clo[b] = (tot * b) / static_cast<int64_t>(gridDim.x);
      __syncthreads();
      sp.v0 = s_v0;
      sp.clo = s_clo;
      sp.V = tot;
      sp.G = static_cast<int>(gridDim.x);
      sp.n_slots = n_slots;
    }
    if (sp.V == 0) break;  // no node left anywhere
    const int64_t my_lo = sp.lo(blockIdx.x), my_hi = sp.lo(blockIdx.x + 1);
    const int t_first = my_hi > my_lo ? sp.slot_of(my_lo) : n_slots;
    // ---- K1: views -> key stems + this CTA's partial reductions per slot
    {
      CPROF_START
      for (int t = t_first; t < n_slots && s_v0[t] < my_hi; ++t) {
        const int64_t a = s_v0[t] > my_lo ? s_v0[t] : my_lo;
        const int64_t z = s_v0[t + 1] < my_hi ? s_v0[t + 1] : my_hi;
        if (z <= a) continue;
        const WgView sv = wg_view(slots + t);
        const Inst wv = wide_view_ctx(P, sv.inst);
        const bool fair = sv.policy == FB_POLICY_FAIRBATCH || sv.policy == FB_POLICY_FAIRBATCH_PAB;
        int64_t r[kK1Vals];
        wide_k1_views(P, wv, a - s_v0[t], z - s_v0[t], sv.now, fair, r, sm, sv.fused != 0, sv.td,
                      sv.tp, &slots[t].ncand, P.wg.cpos + static_cast<size_t>(t) * kWideWin,
                      P.wg.ckey + static_cast<size_t>(t) * kWideWin);
        // each warp folds its reductions into the node's row (P.wg.partial
        // row t, reset by the owner at publish); the warp that completes the
        // node's view count derives init budget, urgency and selection bins
        if (lane_id() == 0 && r[6] > 0) {
          int64_t* row = P.wg.partial + static_cast<int64_t>(t) * kK1Vals;
#pragma unroll
          for (int k = 0; k < 6; ++k)
            if (r[k] != kInf)
              atomicMin(reinterpret_cast<long long*>(row + k), static_cast<long long>(r[k]));
          atomicAdd(reinterpret_cast<unsigned long long*>(row + 7),
                    static_cast<unsigned long long>(r[7]));
          __threadfence();
          const unsigned long long seg = static_cast<unsigned long long>(r[6]);
          if (atomicAdd(&slots[t].k1_done, seg) + seg == static_cast<unsigned long long>(sv.A)) {
            __threadfence();
            int64_t acc[kK1Vals];
#pragma unroll
            for (int k = 0; k < kK1Vals; ++k) acc[k] = __ldcg(row + k);
            const WideStep ss = wide_step(acc, sv.A, sv.policy);
            volatile WideSlot* vs = slots + t;
#pragma unroll
            for (int k = 0; k < kK1Vals; ++k) vs->red[k] = acc[k];
            vs->urgency = ss.urgency;
#pragma unroll
            for (int g = 0; g < 3; ++g) {
              vs->sb.lo[g] = ss.sb.lo[g];
              vs->sb.sh[g] = ss.sb.sh[g];
            }
            vs->sb.urg = ss.sb.urg;
            const int nc = atomicAdd(&slots[t].ncand, 0);
            const bool ok = sv.fused != 0 && wide_fused_ok(ss, sv.policy, sv.fg, sv.td, nc);
            vs->fok = ok ? 1 : 0;
            atomicAdd(&P.wg.bar[ok ? 14 : 15], 1ull);
            if (!ok) vs->ncand = 0;  // K2b gathers the window instead
          }
        }
      }
      CPROF(0)
    }
    wg_barrier(P.wg.bar, ++gen);
    GPROF(13)
    phase(1);
    // the K2 passes only for nodes whose candidates are not a window (every
    // CTA reads the same slots after the barrier: the same decision)
    int need = 0;
    if (threadIdx.x < n_slots) {
      const volatile WideSlot* sl = slots + threadIdx.x;
      need = sl->inst >= 0 && sl->begin && !sl->fok;
    }
    const bool need_k2 = __syncthreads_or(need) != 0;
    if (need_k2) {
    // ---- K2a: histogram of the selection bins
    {
      CPROF_START
      for (int t = t_first; t < n_slots && s_v0[t] < my_hi; ++t) {
        const int64_t a = s_v0[t] > my_lo ? s_v0[t] : my_lo;
        const int64_t z = s_v0[t + 1] < my_hi ? s_v0[t + 1] : my_hi;
        if (z <= a) continue;
        const WgView sv = wg_view(slots + t);
        if (sv.fok) continue;
        const Inst wv = wide_view_ctx(P, sv.inst);
        const WideScratch ws = wide_scratch(P, wv);
        const int64_t p_lo = a - s_v0[t], p_hi = z - s_v0[t];
        if (sv.fused) {  // K1 kept only candidate stems: write them all now
          const bool fair = sv.policy == FB_POLICY_FAIRBATCH || sv.policy == FB_POLICY_FAIRBATCH_PAB;
          wide_write_stems(P, wv, p_lo, p_hi, sv.now, fair, sm);
        }
        for (int k = threadIdx.x; k < kSelBins; k += kWideThreads) sm.hist[k] = 0;
        __syncthreads();
        SPROF(0)
        // each view's bin is kept in shared memory for K2b (index = the
        // view's offset in this CTA's range; beyond kWgBinCap K2b recomputes)
        const int64_t sb0 = s_v0[t] - my_lo;
        const uint64_t pol_keep = l2_evict_last_policy();
        constexpr int U = 8;
        for (int64_t b0 = p_lo; b0 < p_hi; b0 += kWideThreads * U) {
          uint64_t kl[U];
#pragma unroll
          for (int j = 0; j < U; ++j) {
            const int64_t p = b0 + j * kWideThreads + threadIdx.x;
            kl[j] = p < p_hi ? ld_keep_u64(ws.klow + p, pol_keep) : 0;
          }
#pragma unroll
          for (int j = 0; j < U; ++j) {
            const int64_t p = b0 + j * kWideThreads + threadIdx.x;
            if (p < p_hi) {
              const int bin = sel_bin(kl[j], sv.policy, sv.urgency, sv.sb);
              atomicAdd(&sm.hist[bin], 1u);
              if (sb0 + p < kWgBinCap) wg_bins(sm)[sb0 + p] = static_cast<uint16_t>(bin);
            }
          }
        }
        __syncthreads();
        SPROF(1)
        // Flush only up to this segment's own crossing bin (the first whose
        // cumulative count exceeds a window): the node's global crossing bin
        // can only come earlier (counts only add), so every bin up to it is
        // complete in the global histogram.
        uint32_t* gh = P.wg.hist + static_cast<size_t>(t) * kSelBins;
        constexpr int kPer = kSelBins / kWideThreads;
        const int c0 = threadIdx.x * kPer;
        int loc = 0;
#pragma unroll
        for (int k = 0; k < kPer; ++k) loc += static_cast<int>(sm.hist[c0 + k]);
        int tot;
        const int before = block_excl_sum(loc, tot, sm);
        int64_t cross = kSelBins;
        if (before <= kWideWin && before + loc > kWideWin) {
          int cum = before;
          for (int k = 0; k < kPer; ++k) {
            cum += static_cast<int>(sm.hist[c0 + k]);
            if (cum > kWideWin) {
              cross = c0 + k;
              break;
            }
          }
        }
        cross = block_min(cross, sm);
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
          const uint32_t v = sm.hist[c0 + k];
          if (v && c0 + k <= cross) atomicAdd(gh + c0 + k, v);
        }
        __syncthreads();
        SPROF(2)
        // the CTA that completes the node's histogram picks its window once
        if (threadIdx.x == 0) {
          __threadfence();
          const unsigned long long seg = static_cast<unsigned long long>(z - a);
          sm.ibcast[6] =
              atomicAdd(&slots[t].hist_done, seg) + seg == static_cast<unsigned long long>(sv.A);
        }
        __syncthreads();
        if (sm.ibcast[6]) {
          __threadfence();
          int bmax;
          bool all;
          wg_window(P, t, sv.A, bmax, all, sm);
          if (threadIdx.x == 0) {
            volatile WideSlot* vs = slots + t;
            vs->bmax = bmax;
            vs->all = all ? 1 : 0;
          }
        }
        __syncthreads();
        SPROF(3)
      }
      CPROF(1)
    }
    wg_barrier(P.wg.bar, ++gen);
    GPROF(14)
    phase(2);
    // ---- K2b: gather the window's keys
    {
      CPROF_START
      for (int t = t_first; t < n_slots && s_v0[t] < my_hi; ++t) {
        const int64_t a = s_v0[t] > my_lo ? s_v0[t] : my_lo;
        const int64_t z = s_v0[t + 1] < my_hi ? s_v0[t + 1] : my_hi;
        if (z <= a) continue;
        const WgView sv = wg_view(slots + t);
        const int bmax = sv.bmax;
        if (sv.fok || bmax < 0) continue;
        const Inst wv = wide_view_ctx(P, sv.inst);
        const WideScratch ws = wide_scratch(P, wv);
        const int64_t p_lo = a - s_v0[t], p_hi = z - s_v0[t];
        int32_t* cp = P.wg.cpos + static_cast<size_t>(t) * kWideWin;
        int32_t* ncand = &slots[t].ncand;
        // the bins K2a left in shared memory: only the selected views' stems
        // are read again (a window's worth per node, not every view).  Count
        // this CTA's selected views, reserve their slots with one atomic,
        // then write them (any order: the owner sorts the window).
        const int64_t sb0 = s_v0[t] - my_lo;
        const uint16_t* bins = wg_bins(sm);
        SPROF(4)
        int cnt = 0;
        for (int64_t p = p_lo + threadIdx.x; p < p_hi; p += kWideThreads) {
          const bool sel = sb0 + p < kWgBinCap
                               ? static_cast<int>(bins[sb0 + p]) <= bmax
                               : sel_bin(__ldcg(ws.klow + p), sv.policy, sv.urgency, sv.sb) <= bmax;
          cnt += sel;
        }
        int tot;
        int slot = block_excl_sum(cnt, tot, sm);
        if (tot == 0) continue;
        if (threadIdx.x == 0) sm.ibcast[7] = atomicAdd(ncand, tot);
        __syncthreads();
        slot += sm.ibcast[7];
        // positions only: the owner reads the window's stems itself
        for (int64_t p = p_lo + threadIdx.x; cnt > 0 && p < p_hi; p += kWideThreads) {
          const bool sel = sb0 + p < kWgBinCap
                               ? static_cast<int>(bins[sb0 + p]) <= bmax
                               : sel_bin(__ldcg(ws.klow + p), sv.policy, sv.urgency, sv.sb) <= bmax;
          if (sel) {
            cp[slot] = static_cast<int32_t>(p);
            ++slot;
            --cnt;
          }
        }
        __syncthreads();
      }
      SPROF(5)
      CPROF(2)
    }
    wg_barrier(P.wg.bar, ++gen);
    }  // need_k2
    GPROF(15)
    phase(3);
    // ---- owner: the rest of begin_step
    if (s_have) {
      WPROF_START
      Inst w = s_w;
      bool have = true;
      const int t = static_cast<int>(blockIdx.x);
      const volatile WideSlot* vs = my;
      int64_t acc[kK1Vals];
#pragma unroll
      for (int k = 0; k < kK1Vals; ++k) acc[k] = vs->red[k];
      const WideStep ss = wide_step(acc, vs->A, w.policy);
      const int bmax = vs->bmax;
      bool all0 = vs->all != 0;
      int K0 = -1;
      if (vs->fok) {  // K1 gathered the window: its keys, sorted
        K0 = vs->ncand;
        all0 = K0 == vs->A;
        const uint64_t* ck = P.wg.ckey + static_cast<size_t>(t) * kWideWin;
        const int32_t* cp = P.wg.cpos + static_cast<size_t>(t) * kWideWin;
        WPROF(0)
        for (int k = threadIdx.x; k < K0; k += kWideThreads) {
          sm.wkey[k] = wide_key(__ldcg(ck + k), w.policy, ss.urgency);
          sm.wpos[k] = __ldcg(cp + k);
        }
        __syncthreads();
        WPROF(21)
        wide_bitonic_sort(K0, sm);
        WPROF(1)
        WPROF_COUNT(18, K0)
      } else if (bmax >= 0) {
        K0 = vs->ncand;
        WPROF(0)
        wg_bin_sort(P, t, K0, bmax, w.policy, ss, wide_scratch(P, w).klow, sm);
        WPROF(1)
      } else {
        all0 = false;
      }
      wide_finish(P, w, vs->now, ss, K0, all0, sm, s_pred, vs->fok == 0);
      __syncthreads();
      if (w.S.done) wg_release(P, w, have);
      if (threadIdx.x == 0) {
        s_w = w;
        s_have = have ? 1 : 0;
      }
      __syncthreads();
    }
    GPROF(9)
    phase(4);
    if (blockIdx.x == 0 && threadIdx.x == 0) P.wg.bar[13]++;
  }
}

}  // namespace fbgpu
