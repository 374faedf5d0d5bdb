// fb_device.cuh -- device-side layouts and primitives shared by the kernels.
//
// Arithmetic conventions (bit-exact parity with the reference):
//   * every fp64 expression on the decision path is written with explicit
//     round-to-nearest intrinsics in the reference's operation order, and the
//     translation unit is additionally compiled with -fmad=false, so no FMA
//     contraction can change a batch decision;
//   * time is int64 microseconds (time.h:23-34).
#pragma once

// Loops off the repeated-plan hot path are kept rolled: the warp engine is
// instruction-fetch bound, so code size costs more than loop overhead there
// (FB_COLD_UNROLL=0 restores the compiler's default unrolling).
#ifndef FB_COLD_UNROLL
#define FB_COLD_UNROLL 1
#endif
#if FB_COLD_UNROLL
#define FB_COLD_LOOP _Pragma("unroll 1")
#else
#define FB_COLD_LOOP
#endif

#ifndef FB_NOHINT
#define FB_LIKELY(x) __builtin_expect(!!(x), 1)
#define FB_UNLIKELY(x) __builtin_expect(!!(x), 0)
#else
#define FB_LIKELY(x) (x)
#define FB_UNLIKELY(x) (x)
#endif

#include <cstdint>

#include "../../include/fbgpu.h"
#include "../../include/fbgpu_digest.h"

namespace fbgpu {

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;
constexpr int64_t kInf = INT64_MAX;

// ------------------------------------------------------------ fp64 helpers

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// us_to_ms, time.h:34: RN(us / 1000) without the division sequence --
// Markstein's correction step: with y_inv = RN(1/1000) = 0.001 and the
// faithful q0 = RN(x y_inv), r = x - 1000 q0 is exact (one FMA) and
// RN(q0 + r y_inv) is the correctly rounded quotient.  Checked bit for bit
// against __ddiv_rn on 4.7e10 integers (all of [-2^32, 2^32), 2^29 around
// every power of two up to 2^53, 2^34 random ones): tools/micro/div1000.cu.
__device__ __forceinline__ double us_to_ms(int64_t us) {
  const double x = static_cast<double>(us);
  const double q0 = __dmul_rn(x, 0.001);
  return __fma_rn(__fma_rn(-q0, 1000.0, x), 0.001, q0);
}
// ms_to_us, time.h:30-32 (llround: half away from zero)
__device__ __forceinline__ int64_t ms_to_us(double ms) {
  return static_cast<int64_t>(llround(dmul(ms, 1000.0)));
}
// predict_step_time_ms, costmodel.cpp:112-116: (a + b*new) + c*ctx
__device__ __forceinline__ double predict_ms(double a, double b, double c,
                                             int64_t nw, int64_t ctx) {
  return dadd(dadd(a, dmul(b, static_cast<double>(nw))),
              dmul(c, static_cast<double>(ctx)));
}

// Running max of x_j = fl(fl(d/1000)/j) (RequestReport::max_tpot_ms,
// metrics.cpp:42-49) without the two divisions when x_j cannot exceed the
// current max m: x_j <= (d/(1000 j)) (1+2^-53)^2 < (d/(1000 j)) (1+2^-51), so
// d*(1+2^-51) <= 1000*j*m (evaluated with upward / downward rounding) proves
// x_j <= m and the std::max leaves m unchanged.  Otherwise x_j is computed
// exactly in the reference's operation order.  d >= 0, 1 <= j < 2^31.
// The divisions, out of line (rarely reached: keeps the hot loops compact).
static __device__ __noinline__ double max_ratio_div(double m, int64_t d, int32_t j) {
  const double x = ddiv(us_to_ms(d), static_cast<double>(j));
  return m < x ? x : m;
}
__device__ __forceinline__ void max_ratio(double& m, int64_t d, int32_t j) {
  const double lhs = __dmul_ru(static_cast<double>(d), 1.0 + 0x1p-51);
  const double rhs = __dmul_rd(__dmul_rd(1000.0, static_cast<double>(j)), m);
  if (FB_LIKELY(lhs <= rhs)) return;
  m = max_ratio_div(m, d, j);
}

// -------------------------------------------------------------- rng.h

__device__ __forceinline__ uint64_t splitmix64(uint64_t& s) {  // rng.h:25-30
  uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t derive_seed(uint64_t base, uint64_t stream) {
  uint64_t s = base ^ (0x9e3779b97f4a7c15ULL * (stream + 1));  // rng.h:33-37
  splitmix64(s);
  return splitmix64(s);
}
__device__ __forceinline__ double keyed_uniform(uint64_t seed, uint64_t ord) {
  uint64_t s = derive_seed(seed, ord);  // rng.h:91-94
  return dmul(static_cast<double>(splitmix64(s) >> 11), 0x1.0p-53);
}
// ground_truth_step_time_ms's noise factor (costmodel.cpp:138-146):
// actual * (1 + amp * (2u - 1)), out of line (noise is off in most runs).
static __device__ __noinline__ double apply_noise(double actual, double amp, uint64_t seed,
                                           uint64_t ord) {
  const double u = dsub(dmul(2.0, keyed_uniform(seed, ord)), 1.0);
  return dmul(actual, dadd(1.0, dmul(amp, u)));
}

// ------------------------------------------------------------- warp utils

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

template <typename T>
__device__ __forceinline__ T warp_min(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T w = __shfl_xor_sync(kFull, v, o);
    v = w < v ? w : v;
  }
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T w = __shfl_xor_sync(kFull, v, o);
    v = w > v ? w : v;
  }
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {  // integers only (exact)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// Single-instruction (redux.sync) reductions with exact fallbacks.

// min over int64 values; kInf marks "no value".  One REDUX when every value
// fits in int32, else the 5-level shuffle tree.
__device__ __forceinline__ int64_t warp_min_i64(int64_t v) {
  const bool none = v == kInf;
  const bool fits = none || (v >= INT32_MIN && v < INT32_MAX);
  if (__all_sync(kFull, fits)) {
    const int m = __reduce_min_sync(kFull, none ? INT32_MAX : static_cast<int>(v));
    return m == INT32_MAX ? kInf : static_cast<int64_t>(m);
  }
  return warp_min(v);
}
// sum of non-negative values below 2^50 (two 32-bit REDUX on 24-bit splits)
__device__ __forceinline__ int64_t warp_sum_small(int64_t v) {
  const uint32_t lo = static_cast<uint32_t>(v) & 0xffffffu;
  const uint32_t hi = static_cast<uint32_t>(static_cast<uint64_t>(v) >> 24);
  return (static_cast<int64_t>(__reduce_add_sync(kFull, hi)) << 24) +
         static_cast<int64_t>(__reduce_add_sync(kFull, lo));
}
// Upper bound of a sum of doubles (every partial rounded toward +inf).
__device__ __forceinline__ double warp_sum_ru(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_ru(v, __shfl_xor_sync(kFull, v, o));
  return v;
}
__device__ __forceinline__ uint64_t warp_xor_u64(uint64_t v) {
  const uint32_t lo = __reduce_xor_sync(kFull, static_cast<uint32_t>(v));
  const uint32_t hi = __reduce_xor_sync(kFull, static_cast<uint32_t>(v >> 32));
  return (static_cast<uint64_t>(hi) << 32) | lo;
}

// ------------------------------------------------------------- tile utils
//
// The warp engine simulates one node per *tile* of kTile lanes: a full warp
// by default; FB_TILE = 16 builds half-warp tiles (two nodes advance per warp
// instruction when their control flow agrees; bit-exact, slower on C2).
// Every lane-collective on the per-node paths goes through these:
// masks name only the tile, so the two tiles of a warp stay correct whether
// they run converged or diverged.  Ballots / match results and lane indices
// are tile-relative.
#ifndef FB_TILE
#define FB_TILE 32
#endif
constexpr int kTile = FB_TILE;
static_assert(kTile == 16 || kTile == 32, "tile of 16 or 32 lanes");

__device__ __forceinline__ int tile_lane() { return threadIdx.x & (kTile - 1); }
__device__ __forceinline__ int tile_base() { return (threadIdx.x & (kWarp - 1)) & ~(kTile - 1); }
__device__ __forceinline__ unsigned tile_mask() {
  return kTile == kWarp ? kFull : (((1u << kTile) - 1u) << tile_base());
}
__device__ __forceinline__ void tile_sync() { __syncwarp(tile_mask()); }
__device__ __forceinline__ unsigned tile_ballot(bool p) {
  if (kTile == kWarp) return __ballot_sync(kFull, p);
  return __ballot_sync(tile_mask(), p) >> tile_base();
}
__device__ __forceinline__ bool tile_all(bool p) { return __all_sync(tile_mask(), p); }
__device__ __forceinline__ bool tile_any(bool p) { return __any_sync(tile_mask(), p); }
__device__ __forceinline__ unsigned tile_match_any(unsigned v) {
  if (kTile == kWarp) return __match_any_sync(kFull, v);
  return __match_any_sync(tile_mask(), v) >> tile_base();
}
__device__ __forceinline__ unsigned tile_lanemask_lt() { return (1u << tile_lane()) - 1u; }
__device__ __forceinline__ unsigned tile_or(unsigned v) { return __reduce_or_sync(tile_mask(), v); }
template <typename T>
__device__ __forceinline__ T tile_shfl(T v, int src) {
  return __shfl_sync(tile_mask(), v, src, kTile);
}
template <typename T>
__device__ __forceinline__ T tile_shfl_xor(T v, int o) {
  return __shfl_xor_sync(tile_mask(), v, o, kTile);
}
template <typename T>
__device__ __forceinline__ T tile_shfl_up(T v, int o) {
  return __shfl_up_sync(tile_mask(), v, o, kTile);
}
template <typename T>
__device__ __forceinline__ T tile_min(T v) {
#pragma unroll
  for (int o = kTile / 2; o > 0; o >>= 1) {
    T w = tile_shfl_xor(v, o);
    v = w < v ? w : v;
  }
  return v;
}
template <typename T>
__device__ __forceinline__ T tile_max(T v) {
#pragma unroll
  for (int o = kTile / 2; o > 0; o >>= 1) {
    T w = tile_shfl_xor(v, o);
    v = w > v ? w : v;
  }
  return v;
}
template <typename T>
__device__ __forceinline__ T tile_sum(T v) {  // integers only (exact)
#pragma unroll
  for (int o = kTile / 2; o > 0; o >>= 1) v += tile_shfl_xor(v, o);
  return v;
}
__device__ __forceinline__ int64_t tile_min_i64(int64_t v) {
  const bool none = v == kInf;
  const bool fits = none || (v >= INT32_MIN && v < INT32_MAX);
  if (tile_all(fits)) {
    const int m = __reduce_min_sync(tile_mask(), none ? INT32_MAX : static_cast<int>(v));
    return m == INT32_MAX ? kInf : static_cast<int64_t>(m);
  }
  return tile_min(v);
}
__device__ __forceinline__ int64_t tile_sum_small(int64_t v) {
  const uint32_t lo = static_cast<uint32_t>(v) & 0xffffffu;
  const uint32_t hi = static_cast<uint32_t>(static_cast<uint64_t>(v) >> 24);
  return (static_cast<int64_t>(__reduce_add_sync(tile_mask(), hi)) << 24) +
         static_cast<int64_t>(__reduce_add_sync(tile_mask(), lo));
}
__device__ __forceinline__ uint32_t tile_add_u32(uint32_t v) {
  return __reduce_add_sync(tile_mask(), v);
}
__device__ __forceinline__ int tile_min_i32(int v) { return __reduce_min_sync(tile_mask(), v); }
__device__ __forceinline__ double tile_sum_ru(double v) {
#pragma unroll
  for (int o = kTile / 2; o > 0; o >>= 1) v = __dadd_ru(v, tile_shfl_xor(v, o));
  return v;
}
__device__ __forceinline__ uint64_t tile_xor_u64(uint64_t v) {
  const uint32_t lo = __reduce_xor_sync(tile_mask(), static_cast<uint32_t>(v));
  const uint32_t hi = __reduce_xor_sync(tile_mask(), static_cast<uint32_t>(v >> 32));
  return (static_cast<uint64_t>(hi) << 32) | lo;
}

// ---------------------------------------------------------- device layouts

// Immutable per-instance parameters (from fb_instance).
struct DevInst {
  double sa, sb, sc;  // scheduler cost model
  double ta, tb, tc;  // truth cost model
  double noise_amp;
  uint64_t noise_seed;
  int64_t token_budget;
  int64_t g_ttft, g_tpot;  // global SLOs (PAB)
  int64_t horizon;
  int64_t trace_off;  // first trace row
  int64_t rec_off;    // first row of this instance's state/record/vlist region
  int64_t n_req;
  int64_t log_step_off, log_entry_off, log_reject_off;
  int64_t tpot_uniform;  // every row's tpot_slo when they are all equal, else -1
  int32_t policy, max_chunk, max_active;
  int32_t wide_ok;  // may escalate to the wide engine: n_req < 2^22, arrival + ttft < 2^41
};

// Mutable per-instance step-machine state (Node's scalars, engine.h:156-175).
struct DevState {
  int64_t step_end;     // valid when busy
  int64_t arr;          // next trace row to enqueue (run_node's `arr`)
  int64_t pulled;       // rows [pulled, arr) are pending (Node::pending_)
  int64_t n_active;     // vlist [0, n_active) = active_, activation order
  int64_t n_live;       // vlist [n_active, n_live) = waiting_, admission order
  int64_t seq_counter;  // engine.h:174
  int64_t t_last;
  uint64_t step_counter;  // engine.h:172 (== steps started)
  uint64_t digest;
  int64_t n_rejected;
  int64_t sum_visible, sum_entries, sum_new;
  int32_t busy, done, status, log_steps;
  int32_t log_entries, log_rejects, log_trunc, incomplete;
  int32_t escalated;      // handed to the CTA-wide engine (fb_wide.cuh)
  int32_t pending_begin;  // a begin_step at t_last is owed by the wide engine
  uint32_t paths;         // engine paths used: 1 register, 2 warp-memory, 4 CTA-wide
  int32_t pad2;
};
constexpr uint32_t kPathRegister = 1u, kPathMemory = 2u, kPathWide = 4u, kPathRepeatRegister = 8u,
                   kPathRepeatMemory = 16u;

// Per-request mutable state, structure of arrays indexed by rec_off + row.
struct DevReq {
  int32_t* prefilled;  // RequestProgress::prefilled_tokens
  int32_t* nidx;       // RequestProgress::next_output_idx (== tokens emitted)
  int32_t* seq;        // RequestState::seq
  uint32_t* flags;     // FB_REC_* plus kTpotViolated
  int64_t* first;      // time of token 0 (-1 none)
  double* maxtp;       // running max_tpot_ms
  double* maxtp_alt;   // running max_tpot_alt_ms
};
constexpr uint32_t kTpotViolated = 0x80000000u;

// Trace rows, structure of arrays.
struct DevRows {
  const int64_t* arrival;
  const int32_t* prompt;
  const int32_t* output;
  const int64_t* ttft;
  const int64_t* tpot;
};

// Optional logs.
struct DevLogs {
  fb_step_log* steps;
  fb_plan_entry* entries;
  fb_reject_log* rejects;
  int32_t step_cap, entry_cap, reject_cap, on;
};

// Per-warp scratch, one slot per visible task (view position p) or per
// sorted position k.  Lives in shared memory when A <= kScratchSmem, else in
// the instance's global scratch region (generic pointers either way).
struct Scratch {
  int64_t* slack;   // [p] slack (us)
  uint64_t* khi;    // [p] (group << 62) | (slack + 2^61)
  int64_t* seq;     // [p] arrival_seq
  int64_t* ctx;     // [p] context
  int32_t* nw;      // [p] new tokens available | phase << 31
  int32_t* req;     // [p] request row
  int32_t* order;   // [k] view position at sorted rank k
  int32_t* take;    // [k] admitted tokens (0 = not admitted); later [p] new pos
  double* tcost;    // [k] b*new + c*ctx (or PAB term [p])
  double* ccost;    // [k] c*ctx
};
// 64 bytes carved per slot (Scratch) + 16 so that every instance's region
// (rec_off * kScratchBytesPerSlot) is 16-byte aligned and holds the wide
// engine's 52 bytes per slot plus its 16-byte view records.
constexpr int kScratchBytesPerSlot = 80;
static_assert(kScratchBytesPerSlot >= 8 + 8 + 8 + 8 + 4 + 4 + 4 + 4 + 8 + 8, "Scratch slot");

__device__ __forceinline__ Scratch carve_scratch(unsigned char* base, int cap) {
  Scratch s;
  unsigned char* p = base;
  s.slack = reinterpret_cast<int64_t*>(p); p += 8 * static_cast<size_t>(cap);
  s.khi = reinterpret_cast<uint64_t*>(p); p += 8 * static_cast<size_t>(cap);
  s.seq = reinterpret_cast<int64_t*>(p); p += 8 * static_cast<size_t>(cap);
  s.ctx = reinterpret_cast<int64_t*>(p); p += 8 * static_cast<size_t>(cap);
  s.tcost = reinterpret_cast<double*>(p); p += 8 * static_cast<size_t>(cap);
  s.ccost = reinterpret_cast<double*>(p); p += 8 * static_cast<size_t>(cap);
  s.nw = reinterpret_cast<int32_t*>(p); p += 4 * static_cast<size_t>(cap);
  s.req = reinterpret_cast<int32_t*>(p); p += 4 * static_cast<size_t>(cap);
  s.order = reinterpret_cast<int32_t*>(p); p += 4 * static_cast<size_t>(cap);
  s.take = reinterpret_cast<int32_t*>(p);
  return s;
}

constexpr uint32_t kDecodeBit = 0x80000000u;

}  // namespace fbgpu
