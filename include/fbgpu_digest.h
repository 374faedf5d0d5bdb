/*
 * fbgpu_digest.h -- rolling digest of batch decisions, shared by the device
 * engine, the C oracle and the reference shim so that whole runs can be
 * compared bit-for-bit with one 64-bit word per instance.
 *
 * Per begin_step (engine.cpp:153-202) the digest absorbs the step time, the
 * plan entries in admission order (request row, new tokens), the predicted
 * and the ground-truth step times (exact fp64 bit patterns).  Per PAB reject
 * (engine.cpp:134-142) it absorbs the time, the request row and the budget.
 *
 * The entry part is a position-tagged XOR so it can be reduced in any order
 * (one redux.sync per 32-bit half on the device) while staying
 * order-sensitive through the admission position k.
 */
#ifndef FBGPU_DIGEST_H_
#define FBGPU_DIGEST_H_

#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define FB_HD __host__ __device__ __forceinline__
#else
#define FB_HD static inline
#endif

FB_HD uint64_t fb_mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xbf58476d1ce4e5b9ULL;
  z ^= z >> 27;
  z *= 0x94d049bb133111ebULL;
  z ^= z >> 31;
  return z;
}

FB_HD uint64_t fb_rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

/* Hash of the k-th plan entry (k = admission position): a multiply on the
 * (position, request) word -- a bijection -- plus the tokens, one xorshift. */
FB_HD uint64_t fb_digest_entry(uint32_t k, uint32_t req, uint32_t new_tokens) {
  uint64_t z = (((uint64_t)k << 32) | (uint64_t)req) * 0x9e3779b97f4a7c15ULL;
  z ^= (uint64_t)new_tokens * 0xc2b2ae3d27d4eb4fULL;
  return z ^ (z >> 29);
}

FB_HD uint64_t fb_digest_bits(double x) {
  uint64_t u;
#if defined(__CUDA_ARCH__)
  u = (uint64_t)__double_as_longlong(x);
#else
  memcpy(&u, &x, sizeof(u));
#endif
  return u;
}

/* entry_sum = XOR over k of fb_digest_entry(k, req_k, new_k).  One chained
 * step per begin_step over the step's fields (time, entry sum, entry count,
 * predicted and ground-truth step-time bit patterns): the fields are folded
 * into the running state, then one odd multiply and one xorshift -- both
 * bijections, so the new state changes whenever the folded word does.  (The
 * per-step cost matters: the device engine's repeated-plan loop runs ~190
 * warp instructions per step, and the round-1 splitmix chain took ~35.) */
FB_HD uint64_t fb_digest_step(uint64_t h, int64_t t_us, uint32_t n_entries,
                              uint64_t entry_sum, double predicted_ms,
                              double actual_ms) {
  uint64_t x = h ^ (uint64_t)t_us ^ entry_sum ^ ((uint64_t)n_entries << 44) ^
               fb_rotl64(fb_digest_bits(predicted_ms), 21) ^ fb_digest_bits(actual_ms);
  x *= 0x9e3779b97f4a7c15ULL;
  return x ^ (x >> 31);
}

FB_HD uint64_t fb_digest_reject(uint64_t h, int64_t t_us, uint32_t req,
                                int64_t pab_tokens) {
  h = fb_mix64(h ^ 0x52454a4543540000ULL);
  h = fb_mix64(h ^ (uint64_t)t_us);
  h = fb_mix64(h ^ (uint64_t)req);
  h = fb_mix64(h ^ (uint64_t)pab_tokens);
  return h;
}

#define FB_DIGEST_INIT 0x6662677075303031ULL

#endif /* FBGPU_DIGEST_H_ */
