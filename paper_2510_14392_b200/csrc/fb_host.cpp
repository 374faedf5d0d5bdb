// fb_host.cpp -- host-side pieces of the product library: the thread-local
// error slot and trace generation.  Trace generation stays on the host
// (SURVEY §7 hard part 8): it uses libm log/exp/cos/sqrt, whose device
// counterparts round differently.  Compiled with -ffp-contract=off and no
// -march so the arithmetic matches the reference build bit for bit.
#include <cmath>
#include <cstdint>
#include <string>

#include "../../include/fbgpu.h"

namespace fbgpu {

namespace {
thread_local std::string g_error;
}

int set_error(int code, const std::string& msg) {
  g_error = msg;
  return code;
}

namespace {

// splitmix64 / derive_seed / Rng (rng.h:25-86)
uint64_t splitmix64(uint64_t& s) {
  uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

uint64_t derive_seed(uint64_t base, uint64_t stream) {
  uint64_t s = base ^ (0x9e3779b97f4a7c15ULL * (stream + 1));
  splitmix64(s);
  return splitmix64(s);
}

struct Stream {
  uint64_t state;
  double uniform01() { return static_cast<double>(splitmix64(state) >> 11) * 0x1.0p-53; }
  double exponential(double rate) {
    double u;
    do {
      u = uniform01();
    } while (u <= 0.0);
    return -std::log(u) / rate;
  }
  double gaussian() {  // Box-Muller, one draw per call
    double u1;
    do {
      u1 = uniform01();
    } while (u1 <= 0.0);
    const double u2 = uniform01();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
  }
};

int64_t to_us(double ms) { return static_cast<int64_t>(std::llround(ms * 1000.0)); }
double to_ms(int64_t us) { return static_cast<double>(us) / 1000.0; }

// (mean, p90) -> log-normal (mu, sigma), workload.cpp:231-242
bool lognormal_fit(double mean, double p90, double& mu, double& sigma) {
  constexpr double z90 = 1.2815515655446004;
  if (!(mean > 0.0) || !(p90 > 0.0)) return false;
  const double ratio = std::log(p90 / mean);
  const double disc = z90 * z90 - 2.0 * ratio;
  sigma = disc >= 0.0 ? z90 - std::sqrt(disc) : z90;
  if (sigma < 0.0) sigma = 0.0;
  mu = std::log(mean) - 0.5 * sigma * sigma;
  return true;
}

}  // namespace
}  // namespace fbgpu

extern "C" {

const char* fb_last_error(void) { return fbgpu::g_error.c_str(); }

int fb_abi_version(void) { return FBGPU_ABI_VERSION; }

// generate_bursty (workload.cpp:244-298): alternating idle/burst phases with
// Poisson arrivals and log-normal lengths, arrivals already in order.
int fb_generate_bursty(const fb_burst_profile* p, int64_t horizon_us, int64_t cap,
                       int64_t* arrival_us, int32_t* prompt_len, int32_t* output_len,
                       int64_t* ttft_us, int64_t* tpot_us, int64_t* n_out) {
  using namespace fbgpu;
  if (!p || !n_out) return set_error(FB_ERR_USAGE, "fb_generate_bursty: null argument");
  if (horizon_us <= 0) return set_error(FB_ERR_VALIDATION, "horizon must be > 0");
  if (p->base_rate < 0.0 || p->burst_rate < p->base_rate)
    return set_error(FB_ERR_VALIDATION, "require burst_rate >= base_rate >= 0");
  if (p->ttft_us <= 0 || p->tpot_us <= 0)
    return set_error(FB_ERR_VALIDATION, "burst profile SLO targets must be positive");
  double pmu, psig, omu, osig;
  if (!lognormal_fit(p->prompt_mean, p->prompt_p90, pmu, psig) ||
      !lognormal_fit(p->output_mean, p->output_p90, omu, osig))
    return set_error(FB_ERR_VALIDATION, "length distribution mean and p90 must be > 0");
  Stream arrivals{derive_seed(p->seed, 1)};
  Stream lengths{derive_seed(p->seed, 2)};
  int64_t n = 0;
  int64_t phase_start = 0;
  bool burst = false;
  while (phase_start < horizon_us) {
    const int64_t len = burst ? p->burst_duration_us : p->idle_duration_us;
    const double rate = burst ? p->burst_rate : p->base_rate;
    const int64_t phase_end = phase_start + len < horizon_us ? phase_start + len : horizon_us;
    if (rate > 0.0) {
      double t_ms = to_ms(phase_start);
      const double end_ms = to_ms(phase_end);
      for (;;) {
        t_ms += arrivals.exponential(rate) * 1000.0;
        if (t_ms >= end_ms) break;
        const double pl = std::exp(pmu + psig * lengths.gaussian());
        const double ol = std::exp(omu + osig * lengths.gaussian());
        const int64_t pli = std::llround(pl) < 1 ? 1 : std::llround(pl);
        const int64_t oli = std::llround(ol) < 1 ? 1 : std::llround(ol);
        if (n < cap) {
          arrival_us[n] = to_us(t_ms);
          prompt_len[n] = static_cast<int32_t>(pli);
          output_len[n] = static_cast<int32_t>(oli);
          ttft_us[n] = p->ttft_us;
          tpot_us[n] = p->tpot_us;
        }
        ++n;
      }
    }
    phase_start = phase_end;
    burst = !burst;
  }
  *n_out = n;
  if (n > cap) return set_error(FB_ERR_CAPACITY, "fb_generate_bursty: buffer too small");
  return FB_OK;
}

// scale_trace, workload.cpp:211-221
int fb_scale_trace(int64_t* arrival_us, int64_t n, double factor) {
  if (!(factor > 0.0)) return fbgpu::set_error(FB_ERR_VALIDATION, "scale factor must be > 0");
  for (int64_t i = 0; i < n; ++i)
    arrival_us[i] = static_cast<int64_t>(std::llround(static_cast<double>(arrival_us[i]) / factor));
  return FB_OK;
}

// offered_rps, workload.cpp:315-321
int fb_offered_rps(const int64_t* arrival_us, int64_t n, double* rps_out) {
  if (!rps_out) return fbgpu::set_error(FB_ERR_USAGE, "null output");
  if (n <= 0) {
    *rps_out = 0.0;
  } else if (arrival_us[n - 1] <= 0) {
    *rps_out = static_cast<double>(n);
  } else {
    *rps_out = static_cast<double>(n) / (fbgpu::to_ms(arrival_us[n - 1]) / 1000.0);
  }
  return FB_OK;
}

}  // extern "C"
