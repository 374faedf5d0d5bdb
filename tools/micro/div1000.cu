// Exhaustive / sampled check of the FMA-corrected division by 1000 used by
// us_to_ms against the IEEE division __ddiv_rn (dev tool):
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -fmad=false tools/micro/div1000.cu -o /tmp/div1000 && /tmp/div1000
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ double div1000(double x) {
  const double q0 = __dmul_rn(x, 0.001);
  const double r = __fma_rn(-q0, 1000.0, x);
  return __fma_rn(r, 0.001, q0);
}

__device__ unsigned long long bad = 0, first_bad = 0;

__global__ void dense(int64_t lo, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double x = (double)(lo + i);
    const double a = div1000(x), b = __ddiv_rn(x, 1000.0);
    if (__double_as_longlong(a) != __double_as_longlong(b)) {
      if (atomicAdd(&bad, 1ull) == 0) first_bad = (unsigned long long)(lo + i);
    }
  }
}

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// random integers of every magnitude up to 2^53, both signs
__global__ void sampled(uint64_t seed, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t z = mix(seed ^ (uint64_t)i);
    const int sh = (int)(z & 63) % 54;
    int64_t v = (int64_t)((z >> 8) & ((1ull << 53) - 1)) >> (53 - sh);
    if (z & 128) v = -v;
    const double x = (double)v;
    const double a = div1000(x), b = __ddiv_rn(x, 1000.0);
    if (__double_as_longlong(a) != __double_as_longlong(b)) {
      if (atomicAdd(&bad, 1ull) == 0) first_bad = (unsigned long long)v;
    }
  }
}

int main() {
  const int64_t span = int64_t(1) << 33;  // [-2^32, 2^32)
  dense<<<148 * 16, 256>>>(-(int64_t(1) << 32), span);
  // top of the exact range and around powers of two
  for (int e = 34; e <= 53; ++e) {
    dense<<<148 * 16, 256>>>((int64_t(1) << e) - (int64_t(1) << 28), int64_t(1) << 29);
    dense<<<148 * 16, 256>>>(-(int64_t(1) << e) - (int64_t(1) << 28), int64_t(1) << 29);
  }
  sampled<<<148 * 16, 256>>>(12345, int64_t(1) << 34);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long nb = 0, fb = 0;
  cudaMemcpyFromSymbol(&nb, bad, sizeof(nb));
  cudaMemcpyFromSymbol(&fb, first_bad, sizeof(fb));
  const double checked = (double)span + 40.0 * (1 << 29) + (double)(int64_t(1) << 34);
  printf("div1000: %s, %.3g values checked, mismatches %llu (first %lld)\n",
         cudaGetErrorString(e), checked, nb, (long long)fb);
  return nb != 0;
}
