// Micro-benchmark of the wide engine's window sort (dev tool, not product):
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2510_14392_b200/csrc
//        -I include tools/micro/sortbench.cu -o build/sortbench
#include <cstdio>
#include <vector>
#include <random>
#include <algorithm>
#include "fb_engine_dev.cuh"
#include "fb_wide.cuh"
using namespace fbgpu;

template <int ALG>
__global__ void __launch_bounds__(kWideThreads, 1)
k_sort(const uint64_t* in, int K, uint64_t* out, long long* clk, int reps) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WideSmem& sm = *reinterpret_cast<WideSmem*>(smem_raw);
  long long tot = 0;
  for (int r = 0; r < reps; ++r) {
    for (int k = threadIdx.x; k < K; k += kWideThreads) {
      sm.wkey[k] = in[blockIdx.x * (size_t)K + k];
      sm.wpos[k] = k;
    }
    __syncthreads();
    long long t0 = clock64();
    wide_bitonic_sort(K, sm);
    long long t1 = clock64();
    tot += t1 - t0;
    __syncthreads();
  }
  for (int k = threadIdx.x; k < K; k += kWideThreads) out[blockIdx.x * (size_t)K + k] = sm.wkey[k];
  if (threadIdx.x == 0) clk[blockIdx.x] = tot / reps;
}

int main(int argc, char** argv) {
  int K = argc > 1 ? atoi(argv[1]) : 1040;
  int G = argc > 2 ? atoi(argv[2]) : 64;
  std::mt19937_64 rng(1);
  std::vector<uint64_t> h((size_t)G * K);
  for (auto& x : h) x = rng() >> 2;
  uint64_t *din, *dout; long long* dclk;
  cudaMalloc(&din, h.size() * 8); cudaMalloc(&dout, h.size() * 8); cudaMalloc(&dclk, G * 8);
  cudaMemcpy(din, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  size_t smem = sizeof(WideSmem);
  int alg = argc > 3 ? atoi(argv[3]) : 0;
  cudaFuncSetAttribute(k_sort<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_sort<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (alg == 0) k_sort<0><<<G, kWideThreads, smem>>>(din, K, dout, dclk, 20);
  else k_sort<1><<<G, kWideThreads, smem>>>(din, K, dout, dclk, 20);
  cudaError_t e = cudaDeviceSynchronize();
  if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<long long> c(G);
  cudaMemcpy(c.data(), dclk, G * 8, cudaMemcpyDeviceToHost);
  std::vector<uint64_t> o(h.size());
  cudaMemcpy(o.data(), dout, o.size() * 8, cudaMemcpyDeviceToHost);
  bool ok = true;
  for (int b = 0; b < G; ++b) {
    std::vector<uint64_t> s(h.begin() + (size_t)b * K, h.begin() + (size_t)(b + 1) * K);
    std::sort(s.begin(), s.end());
    ok &= std::equal(s.begin(), s.end(), o.begin() + (size_t)b * K);
  }
  printf("alg=%d K=%d G=%d sorted=%d cycles=%lld (%.2f us at 1.965 GHz)\n", alg, K, G, ok, c[0], c[0] / 1965.0);
  return 0;
}
