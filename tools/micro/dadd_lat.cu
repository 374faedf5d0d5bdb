// Dependent-chain latency of fp64 add / mul / fma and of a shared-memory-fed
// subtraction chain (the wide engine's exact budget fold), one thread (dev tool):
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -fmad=false tools/micro/dadd_lat.cu -o /tmp/dl
#include <cstdio>
__global__ void k(double* out, long long* cyc, int n, double a) {
  __shared__ double sm[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = 1e-3 * (i + 1);
  __syncthreads();
  if (threadIdx.x) return;
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, 1e-9);
  long long t1 = clock64();
  double y = a;
  for (int i = 0; i < n; ++i) y = __dmul_rn(y, 1.0000001);
  long long t2 = clock64();
  double z = a;
  for (int i = 0; i < n; i += 4) {
    const int j = i & 2047;
    const double a0 = sm[j], a1 = sm[(j + 1) & 2047], a2 = sm[(j + 2) & 2047], a3 = sm[(j + 3) & 2047];
    z = __dsub_rn(__dsub_rn(__dsub_rn(__dsub_rn(z, a0), a1), a2), a3);
  }
  long long t3 = clock64();
  out[0] = x + y + z;
  cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 24);
  const int n = 1 << 20;
  k<<<1, 256>>>(o, c, n, 1.0);
  k<<<1, 256>>>(o, c, n, 1.0);
  long long h[3]; cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
  printf("cycles per dependent op: dadd %.2f dmul %.2f smem-fed dsub chain %.2f\n",
         (double)h[0] / n, (double)h[1] / n, (double)h[2] / n);
}
