// MUFU.EX2 and FFMA throughput per SM (B200): independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
template <int MODE>
__global__ void k(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = ex2(a[i]) - 1.0f;
      else a[i] = fmaf(a[i], 0.999f, 1e-4f);
    }
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.f) out[0] = s;
}
int main() {
  float* d;
  cudaMalloc(&d, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  for (int mode = 0; mode < 2; ++mode) {
    for (int threads : {256, 512, 1024}) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (mode == 0) k<0><<<sms * 2, threads>>>(d, iters);
        else k<1><<<sms * 2, threads>>>(d, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double ops = 2.0 * sms * threads * iters * 8;
        if (rep) printf("%s threads/CTA %d: %.2f ops/clk/SM (at %d MHz nominal), %.3f ms\n",
                        mode ? "FFMA" : "EX2 ", threads, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000, ms);
      }
    }
  }
  return 0;
}
