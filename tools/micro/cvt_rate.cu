// Throughput per SM of the softmax's non-FMA instructions: F2FP (fp32 pair ->
// f16x2), MUFU.EX2, and a 64-element mix as in the attention kernel.
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
template <int MODE>
__global__ void k(unsigned* out, int iters) {
  float a[8];
  unsigned acc = 0;
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      if (MODE == 0) {  // F2FP only
        __half2 h = __floats2half2_rn(a[i], a[i + 1]);
        acc ^= *reinterpret_cast<unsigned*>(&h);
        a[i] += 1e-7f;
      } else if (MODE == 1) {  // EX2 + F2FP per pair
        const float x = ex2(a[i]), y = ex2(a[i + 1]);
        __half2 h = __floats2half2_rn(x, y);
        acc ^= *reinterpret_cast<unsigned*>(&h);
        a[i] += 1e-7f;
        a[i + 1] += 1e-7f;
      }
    }
  }
  if (acc == 12345u) out[0] = acc;
}
int main() {
  unsigned* d;
  cudaMalloc(&d, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096, threads = 512;
  for (int mode = 0; mode < 2; ++mode)
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<sms * 2, threads>>>(d, iters);
      else k<1><<<sms * 2, threads>>>(d, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double pairs = 2.0 * sms * threads * iters * 4;
      if (rep)
        printf("%s: %.2f pairs/clk/SM at 1.965 GHz (%.3f ms)\n",
               mode ? "EX2 x2 + F2FP" : "F2FP         ", pairs / (ms * 1e-3) / sms / 1.965e9, ms);
    }
  return 0;
}
