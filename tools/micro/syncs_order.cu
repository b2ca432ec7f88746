// Does an mbarrier test/try_wait issued after tcgen05.commit stall until the
// committed MMAs complete? One CTA, one issuing thread.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2508_17137_b200/csrc/tc_sm100.cuh"
using namespace moeb::tc;
__device__ __forceinline__ uint32_t test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
               "selp.b32 %0, 1, 0, p;\n}\n" : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return done;
}
__global__ void k(long long* out, int mode) {
  __shared__ __align__(1024) unsigned char sm[32768];
  __shared__ uint64_t bars[2];
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc<128>(&slot);
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    mbar_arrive(&bars[1]);  // bars[1] phase 0 complete
    const uint64_t da = umma_desc_sw128(smem_u32(sm)), db = umma_desc_sw128(smem_u32(sm + 16384));
    const uint32_t idesc = umma_idesc_f16(128, 64, 0);
    long long acc = 0, acc2 = 0;
    for (int it = 0; it < 64; ++it) {
      for (int k = 0; k < 4; ++k) mma_f16_ss(tmem, da + 2 * k, db + 2 * k, idesc, k > 0);
      if (mode >= 1) mma_commit(&bars[0]);
      const long long t0 = clock64();
      uint32_t d = test_wait(&bars[1], 0);
      const long long t1 = clock64();
      acc += t1 - t0 + (d ? 0 : 1000000);
      if (mode >= 1) mbar_wait(&bars[0], it & 1);
      const long long t2 = clock64();
      acc2 += t2 - t1;
    }
    out[2 * mode] = acc / 64;
    out[2 * mode + 1] = acc2 / 64;
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<128>(tmem);
}
int main() {
  long long* d;
  cudaMalloc(&d, 64);
  for (int mode = 0; mode < 2; ++mode) k<<<1, 128>>>(d, mode);
  long long h[4];
  cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  printf("test_wait on a completed barrier after 4 MMAs: no commit %lld clk; after commit %lld clk (then commit wait %lld)\n",
         h[0], h[2], h[3]);
  return 0;
}
