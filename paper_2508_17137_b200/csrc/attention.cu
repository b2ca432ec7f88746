// K5 -- windowed bidirectional multi-head attention for the transformer
// predictor (8 heads x 64, windows of <= 512 trace rows, key padding).
//
// qkv [rows][1536] 16-bit from the QKV GEMM (q | k | v, head h at columns
// 64h..64h+63 of each third); out [rows][512] 16-bit. One CTA = (window,
// head, 128-query block); key blocks of 64 staged in
// XOR-swizzled shared memory, double-buffered with cp.async (zero-filled
// beyond the window); 8 warps x 16 queries = 128 queries per CTA; S = Q K^T
// and O += P V with mma.sync m16n8k16 (fp32 accumulate), online softmax in
// fp32 (exp2 form).
// (Round-1 kernel: the tcgen05/TMEM attention is the DESIGN.md next step.)
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"

namespace {

constexpr int D = 64;
constexpr int QB = 128;  // queries per CTA (8 warps x 16)
constexpr int KB = 64;  // keys per block

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// element offset of (row, col) in a [64][64] 16-bit tile with 16-byte chunks
// XOR-swizzled by row (conflict-free ldmatrix)
__device__ __forceinline__ int swz(int row, int col) {
  return row * 64 + ((((col >> 3) ^ (row & 7)) << 3) | (col & 7));
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1,
                                          uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

template <bool FP16>
__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  if (FP16) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  } else {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
}

template <bool FP16>
__device__ __forceinline__ uint32_t pack2(float x, float y) {
  if (FP16) {
    const __half2 h = __floats2half2_rn(x, y);
    return *reinterpret_cast<const uint32_t*>(&h);
  }
  const __nv_bfloat162 h = __floats2bfloat162_rn(x, y);
  return *reinterpret_cast<const uint32_t*>(&h);
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// asynchronously copy a [64 rows][64] 16-bit block (rows >= n zero-filled)
__device__ __forceinline__ void load_tile_async(uint16_t* tile, const uint16_t* src, int ld,
                                                int n) {
  for (int i = threadIdx.x; i < 64 * 8; i += blockDim.x) {
    const int row = i >> 3, ch = i & 7;
    const bool v = row < n;
    cp_async16(smem_u32(tile + swz(row, ch * 8)), src + (int64_t)(v ? row : 0) * ld + ch * 8, v);
  }
}

// copy a [rows][64] 16-bit block (rows beyond n zero-filled) into a
// swizzled tile
template <int ROWS = 64>
__device__ __forceinline__ void load_tile(uint16_t* tile, const uint16_t* src, int ld, int n) {
  for (int i = threadIdx.x; i < ROWS * 8; i += blockDim.x) {
    const int row = i >> 3, ch = i & 7;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (row < n) v = *reinterpret_cast<const uint4*>(src + (int64_t)row * ld + ch * 8);
    *reinterpret_cast<uint4*>(tile + swz(row, ch * 8)) = v;
  }
}

template <bool FP16>
__global__ void __launch_bounds__(256, 2) k_window_attention(const uint16_t* __restrict__ qkv,
                                                             uint16_t* __restrict__ out,
                                                             const int64_t* __restrict__ win_start,
                                                             const int32_t* __restrict__ win_len) {
  __shared__ __align__(128) uint16_t sQ[QB * D];
  __shared__ __align__(128) uint16_t sK[2][KB * D];
  __shared__ __align__(128) uint16_t sV[2][KB * D];
  const int w = blockIdx.x, head = blockIdx.y, qb = blockIdx.z;
  const int n = win_len[w];
  if (qb * QB >= n) return;
  const int64_t r0 = win_start[w];
  const int ld = 3 * 512;
  const uint16_t* Qg = qkv + (r0 + qb * QB) * ld + head * D;
  const uint16_t* Kg = qkv + r0 * ld + 512 + head * D;
  const uint16_t* Vg = qkv + r0 * ld + 1024 + head * D;
  const int nq = min(QB, n - qb * QB);
  load_tile_async(sK[0], Kg, ld, n);
  load_tile_async(sV[0], Vg, ld, n);
  cp_async_commit();
  load_tile<QB>(sQ, Qg, ld, nq);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const float scale_log2 = 0.125f * 1.4426950408889634f;  // 1/sqrt(64) * log2(e)

  float o[8][4];
#pragma unroll
  for (int j = 0; j < 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  uint32_t qa[4][4];  // Q fragments for the 4 k-steps of d = 64
  __syncthreads();
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    const int row = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
    const int col = ks * 16 + (lane >> 4) * 8;
    ldsm_x4(smem_u32(sQ + swz(row, col)), qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3]);
  }

  int buf = 0;
  for (int kb0 = 0; kb0 < n; kb0 += KB, buf ^= 1) {
    const int nk = min(KB, n - kb0);
    if (kb0 + KB < n) {  // prefetch the next key block into the other buffer
      load_tile_async(sK[buf ^ 1], Kg + (int64_t)(kb0 + KB) * ld, ld, n - kb0 - KB);
      load_tile_async(sV[buf ^ 1], Vg + (int64_t)(kb0 + KB) * ld, ld, n - kb0 - KB);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const uint16_t* cK = sK[buf];
    const uint16_t* cV = sV[buf];
    // S = Q K^T : 16 x 64 per warp
    float s[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
#pragma unroll
      for (int jp = 0; jp < 4; ++jp) {  // pairs of 8-key n-tiles
        uint32_t b0, b1, b2, b3;
        const int key = jp * 16 + (lane & 7) + (lane >> 4) * 8;
        const int col = ks * 16 + ((lane >> 3) & 1) * 8;
        ldsm_x4(smem_u32(cK + swz(key, col)), b0, b1, b2, b3);
        mma16816<FP16>(s[2 * jp], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b0, b1);
        mma16816<FP16>(s[2 * jp + 1], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b2, b3);
      }
    }
    // mask padded keys, online softmax (rows g and g + 8 of this warp)
    float mnew[2] = {mrow[0], mrow[1]};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int key = j * 8 + tig * 2 + (u & 1);
        s[j][u] = key < nk ? s[j][u] * scale_log2 : -INFINITY;
        mnew[u >> 1] = fmaxf(mnew[u >> 1], s[j][u]);
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      mnew[h] = fmaxf(mnew[h], __shfl_xor_sync(0xffffffffu, mnew[h], 1));
      mnew[h] = fmaxf(mnew[h], __shfl_xor_sync(0xffffffffu, mnew[h], 2));
    }
    float corr[2], lsum[2] = {0.f, 0.f};
#pragma unroll
    for (int h = 0; h < 2; ++h) corr[h] = exp2f(mrow[h] - mnew[h]);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        s[j][u] = exp2f(s[j][u] - mnew[u >> 1]);
        lsum[u >> 1] += s[j][u];
      }
      o[j][0] *= corr[0];
      o[j][1] *= corr[0];
      o[j][2] *= corr[1];
      o[j][3] *= corr[1];
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      lrow[h] = lrow[h] * corr[h] + lsum[h];
      mrow[h] = mnew[h];
    }
    // O += P V : P from the S accumulators, V via transposed ldmatrix
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {  // 16 keys per k-step
      const uint32_t a0 = pack2<FP16>(s[2 * ks][0], s[2 * ks][1]);
      const uint32_t a1 = pack2<FP16>(s[2 * ks][2], s[2 * ks][3]);
      const uint32_t a2 = pack2<FP16>(s[2 * ks + 1][0], s[2 * ks + 1][1]);
      const uint32_t a3 = pack2<FP16>(s[2 * ks + 1][2], s[2 * ks + 1][3]);
#pragma unroll
      for (int jp = 0; jp < 4; ++jp) {  // pairs of 8-dim n-tiles
        uint32_t b0, b1, b2, b3;
        const int key = ks * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int col = jp * 16 + (lane >> 4) * 8;
        ldsm_x4_t(smem_u32(cV + swz(key, col)), b0, b1, b2, b3);
        mma16816<FP16>(o[2 * jp], a0, a1, a2, a3, b0, b1);
        mma16816<FP16>(o[2 * jp + 1], a0, a1, a2, a3, b2, b3);
      }
    }
    __syncthreads();  // buffer `buf` is refilled two iterations later
  }
  // finalize: row sums across the 4 threads of a row group
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    lrow[h] += __shfl_xor_sync(0xffffffffu, lrow[h], 1);
    lrow[h] += __shfl_xor_sync(0xffffffffu, lrow[h], 2);
  }
  const float inv0 = 1.f / lrow[0], inv1 = 1.f / lrow[1];
  const int q0 = qb * QB + warp * 16 + g;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int col = head * D + j * 8 + tig * 2;
    if (q0 < n)
      *reinterpret_cast<uint32_t*>(out + (r0 + q0) * 512 + col) =
          pack2<FP16>(o[j][0] * inv0, o[j][1] * inv0);
    if (q0 + 8 < n)
      *reinterpret_cast<uint32_t*>(out + (r0 + q0 + 8) * 512 + col) =
          pack2<FP16>(o[j][2] * inv1, o[j][3] * inv1);
  }
}

}  // namespace

extern "C" int moeb_window_attention(const void* qkv, void* out, const int64_t* win_start,
                                     const int32_t* win_len, int n_windows, int max_len, int fp16,
                                     void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(qkv && out && win_start && win_len, "null argument");
  MOEB_REQUIRE(n_windows >= 0 && max_len >= 1 && max_len <= 4096, "bad window arguments");
  if (n_windows == 0) return MOEB_OK;
  dim3 grid((unsigned)n_windows, 8, (unsigned)((max_len + QB - 1) / QB));
  cudaStream_t s = moeb::as_stream(stream);
  if (fp16)
    k_window_attention<true><<<grid, 256, 0, s>>>(static_cast<const uint16_t*>(qkv),
                                                  static_cast<uint16_t*>(out), win_start, win_len);
  else
    k_window_attention<false><<<grid, 256, 0, s>>>(static_cast<const uint16_t*>(qkv),
                                                   static_cast<uint16_t*>(out), win_start, win_len);
  return moeb::check_launch("k_window_attention");
}
