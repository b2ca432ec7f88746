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
//
// k_window_attention_fb (default, below) is a persistent one-pass tcgen05
// kernel: S = Q K^T and O += P V on the tensor cores with S, P and O in
// tensor memory, a lazily advanced running max, two CTAs per SM (one
// 128-query tile each). k_window_attention_fa (MOEB_ATTN=fa) is the
// two-pass warp-specialised kernel it replaced, k_window_attention_tc
// (MOEB_ATTN=tc1) the whole-window single-CTA kernel (S for all 512 keys in
// the 512 TMEM columns, an exact two-pass softmax, P through shared memory),
// and the mma.sync kernel above (MOEB_ATTN=mma) the comparison baseline.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cuda.h>

#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "tc_sm100.cuh"

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

// ---------------------------------------------------------------------------
// tcgen05 attention (one CTA = window x head x 128-query block, 8 warps: warp
// w reads TMEM lane quarter w % 4 and the column half w / 4 of every 64-key
// block; row max / row sum are combined through shared memory). CTAs of the
// same (window, head) are adjacent in the 1-D grid so K/V stay in L2.
// ---------------------------------------------------------------------------
constexpr int TQ = 128;        // queries per CTA = TMEM lanes
constexpr int TKMAX = 512;     // keys per window
constexpr int kTcThreads = 256;

// 128-byte swizzle of one 16-byte chunk (K-major rows of 64 16-bit elements)
__device__ __forceinline__ uint32_t sw128(int row, int chunk) {
  return (uint32_t)(row * 128 + ((chunk ^ (row & 7)) << 4));
}

__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// [rows][64] 16-bit rows from global (row stride ld elements) into a SW128
// tile; rows >= n zero-filled
__device__ __forceinline__ void load_sw128_async(unsigned char* tile, const uint16_t* src, int ld,
                                                 int rows, int n) {
  for (int i = threadIdx.x; i < rows * 8; i += kTcThreads) {
    const int row = i >> 3, ch = i & 7;
    const bool v = row < n;
    cp_async16(smem_u32(tile + sw128(row, ch)), src + (int64_t)(v ? row : 0) * ld + ch * 8, v);
  }
}

template <bool FP16>
__global__ void __launch_bounds__(kTcThreads, 1) k_window_attention_tc(
    const uint16_t* __restrict__ qkv, uint16_t* __restrict__ out,
    const int64_t* __restrict__ win_start, const int32_t* __restrict__ win_len, int nqb) {
  using namespace moeb::tc;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sQ = smem_raw;                 // [128][64]  16 KB
  unsigned char* sK = sQ + TQ * 128;            // [512][64]  64 KB, later P (4 x [128][64])
  unsigned char* sV = sK + TKMAX * 128;         // [512][64]  64 KB (MN-major B of P V)
  float* red = reinterpret_cast<float*>(sV + TKMAX * 128);  // [2][128] row max / sum halves
  uint64_t* bar = reinterpret_cast<uint64_t*>(red + 2 * TQ);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 1);

  const int qb = blockIdx.x % nqb;
  const int head = (blockIdx.x / nqb) % 8;
  const int w = blockIdx.x / (nqb * 8);
  const int n = win_len[w];
  if (qb * TQ >= n) return;
  const int64_t r0 = win_start[w];
  const int ld = 3 * 512;
  const int nq = min(TQ, n - qb * TQ);
  const int nkp = (n + 63) & ~63;  // keys padded to the 64-key blocks
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int quarter = warp & 3, hh = warp >> 2;

  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  load_sw128_async(sQ, qkv + (r0 + qb * TQ) * ld + head * 64, ld, TQ, nq);
  load_sw128_async(sK, qkv + r0 * ld + 512 + head * 64, ld, nkp, n);
  load_sw128_async(sV, qkv + r0 * ld + 1024 + head * 64, ld, nkp, n);
  cp_async_commit();
  cp_async_wait<0>();
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int ab = FP16 ? 0 : 1;
  uint32_t phase = 0;

  // ---- S = Q K^T into TMEM columns [0, nkp) ----
  if (threadIdx.x == 0) {
    for (int nb = 0; nb < nkp; nb += 256) {
      const int nn = min(256, nkp - nb);
      const uint32_t idesc = umma_idesc_f16(TQ, nn, ab);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        mma_f16_ss(tmem + nb, umma_desc_sw128(smem_u32(sQ) + k * 32),
                   umma_desc_sw128(smem_u32(sK) + nb * 128 + k * 32), idesc, k > 0);
    }
    mma_commit(bar);
  }
  mbar_wait(bar, phase);
  phase ^= 1;
  tc_fence_after();

  const int row = quarter * 32 + lane;                      // query row = TMEM lane
  const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16) + hh * 32;
  const float sl2 = 0.125f * 1.4426950408889634f;         // 1/sqrt(64) * log2(e)

  // ---- pass 1: row max over the valid keys (this warp's column halves) ----
  float mx = -INFINITY;
  for (int c = 0; c < nkp; c += 128) {
    uint32_t r0v[32], r1v[32];
    tmem_ld32(trow + c, r0v);
    const bool two = c + 64 < nkp;
    if (two) tmem_ld32(trow + c + 64, r1v);
    tmem_ld_wait();
    const int k0 = c + hh * 32, k1 = c + 64 + hh * 32;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (k0 + j < n) mx = fmaxf(mx, __uint_as_float(r0v[j]));
      if (two && k1 + j < n) mx = fmaxf(mx, __uint_as_float(r1v[j]));
    }
  }
  red[hh * TQ + row] = mx;
  __syncthreads();
  mx = fmaxf(red[row], red[TQ + row]);
  const float ms = mx * sl2;

  // ---- pass 2 per 256-key half: P = exp2(S*sl2 - ms) -> smem, O += P V ----
  float sum = 0.f;
  unsigned char* sP = sK;
  for (int h0 = 0; h0 < nkp; h0 += 256) {
    const int hn = min(256, nkp - h0);
    for (int c = 0; c < hn; c += 64) {
      uint32_t rv[32];
      tmem_ld32(trow + h0 + c, rv);
      tmem_ld_wait();
      unsigned char* blk = sP + (c >> 6) * (TQ * 128);
      const int kb = h0 + c + hh * 32;
#pragma unroll
      for (int q = 0; q < 4; ++q) {  // 4 chunks of 8 keys
        uint32_t pk[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = q * 8 + u * 2;
          const float x0 = kb + j < n ? exp2f(__uint_as_float(rv[j]) * sl2 - ms) : 0.f;
          const float x1 = kb + j + 1 < n ? exp2f(__uint_as_float(rv[j + 1]) * sl2 - ms) : 0.f;
          sum += x0 + x1;
          pk[u] = pack2<FP16>(x0, x1);
        }
        *reinterpret_cast<uint4*>(blk + sw128(row, hh * 4 + q)) =
            make_uint4(pk[0], pk[1], pk[2], pk[3]);
      }
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) {
      tc_fence_after();
      // O (TMEM columns [0, 64), free once S's first half was read) += P V
      const uint32_t idesc = umma_idesc_f16(TQ, 64, ab) | (1u << 16);  // B MN-major
      for (int c = 0; c < hn; c += 64) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          mma_f16_ss(tmem, umma_desc_sw128(smem_u32(sP) + (c >> 6) * (TQ * 128) + k * 32),
                     umma_desc_sw128(smem_u32(sV) + (h0 + c + k * 16) * 128), idesc,
                     (h0 | c | k) != 0);
      }
      mma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();
  }

  // ---- O / rowsum -> out (this warp's 32 of the 64 dims) ----
  red[hh * TQ + row] = sum;  // max reads finished at the pass-2 barriers
  __syncthreads();
  sum = red[row] + red[TQ + row];
  {
    uint32_t o0[32];
    tmem_ld32(trow, o0);
    tmem_ld_wait();
    const float inv = 1.f / sum;
    if (row < nq) {
      uint16_t* dst = out + (r0 + qb * TQ + row) * 512 + head * 64 + hh * 32;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t pk[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = q * 8 + u * 2;
          pk[u] = pack2<FP16>(__uint_as_float(o0[j]) * inv, __uint_as_float(o0[j + 1]) * inv);
        }
        reinterpret_cast<uint4*>(dst)[q] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

// ---------------------------------------------------------------------------
// Warp-specialised tcgen05 attention (default): one CTA = (window, head,
// 128-query block), two CTAs per SM (97 KB shared memory, 256 TMEM columns
// each). Keys stream in 64-key chunks through a 3-stage TMA ring;
//   warp 0   TMA producer: Q (2 boxes), then K chunks (pass 1), then K + V
//            chunks (pass 2)
//   warp 1   MMA issuer: S_c = Q K_c^T into one of two 64-column TMEM
//            buffers; in pass 2 also O += P_c V_c (V MN-major from its
//            natural layout) into 64 more columns
//   warps 2-9 softmax: two warps per TMEM lane quarter, 32 keys each; pass 1
//            row max, pass 2 P = exp2(S - max) (16-bit, SW128 shared memory,
//            two buffers) and the row sum; final O / sum
// Exact two-pass softmax (S recomputed: the MMAs are cheap, TMEM holds only
// two S chunks); every hand-off is an mbarrier (TMA complete_tx,
// tcgen05.commit, or 8 softmax-warp arrivals).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float ex2_ftz(float x) {  // one MUFU.EX2
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

constexpr int FA_CK = 64;      // keys per chunk
constexpr int FA_NST = 3;      // ring stages (K 8 KB + V 8 KB each)
constexpr int FA_NS = 2;       // S buffers in tensor memory (64 columns each)
__device__ __forceinline__ uint32_t s_col(int b) { return b == 2 ? 192u : (uint32_t)b * 64u; }
constexpr int FA_THREADS = 320;

struct FaSmem {
  static constexpr int Q = 0;                         // 16 KB
  static constexpr int RING = 16384;                  // FA_NST x 16 KB
  static constexpr int P = RING + FA_NST * 16384;     // 2 x 16 KB
  static constexpr int RED = P + 2 * 16384;           // 4 x 128 floats
  static constexpr int BAR = RED + 4 * 128 * 4;       // 17 mbarriers
  static constexpr int SLOT = BAR + 8 * 24;
  static constexpr int BYTES = SLOT + 16;
};

template <bool FP16>
__global__ void __launch_bounds__(FA_THREADS, 2) k_window_attention_fa(
    const __grid_constant__ CUtensorMap tm, uint16_t* __restrict__ out,
    const int64_t* __restrict__ win_start, const int32_t* __restrict__ win_len, int nqb) {
  using namespace moeb::tc;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sQ = smem_raw + FaSmem::Q;
  unsigned char* ring = smem_raw + FaSmem::RING;
  unsigned char* sP = smem_raw + FaSmem::P;
  float* red = reinterpret_cast<float*>(smem_raw + FaSmem::RED);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + FaSmem::BAR);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;             // [FA_NST]
  uint64_t* kv_empty = kv_full + FA_NST;    // [FA_NST]
  uint64_t* s_full = kv_empty + FA_NST;     // [FA_NS]
  uint64_t* s_empty = s_full + FA_NS;       // [FA_NS]
  uint64_t* p_full = s_empty + FA_NS;       // [2]
  uint64_t* p_empty = p_full + 2;           // [2]
  uint64_t* o_full = p_empty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_raw + FaSmem::SLOT);

  const int qb = blockIdx.x % nqb;
  const int head = (blockIdx.x / nqb) % 8;
  const int w = blockIdx.x / (nqb * 8);
  const int n = win_len[w];
  if (qb * TQ >= n) return;
  const int r0 = (int)win_start[w];
  const int nq = min(TQ, n - qb * TQ);
  const int nch = (n + FA_CK - 1) / FA_CK;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tm);
    mbar_init(q_full, 1);
    for (int i = 0; i < FA_NST; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int b = 0; b < FA_NS; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&s_empty[b], 8);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&p_full[b], 8);
      mbar_init(&p_empty[b], 1);
    }
    mbar_init(o_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // S buffers at +0 / +64 / +192, O at +128

  if (warp == 0) {
    if (lane == 0) {  // ===== TMA producer =====
      mbar_expect_tx(q_full, TQ * 128);
      tma_load_2d(sQ, &tm, q_full, head * 64, r0 + qb * TQ);
      tma_load_2d(sQ + 64 * 128, &tm, q_full, head * 64, r0 + qb * TQ + 64);
      for (int g = 0; g < 2 * nch; ++g) {
        const int c = g < nch ? g : g - nch;
        const bool v = g >= nch;
        const int st = g % FA_NST;
        mbar_wait_sleep(&kv_empty[st], ((g / FA_NST) & 1) ^ 1);
        unsigned char* stg = ring + st * 16384;
        mbar_expect_tx(&kv_full[st], v ? 16384 : 8192);
        tma_load_2d(stg, &tm, &kv_full[st], 512 + head * 64, r0 + c * FA_CK);
        if (v) tma_load_2d(stg + 8192, &tm, &kv_full[st], 1024 + head * 64, r0 + c * FA_CK);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ===== MMA issuer =====
      const int ab = FP16 ? 0 : 1;
      const uint32_t idesc_s = umma_idesc_f16(TQ, FA_CK, ab);
      const uint32_t idesc_o = umma_idesc_f16(TQ, 64, ab) | (1u << 16);  // V MN-major
      int s_use = 0;
      mbar_wait_sleep(q_full, 0);
      auto issue_s = [&](int g) {
        const int st = g % FA_NST;
        mbar_wait_sleep(&kv_full[st], (g / FA_NST) & 1);
        const int b = s_use % FA_NS;
        mbar_wait_sleep(&s_empty[b], ((s_use / FA_NS) & 1) ^ 1);
        tc_fence_after();
        const uint32_t kb = smem_u32(ring + st * 16384);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          mma_f16_ss(tmem + s_col(b), umma_desc_sw128(smem_u32(sQ) + k * 32),
                     umma_desc_sw128(kb + k * 32), idesc_s, k > 0);
        mma_commit(&s_full[b]);
        if (g < nch) mma_commit(&kv_empty[st]);  // pass 1: K chunk consumed
        ++s_use;
      };
      for (int g = 0; g < nch; ++g) issue_s(g);
      for (int c = 0; c < FA_NS - 1 && c < nch; ++c) issue_s(nch + c);
      for (int c = 0; c < nch; ++c) {
        const int g = nch + c;
        if (c + FA_NS - 1 < nch) issue_s(g + FA_NS - 1);
        mbar_wait_sleep(&p_full[c & 1], (c >> 1) & 1);
        tc_fence_after();
        const uint32_t vb = smem_u32(ring + (g % FA_NST) * 16384 + 8192);
        const uint32_t pb = smem_u32(sP + (c & 1) * 16384);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          mma_f16_ss(tmem + 128, umma_desc_sw128(pb + k * 32), umma_desc_sw128(vb + k * 2048),
                     idesc_o, (c | k) != 0);
        mma_commit(&p_empty[c & 1]);
        mma_commit(&kv_empty[g % FA_NST]);  // pass 2: K + V chunk consumed
      }
      mma_commit(o_full);
    }
  } else {
    // ===== softmax warps 2..9 =====
    const int quarter = warp & 3, half = (warp - 2) >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t tq = tmem + ((uint32_t)(quarter * 32) << 16) + half * 32;
    const float sl2 = 0.125f * 1.4426950408889634f;
    int s_use = 0;
    float mx = -INFINITY;
    for (int c = 0; c < nch; ++c) {  // pass 1: row max
      const int b = s_use % FA_NS;
      mbar_wait(&s_full[b], (s_use / FA_NS) & 1);
      tc_fence_after();
      uint32_t r[32];
      tmem_ld32(tq + s_col(b), r);
      tmem_ld_wait();
      const int k0 = c * FA_CK + half * 32;
      if (k0 + 32 <= n) {  // full chunk: no key mask
#pragma unroll
        for (int j = 0; j < 32; ++j) mx = fmaxf(mx, __uint_as_float(r[j]));
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (k0 + j < n) mx = fmaxf(mx, __uint_as_float(r[j]));
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[b]);
      ++s_use;
    }
    red[half * TQ + row] = mx;
    asm volatile("bar.sync 1, 256;" ::: "memory");
    mx = fmaxf(red[row], red[TQ + row]);
    const float ms = mx * sl2;
    float sum = 0.f;
    for (int c = 0; c < nch; ++c) {  // pass 2: P and row sum
      const int b = s_use % FA_NS;
      mbar_wait(&s_full[b], (s_use / FA_NS) & 1);
      tc_fence_after();
      uint32_t r[32];
      tmem_ld32(tq + s_col(b), r);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[b]);
      ++s_use;
      const int k0 = c * FA_CK + half * 32;
      uint32_t pk[16];
      if (k0 + 32 <= n) {  // full chunk: no key mask
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const float x0 = ex2_ftz(fmaf(__uint_as_float(r[j]), sl2, -ms));
          const float x1 = ex2_ftz(fmaf(__uint_as_float(r[j + 1]), sl2, -ms));
          sum += x0 + x1;
          pk[j >> 1] = pack2<FP16>(x0, x1);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const float x0 = k0 + j < n ? ex2_ftz(fmaf(__uint_as_float(r[j]), sl2, -ms)) : 0.f;
          const float x1 =
              k0 + j + 1 < n ? ex2_ftz(fmaf(__uint_as_float(r[j + 1]), sl2, -ms)) : 0.f;
          sum += x0 + x1;
          pk[j >> 1] = pack2<FP16>(x0, x1);
        }
      }
      const int pb = c & 1;
      if (c >= 2) mbar_wait(&p_empty[pb], ((c >> 1) - 1) & 1);  // PV of chunk c - 2 done
      unsigned char* dst = sP + pb * 16384;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<uint4*>(dst + sw128(row, half * 4 + q)) =
            make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[pb]);
    }
    red[2 * TQ + half * TQ + row] = sum;
    asm volatile("bar.sync 1, 256;" ::: "memory");
    sum = red[2 * TQ + row] + red[3 * TQ + row];
    mbar_wait(o_full, 0);
    tc_fence_after();
    uint32_t o[32];
    tmem_ld32(tq + 128, o);
    tmem_ld_wait();
    const float inv = 1.f / sum;
    if (row < nq) {
      uint16_t* dst = out + ((int64_t)r0 + qb * TQ + row) * 512 + head * 64 + half * 32;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t pk[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = q * 8 + u * 2;
          pk[u] = pack2<FP16>(__uint_as_float(o[j]) * inv, __uint_as_float(o[j + 1]) * inv);
        }
        reinterpret_cast<uint4*>(dst)[q] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<256>(tmem);
}

// ---------------------------------------------------------------------------
// One-pass persistent tcgen05 attention (default). Persistent CTAs loop over
// work items = (window, head, group of NT 128-query tiles); NT = 1 by default
// (two CTAs per SM whose softmax warps run out of phase), NT = 2 shares each
// K / V chunk between two tiles of one CTA (MOEB_ATTN_NT=2). 64 + 128 NT
// threads:
//   warp 0   TMA: the group's Q tiles (double-buffered: the next item's Q
//            lands while this item runs), then 64-key K + V chunks through
//            a 4-stage ring that runs ahead across items
//   warp 1   MMA: S_t = Q_t K_c^T two chunks ahead of the softmax (three
//            64-column TMEM buffers per tile), O_t += P_t V_c behind it with
//            P read from tensor memory (A operand in TMEM, V MN-major from
//            its natural layout); the S buffer is released by the commit
//            after its P V
//   4 warps per tile  softmax, thread = query row = TMEM lane, all 64 keys
//            of a chunk per thread, the next chunk's S loaded while this
//            chunk's exponentials run: online softmax with a lazily advanced
//            running max (the max only moves, and O in TMEM is only
//            rescaled, when a chunk's max exceeds it by more than 2^8 -- P
//            <= 256 stays exact in 16 bits, O / rowsum is shift-invariant);
//            P = exp2(S - m) 16-bit written over the chunk's S columns
//            (tcgen05.st); O / rowsum on the way out
// Every role is a whole warp (warp-uniform control flow, one elected lane
// issues TMA / MMA / commits); no runtime integer division or MUFU
// reciprocal outside the exponentials (their XU queue is the busiest pipe).
// TMEM: tile t has S buffers at 256t + {0, 64, 128} and O at 256t + 192.
// ---------------------------------------------------------------------------
constexpr int FB_CK = 64;
constexpr int FB_NST = 4;
constexpr int FB_NS = 3;
#ifndef FB_NT_DEFAULT
#define FB_NT_DEFAULT 1
#endif
constexpr float FB_SLACK = 8.f;  // log2 headroom of the lazily advanced max
#ifndef FB_EMU
#define FB_EMU 0
#endif
// 2^x for a pair on the FMA pipe (x <= 2^8; clamped at -126: the exponent
// field cannot wrap): the integer part by the 1.5 * 2^23 rounding trick, 2^f
// on [-1/2, 1/2] by a degree-4 polynomial (relative error 2.7e-6, below the
// 16-bit P rounding), the exponent added into the bits. Can take part of
// the softmax's exponentials off the 16-per-clock MUFU (FB_EMU pairs of 8).
__device__ __forceinline__ float2 exp2_fma2(float2 x) {
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 big = make_float2(12582912.f, 12582912.f);
  const float2 t = __fadd2_rn(x, big);
  const float2 f = __fadd2_rn(x, __fadd2_rn(big, make_float2(-t.x, -t.y)));
  float2 p = __ffma2_rn(f, make_float2(0.009570102207362652f, 0.009570102207362652f),
                        make_float2(0.05591786280274391f, 0.05591786280274391f));
  p = __ffma2_rn(p, f, make_float2(0.240247443318367f, 0.240247443318367f));
  p = __ffma2_rn(p, f, make_float2(0.6931217908859253f, 0.6931217908859253f));
  p = __ffma2_rn(p, f, make_float2(0.9999992847442627f, 0.9999992847442627f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

// NT query tiles per CTA: NT = 2 (one CTA per SM, 512 TMEM columns) or
// NT = 1 (two CTAs per SM, 256 columns each)
template <int NT>
struct FbSmem {
  static constexpr int Q = 0;                        // [2 bufs][NT tiles] 16 KB
  static constexpr int RING = 2 * NT * 16384;        // FB_NST x (K 8 KB + V 8 KB)
  static constexpr int BAR = RING + FB_NST * 16384;
  static constexpr int NBAR = 2 * FB_NST + 2 * 4 + 2 * 2 * FB_NS + 2 * 2 * 2 + 2 * 2;
  static constexpr int SLOT = BAR + NBAR * 8;
  static constexpr int BYTES = SLOT + 16;
  static constexpr int THREADS = 64 + 128 * NT;
};

#ifdef FB_TRACE
__device__ unsigned long long g_fbtrace[16384];
// per-role slices of 4096 events, no atomics (a store does not stall the role)
#define FBT(code, c)                                                                   \
  do {                                                                                 \
    if (blockIdx.x == 0 && it < (int)gridDim.x * 4 && fbt_i < 4096)                    \
      g_fbtrace[fbt_base + fbt_i++] = ((unsigned long long)(code) << 56) |             \
          ((unsigned long long)((c) & 0xff) << 48) | (clock64() & 0xffffffffffffull);   \
  } while (0)
#else
#define FBT(code, c) do {} while (0)
#endif

// 1/x for x in [1, 2^127) on the FMA pipe (bit-trick seed, three Newton
// steps: relative error ~1e-7): a MUFU.RCP would queue behind the softmax's
// EX2 stream
__device__ __forceinline__ float rcp_fma(float x) {
  float y = __int_as_float(0x7EF311C3 - __float_as_int(x));
  y = y * fmaf(-x, y, 2.f);
  y = y * fmaf(-x, y, 2.f);
  y = y * fmaf(-x, y, 2.f);
  return y;
}

struct FbItem {
  int r0, n, q0, ntile, head;
};

template <bool FP16, int NT>
__global__ void __launch_bounds__(FbSmem<NT>::THREADS, 2 / NT) k_window_attention_fb(
    const __grid_constant__ CUtensorMap tm, uint16_t* __restrict__ out,
    const int64_t* __restrict__ win_start, const int32_t* __restrict__ win_len, int n_items,
    int pshift) {
  using namespace moeb::tc;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // no runtime integer division anywhere in this kernel: it compiles to
  // I2F / MUFU.RCP / F2I, and the MUFU queue is full of the softmax's EX2
  using Smem = FbSmem<NT>;
  const int npair = 1 << pshift;  // groups of NT query tiles per (window, head)
  unsigned char* sQ = smem_raw + Smem::Q;
  unsigned char* ring = smem_raw + Smem::RING;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + Smem::BAR);
  uint64_t* kv_full = bars;                  // [FB_NST]
  uint64_t* kv_empty = kv_full + FB_NST;     // [FB_NST]
  uint64_t* q_full = kv_empty + FB_NST;      // [2 tiles][2 bufs]
  uint64_t* q_empty = q_full + 4;            // [2][2]
  uint64_t* s_full = q_empty + 4;            // [2 tiles][FB_NS]
  uint64_t* s_empty = s_full + 2 * FB_NS;    // [2][FB_NS]
  uint64_t* p_full = s_empty + 2 * FB_NS;    // [2 tiles][2 bufs]
  uint64_t* o_full = p_full + 4;             // [2]
  uint64_t* o_empty = o_full + 2;            // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_raw + Smem::SLOT);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tm);
    for (int i = 0; i < FB_NST; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&o_full[t], 1);
      mbar_init(&o_empty[t], 4);
      for (int b = 0; b < 2; ++b) {
        mbar_init(&q_full[2 * t + b], 1);
        mbar_init(&q_empty[2 * t + b], 1);
        mbar_init(&p_full[2 * t + b], 4);
      }
      for (int b = 0; b < FB_NS; ++b) {
        mbar_init(&s_full[FB_NS * t + b], 1);
        mbar_init(&s_empty[FB_NS * t + b], 1);
      }
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<256 * NT>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // a work item's geometry, identical in every role. Each role is a whole
  // warp; lane i holds the window length / start of local item k0 + i, so
  // the global loads are waited on once per 32 items (an mbarrier wait
  // behind an outstanding load otherwise stalls on it)
  struct GeoCache {
    int k0, n, r0;
  };
  auto fetch = [&](GeoCache& gc, int k) {
    FbItem g{0, 0, 0, 0, 0};
    const int it = blockIdx.x + k * gridDim.x;
    if (it >= n_items) return g;
    const int kb = k & ~31;
    if (kb != gc.k0) {
      gc.k0 = kb;
      const int itl = blockIdx.x + (kb + lane) * gridDim.x;
      if (itl < n_items) {
        const int w = itl >> (pshift + 3);
        gc.n = __ldg(win_len + w);
        gc.r0 = (int)__ldg(win_start + w);
      }
    }
    g.n = __shfl_sync(0xffffffffu, gc.n, k & 31);
    g.r0 = __shfl_sync(0xffffffffu, gc.r0, k & 31);
    const int pair = it & (npair - 1);
    g.head = (it >> pshift) & 7;
    g.q0 = pair * NT * TQ;
    g.ntile = g.q0 >= g.n ? 0 : (NT == 1 || g.q0 + TQ >= g.n ? 1 : 2);
    return g;
  };

  if (warp == 0) {
    {  // ===== TMA producer: the whole warp, one elected lane issues =====
      uint32_t g = 0, qi[2] = {0, 0};
#ifdef FB_TRACE
      int fbt_i = 0;
      const int fbt_base = 3 * 4096;
#endif
      int it = 0;
      auto load_q = [&](const FbItem& w) {
        for (int t = 0; t < w.ntile; ++t) {
          const int qb = qi[t] & 1;
          FBT(12, t);
          mbar_wait_sleep(&q_empty[2 * t + qb], ((qi[t] >> 1) & 1) ^ 1);
          FBT(13, t);
          if (elect_one()) {
            mbar_expect_tx(&q_full[2 * t + qb], TQ * 128);
            unsigned char* dq = sQ + (NT * qb + t) * 16384;
            tma_load_2d(dq, &tm, &q_full[2 * t + qb], w.head * 64, w.r0 + w.q0 + t * TQ);
            tma_load_2d(dq + 8192, &tm, &q_full[2 * t + qb], w.head * 64,
                        w.r0 + w.q0 + t * TQ + 64);
          }
          __syncwarp();
          ++qi[t];
        }
      };
      GeoCache gc{-32, 0, 0};
      bool q_ahead = false;  // the current item's Q was issued during the previous item
      for (int k = 0; (it = blockIdx.x + k * gridDim.x) < n_items; ++k) {
        const FbItem cur = fetch(gc, k);
        if (cur.ntile == 0) continue;
        if (!q_ahead) load_q(cur);
        q_ahead = false;
        const int nch = (cur.n + FB_CK - 1) / FB_CK;
        for (int c = 0; c < nch; ++c, ++g) {
          const int st = g % FB_NST;
          FBT(14, c);
          mbar_wait_sleep(&kv_empty[st], ((g / FB_NST) & 1) ^ 1);
          FBT(15, c);
          if (elect_one()) {
            unsigned char* stg = ring + st * 16384;
            mbar_expect_tx(&kv_full[st], 16384);
            tma_load_2d(stg, &tm, &kv_full[st], 512 + cur.head * 64, cur.r0 + c * FB_CK);
            tma_load_2d(stg + 8192, &tm, &kv_full[st], 1024 + cur.head * 64, cur.r0 + c * FB_CK);
          }
          __syncwarp();
          // the next item's Q (double-buffered) a few chunks before it is needed
          if (c == (nch > 2 ? 2 : nch - 1)) {
            const FbItem nxt = fetch(gc, k + 1);
            if (nxt.ntile > 0) {
              load_q(nxt);
              q_ahead = true;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    {  // ===== MMA issuer: the whole warp, one elected lane issues =====
#ifdef FB_TRACE
      int fbt_i = 0;
      const int fbt_base = 0;
#endif
      const int ab = FP16 ? 0 : 1;
      const uint32_t idesc_s = umma_idesc_f16(TQ, FB_CK, ab);
      const uint32_t idesc_o = umma_idesc_f16(TQ, 64, ab) | (1u << 16);  // V MN-major
      // descriptors advance by (bytes >> 4) in their low bits (no carry:
      // shared addresses < 256 KB)
      const uint64_t dq0 = umma_desc_sw128(smem_u32(sQ));
      const uint64_t dring = umma_desc_sw128(smem_u32(ring));
      uint32_t g = 0, qi[2] = {0, 0}, su[2] = {0, 0}, pu[2] = {0, 0}, oi[2] = {0, 0};
      GeoCache gcache{-32, 0, 0};
      for (int k = 0, it; (it = blockIdx.x + k * gridDim.x) < n_items; ++k) {
        const FbItem cur = fetch(gcache, k);
        if (cur.ntile == 0) continue;
        const int ntile = cur.ntile;
        const int nch = (cur.n + FB_CK - 1) / FB_CK;
        uint64_t dq[2];
        FBT(8, 0);
        for (int t = 0; t < ntile; ++t) {
          const int qb = qi[t] & 1;
#ifdef FB_TRACE
          {
            uint32_t done;
            asm volatile(
                "{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                "selp.b32 %0, 1, 0, p;\n}\n"
                : "=r"(done)
                : "r"(smem_u32(&q_full[2 * t + qb])), "r"((qi[t] >> 1) & 1)
                : "memory");
            FBT(7, done + 2 * t);
          }
#endif
          mbar_wait(&q_full[2 * t + qb], (qi[t] >> 1) & 1);
          FBT(9 + t, 0);
          dq[t] = dq0 + (uint64_t)((NT * qb + t) * (16384 >> 4));
        }
        auto issue_s = [&](int c) {  // S_t = Q_t K_c^T for both tiles
          FBT(1, c);
          const uint32_t gc = g + c;
          const int st = gc % FB_NST;
          mbar_wait(&kv_full[st], (gc / FB_NST) & 1);
          FBT(11, c);
          const uint64_t dk = dring + (uint64_t)(st * (16384 >> 4));
          for (int t = 0; t < ntile; ++t) {
            const int b = su[t] % FB_NS;
            mbar_wait(&s_empty[FB_NS * t + b], ((su[t] / FB_NS) & 1) ^ 1);
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
              for (int k = 0; k < 4; ++k)
                mma_f16_ss(tmem + 256 * t + 64 * b, dq[t] + 2 * k, dk + 2 * k, idesc_s, k > 0);
              mma_commit(&s_full[FB_NS * t + b]);
              if (c == nch - 1) mma_commit(&q_empty[2 * t + (qi[t] & 1)]);
            }
            __syncwarp();
            FBT(2 + t, c);
            ++su[t];
          }
        };
        auto issue_pv = [&](int c) {  // O_t += P_t V_c for both tiles
          FBT(4, c);
          const uint32_t gc = g + c;
          const int st = gc % FB_NST;
          const uint64_t dv = dring + (uint64_t)((st * 16384 + 8192) >> 4);
          for (int t = 0; t < ntile; ++t) {
            const int b = pu[t] & 1;
            const int sb = pu[t] % FB_NS;  // P sits in its S buffer's first 32 columns
            mbar_wait(&p_full[2 * t + b], (pu[t] >> 1) & 1);
            if (c == 0) mbar_wait(&o_empty[t], (oi[t] & 1) ^ 1);
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
              for (int k = 0; k < 4; ++k)
                mma_f16_ts(tmem + 256 * t + 192, tmem + 256 * t + 64 * sb + 8 * k,
                           dv + k * (2048 >> 4), idesc_o, (c | k) != 0);
              mma_commit(&s_empty[FB_NS * t + sb]);  // S/P buffer free once P V ran
            }
            __syncwarp();
            FBT(5 + t, c);
            ++pu[t];
          }
          if (elect_one()) mma_commit(&kv_empty[st]);
          __syncwarp();
        };
        issue_s(0);
        if (nch > 1) issue_s(1);
        for (int c = 0; c < nch; ++c) {
          if (c + 2 < nch) issue_s(c + 2);
          issue_pv(c);
        }
        g += nch;
        if (elect_one())
          for (int t = 0; t < ntile; ++t) mma_commit(&o_full[t]);
        __syncwarp();
        for (int t = 0; t < ntile; ++t) {
          ++oi[t];
          ++qi[t];
        }
      }
    }
  } else {
    // ===== softmax: warps 2-5 tile 0, warps 6-9 tile 1 =====
    // thread = query row = TMEM lane, all 64 keys of a chunk; software
    // pipelined: chunk c+1's S is loaded from TMEM while chunk c's
    // exponentials run, so the load and its barrier wait leave the MUFU
    // phase's critical path
    const int t = (warp - 2) >> 2, quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t tq = tmem + ((uint32_t)(quarter * 32) << 16) + 256 * t;
    const float sl2 = 0.125f * 1.4426950408889634f;  // 1/sqrt(64) * log2(e)
    uint32_t j = 0, oi = 0;
#ifdef FB_TRACE
    int fbt_i = 0;
    const int fbt_base = 4096 * (1 + t);
#endif
    auto load_s = [&](uint32_t jj, uint32_t (&r)[64]) {
      const int sb = jj % FB_NS;
      mbar_wait(&s_full[FB_NS * t + sb], (jj / FB_NS) & 1);
      tc_fence_after();
      tmem_ld64(tq + 64 * sb, r);
    };
    auto release_s = [&](uint32_t jj, uint32_t (&r)[64]) {  // S of chunk jj in registers
      tmem_ld_wait_regs(*reinterpret_cast<uint32_t(*)[32]>(r));
      reg_barrier32(*reinterpret_cast<uint32_t(*)[32]>(r + 32));
    };
    GeoCache gcache{-32, 0, 0};
    for (int k = 0, it; (it = blockIdx.x + k * gridDim.x) < n_items; ++k) {
      const FbItem cur = fetch(gcache, k);
      if (t >= cur.ntile) continue;
      const int n = cur.n;
      const int nch = (n + FB_CK - 1) / FB_CK;
      float m = 0.f, l0 = 0.f, l1 = 0.f, l2 = 0.f, l3 = 0.f;
      uint32_t r[64];
      load_s(j, r);
      release_s(j, r);
      for (int c = 0; c < nch; ++c, ++j) {
        if (lane == 0 && quarter == 2) FBT(18 + 8 * t, c);
        const int kv = n - c * FB_CK;  // valid keys in this chunk
        if (kv < FB_CK) {
#pragma unroll
          for (int i = 0; i < 64; ++i)
            if (i >= kv) r[i] = __float_as_uint(-INFINITY);
        }
        float mm[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float a = __uint_as_float(r[16 * q]);
#pragma unroll
          for (int i = 1; i < 16; ++i) a = fmaxf(a, __uint_as_float(r[16 * q + i]));
          mm[q] = a;
        }
        const float cm = fmaxf(fmaxf(mm[0], mm[1]), fmaxf(mm[2], mm[3])) * sl2;
        float alpha = 1.f;
        if (c == 0) {
          m = cm;
        } else if (cm > m + FB_SLACK) {
          alpha = ex2_ftz(m - cm);
          l0 *= alpha;
          l1 *= alpha;
          l2 *= alpha;
          l3 *= alpha;
          m = cm;
        }
        if (c > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
          // rescale this warp's O rows once the previous chunk's P V landed
          const uint32_t jp = j - 1;
          // (the S buffer's release is committed after that P V; its next
          // release needs P of chunk jp + FB_NS, not produced yet)
          mbar_wait(&s_empty[FB_NS * t + jp % FB_NS], (jp / FB_NS) & 1);
          tc_fence_after();
          uint32_t o[32];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            tmem_ld32(tq + 192 + 32 * h, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st32(tq + 192 + 32 * h, o);
          }
          tmem_st_wait();
        }
        uint32_t pk[32];
        float2 la = make_float2(0.f, 0.f), lb = make_float2(0.f, 0.f);
        const float2 sl22 = make_float2(sl2, sl2), nm2 = make_float2(-m, -m);
#pragma unroll
        for (int u = 0; u < 32; ++u) {  // pairs; the last FB_EMU of 8 on the FMA pipe
          float2 x = __ffma2_rn(make_float2(__uint_as_float(r[2 * u]), __uint_as_float(r[2 * u + 1])),
                                sl22, nm2);
          if ((u & 7) >= 8 - FB_EMU) {
            x = exp2_fma2(x);
          } else {
            x.x = ex2_ftz(x.x);
            x.y = ex2_ftz(x.y);
          }
          if (u & 1)
            lb = __fadd2_rn(lb, x);
          else
            la = __fadd2_rn(la, x);
          pk[u] = pack2<FP16>(x.x, x.y);
        }
        l0 += la.x;
        l1 += la.y;
        l2 += lb.x;
        l3 += lb.y;
        // next chunk's S: its wait and TMEM load overlap the P store below
        if (c + 1 < nch) load_s(j + 1, r);
        if (lane == 0 && quarter == 2) FBT(19 + 8 * t, c);
        const int pb = j & 1;
        if (lane == 0 && quarter == 2) FBT(20 + 8 * t, c);
        // P (16-bit pairs) over the first 32 columns of this chunk's S
        // buffer: the A operand of P V straight from tensor memory
        tmem_st32(tq + 64 * (j % FB_NS), pk);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[2 * t + pb]);
        if (lane == 0 && quarter == 2) FBT(21 + 8 * t, c);
        if (c + 1 < nch) release_s(j + 1, r);
      }
      // ---- O / rowsum -> out ----
      if (lane == 0 && quarter == 2) FBT(22 + 8 * t, 0);
      mbar_wait(&o_full[t], oi & 1);
      if (lane == 0 && quarter == 2) FBT(23 + 8 * t, 0);
      ++oi;
      tc_fence_after();
      uint32_t o0[32], o1[32];
      tmem_ld32(tq + 192, o0);
      tmem_ld32(tq + 224, o1);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_empty[t]);
      const float inv = rcp_fma((l0 + l1) + (l2 + l3));
      if (cur.q0 + t * TQ + row < n) {
        uint4* dst = reinterpret_cast<uint4*>(
            out + ((int64_t)cur.r0 + cur.q0 + t * TQ + row) * 512 + cur.head * 64);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint32_t* o = q < 4 ? o0 + 8 * q : o1 + 8 * (q - 4);
          dst[q] = make_uint4(
              pack2<FP16>(__uint_as_float(o[0]) * inv, __uint_as_float(o[1]) * inv),
              pack2<FP16>(__uint_as_float(o[2]) * inv, __uint_as_float(o[3]) * inv),
              pack2<FP16>(__uint_as_float(o[4]) * inv, __uint_as_float(o[5]) * inv),
              pack2<FP16>(__uint_as_float(o[6]) * inv, __uint_as_float(o[7]) * inv));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<256 * NT>(tmem);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// qkv [rows][1536] 16-bit, 64 x 64 boxes, 128-byte swizzle
int qkv_map(CUtensorMap* m, const void* qkv, int64_t rows, bool fp16) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess || q != cudaDriverEntryPointSuccess)
      return moeb::fail(MOEB_ECUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  cuuint64_t dims[2] = {1536, (cuuint64_t)rows};
  cuuint64_t strides[1] = {1536 * 2};
  cuuint32_t box[2] = {64, 64};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, fp16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                  const_cast<void*>(qkv), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return moeb::fail(MOEB_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return MOEB_OK;
}

}  // namespace

#ifdef FB_TRACE
// debug builds only (-DFB_TRACE, tools/fb_trace_probe.py): CTA 0's event
// timeline of the last k_window_attention_fb launch
extern "C" int moeb_debug_fb_trace(unsigned long long* dst, int n) {
  cudaMemcpyFromSymbol(dst, g_fbtrace, sizeof(unsigned long long) * (size_t)n);
  return n;
}
#endif

extern "C" int moeb_window_attention(const void* qkv, void* out, const int64_t* win_start,
                                     const int32_t* win_len, int n_windows, int max_len,
                                     int64_t rows, int fp16, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(qkv && out && win_start && win_len, "null argument");
  MOEB_REQUIRE(n_windows >= 0 && max_len >= 1 && max_len <= 4096 && rows >= 1,
               "bad window arguments");
  if (n_windows == 0) return MOEB_OK;
  dim3 grid((unsigned)n_windows, 8, (unsigned)((max_len + QB - 1) / QB));
  cudaStream_t s = moeb::as_stream(stream);
  // MOEB_ATTN: unset / "fb" persistent one-pass (default), "fa" two-pass
  // warp-specialised, "tc1" whole-window single CTA, "mma" mma.sync baseline
  const char* env = getenv("MOEB_ATTN");
  const char mode = !env || !strcmp(env, "fb") ? 'p' : !strcmp(env, "fa") ? 'f'
                    : !strcmp(env, "tc1") ? 't' : 'm';
  const int nqb = (max_len + TQ - 1) / TQ;
  if (mode == 'p' && max_len <= TKMAX && rows < (1ll << 31)) {
    CUtensorMap tm;
    if (int rc = qkv_map(&tm, qkv, rows, fp16 != 0)) return rc;
    // MOEB_ATTN_NT: 1 = one query tile per CTA, two CTAs per SM (default); 2 =
    // two tiles sharing each K / V chunk, one CTA per SM
    const char* nte = getenv("MOEB_ATTN_NT");
    const int nt = nte ? (nte[0] == '1' ? 1 : 2) : FB_NT_DEFAULT;
    auto k = nt == 1 ? (fp16 ? k_window_attention_fb<true, 1> : k_window_attention_fb<false, 1>)
                     : (fp16 ? k_window_attention_fb<true, 2> : k_window_attention_fb<false, 2>);
    const int bytes = nt == 1 ? FbSmem<1>::BYTES : FbSmem<2>::BYTES;
    const int threads = nt == 1 ? FbSmem<1>::THREADS : FbSmem<2>::THREADS;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    // groups of nt 128-query tiles per (window, head), a power of two
    const int groups = (nqb + nt - 1) / nt;
    const int pshift = groups > 2 ? 2 : groups > 1 ? 1 : 0;
    const int64_t items = (int64_t)n_windows * 8 << pshift;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t slots = (int64_t)sms * (2 / nt);
    const int grid = (int)(items < slots ? items : slots);
    k<<<grid, threads, bytes, s>>>(tm, static_cast<uint16_t*>(out), win_start, win_len, (int)items,
                                   pshift);
    return moeb::check_launch("k_window_attention_fb");
  }
  if (mode == 'f' && max_len <= TKMAX && rows < (1ll << 31)) {
    CUtensorMap tm;
    if (int rc = qkv_map(&tm, qkv, rows, fp16 != 0)) return rc;
    auto k = fp16 ? k_window_attention_fa<true> : k_window_attention_fa<false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, FaSmem::BYTES);
    k<<<(unsigned)((int64_t)n_windows * 8 * nqb), FA_THREADS, FaSmem::BYTES, s>>>(
        tm, static_cast<uint16_t*>(out), win_start, win_len, nqb);
    return moeb::check_launch("k_window_attention_fa");
  }
  if (mode == 't' && max_len <= TKMAX) {
    const size_t smem = TQ * 128 + 2 * TKMAX * 128 + 2 * TQ * 4 + 64;
    auto k = fp16 ? k_window_attention_tc<true> : k_window_attention_tc<false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<(unsigned)((int64_t)n_windows * 8 * nqb), kTcThreads, smem, s>>>(
        static_cast<const uint16_t*>(qkv), static_cast<uint16_t*>(out), win_start, win_len, nqb);
    return moeb::check_launch("k_window_attention_tc");
  }
  if (fp16)
    k_window_attention<true><<<grid, 256, 0, s>>>(static_cast<const uint16_t*>(qkv),
                                                  static_cast<uint16_t*>(out), win_start, win_len);
  else
    k_window_attention<false><<<grid, 256, 0, s>>>(static_cast<const uint16_t*>(qkv),
                                                   static_cast<uint16_t*>(out), win_start, win_len);
  return moeb::check_launch("k_window_attention");
}
