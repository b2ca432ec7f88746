// K4 -- tcgen05 GEMM for the transformer predictor (sm_100a).
//
//   C[M x N] = A[M x K] . B[N x K]^T   (both K-major, 16-bit bf16/fp16, fp32
//   accumulation in tensor memory), with a fused epilogue:
//     EPI_F32        C + bias -> fp32
//     EPI_BIAS       C + bias -> 16-bit
//     EPI_BIAS_RELU  relu(C + bias) -> 16-bit
//     EPI_BIAS_GELU  gelu(C + bias) -> 16-bit (erf form, as torch)
//     EPI_RESID_LN   x = resid + C + bias; y = LayerNorm(x) -> fp32 resid
//                    (in place) and a 16-bit copy (post-norm encoder layers;
//                    needs the whole row: BN = N = 512)
// Persistent, warp-specialised: warp 0 = TMA producer (128-byte-swizzled
// tiles, mbarrier ring of STAGES), warp 1 = MMA issuer (one elected thread,
// tcgen05.mma.cta_group::1.kind::f16, M = 128, N <= 256 per instruction),
// warps 2..9 = epilogue (tcgen05.ld 32x32b, one TMEM lane = one output row;
// two warps per lane quarter split the columns).
// Two TMEM accumulators (when BN <= 256) let the epilogue of tile i overlap
// the mainloop of tile i+1.
#include <cuda.h>
#include <cstdlib>
#include <cstring>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"
#include "tc_sm100.cuh"

namespace {

using namespace moeb::tc;

enum : int {
  EPI_F32 = 0,
  EPI_BIAS = 1,
  EPI_BIAS_RELU = 2,
  EPI_BIAS_GELU = 3,
  EPI_RESID_LN = 4,
  EPI_ROWMAX = 5,  // per (row, N-tile): max value (out32) and first argmax column (out16 as int32)
  EPI_RESID_ADD = 6,   // out32 += C + bias (fp32 residual stream, in place; LN runs separately)
  EPI_RESID_ADD16 = 7  // out16 += C + bias (16-bit residual stream, in place)
};

struct GemmArgs {
  int M, N, K;
  const float* bias;   // [N] (nullable for EPI_F32)
  float* out32;        // [M][N]: EPI_F32 output / EPI_RESID_LN residual (in place)
  void* out16;         // [M][ld16] 16-bit output
  int ld16;
  const float* ln_w;
  const float* ln_b;
  float ln_eps;
  int raster_m;  // 1: m-fastest tile order (B tiles stream from HBM once)
};

constexpr int BM = 128;
constexpr int kBiasMax = 4096;  // bias entries staged in shared memory
constexpr int BK = 64;  // 64 16-bit elements = one 128-byte swizzle row

__device__ __forceinline__ uint16_t to16(float x, bool fp16) {
  if (fp16) return __half_as_ushort(__float2half_rn(x));
  return __bfloat16_as_ushort(__float2bfloat16_rn(x));
}

__device__ __forceinline__ float gelu_erf(float x) {
  return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f));
}

// PAIR: a cluster of two CTAs on one TPC computes a 256 x BN tile with
// tcgen05.mma.cta_group::2 (M = 256): each CTA loads its 128 rows of A and
// half of the BN rows of B (the 2-SM TMA completes on the leader's barrier),
// the leader issues the MMAs and multicasts their completion; each CTA's
// epilogue drains its own 128 accumulator rows. Per-SM operand traffic per
// output tile drops from (A + B) to (A + B / 2).
template <int BN, int STAGES, int EPI, bool FP16, bool PAIR = false>
__global__ void __launch_bounds__(320, 1)
    k_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
           const __grid_constant__ CUtensorMap tmC, const GemmArgs g) {
  constexpr int ACC = BN <= 256 ? 2 : 1;           // TMEM accumulator buffers
  constexpr bool kTbuf = EPI == EPI_RESID_LN || EPI == EPI_RESID_ADD;  // 32x33 transposes
  constexpr uint32_t TMEM_COLS = BN * ACC <= 32 ? 32 : BN * ACC;
  constexpr int BROWS = PAIR ? BN / 2 : BN;        // B rows held by this CTA
  constexpr int TM = PAIR ? 2 * BM : BM;            // output rows per tile
  constexpr int A_BYTES = BM * BK * 2;
  constexpr int B_BYTES = BROWS * BK * 2;
  constexpr int BOX_N = BROWS < 256 ? BROWS : 256;  // TMA box rows for B
  constexpr int UMMA_N = BN < 256 ? BN : 256;
  constexpr uint32_t IDESC = umma_idesc_f16(TM, UMMA_N, FP16 ? 0 : 1);
  static_assert(!PAIR || BN <= 256, "pair tiles use one accumulator per N <= 256");

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // The dynamic shared-memory window starts 1024-byte aligned (no static
  // shared memory here), as SW128 atoms require; keeping smem_raw as the base
  // lets the compiler emit shared (not generic) loads/stores.
  unsigned char* base = smem_raw;
  unsigned char* sA = base;
  unsigned char* sB = base + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + ACC;
  uint32_t* tmem_base_smem = reinterpret_cast<uint32_t*>(tempty + ACC);
  // per-epilogue-warp 32 x 33 fp32 transpose tiles (LayerNorm epilogue),
  // then the pair-exchange area (8 warps x 32 lanes x 8 bytes)
  float* tbuf = reinterpret_cast<float*>(tmem_base_smem + 4);
  // bias staged once per CTA (N <= kBiasMax): epilogue reads are smem broadcasts
  // (offset arithmetic on the shared window keeps LDS, not generic loads)
  float* sbias0 = tbuf + (kTbuf ? 8 * 32 * 33 : 0) + 8 * 32 * 2;
  const uint32_t mis = smem_u32(sbias0) & 15u;
  float* sbias = sbias0 + (mis ? (16u - mis) / 4u : 0u);
  const bool bias_smem = g.bias != nullptr && g.N <= kBiasMax;
  // 16-bit output staging for TMA stores: per epilogue warp two [32][32] boxes
  constexpr bool kTmaOut = PAIR && (EPI == EPI_BIAS || EPI == EPI_BIAS_RELU ||
                                    EPI == EPI_BIAS_GELU || EPI == EPI_RESID_ADD16);
  unsigned char* stg0 = reinterpret_cast<unsigned char*>(sbias + kBiasMax);
  unsigned char* sstage = stg0 + ((128u - (smem_u32(stg0) & 127u)) & 127u);
  if (bias_smem)
    for (int i = threadIdx.x; i < g.N; i += blockDim.x) sbias[i] = __ldg(g.bias + i);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_m = (g.M + TM - 1) / TM, tiles_n = g.N / BN;
  const int num_tiles = tiles_m * tiles_n;
  const int nk = g.K / BK;
  const int rank = PAIR ? (int)cluster_ctarank() : 0;
  const bool leader = rank == 0;
  const int tile0 = PAIR ? (int)blockIdx.x / 2 : (int)blockIdx.x;
  const int tstride = PAIR ? (int)gridDim.x / 2 : (int)gridDim.x;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < ACC; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], PAIR ? 16 : 8);  // one arrive per epilogue warp (of both CTAs)
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    if (PAIR) tmem_alloc_pair<TMEM_COLS>(tmem_base_smem);
    else tmem_alloc<TMEM_COLS>(tmem_base_smem);
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync();  // peer barriers initialised before any remote arrive / TMA
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_smem;

  if (warp == 0) {
    // ===== TMA producer =====
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = tile0; tile < num_tiles; tile += tstride) {
        // n-fastest raster: consecutive CTAs share the A tile in L2 (m-fastest
        // when B is the large streamed operand)
        const int tn = g.raster_m ? tile / tiles_m : tile % tiles_n;
        const int tm = g.raster_m ? tile % tiles_m : tile / tiles_n;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (PAIR) {
            // both CTAs' bytes complete on the leader's barrier
            if (leader) mbar_expect_tx(&full[stage], 2 * (A_BYTES + B_BYTES));
            tma_load_2d_pair(sA + stage * A_BYTES, &tmA, &full[stage], kb * BK,
                             tm * TM + rank * BM);
#pragma unroll
            for (int j = 0; j < BROWS / BOX_N; ++j)
              tma_load_2d_pair(sB + stage * B_BYTES + j * BOX_N * 128, &tmB, &full[stage],
                               kb * BK, tn * BN + rank * BROWS + j * BOX_N);
          } else {
          mbar_expect_tx(&full[stage], A_BYTES + B_BYTES);
          tma_load_2d(sA + stage * A_BYTES, &tmA, &full[stage], kb * BK, tm * BM);
#pragma unroll
          for (int j = 0; j < BN / BOX_N; ++j)
            tma_load_2d(sB + stage * B_BYTES + j * BOX_N * 128, &tmB, &full[stage], kb * BK,
                        tn * BN + j * BOX_N);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer (the leader CTA of a pair): the whole warp runs the
    // loop in warp-uniform control flow (descriptors in uniform registers),
    // one elected lane issues
    if (leader) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      const uint64_t da0 = umma_desc_sw128(smem_u32(sA));
      const uint64_t db0 = umma_desc_sw128(smem_u32(sB));
      for (int tile = tile0; tile < num_tiles; tile += tstride) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);  // epilogue drained this buffer
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          // descriptors advance by (bytes >> 4) in their low bits
          const uint64_t a0 = da0 + (uint64_t)((stage * A_BYTES) >> 4);
          const uint64_t b0 = db0 + (uint64_t)((stage * B_BYTES) >> 4);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
#pragma unroll
              for (int j = 0; j < BN / UMMA_N; ++j) {
                const uint64_t ad = a0 + 2 * k;
                const uint64_t bd = b0 + (uint64_t)((j * UMMA_N * 128) >> 4) + 2 * k;
                if (PAIR) mma_f16_ss_pair(d_tmem + j * UMMA_N, ad, bd, IDESC, (kb | k) != 0);
                else mma_f16_ss(d_tmem + j * UMMA_N, ad, bd, IDESC, (kb | k) != 0);
              }
            }
            // frees the smem stage (of both CTAs) when these MMAs finish
            if (PAIR) mma_commit_pair(&empty[stage], 3);
            else mma_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        // accumulator ready for the epilogue(s)
        if (elect_one()) {
          if (PAIR) mma_commit_pair(&tfull[acc], 3);
          else mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++acc == ACC) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // ===== epilogue warps 2..9: TMEM lane quarter = warp % 4; the two warps
    // of a quarter split the tile's columns (half = (warp - 2) / 4) =====
    const int quarter = warp & 3;
    const int ew = warp - 2;
    const int half = ew >> 2;
    constexpr int HC = BN / 2;  // columns per epilogue warp
    const int cb = half * HC;
    float2* xch = reinterpret_cast<float2*>(tbuf + (kTbuf ? 8 * 32 * 33 : 0));
    auto pair_sync = [&]() {  // the two warps sharing this lane quarter
      asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");
    };
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = tile0; tile < num_tiles; tile += tstride) {
      const int tn = g.raster_m ? tile / tiles_m : tile % tiles_n;
      const int tm = g.raster_m ? tile % tiles_m : tile / tiles_n;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = tm * TM + rank * BM + quarter * 32 + lane;
      const bool rv = row < g.M;
      const uint32_t t0 = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN;
      if (EPI == EPI_RESID_LN) {
        // pass 1: x = resid + acc + bias, stashed back into TMEM; partial row
        // stats over this warp's columns. Residual chunks [32 rows x 32 cols]
        // are read coalesced (lane = column) and transposed via shared memory.
        float* T = tbuf + ew * (32 * 33);
        const int rowbase = tm * BM + quarter * 32;
        float s1 = 0.f, s2 = 0.f;
        float nxt[32];  // next chunk's residual column (software pipelined)
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int rr = rowbase + i;
          nxt[i] = rr < g.M ? __ldg(g.out32 + (int64_t)rr * g.N + cb + lane) : 0.f;
        }
        for (int c0 = cb; c0 < cb + HC; c0 += 32) {
          uint32_t r[32];
          tmem_ld32(t0 + c0, r);
#pragma unroll
          for (int i = 0; i < 32; ++i) T[i * 33 + lane] = nxt[i];
          if (c0 + 32 < cb + HC) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const int rr = rowbase + i;
              nxt[i] = rr < g.M ? __ldg(g.out32 + (int64_t)rr * g.N + c0 + 32 + lane) : 0.f;
            }
          }
          __syncwarp();
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float x = __uint_as_float(r[j]) + (bias_smem ? sbias[c0 + j] : __ldg(g.bias + c0 + j)) +
                            T[lane * 33 + j];
            r[j] = __float_as_uint(x);
            s1 += x;
            s2 += x * x;
          }
          __syncwarp();
          tmem_st32(t0 + c0, r);
        }
        tmem_st_wait();
        xch[ew * 32 + lane] = make_float2(s1, s2);
        pair_sync();
        const float2 o = xch[(ew ^ 4) * 32 + lane];
        pair_sync();  // partner read done before the next tile overwrites
        s1 += o.x;
        s2 += o.y;
        const float mean = s1 / BN;
        const float var = fmaxf(s2 / BN - mean * mean, 0.f);
        const float rstd = rsqrtf(var + g.ln_eps);
        // pass 2: y = LN(x); coalesced stores of fp32 (in place) and 16-bit
        for (int c0 = cb; c0 < cb + HC; c0 += 32) {
          uint32_t r[32];
          tmem_ld32(t0 + c0, r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j)
            T[lane * 33 + j] = (__uint_as_float(r[j]) - mean) * rstd * __ldg(g.ln_w + c0 + j) +
                               __ldg(g.ln_b + c0 + j);
          __syncwarp();
          uint16_t* o16 = reinterpret_cast<uint16_t*>(g.out16);
#pragma unroll 8
          for (int i = 0; i < 32; ++i) {
            const int rr = rowbase + i;
            if (rr < g.M) {
              const float y = T[i * 33 + lane];
              g.out32[(int64_t)rr * g.N + c0 + lane] = y;
              o16[(int64_t)rr * g.ld16 + c0 + lane] = to16(y, FP16);
            }
          }
          __syncwarp();
        }
      } else if (EPI == EPI_ROWMAX) {
        float best = -INFINITY;
        int bi = 0;
        for (int c0 = cb; c0 < cb + HC; c0 += 32) {
          uint32_t r[32];
          tmem_ld32(t0 + c0, r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float v = __uint_as_float(r[j]);
            if (v > best) {  // ascending columns: first maximum
              best = v;
              bi = tn * BN + c0 + j;
            }
          }
        }
        xch[ew * 32 + lane] = make_float2(best, __int_as_float(bi));
        pair_sync();
        if (half == 0) {
          const float2 o = xch[(ew ^ 4) * 32 + lane];  // upper columns: wins only if larger
          if (o.x > best) {
            best = o.x;
            bi = __float_as_int(o.y);
          }
          if (rv) {
            const int ntl = g.N / BN;
            g.out32[(int64_t)row * ntl + tn] = best;
            reinterpret_cast<int32_t*>(g.out16)[(int64_t)row * ntl + tn] = bi;
          }
        }
        pair_sync();
      } else if (EPI == EPI_RESID_ADD) {
        // out32 += acc + bias with coalesced residual I/O: each 32 x 32
        // accumulator chunk goes through a padded shared-memory transpose and
        // lanes walk columns (the 32 residual loads are issued under the
        // TMEM load)
        float* T = tbuf + ew * (32 * 33);
        const int rowbase = tm * TM + rank * BM + quarter * 32;
        for (int c0 = cb; c0 < cb + HC; c0 += 32) {
          uint32_t r[32];
          tmem_ld32(t0 + c0, r);
          const int col = tn * BN + c0 + lane;
          const float bl = bias_smem ? sbias[col] : (g.bias ? __ldg(g.bias + col) : 0.f);
          float res[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int rr = rowbase + i;
            res[i] = rr < g.M ? g.out32[(int64_t)rr * g.N + col] : 0.f;
          }
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) T[lane * 33 + j] = __uint_as_float(r[j]);
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int rr = rowbase + i;
            if (rr < g.M) g.out32[(int64_t)rr * g.N + col] = res[i] + (T[i * 33 + lane] + bl);
          }
          __syncwarp();
        }
      } else {
        unsigned char* wstage = sstage + ew * 4096;  // this warp's two 2 KB boxes
        // 16-bit residual rows (in place) are loaded one 32-column chunk
        // ahead, so their HBM latency overlaps the previous chunk
        const uint4* res_row = reinterpret_cast<const uint4*>(
            reinterpret_cast<const uint16_t*>(g.out16) + (int64_t)row * g.ld16 + tn * BN);
        uint4 rnext[4];
        if (EPI == EPI_RESID_ADD16 && rv) {
#pragma unroll
          for (int q = 0; q < 4; ++q) rnext[q] = res_row[(cb >> 3) + q];
        }
        for (int c0 = cb; c0 < cb + HC; c0 += 32) {
          uint32_t r[32];
          tmem_ld32(t0 + c0, r);
          const int col = tn * BN + c0;
          uint4 rcur[4];
          if (EPI == EPI_RESID_ADD16 && rv) {
#pragma unroll
            for (int q = 0; q < 4; ++q) rcur[q] = rnext[q];
            if (c0 + 32 < cb + HC) {
#pragma unroll
              for (int q = 0; q < 4; ++q) rnext[q] = res_row[((c0 + 32) >> 3) + q];
            }
          }
          float4 bb[8];
#pragma unroll
          for (int q = 0; q < 8; ++q)
            bb[q] = bias_smem ? reinterpret_cast<const float4*>(sbias + col)[q]
                    : g.bias  ? __ldg(reinterpret_cast<const float4*>(g.bias + col) + q)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
          if (EPI == EPI_RESID_ADD16 && rv) {  // 16-bit residual row chunk (64 B), in place
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint4 u = rcur[q];
              const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
              for (int h = 0; h < 2; ++h) {  // elements 8q + 4h .. + 3 -> bb[2q + h]
                float2 f0, f1;
                if (FP16) {
                  f0 = __half22float2(*reinterpret_cast<const __half2*>(&w4[2 * h]));
                  f1 = __half22float2(*reinterpret_cast<const __half2*>(&w4[2 * h + 1]));
                } else {
                  f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w4[2 * h]));
                  f1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w4[2 * h + 1]));
                }
                float4& b4 = bb[2 * q + h];
                b4 = make_float4(b4.x + f0.x, b4.y + f0.y, b4.z + f1.x, b4.w + f1.y);
              }
            }
          }
          if (EPI == EPI_RESID_ADD && rv) {  // residual row chunk, loaded under the TMEM load
            const float4* res = reinterpret_cast<const float4*>(g.out32 + (int64_t)row * g.N + col);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float4 x = res[q];
              bb[q] = make_float4(bb[q].x + x.x, bb[q].y + x.y, bb[q].z + x.z, bb[q].w + x.w);
            }
          }
          tmem_ld_wait();
          if (!kTmaOut && !rv) continue;
          float v[32];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            v[4 * q] = __uint_as_float(r[4 * q]) + bb[q].x;
            v[4 * q + 1] = __uint_as_float(r[4 * q + 1]) + bb[q].y;
            v[4 * q + 2] = __uint_as_float(r[4 * q + 2]) + bb[q].z;
            v[4 * q + 3] = __uint_as_float(r[4 * q + 3]) + bb[q].w;
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            if (EPI == EPI_BIAS_RELU) v[j] = fmaxf(v[j], 0.f);
            if (EPI == EPI_BIAS_GELU) v[j] = gelu_erf(v[j]);
          }
          if (EPI == EPI_F32 || EPI == EPI_RESID_ADD) {
            float4* o = reinterpret_cast<float4*>(g.out32 + (int64_t)row * g.N + col);
#pragma unroll
            for (int q = 0; q < 8; ++q) o[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          } else if (kTmaOut) {
            // stage [32 rows][32 cols] 16-bit, then one TMA store per warp
            // (rows past M are clipped by the tensor map)
            const int buf = (c0 >> 5) & 1;
            unsigned char* box = wstage + buf * 2048;
            if (c0 - cb >= 64) {  // the box written two chunks ago has been read
              if (lane == 0) bulk_wait_read<1>();
              __syncwarp();
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint32_t w[4];
#pragma unroll
              for (int u = 0; u < 4; ++u)
                w[u] = to16(v[8 * q + 2 * u], FP16) | ((uint32_t)to16(v[8 * q + 2 * u + 1], FP16) << 16);
              *reinterpret_cast<uint4*>(box + lane * 64 + q * 16) = make_uint4(w[0], w[1], w[2], w[3]);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&tmC, box, col, tm * TM + rank * BM + quarter * 32);
              bulk_commit();
            }
          } else {
            uint4* o = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(g.out16) +
                                                (int64_t)row * g.ld16 + col);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint32_t w[4];
#pragma unroll
              for (int u = 0; u < 4; ++u)
                w[u] = to16(v[8 * q + 2 * u], FP16) | ((uint32_t)to16(v[8 * q + 2 * u + 1], FP16) << 16);
              o[q] = make_uint4(w[0], w[1], w[2], w[3]);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (kTmaOut) {  // the next tile reuses this warp's staging boxes
        if (lane == 0) bulk_wait_read<0>();
        __syncwarp();
      }
      if (lane == 0) {
        if (PAIR && !leader) mbar_arrive_cluster(&tempty[acc], 0);  // the leader's MMA waits
        else mbar_arrive(&tempty[acc]);
      }
      if (++acc == ACC) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  if (kTmaOut && warp >= 2 && lane == 0) bulk_wait<0>();  // stores complete before exit
  tc_fence_before();
  __syncthreads();
  if (PAIR) {
    cluster_sync();  // both CTAs done with TMEM and each other's barriers
    if (warp == 1) tmem_dealloc_pair<TMEM_COLS>(tmem_base);
  } else if (warp == 1) {
    tmem_dealloc<TMEM_COLS>(tmem_base);
  }
}

// ---------------------------------------------------------------------------
// Host side: tensor maps and launch.
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                             const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                             const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  }
  return fn;
}

// 2-D K-major tensor [rows][K] (row stride ld elements), box [box_rows][64].
int make_map(CUtensorMap* m, const void* ptr, int rows, int K, int ld, int box_rows, bool fp16) {
  EncodeFn enc = encode_fn();
  if (!enc) return moeb::fail(MOEB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, fp16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return moeb::fail(MOEB_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return MOEB_OK;
}

// 16-bit output [rows][ld] (N columns), 32 x 32 boxes, no swizzle (TMA store)
int make_out_map(CUtensorMap* m, const void* ptr, int rows, int N, int ld, bool fp16) {
  EncodeFn enc = encode_fn();
  if (!enc) return moeb::fail(MOEB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, fp16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return moeb::fail(MOEB_ECUDA, "cuTensorMapEncodeTiled (out) failed (%d)", (int)r);
  return MOEB_OK;
}

template <int BN, int STAGES, int EPI, bool FP16>
int launch_gemm_pair(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc,
                     const GemmArgs& g, cudaStream_t s) {
  constexpr int ACC = BN <= 256 ? 2 : 1;
  const size_t smem = 1024 + (size_t)STAGES * (BM * BK * 2 + (BN / 2) * BK * 2) +
                      8 * (2 * STAGES + 2 * ACC) + 16 +
                      ((EPI == EPI_RESID_LN || EPI == EPI_RESID_ADD) ? 8 * 32 * 33 * sizeof(float)
                                                                     : 0) +
                      8 * 32 * 8 + kBiasMax * sizeof(float) + 16 +
                      ((EPI == EPI_BIAS || EPI == EPI_BIAS_RELU || EPI == EPI_BIAS_GELU ||
                        EPI == EPI_RESID_ADD16)
                           ? 8 * 4096 + 128
                           : 0);
  auto k = k_gemm<BN, STAGES, EPI, FP16, true>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int tiles = ((g.M + 2 * BM - 1) / (2 * BM)) * (g.N / BN);
  const int pairs = tiles < moeb::num_sms() / 2 ? tiles : moeb::num_sms() / 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * pairs));
  cfg.blockDim = dim3(320);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, k, ta, tb, tc, g) != cudaSuccess)
    return moeb::check_launch("k_gemm (pair launch)");
  return moeb::check_launch("k_gemm (pair)");
}

template <int BN, int STAGES, int EPI, bool FP16>
int launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc,
                const GemmArgs& g, cudaStream_t s) {
  constexpr int ACC = BN <= 256 ? 2 : 1;
  const size_t smem = 1024 + (size_t)STAGES * (BM * BK * 2 + BN * BK * 2) +
                      8 * (2 * STAGES + 2 * ACC) + 16 +
                      ((EPI == EPI_RESID_LN || EPI == EPI_RESID_ADD) ? 8 * 32 * 33 * sizeof(float)
                                                                     : 0) +
                      8 * 32 * 8 +
                      kBiasMax * sizeof(float) + 16;
  auto k = k_gemm<BN, STAGES, EPI, FP16>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int tiles = ((g.M + BM - 1) / BM) * (g.N / BN);
  const int grid = tiles < moeb::num_sms() ? tiles : moeb::num_sms();
  k<<<grid, 320, smem, s>>>(ta, tb, tc, g);
  return moeb::check_launch("k_gemm");
}

// MOEB_GEMM_PAIR=0 disables the 2-SM tiles (single-CTA M = 128 tiles)
bool pair_mode() {
  const char* e = getenv("MOEB_GEMM_PAIR");
  return !(e && e[0] == '0');
}

template <int EPI, bool FP16>
int dispatch(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc,
             const GemmArgs& g, int bn,
             cudaStream_t s) {
  if (bn == 512) return launch_gemm<512, 2, EPI, FP16>(ta, tb, tc, g, s);
  if (bn == 256) {
    if (pair_mode()) {  // 2-SM tiles (M = 256): B tile split across the CTA pair
      if (EPI == EPI_RESID_ADD) return launch_gemm_pair<256, 4, EPI, FP16>(ta, tb, tc, g, s);
      return launch_gemm_pair<256, 5, EPI, FP16>(ta, tb, tc, g, s);
    }
    if (EPI == EPI_RESID_ADD) return launch_gemm<256, 3, EPI, FP16>(ta, tb, tc, g, s);  // + transposes
    return launch_gemm<256, 4, EPI, FP16>(ta, tb, tc, g, s);
  }
  if (bn == 128) return launch_gemm<128, 6, EPI, FP16>(ta, tb, tc, g, s);
  return launch_gemm<64, 8, EPI, FP16>(ta, tb, tc, g, s);
}

}  // namespace

extern "C" int moeb_gemm(const void* A, int lda, const void* B, int ldb, int M, int N, int K,
                         int fp16, int epi, const float* bias, float* out32, void* out16,
                         int ld16, const float* ln_w, const float* ln_b, float ln_eps,
                         void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(A && B && M >= 1 && N >= 1 && K >= 1, "bad GEMM arguments");
  MOEB_REQUIRE(K % BK == 0, "K must be a multiple of %d (got %d)", BK, K);
  MOEB_REQUIRE(epi >= EPI_F32 && epi <= EPI_RESID_ADD16, "unknown epilogue %d", epi);
  int bn;
  if (epi == EPI_RESID_LN) {
    MOEB_REQUIRE(N == 512, "LayerNorm epilogue needs N == 512");
    MOEB_REQUIRE(out32 && out16 && bias && ln_w && ln_b, "LayerNorm epilogue arguments");
    bn = 512;
  } else {
    bn = N % 256 == 0 ? 256 : N % 128 == 0 ? 128 : N % 64 == 0 ? 64 : 0;
    MOEB_REQUIRE(bn, "N must be a multiple of 64 (got %d)", N);
    MOEB_REQUIRE((epi == EPI_F32 || epi == EPI_RESID_ADD) ? out32 != nullptr : out16 != nullptr,
                 "missing output");
    MOEB_REQUIRE(epi != EPI_ROWMAX || (out32 && bn == 256), "row-max epilogue needs N % 256 == 0");
  }
  CUtensorMap ta, tb, tc;
  if (int rc = make_map(&ta, A, M, K, lda, BM, fp16)) return rc;
  memset(&tc, 0, sizeof(tc));
  const bool tma_out = ((epi >= EPI_BIAS && epi <= EPI_BIAS_GELU) || epi == EPI_RESID_ADD16) &&
                       bn == 256 && pair_mode();
  if (tma_out) {  // 16-bit output tile stores by TMA (32 x 32 boxes)
    if (int rc = make_out_map(&tc, out16, M, N, ld16, fp16)) return rc;
  }
  // pair tiles (dispatch, N-tile 256) load half of the B tile per CTA
  const bool pair_b = bn == 256 && epi != EPI_RESID_LN && epi != EPI_ROWMAX && pair_mode();
  if (int rc = make_map(&tb, B, N, K, ldb, pair_b ? 128 : (bn < 256 ? bn : 256), fp16)) return rc;
  GemmArgs g{M, N, K, bias, out32, out16, ld16, ln_w, ln_b, ln_eps, epi == EPI_ROWMAX ? 1 : 0};
  cudaStream_t s = moeb::as_stream(stream);
  switch (epi) {
    case EPI_F32: return fp16 ? dispatch<EPI_F32, true>(ta, tb, tc, g, bn, s) : dispatch<EPI_F32, false>(ta, tb, tc, g, bn, s);
    case EPI_BIAS: return fp16 ? dispatch<EPI_BIAS, true>(ta, tb, tc, g, bn, s) : dispatch<EPI_BIAS, false>(ta, tb, tc, g, bn, s);
    case EPI_BIAS_RELU: return fp16 ? dispatch<EPI_BIAS_RELU, true>(ta, tb, tc, g, bn, s) : dispatch<EPI_BIAS_RELU, false>(ta, tb, tc, g, bn, s);
    case EPI_BIAS_GELU: return fp16 ? dispatch<EPI_BIAS_GELU, true>(ta, tb, tc, g, bn, s) : dispatch<EPI_BIAS_GELU, false>(ta, tb, tc, g, bn, s);
    case EPI_RESID_ADD: return fp16 ? dispatch<EPI_RESID_ADD, true>(ta, tb, tc, g, bn, s) : dispatch<EPI_RESID_ADD, false>(ta, tb, tc, g, bn, s);
    case EPI_RESID_ADD16: return fp16 ? dispatch<EPI_RESID_ADD16, true>(ta, tb, tc, g, bn, s) : dispatch<EPI_RESID_ADD16, false>(ta, tb, tc, g, bn, s);
    case EPI_ROWMAX: return fp16 ? launch_gemm<256, 4, EPI_ROWMAX, true>(ta, tb, tc, g, s) : launch_gemm<256, 4, EPI_ROWMAX, false>(ta, tb, tc, g, s);
    default: return fp16 ? launch_gemm<512, 2, EPI_RESID_LN, true>(ta, tb, tc, g, s) : launch_gemm<512, 2, EPI_RESID_LN, false>(ta, tb, tc, g, s);
  }
}
