// Transformer predictor glue kernels (the GEMMs are K4, attention K5).
//
// Input projection, factorised: Linear(2560 -> 512) over [tok_emb | layer_emb]
// equals tok_emb . W_tok^T + (layer_emb . W_lay^T + b), so with
// the per-vocabulary table P_tok[32000][512] and the per-layer table
// P_lay[L][512] (both computed once per model by K4) the projected input of a
// trace row is a two-row gather-add.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>

#include "common.cuh"

namespace {

template <bool FP16>
__global__ void __launch_bounds__(128) k_embed_rows(const float* __restrict__ ptok,
                                                    const float* __restrict__ play,
                                                    const int32_t* __restrict__ tok, int L,
                                                    int64_t rows, float* __restrict__ out32,
                                                    uint16_t* __restrict__ out16) {
  // one warp per row, 512 columns = 32 lanes x 16 floats
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= rows) return;
  const int lane = threadIdx.x & 31;
  const int t = tok[r / L], l = (int)(r % L);
  const float4* a = reinterpret_cast<const float4*>(ptok + (int64_t)t * 512) + lane * 4;
  const float4* b = reinterpret_cast<const float4*>(play + (int64_t)l * 512) + lane * 4;
  float4* o = out32 ? reinterpret_cast<float4*>(out32 + r * 512) + lane * 4 : nullptr;
  uint32_t p[8];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float4 x = a[q], y = b[q];
    const float4 v = make_float4(x.x + y.x, x.y + y.y, x.z + y.z, x.w + y.w);
    if (o) o[q] = v;
    if (FP16) {
      const __half2 h0 = __floats2half2_rn(v.x, v.y), h1 = __floats2half2_rn(v.z, v.w);
      p[2 * q] = *reinterpret_cast<const uint32_t*>(&h0);
      p[2 * q + 1] = *reinterpret_cast<const uint32_t*>(&h1);
    } else {
      const __nv_bfloat162 h0 = __floats2bfloat162_rn(v.x, v.y), h1 = __floats2bfloat162_rn(v.z, v.w);
      p[2 * q] = *reinterpret_cast<const uint32_t*>(&h0);
      p[2 * q + 1] = *reinterpret_cast<const uint32_t*>(&h1);
    }
  }
  uint4* o16 = reinterpret_cast<uint4*>(out16 + r * 512) + lane * 2;
  o16[0] = make_uint4(p[0], p[1], p[2], p[3]);
  o16[1] = make_uint4(p[4], p[5], p[6], p[7]);
}

template <bool FP16>
__global__ void k_to16(const float* __restrict__ x, uint16_t* __restrict__ y, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    y[i] = FP16 ? __half_as_ushort(__float2half_rn(x[i]))
                : __bfloat16_as_ushort(__float2bfloat16_rn(x[i]));
}

// Post-norm LayerNorm of the residual stream, one warp per 512-wide row:
// two-pass mean / variance in registers, y = (x - mean) rsqrt(var + eps) w + b
// written back in fp32 (in place) and as the 16-bit GEMM operand.
template <bool FP16>
__global__ void __launch_bounds__(256) k_layernorm_rows(float* __restrict__ x32,
                                                        uint16_t* __restrict__ out16,
                                                        const float* __restrict__ w,
                                                        const float* __restrict__ b,
                                                        int64_t rows, float eps) {
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= rows) return;
  const int lane = threadIdx.x & 31;
  float4* xr = reinterpret_cast<float4*>(x32 + r * 512);
  float4 v[4];
  float s = 0.f;
#pragma unroll
  for (int q = 0; q < 4; ++q) {  // lane owns columns [128 q + 4 lane, +4)
    v[q] = xr[q * 32 + lane];
    s += (v[q].x + v[q].y) + (v[q].z + v[q].w);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float mean = s * (1.f / 512.f);
  float s2 = 0.f;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float a0 = v[q].x - mean, a1 = v[q].y - mean, a2 = v[q].z - mean, a3 = v[q].w - mean;
    s2 += (a0 * a0 + a1 * a1) + (a2 * a2 + a3 * a3);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  const float rstd = rsqrtf(s2 * (1.f / 512.f) + eps);
  const float4* w4 = reinterpret_cast<const float4*>(w);
  const float4* b4 = reinterpret_cast<const float4*>(b);
  uint2* o16 = reinterpret_cast<uint2*>(out16 + r * 512);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float4 ww = __ldg(w4 + q * 32 + lane), bb = __ldg(b4 + q * 32 + lane);
    const float4 y = make_float4((v[q].x - mean) * rstd * ww.x + bb.x,
                                 (v[q].y - mean) * rstd * ww.y + bb.y,
                                 (v[q].z - mean) * rstd * ww.z + bb.z,
                                 (v[q].w - mean) * rstd * ww.w + bb.w);
    xr[q * 32 + lane] = y;
    uint32_t p0, p1;
    if (FP16) {
      const __half2 h0 = __floats2half2_rn(y.x, y.y), h1 = __floats2half2_rn(y.z, y.w);
      p0 = *reinterpret_cast<const uint32_t*>(&h0);
      p1 = *reinterpret_cast<const uint32_t*>(&h1);
    } else {
      const __nv_bfloat162 h0 = __floats2bfloat162_rn(y.x, y.y), h1 = __floats2bfloat162_rn(y.z, y.w);
      p0 = *reinterpret_cast<const uint32_t*>(&h0);
      p1 = *reinterpret_cast<const uint32_t*>(&h1);
    }
    o16[q * 32 + lane] = make_uint2(p0, p1);
  }
}

// The 16-bit residual stream's LayerNorm: x16 [rows][512] normalised in
// place (fp32 statistics and arithmetic, one 16-bit read and write per
// element: 4 B/element instead of the fp32 stream's 10). A warp owns LN_RPW
// consecutive rows, lane = columns [8 lane + 256 q, +8): all of its rows'
// loads are issued before the first row is reduced (LN_RPW x 1 KB in flight
// per warp), and gamma / beta stay in registers across its rows.
constexpr int LN_RPW = 4;

template <bool FP16>
__device__ __forceinline__ void unpack8(const uint4 u, float* v) {
  const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float2 f;
    if (FP16)
      f = __half22float2(*reinterpret_cast<const __half2*>(&w4[j]));
    else
      f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w4[j]));
    v[2 * j] = f.x;
    v[2 * j + 1] = f.y;
  }
}

template <bool FP16>
__global__ void __launch_bounds__(256) k_layernorm_rows16(uint16_t* __restrict__ x16,
                                                          const float* __restrict__ w,
                                                          const float* __restrict__ b,
                                                          int64_t rows, float eps) {
  const int64_t r0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * LN_RPW;
  if (r0 >= rows) return;
  const int lane = threadIdx.x & 31;
  const int nr = rows - r0 < LN_RPW ? (int)(rows - r0) : LN_RPW;
  uint4 u[LN_RPW][2];
#pragma unroll
  for (int i = 0; i < LN_RPW; ++i)
    if (i < nr) {
      const uint4* xr = reinterpret_cast<const uint4*>(x16 + (r0 + i) * 512);
      u[i][0] = xr[lane];
      u[i][1] = xr[32 + lane];
    }
  float ww[16], bb[16];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int c = q * 256 + lane * 8;
    const float4 w0 = __ldg(reinterpret_cast<const float4*>(w + c));
    const float4 w1 = __ldg(reinterpret_cast<const float4*>(w + c + 4));
    const float4 b0 = __ldg(reinterpret_cast<const float4*>(b + c));
    const float4 b1 = __ldg(reinterpret_cast<const float4*>(b + c + 4));
    const float wq[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
    const float bq[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      ww[q * 8 + j] = wq[j];
      bb[q * 8 + j] = bq[j];
    }
  }
#pragma unroll
  for (int i = 0; i < LN_RPW; ++i) {
    if (i >= nr) break;
    float v[16];
    unpack8<FP16>(u[i][0], v);
    unpack8<FP16>(u[i][1], v + 8);
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += v[k];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float mean = s * (1.f / 512.f);
    float s2 = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k) s2 += (v[k] - mean) * (v[k] - mean);
#pragma unroll
    for (int o = 16; o; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    const float rstd = rsqrtf(s2 * (1.f / 512.f) + eps);
    uint4* xr = reinterpret_cast<uint4*>(x16 + (r0 + i) * 512);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      uint32_t p[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int k = q * 8 + 2 * j;
        const float y0 = (v[k] - mean) * rstd * ww[k] + bb[k];
        const float y1 = (v[k + 1] - mean) * rstd * ww[k + 1] + bb[k + 1];
        if (FP16) {
          const __half2 h = __floats2half2_rn(y0, y1);
          p[j] = *reinterpret_cast<const uint32_t*>(&h);
        } else {
          const __nv_bfloat162 h = __floats2bfloat162_rn(y0, y1);
          p[j] = *reinterpret_cast<const uint32_t*>(&h);
        }
      }
      xr[q * 32 + lane] = make_uint4(p[0], p[1], p[2], p[3]);
    }
  }
}

}  // namespace

extern "C" int moeb_layernorm_rows16(void* x16, const float* w, const float* b, int64_t rows,
                                     float eps, int fp16, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(x16 && w && b && rows >= 0, "bad args");
  if (rows == 0) return MOEB_OK;
  const unsigned blocks = (unsigned)(((rows + LN_RPW - 1) / LN_RPW * 32 + 255) / 256);
  cudaStream_t s = moeb::as_stream(stream);
  if (fp16)
    k_layernorm_rows16<true><<<blocks, 256, 0, s>>>(static_cast<uint16_t*>(x16), w, b, rows, eps);
  else
    k_layernorm_rows16<false><<<blocks, 256, 0, s>>>(static_cast<uint16_t*>(x16), w, b, rows, eps);
  return moeb::check_launch("k_layernorm_rows16");
}

extern "C" int moeb_layernorm_rows(float* x32, void* out16, const float* w, const float* b,
                                   int64_t rows, float eps, int fp16, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(x32 && out16 && w && b && rows >= 0, "bad args");
  if (rows == 0) return MOEB_OK;
  const unsigned blocks = (unsigned)((rows * 32 + 255) / 256);
  cudaStream_t s = moeb::as_stream(stream);
  if (fp16)
    k_layernorm_rows<true><<<blocks, 256, 0, s>>>(x32, static_cast<uint16_t*>(out16), w, b, rows,
                                                  eps);
  else
    k_layernorm_rows<false><<<blocks, 256, 0, s>>>(x32, static_cast<uint16_t*>(out16), w, b,
                                                   rows, eps);
  return moeb::check_launch("k_layernorm_rows");
}

extern "C" int moeb_embed_rows(const float* ptok, const float* play, const int32_t* token_ids,
                               int L, int64_t rows, float* out32, void* out16, int fp16,
                               void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(ptok && play && token_ids && out16 && L >= 1 && rows >= 0, "bad args");
  if (rows == 0) return MOEB_OK;
  const unsigned blocks = (unsigned)((rows * 32 + 127) / 128);
  cudaStream_t s = moeb::as_stream(stream);
  if (fp16)
    k_embed_rows<true><<<blocks, 128, 0, s>>>(ptok, play, token_ids, L, rows, out32,
                                              static_cast<uint16_t*>(out16));
  else
    k_embed_rows<false><<<blocks, 128, 0, s>>>(ptok, play, token_ids, L, rows, out32,
                                               static_cast<uint16_t*>(out16));
  return moeb::check_launch("k_embed_rows");
}

extern "C" int moeb_to16(const float* x, void* y, int64_t n, int fp16, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(x && y && n >= 0, "bad args");
  if (n == 0) return MOEB_OK;
  cudaStream_t s = moeb::as_stream(stream);
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  if (fp16)
    k_to16<true><<<blocks, 256, 0, s>>>(x, static_cast<uint16_t*>(y), n);
  else
    k_to16<false><<<blocks, 256, 0, s>>>(x, static_cast<uint16_t*>(y), n);
  return moeb::check_launch("k_to16");
}
