// Transformer predictor training: the
// backward pass and the optimiser step around the forward kernels.
//
// The dense products of the backward pass are K4 (tcgen05) GEMMs:
// dX = dY W uses the transposed 16-bit weight, dW = dY^T X the transposed
// 16-bit activations (moeb_transpose16); everything else is here:
//   moeb_transpose16        [R][C] -> [C][R] 16-bit (32 x 32 smem tiles)
//   moeb_colsum16           bias gradients: out[N] += column sums of [M][N]
//   moeb_layernorm_bwd16    post-norm LayerNorm backward from the saved
//                           pre-norm rows (statistics recomputed in fp32),
//                           dgamma / dbeta column sums
//   moeb_relu_bwd16         d *= (activation > 0)
//   moeb_gelu_fwd16/bwd16   erf GELU of the head's hidden layer and its
//                           derivative
//   moeb_bce_logits_grad    BCEWithLogits (mean over rows x experts) loss and
//                           its gradient, scaled by the loss scale, 16-bit
//   moeb_attention_bwd      windowed multi-head attention backward: per
//                           (window, head, 64-query block) the softmax
//                           statistics and dQ; per (window, head, 64-key
//                           block) dK and dV (scores recomputed, fp32 math)
//   moeb_gather_inputs16    per-row [token embedding | layer embedding] rows
//   moeb_layer_emb_grad     layer-embedding gradient (rows summed per layer)
//   moeb_cast_f32_to_16     fp32 master weights -> 16-bit GEMM operands
//   moeb_sumsq_f32          squared gradient norm (clipping, overflow check)
//   moeb_adamw_f32          torch.optim.AdamW step (decoupled weight decay)
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cmath>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace {

template <bool FP16>
__device__ __forceinline__ float ld16(const uint16_t* p) {
  return FP16 ? __half2float(__ushort_as_half(*p)) : __bfloat162float(__ushort_as_bfloat16(*p));
}
template <bool FP16>
__device__ __forceinline__ float cvt16(uint16_t v) {
  return FP16 ? __half2float(__ushort_as_half(v)) : __bfloat162float(__ushort_as_bfloat16(v));
}
template <bool FP16>
__device__ __forceinline__ uint16_t st16(float x) {
  return FP16 ? __half_as_ushort(__float2half_rn(x)) : __bfloat16_as_ushort(__float2bfloat16_rn(x));
}

// ---------------------------------------------------------------------------
__global__ void k_transpose16(const uint16_t* __restrict__ in, int64_t R, int C, int ld_in,
                              uint16_t* __restrict__ out, int ld_out) {
  __shared__ uint16_t t[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32;
  const int c0 = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = r0 + i;
    const int c = c0 + threadIdx.x;
    t[i][threadIdx.x] = (r < R && c < C) ? in[r * ld_in + c] : (uint16_t)0;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int c = c0 + i;
    const int64_t r = r0 + threadIdx.x;
    if (c < C && r < R) out[(int64_t)c * ld_out + r] = t[threadIdx.x][i];
  }
}

// out[N] += column sums of in [M][N] (ld); thread per column, rows split
// over gridDim.y
template <bool FP16>
__global__ void k_colsum16(const uint16_t* __restrict__ in, int64_t M, int N, int ld,
                           float* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  const int64_t per = (M + gridDim.y - 1) / gridDim.y;
  const int64_t a = (int64_t)blockIdx.y * per, b = min(M, a + per);
  float s = 0.f;
  for (int64_t r = a; r < b; ++r) s += ld16<FP16>(in + r * ld + c);
  if (b > a) atomicAdd(out + c, s);
}

// LayerNorm backward over 512-wide rows. y = (x - mean) rstd w + b; with
// g = dy w: dx = rstd (g - mean(g) - xhat mean(g xhat)); dw += dy xhat,
// db += dy. Warp per row; per-block column partials in shared memory.
template <bool FP16>
__global__ void __launch_bounds__(256) k_layernorm_bwd16(
    const uint16_t* __restrict__ dy16, const uint16_t* __restrict__ x16,
    const float* __restrict__ w, int64_t M, float eps, uint16_t* __restrict__ dx16,
    float* __restrict__ dw, float* __restrict__ db) {
  __shared__ float sdw[512], sdb[512];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) sdw[i] = sdb[i] = 0.f;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  for (int64_t r = (int64_t)blockIdx.x * nw + warp; r < M; r += (int64_t)gridDim.x * nw) {
    float x[16], dy[16];
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int c = j * 32 + lane;
      x[j] = ld16<FP16>(x16 + r * 512 + c);
      dy[j] = ld16<FP16>(dy16 + r * 512 + c);
      s += x[j];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float mean = s * (1.f / 512.f);
    float s2 = 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) s2 += (x[j] - mean) * (x[j] - mean);
#pragma unroll
    for (int o = 16; o; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    const float rstd = rsqrtf(s2 * (1.f / 512.f) + eps);
    float mg = 0.f, mgx = 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int c = j * 32 + lane;
      const float xh = (x[j] - mean) * rstd;
      const float g = dy[j] * w[c];
      mg += g;
      mgx += g * xh;
      atomicAdd(&sdw[c], dy[j] * xh);
      atomicAdd(&sdb[c], dy[j]);
      x[j] = xh;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      mg += __shfl_xor_sync(0xffffffffu, mg, o);
      mgx += __shfl_xor_sync(0xffffffffu, mgx, o);
    }
    mg *= (1.f / 512.f);
    mgx *= (1.f / 512.f);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int c = j * 32 + lane;
      const float g = dy[j] * w[c];
      dx16[r * 512 + c] = st16<FP16>(rstd * (g - mg - x[j] * mgx));
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 512; i += blockDim.x) {
    if (sdw[i] != 0.f) atomicAdd(dw + i, sdw[i]);
    if (sdb[i] != 0.f) atomicAdd(db + i, sdb[i]);
  }
}

template <bool FP16>
__global__ void k_relu_bwd16(uint16_t* __restrict__ d, const uint16_t* __restrict__ act,
                             int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (!(ld16<FP16>(act + i) > 0.f)) d[i] = 0;
}

__device__ __forceinline__ float gelu_erf_f(float u) {
  return 0.5f * u * (1.f + erff(u * 0.70710678118654752f));
}

template <bool FP16>
__global__ void k_gelu_fwd16(const uint16_t* __restrict__ u, uint16_t* __restrict__ g, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    g[i] = st16<FP16>(gelu_erf_f(ld16<FP16>(u + i)));
}

// d <- d * gelu'(u), gelu'(u) = Phi(u) + u phi(u)
template <bool FP16>
__global__ void k_gelu_bwd16(uint16_t* __restrict__ d, const uint16_t* __restrict__ u, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float x = ld16<FP16>(u + i);
    const float cdf = 0.5f * (1.f + erff(x * 0.70710678118654752f));
    const float pdf = 0.39894228040143268f * expf(-0.5f * x * x);
    d[i] = st16<FP16>(ld16<FP16>(d + i) * (cdf + x * pdf));
  }
}

// BCEWithLogits, reduction mean over M x E: loss = softplus(z) - y z (stable
// form max(z, 0) - y z + log1p(exp(-|z|))); dz = (sigmoid(z) - y) / (M E),
// times the loss scale, 16-bit. y = bit e of the row's truth mask.
template <bool FP16>
__global__ void k_bce_grad(const float* __restrict__ z, const uint64_t* __restrict__ truth, int W,
                           int64_t M, int E, float scale, uint16_t* __restrict__ dz,
                           double* __restrict__ loss_sum) {
  __shared__ double red[32];
  double acc = 0.0;
  const float inv = 1.f / (float)((double)M * E);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M * E;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / E;
    const int e = (int)(i % E);
    const float y = (float)((truth[r * W + (e >> 6)] >> (e & 63)) & 1ull);
    const float x = z[i];
    acc += (double)(fmaxf(x, 0.f) - y * x + log1pf(expf(-fabsf(x))));
    const float sg = 1.f / (1.f + expf(-x));
    dz[i] = st16<FP16>((sg - y) * inv * scale);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
    atomicAdd(loss_sum, t);
  }
}

// ---------------------------------------------------------------------------
// Attention backward. qkv [rows][1536] (q | k | v, head h at 64h), o / dO
// [rows][512] (the forward output and its gradient), dqkv [rows][1536].
// Scores s = q.k / 8 in the log2 domain (s2 = q.k * 0.125 log2 e), P =
// exp2(s2 - lse2) with lse2 = m + log2(sum exp2(s2 - m)) per query row.
// 64 x 64 tiles, 256 threads = 16 x 16, thread (ty, tx) owns rows 4 ty.. and
// columns 4 tx.. of a tile.
// ---------------------------------------------------------------------------
constexpr int AT = 64;
constexpr float kSl2 = 0.125f * 1.4426950408889634f;

template <bool FP16>
__device__ __forceinline__ void load_tile(float (*dst)[AT + 1], const uint16_t* __restrict__ base,
                                          int64_t row0, int n, int ld, int col0) {
  for (int i = threadIdx.x; i < AT * AT; i += blockDim.x) {
    const int r = i / AT, c = i % AT;
    dst[r][c] = r < n ? ld16<FP16>(base + (row0 + r) * ld + col0 + c) : 0.f;
  }
}

// acc[a][b] = sum_d X[4ty + a][d] Y[4tx + b][d]
__device__ __forceinline__ void tile_abt(float (&acc)[4][4], const float (*X)[AT + 1],
                                         const float (*Y)[AT + 1], int ty, int tx) {
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
#pragma unroll 8
  for (int d = 0; d < AT; ++d) {
    float xa[4], yb[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) xa[a] = X[4 * ty + a][d];
#pragma unroll
    for (int b = 0; b < 4; ++b) yb[b] = Y[4 * tx + b][d];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(xa[a], yb[b], acc[a][b]);
  }
}

// per (window, head, query block): lse2, dsum = rowsum(dO o O), dQ
template <bool FP16>
__global__ void __launch_bounds__(256) k_attn_bwd_q(
    const uint16_t* __restrict__ qkv, const uint16_t* __restrict__ o,
    const uint16_t* __restrict__ dout, const int64_t* __restrict__ win_start,
    const int32_t* __restrict__ win_len, int nqb, uint16_t* __restrict__ dqkv,
    float* __restrict__ lse2_out, float* __restrict__ dsum_out) {
  extern __shared__ float sm[];
  float(*Q)[AT + 1] = reinterpret_cast<float(*)[AT + 1]>(sm);
  float(*dO)[AT + 1] = Q + AT;
  float(*K)[AT + 1] = dO + AT;
  float(*V)[AT + 1] = K + AT;
  float(*S)[AT + 1] = V + AT;
  float* lse = reinterpret_cast<float*>(S + AT);
  float* dsum = lse + AT;
  const int qb = blockIdx.x % nqb, head = (blockIdx.x / nqb) % 8, w = blockIdx.x / (nqb * 8);
  const int n = win_len[w];
  if (qb * AT >= n) return;
  const int64_t r0 = win_start[w];
  const int64_t q0 = r0 + qb * AT;
  const int nq = min(AT, n - qb * AT);
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  load_tile<FP16>(Q, qkv, q0, nq, 1536, head * 64);
  load_tile<FP16>(dO, dout, q0, nq, 512, head * 64);
  __syncthreads();
  if (tid < AT) {  // dsum = sum_d dO o O (O read from global, fp32 math)
    float acc = 0.f;
    if (tid < nq)
      for (int d = 0; d < 64; ++d) acc += dO[tid][d] * ld16<FP16>(o + (q0 + tid) * 512 + head * 64 + d);
    dsum[tid] = acc;
  }
  // pass A: online max / sum of exp2 per query row
  float m[4], l[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    m[a] = -INFINITY;
    l[a] = 0.f;
  }
  const int nkb = (n + AT - 1) / AT;
  for (int kb = 0; kb < nkb; ++kb) {
    __syncthreads();
    load_tile<FP16>(K, qkv, r0 + kb * AT, min(AT, n - kb * AT), 1536, 512 + head * 64);
    __syncthreads();
    float s[4][4];
    tile_abt(s, Q, K, ty, tx);
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      float mx = -INFINITY;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        s[a][b] = kb * AT + 4 * tx + b < n ? s[a][b] * kSl2 : -INFINITY;
        mx = fmaxf(mx, s[a][b]);
      }
#pragma unroll
      for (int off = 8; off; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      const float mn = fmaxf(m[a], mx);
      float sum = 0.f;
#pragma unroll
      for (int b = 0; b < 4; ++b) sum += exp2f(s[a][b] - mn);
#pragma unroll
      for (int off = 8; off; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
      l[a] = l[a] * exp2f(m[a] - mn) + sum;
      m[a] = mn;
    }
  }
  if (tx == 0) {
#pragma unroll
    for (int a = 0; a < 4; ++a) lse[4 * ty + a] = m[a] + log2f(l[a]);
  }
  __syncthreads();
  // pass B: dS = P (dO V^T - dsum), dQ = dS K / 8
  float dq[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) dq[a][b] = 0.f;
  for (int kb = 0; kb < nkb; ++kb) {
    __syncthreads();
    const int nk = min(AT, n - kb * AT);
    load_tile<FP16>(K, qkv, r0 + kb * AT, nk, 1536, 512 + head * 64);
    load_tile<FP16>(V, qkv, r0 + kb * AT, nk, 1536, 1024 + head * 64);
    __syncthreads();
    float s[4][4], dp[4][4];
    tile_abt(s, Q, K, ty, tx);
    tile_abt(dp, dO, V, ty, tx);
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int row = 4 * ty + a, col = 4 * tx + b;
        const float p = col < nk ? exp2f(s[a][b] * kSl2 - lse[row]) : 0.f;
        S[row][col] = p * (dp[a][b] - dsum[row]);
      }
    __syncthreads();
    // dq[a][b] += sum_k dS[4ty + a][k] K[k][4tx + b]
#pragma unroll 8
    for (int k = 0; k < AT; ++k) {
      float sa[4], kb4[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) sa[a] = S[4 * ty + a][k];
#pragma unroll
      for (int b = 0; b < 4; ++b) kb4[b] = K[k][4 * tx + b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dq[a][b] = fmaf(sa[a], kb4[b], dq[a][b]);
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int row = 4 * ty + a;
    if (row >= nq) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b)
      dqkv[(q0 + row) * 1536 + head * 64 + 4 * tx + b] = st16<FP16>(dq[a][b] * 0.125f);
  }
  if (tid < nq) {
    lse2_out[(q0 + tid) * 8 + head] = lse[tid];
    dsum_out[(q0 + tid) * 8 + head] = dsum[tid];
  }
}

// per (window, head, key block): dV = P^T dO, dK = dS^T Q / 8
template <bool FP16>
__global__ void __launch_bounds__(256) k_attn_bwd_kv(
    const uint16_t* __restrict__ qkv, const uint16_t* __restrict__ dout,
    const int64_t* __restrict__ win_start, const int32_t* __restrict__ win_len, int nkb,
    const float* __restrict__ lse2, const float* __restrict__ dsum_in,
    uint16_t* __restrict__ dqkv) {
  extern __shared__ float sm[];
  float(*K)[AT + 1] = reinterpret_cast<float(*)[AT + 1]>(sm);
  float(*V)[AT + 1] = K + AT;
  float(*Q)[AT + 1] = V + AT;
  float(*dO)[AT + 1] = Q + AT;
  float(*P)[AT + 1] = dO + AT;   // [q][k]
  float(*dS)[AT + 1] = P + AT;   // [q][k]
  float* lse = reinterpret_cast<float*>(dS + AT);
  float* dsum = lse + AT;
  const int kb = blockIdx.x % nkb, head = (blockIdx.x / nkb) % 8, w = blockIdx.x / (nkb * 8);
  const int n = win_len[w];
  if (kb * AT >= n) return;
  const int64_t r0 = win_start[w];
  const int64_t k0 = r0 + kb * AT;
  const int nk = min(AT, n - kb * AT);
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  load_tile<FP16>(K, qkv, k0, nk, 1536, 512 + head * 64);
  load_tile<FP16>(V, qkv, k0, nk, 1536, 1024 + head * 64);
  float dk[4][4], dv[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) dk[a][b] = dv[a][b] = 0.f;
  const int nqb = (n + AT - 1) / AT;
  for (int qb = 0; qb < nqb; ++qb) {
    __syncthreads();
    const int64_t q0 = r0 + qb * AT;
    const int nq = min(AT, n - qb * AT);
    load_tile<FP16>(Q, qkv, q0, nq, 1536, head * 64);
    load_tile<FP16>(dO, dout, q0, nq, 512, head * 64);
    if (tid < AT) {
      lse[tid] = tid < nq ? lse2[(q0 + tid) * 8 + head] : 0.f;
      dsum[tid] = tid < nq ? dsum_in[(q0 + tid) * 8 + head] : 0.f;
    }
    __syncthreads();
    float s[4][4], dp[4][4];
    tile_abt(s, Q, K, ty, tx);   // [q = 4ty + a][k = 4tx + b]
    tile_abt(dp, dO, V, ty, tx);
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int q = 4 * ty + a, k = 4 * tx + b;
        const float p = (q < nq && k < nk) ? exp2f(s[a][b] * kSl2 - lse[q]) : 0.f;
        P[q][k] = p;
        dS[q][k] = p * (dp[a][b] - dsum[q]);
      }
    __syncthreads();
    // dv[k = 4ty + a][d = 4tx + b] += sum_q P[q][k] dO[q][d]; dk likewise with dS, Q
#pragma unroll 8
    for (int q = 0; q < AT; ++q) {
      float pa[4], sa[4], ob[4], qb4[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        pa[a] = P[q][4 * ty + a];
        sa[a] = dS[q][4 * ty + a];
      }
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        ob[b] = dO[q][4 * tx + b];
        qb4[b] = Q[q][4 * tx + b];
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          dv[a][b] = fmaf(pa[a], ob[b], dv[a][b]);
          dk[a][b] = fmaf(sa[a], qb4[b], dk[a][b]);
        }
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int k = 4 * ty + a;
    if (k >= nk) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      dqkv[(k0 + k) * 1536 + 512 + head * 64 + 4 * tx + b] = st16<FP16>(dk[a][b] * 0.125f);
      dqkv[(k0 + k) * 1536 + 1024 + head * 64 + 4 * tx + b] = st16<FP16>(dv[a][b]);
    }
  }
}

// ---------------------------------------------------------------------------
// Attention backward on the tensor cores (default): the same two passes as
// the fp32 SIMT kernels above, with every product an mma.sync m16n8k16 (16-bit
// operands, fp32 accumulation): per (window, head, 64-query block) 4 warps x
// 16 query rows -- S = Q K^T twice (row statistics, then P), dP = dO V^T,
// dS = P (dP - dsum), dQ += dS K; per (window, head, 64-key block) 4 warps x
// 16 key rows -- S^T = K Q^T, dP^T = V dO^T, dV += P^T dO, dK += dS^T Q. P
// and dS enter the second products as 16-bit A fragments straight from the
// accumulators; K / V / Q / dO tiles are staged by cp.async (double-buffered
// key / query blocks) in XOR-swizzled shared memory and read with ldmatrix
// (.trans for the [key][d] operands of dQ, dV and dK). MOEB_ATTN_BWD=simt
// selects the fp32 kernels.
// ---------------------------------------------------------------------------
template <bool FP16>
__device__ __forceinline__ void bmma(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                     uint32_t a3, uint32_t b0, uint32_t b1) {
  if (FP16)
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  else
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
template <bool FP16>
__device__ __forceinline__ uint32_t bpack2(float x, float y) {
  if (FP16) {
    const __half2 h = __floats2half2_rn(x, y);
    return *reinterpret_cast<const uint32_t*>(&h);
  }
  const __nv_bfloat162 h = __floats2bfloat162_rn(x, y);
  return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ void bcp16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void bcp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bcp_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ int bswz(int row, int col) {  // [64][64] 16-bit, 16-B chunks
  return row * 64 + ((((col >> 3) ^ (row & 7)) << 3) | (col & 7));
}
__device__ __forceinline__ uint32_t bsmem(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bldsm(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void bldsm_t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
// [64 rows][64] 16-bit block (rows >= n zero-filled) -> swizzled tile, async
__device__ __forceinline__ void btile_async(uint16_t* tile, const uint16_t* src, int ld, int n) {
  for (int i = threadIdx.x; i < 64 * 8; i += blockDim.x) {
    const int row = i >> 3, ch = i & 7;
    const bool v = row < n;
    bcp16(bsmem(tile + bswz(row, ch * 8)), src + (int64_t)(v ? row : 0) * ld + ch * 8,
                     v);
  }
}
// A fragments (16 rows of this warp x 64 columns, 4 k-steps) of a swizzled tile
__device__ __forceinline__ void a_frags(const uint16_t* tile, int warp, int lane,
                                        uint32_t (&fr)[4][4]) {
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    const int row = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
    const int col = ks * 16 + (lane >> 4) * 8;
    bldsm(bsmem(tile + bswz(row, col)), fr[ks]);
  }
}
// acc[16 x 64] = A (fragments, 16 x 64) . B^T with B a [64 rows][64] tile
// (row = output column): the S = Q K^T pattern
template <bool FP16>
__device__ __forceinline__ void mm_abt(float (&acc)[8][4], const uint32_t (&fa)[4][4],
                                       const uint16_t* B, int lane) {
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
#pragma unroll
  for (int ks = 0; ks < 4; ++ks)
#pragma unroll
    for (int jp = 0; jp < 4; ++jp) {
      uint32_t b[4];
      const int row = jp * 16 + (lane & 7) + (lane >> 4) * 8;
      const int col = ks * 16 + ((lane >> 3) & 1) * 8;
      bldsm(bsmem(B + bswz(row, col)), b);
      bmma<FP16>(acc[2 * jp], fa[ks][0], fa[ks][1], fa[ks][2], fa[ks][3], b[0], b[1]);
      bmma<FP16>(acc[2 * jp + 1], fa[ks][0], fa[ks][1], fa[ks][2], fa[ks][3], b[2],
                           b[3]);
    }
}
// acc[16 x 64] += X (16 x 64 accumulator-layout values, packed to A
// fragments) . B with B a [64 rows = k][64 cols = n] tile: the O += P V pattern
template <bool FP16>
__device__ __forceinline__ void mm_acc_ab(float (&acc)[8][4], const float (&x)[8][4],
                                          const uint16_t* B, int lane) {
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    const uint32_t a0 = bpack2<FP16>(x[2 * ks][0], x[2 * ks][1]);
    const uint32_t a1 = bpack2<FP16>(x[2 * ks][2], x[2 * ks][3]);
    const uint32_t a2 = bpack2<FP16>(x[2 * ks + 1][0], x[2 * ks + 1][1]);
    const uint32_t a3 = bpack2<FP16>(x[2 * ks + 1][2], x[2 * ks + 1][3]);
#pragma unroll
    for (int jp = 0; jp < 4; ++jp) {
      uint32_t b[4];
      const int row = ks * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
      const int col = jp * 16 + (lane >> 4) * 8;
      bldsm_t(bsmem(B + bswz(row, col)), b);
      bmma<FP16>(acc[2 * jp], a0, a1, a2, a3, b[0], b[1]);
      bmma<FP16>(acc[2 * jp + 1], a0, a1, a2, a3, b[2], b[3]);
    }
  }
}

template <bool FP16>
__global__ void __launch_bounds__(128) k_attn_bwd_q_mma(
    const uint16_t* __restrict__ qkv, const uint16_t* __restrict__ o,
    const uint16_t* __restrict__ dout, const int64_t* __restrict__ win_start,
    const int32_t* __restrict__ win_len, int nqb, uint16_t* __restrict__ dqkv,
    float* __restrict__ lse2_out, float* __restrict__ dsum_out) {
  extern __shared__ __align__(128) unsigned char bsm_q[];  // 48 KB tiles + row sums
  uint16_t* sQ = reinterpret_cast<uint16_t*>(bsm_q);
  uint16_t* sdO = sQ + 64 * 64;
  uint16_t(*sK)[64 * 64] = reinterpret_cast<uint16_t(*)[64 * 64]>(sdO + 64 * 64);
  uint16_t(*sV)[64 * 64] = sK + 2;
  float* sdsum = reinterpret_cast<float*>(sV + 2);
  const int qb = blockIdx.x % nqb, head = (blockIdx.x / nqb) % 8, w = blockIdx.x / (nqb * 8);
  const int n = win_len[w];
  if (qb * 64 >= n) return;
  const int64_t r0 = win_start[w];
  const int64_t q0 = r0 + qb * 64;
  const int nq = min(64, n - qb * 64);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tig = lane & 3;
  const uint16_t* Kg = qkv + r0 * 1536 + 512 + head * 64;
  const uint16_t* Vg = qkv + r0 * 1536 + 1024 + head * 64;
  btile_async(sQ, qkv + q0 * 1536 + head * 64, 1536, nq);
  btile_async(sdO, dout + q0 * 512 + head * 64, 512, nq);
  btile_async(sK[0], Kg, 1536, n);
  bcp_commit();
  if (threadIdx.x < 64) {  // dsum = rowsum(dO o O), fp32 from global
    float acc = 0.f;
    if (threadIdx.x < nq) {
      const uint16_t* orow = o + (q0 + threadIdx.x) * 512 + head * 64;
      const uint16_t* drow = dout + (q0 + threadIdx.x) * 512 + head * 64;
      for (int d = 0; d < 64; ++d) acc += ld16<FP16>(orow + d) * ld16<FP16>(drow + d);
    }
    sdsum[threadIdx.x] = acc;
  }
  bcp_wait0();
  __syncthreads();
  uint32_t qa[4][4], da[4][4];
  a_frags(sQ, warp, lane, qa);
  a_frags(sdO, warp, lane, da);
  const int nkb = (n + 63) / 64;
  // pass A: running max / sum of exp2 per query row (rows g, g + 8)
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  for (int kb = 0; kb < nkb; ++kb) {
    const int cur = kb & 1;
    if (kb + 1 < nkb) btile_async(sK[cur ^ 1], Kg + (int64_t)(kb + 1) * 64 * 1536, 1536,
                                  n - (kb + 1) * 64);
    bcp_commit();
    float s[8][4];
    mm_abt<FP16>(s, qa, sK[cur], lane);
    const int nk = min(64, n - kb * 64);
    float mnew[2] = {mrow[0], mrow[1]};
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int key = j * 8 + tig * 2 + (u & 1);
        s[j][u] = key < nk ? s[j][u] * kSl2 : -INFINITY;
        mnew[u >> 1] = fmaxf(mnew[u >> 1], s[j][u]);
      }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      mnew[h] = fmaxf(mnew[h], __shfl_xor_sync(0xffffffffu, mnew[h], 1));
      mnew[h] = fmaxf(mnew[h], __shfl_xor_sync(0xffffffffu, mnew[h], 2));
    }
    float sum[2] = {0.f, 0.f};
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int u = 0; u < 4; ++u) sum[u >> 1] += exp2f(s[j][u] - mnew[u >> 1]);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      lrow[h] = lrow[h] * exp2f(mrow[h] - mnew[h]) + sum[h];
      mrow[h] = mnew[h];
    }
    bcp_wait0();
    __syncthreads();
  }
  float lse[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    lrow[h] += __shfl_xor_sync(0xffffffffu, lrow[h], 1);
    lrow[h] += __shfl_xor_sync(0xffffffffu, lrow[h], 2);
    lse[h] = mrow[h] + log2f(lrow[h]);
  }
  const int rl[2] = {warp * 16 + g, warp * 16 + g + 8};
  const float ds[2] = {sdsum[rl[0]], sdsum[rl[1]]};
  // pass B: P, dP = dO V^T, dS = P (dP - dsum), dQ += dS K
  float dq[8][4];
#pragma unroll
  for (int j = 0; j < 8; ++j) dq[j][0] = dq[j][1] = dq[j][2] = dq[j][3] = 0.f;
  btile_async(sK[0], Kg, 1536, n);
  btile_async(sV[0], Vg, 1536, n);
  bcp_commit();
  bcp_wait0();
  __syncthreads();
  for (int kb = 0; kb < nkb; ++kb) {
    const int cur = kb & 1;
    if (kb + 1 < nkb) {
      btile_async(sK[cur ^ 1], Kg + (int64_t)(kb + 1) * 64 * 1536, 1536, n - (kb + 1) * 64);
      btile_async(sV[cur ^ 1], Vg + (int64_t)(kb + 1) * 64 * 1536, 1536, n - (kb + 1) * 64);
    }
    bcp_commit();
    float s[8][4], dp[8][4];
    mm_abt<FP16>(s, qa, sK[cur], lane);
    mm_abt<FP16>(dp, da, sV[cur], lane);
    const int nk = min(64, n - kb * 64);
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int key = j * 8 + tig * 2 + (u & 1);
        const float p = key < nk ? exp2f(s[j][u] * kSl2 - lse[u >> 1]) : 0.f;
        s[j][u] = p * (dp[j][u] - ds[u >> 1]);
      }
    mm_acc_ab<FP16>(dq, s, sK[cur], lane);
    bcp_wait0();
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int col = head * 64 + j * 8 + tig * 2;
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (rl[h] < nq)
        *reinterpret_cast<uint32_t*>(dqkv + (q0 + rl[h]) * 1536 + col) =
            bpack2<FP16>(dq[j][2 * h] * 0.125f, dq[j][2 * h + 1] * 0.125f);
  }
  if (tig == 0)
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (rl[h] < nq) {
        lse2_out[(q0 + rl[h]) * 8 + head] = lse[h];
        dsum_out[(q0 + rl[h]) * 8 + head] = ds[h];
      }
}

template <bool FP16>
__global__ void __launch_bounds__(128) k_attn_bwd_kv_mma(
    const uint16_t* __restrict__ qkv, const uint16_t* __restrict__ dout,
    const int64_t* __restrict__ win_start, const int32_t* __restrict__ win_len, int nkb,
    const float* __restrict__ lse2, const float* __restrict__ dsum_in,
    uint16_t* __restrict__ dqkv) {
  extern __shared__ __align__(128) unsigned char bsm_kv[];  // 48 KB tiles + row statistics
  uint16_t* sK = reinterpret_cast<uint16_t*>(bsm_kv);
  uint16_t* sV = sK + 64 * 64;
  uint16_t(*sQ)[64 * 64] = reinterpret_cast<uint16_t(*)[64 * 64]>(sV + 64 * 64);
  uint16_t(*sdO)[64 * 64] = sQ + 2;
  float(*slse)[64] = reinterpret_cast<float(*)[64]>(sdO + 2);
  float(*sds)[64] = slse + 2;
  const int kb = blockIdx.x % nkb, head = (blockIdx.x / nkb) % 8, w = blockIdx.x / (nkb * 8);
  const int n = win_len[w];
  if (kb * 64 >= n) return;
  const int64_t r0 = win_start[w];
  const int64_t k0 = r0 + kb * 64;
  const int nk = min(64, n - kb * 64);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tig = lane & 3;
  const uint16_t* Qg = qkv + r0 * 1536 + head * 64;
  const uint16_t* dOg = dout + r0 * 512 + head * 64;
  auto stage = [&](int qb, int buf) {
    btile_async(sQ[buf], Qg + (int64_t)qb * 64 * 1536, 1536, n - qb * 64);
    btile_async(sdO[buf], dOg + (int64_t)qb * 64 * 512, 512, n - qb * 64);
    if (threadIdx.x < 64) {
      const int q = qb * 64 + threadIdx.x;
      slse[buf][threadIdx.x] = q < n ? lse2[(r0 + q) * 8 + head] : 0.f;
      sds[buf][threadIdx.x] = q < n ? dsum_in[(r0 + q) * 8 + head] : 0.f;
    }
  };
  btile_async(sK, qkv + k0 * 1536 + 512 + head * 64, 1536, nk);
  btile_async(sV, qkv + k0 * 1536 + 1024 + head * 64, 1536, nk);
  stage(0, 0);
  bcp_commit();
  bcp_wait0();
  __syncthreads();
  uint32_t ka[4][4], va[4][4];
  a_frags(sK, warp, lane, ka);
  a_frags(sV, warp, lane, va);
  const int kl[2] = {warp * 16 + g, warp * 16 + g + 8};  // this thread's key rows
  float dk[8][4], dv[8][4];
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int u = 0; u < 4; ++u) dk[j][u] = dv[j][u] = 0.f;
  const int nqb = (n + 63) / 64;
  for (int qb = 0; qb < nqb; ++qb) {
    const int cur = qb & 1;
    if (qb + 1 < nqb) stage(qb + 1, cur ^ 1);
    bcp_commit();
    float s[8][4], dp[8][4];
    mm_abt<FP16>(s, ka, sQ[cur], lane);   // S^T [key][query]
    mm_abt<FP16>(dp, va, sdO[cur], lane); // dP^T
    const int nq = min(64, n - qb * 64);
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = j * 8 + tig * 2 + (u & 1);
        const bool ok = q < nq && kl[u >> 1] < nk;
        const float p = ok ? exp2f(s[j][u] * kSl2 - slse[cur][q]) : 0.f;
        s[j][u] = p;                                   // P^T
        dp[j][u] = p * (dp[j][u] - sds[cur][q]);      // dS^T
      }
    mm_acc_ab<FP16>(dv, s, sdO[cur], lane);
    mm_acc_ab<FP16>(dk, dp, sQ[cur], lane);
    bcp_wait0();
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int col = head * 64 + j * 8 + tig * 2;
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (kl[h] < nk) {
        uint16_t* row = dqkv + (k0 + kl[h]) * 1536;
        *reinterpret_cast<uint32_t*>(row + 512 + col) =
            bpack2<FP16>(dk[j][2 * h] * 0.125f, dk[j][2 * h + 1] * 0.125f);
        *reinterpret_cast<uint32_t*>(row + 1024 + col) =
            bpack2<FP16>(dv[j][2 * h], dv[j][2 * h + 1]);
      }
  }
}

// F[row] = [tok16[token[row]] (2048) | lay16[layer[row]] (512)], 16-bit
__global__ void k_gather_inputs16(const uint16_t* __restrict__ tok16,
                                  const uint16_t* __restrict__ lay16,
                                  const int32_t* __restrict__ token, const int32_t* __restrict__ layer,
                                  int64_t M, uint16_t* __restrict__ F) {
  const int64_t r = blockIdx.x;
  if (r >= M) return;
  const uint4* t = reinterpret_cast<const uint4*>(tok16 + (int64_t)token[r] * 2048);
  const uint4* l = reinterpret_cast<const uint4*>(lay16 + (int64_t)layer[r] * 512);
  uint4* o = reinterpret_cast<uint4*>(F + r * 2560);
  for (int i = threadIdx.x; i < 320; i += blockDim.x) o[i] = i < 256 ? t[i] : l[i - 256];
}

// dlay[layer[row]][c] += d[row][c] (d [M][ld] 16-bit, 512 columns): block =
// 32 columns x a row range, per-layer partials in shared memory
template <bool FP16>
__global__ void k_layer_emb_grad(const uint16_t* __restrict__ d, int ld, int64_t M,
                                 const int32_t* __restrict__ layer, int nl,
                                 float* __restrict__ dlay) {
  extern __shared__ float acc[];  // [nl][32]
  for (int i = threadIdx.x; i < nl * 32; i += blockDim.x) acc[i] = 0.f;
  __syncthreads();
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  const int64_t per = (M + gridDim.y - 1) / gridDim.y;
  const int64_t a = (int64_t)blockIdx.y * per, b = min(M, a + per);
  for (int64_t r = a + (threadIdx.x >> 5); r < b; r += blockDim.x >> 5)
    atomicAdd(&acc[layer[r] * 32 + (threadIdx.x & 31)], ld16<FP16>(d + r * ld + c));
  __syncthreads();
  for (int i = threadIdx.x; i < nl * 32; i += blockDim.x)
    if (acc[i] != 0.f) atomicAdd(dlay + (i / 32) * 512 + blockIdx.x * 32 + (i % 32), acc[i]);
}

template <bool FP16>
__global__ void k_cast16(const float* __restrict__ x, int64_t n, uint16_t* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = st16<FP16>(x[i]);
}

__global__ void k_sumsq(const float* __restrict__ g, int64_t n, double* __restrict__ out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    acc += (double)g[i] * (double)g[i];
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
    atomicAdd(out, t);
  }
}

// torch.optim.AdamW (maximize=False, amsgrad=False): p *= 1 - lr wd;
// m = b1 m + (1 - b1) g; v = b2 v + (1 - b2) g^2;
// p -= lr / bc1 * m / (sqrt(v) / sqrt(bc2) + eps); g = grad * gscale
__global__ void k_adamw(float* __restrict__ p, const float* __restrict__ grad,
                        float* __restrict__ m, float* __restrict__ v, int64_t n, float lr,
                        float b1, float b2, float eps, float wd, float bc1, float bc2,
                        float gscale) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float g = grad[i] * gscale;
    float pi = p[i] * (1.f - lr * wd);
    const float mi = fmaf(1.f - b1, g - m[i], m[i]);  // torch: exp_avg.lerp_(grad, 1 - beta1)
    const float vi = b2 * v[i] + (1.f - b2) * g * g;
    m[i] = mi;
    v[i] = vi;
    const float denom = sqrtf(vi) / sqrtf(bc2) + eps;
    pi -= (lr / bc1) * mi / denom;
    p[i] = pi;
  }
}

inline unsigned grid_for(int64_t n, int threads = 256) {
  const int64_t b = (n + threads - 1) / threads;
  const int64_t cap = 16LL * moeb::num_sms();
  return (unsigned)(b < cap ? (b > 0 ? b : 1) : cap);
}

}  // namespace

#define MOEB_FP16_SWITCH(fp16, KERNEL, ...) \
  do {                                      \
    if (fp16)                               \
      KERNEL<true> __VA_ARGS__;             \
    else                                    \
      KERNEL<false> __VA_ARGS__;            \
  } while (0)

extern "C" int moeb_transpose16(const void* in, int64_t R, int C, int ld_in, void* out,
                                int ld_out, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(in && out && R >= 0 && C >= 1, "bad arguments");
  if (R == 0) return MOEB_OK;
  dim3 grid((unsigned)((C + 31) / 32), (unsigned)((R + 31) / 32));
  k_transpose16<<<grid, dim3(32, 8), 0, moeb::as_stream(stream)>>>(
      static_cast<const uint16_t*>(in), R, C, ld_in, static_cast<uint16_t*>(out), ld_out);
  return moeb::check_launch("k_transpose16");
}

extern "C" int moeb_colsum16(const void* in, int64_t M, int N, int ld, float* out, int fp16,
                             void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(in && out && M >= 0 && N >= 1, "bad arguments");
  if (M == 0) return MOEB_OK;
  dim3 grid((unsigned)((N + 127) / 128), (unsigned)std::min<int64_t>(256, (M + 255) / 256));
  MOEB_FP16_SWITCH(fp16, k_colsum16, <<<grid, 128, 0, moeb::as_stream(stream)>>>(
                                         static_cast<const uint16_t*>(in), M, N, ld, out));
  return moeb::check_launch("k_colsum16");
}

extern "C" int moeb_layernorm_bwd16(const void* dy16, const void* x16, const float* w, int64_t M,
                                    float eps, void* dx16, float* dw, float* db, int fp16,
                                    void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(dy16 && x16 && w && dx16 && dw && db && M >= 0, "bad arguments");
  if (M == 0) return MOEB_OK;
  MOEB_FP16_SWITCH(fp16, k_layernorm_bwd16, <<<grid_for(M * 32), 256, 0, moeb::as_stream(stream)>>>(
                                                static_cast<const uint16_t*>(dy16),
                                                static_cast<const uint16_t*>(x16), w, M, eps,
                                                static_cast<uint16_t*>(dx16), dw, db));
  return moeb::check_launch("k_layernorm_bwd16");
}

extern "C" int moeb_relu_bwd16(void* d, const void* act, int64_t n, int fp16, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(d && act && n >= 0, "bad arguments");
  if (n == 0) return MOEB_OK;
  MOEB_FP16_SWITCH(fp16, k_relu_bwd16, <<<grid_for(n), 256, 0, moeb::as_stream(stream)>>>(
                                           static_cast<uint16_t*>(d),
                                           static_cast<const uint16_t*>(act), n));
  return moeb::check_launch("k_relu_bwd16");
}

extern "C" int moeb_gelu_fwd16(const void* u, void* g, int64_t n, int fp16, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(u && g && n >= 0, "bad arguments");
  if (n == 0) return MOEB_OK;
  MOEB_FP16_SWITCH(fp16, k_gelu_fwd16, <<<grid_for(n), 256, 0, moeb::as_stream(stream)>>>(
                                           static_cast<const uint16_t*>(u),
                                           static_cast<uint16_t*>(g), n));
  return moeb::check_launch("k_gelu_fwd16");
}

extern "C" int moeb_gelu_bwd16(void* d, const void* u, int64_t n, int fp16, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(d && u && n >= 0, "bad arguments");
  if (n == 0) return MOEB_OK;
  MOEB_FP16_SWITCH(fp16, k_gelu_bwd16, <<<grid_for(n), 256, 0, moeb::as_stream(stream)>>>(
                                           static_cast<uint16_t*>(d),
                                           static_cast<const uint16_t*>(u), n));
  return moeb::check_launch("k_gelu_bwd16");
}

extern "C" int moeb_bce_logits_grad(const float* z, const uint64_t* truth, int64_t M, int E,
                                    float scale, void* dz16, double* loss_sum, int fp16,
                                    void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(z && truth && dz16 && loss_sum && M >= 0 && E >= 1 && E <= 256, "bad arguments");
  if (M == 0) return MOEB_OK;
  const int W = (E + 63) / 64;
  MOEB_FP16_SWITCH(fp16, k_bce_grad, <<<grid_for(M * E), 256, 0, moeb::as_stream(stream)>>>(
                                         z, truth, W, M, E, scale,
                                         static_cast<uint16_t*>(dz16), loss_sum));
  return moeb::check_launch("k_bce_grad");
}

extern "C" int moeb_attention_bwd(const void* qkv, const void* o, const void* dout,
                                  const int64_t* win_start, const int32_t* win_len, int n_windows,
                                  int max_len, void* dqkv, float* lse2, float* dsum, int fp16,
                                  void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(qkv && o && dout && win_start && win_len && dqkv && lse2 && dsum, "null argument");
  MOEB_REQUIRE(n_windows >= 0 && max_len >= 1 && max_len <= 4096, "bad window arguments");
  if (n_windows == 0) return MOEB_OK;
  cudaStream_t s = moeb::as_stream(stream);
  const int nb = (max_len + AT - 1) / AT;
  const char* env = getenv("MOEB_ATTN_BWD");
  if (!(env && !strcmp(env, "simt"))) {  // tensor cores (mma.sync)
    const unsigned grid = (unsigned)((int64_t)n_windows * 8 * nb);
    const int sq = 6 * 64 * 64 * 2 + 64 * 4, skv = 6 * 64 * 64 * 2 + 4 * 64 * 4;
    moeb::set_smem(k_attn_bwd_q_mma<true>, sq);
    moeb::set_smem(k_attn_bwd_q_mma<false>, sq);
    moeb::set_smem(k_attn_bwd_kv_mma<true>, skv);
    moeb::set_smem(k_attn_bwd_kv_mma<false>, skv);
    MOEB_FP16_SWITCH(fp16, k_attn_bwd_q_mma, <<<grid, 128, sq, s>>>(
                                                 static_cast<const uint16_t*>(qkv),
                                                 static_cast<const uint16_t*>(o),
                                                 static_cast<const uint16_t*>(dout), win_start,
                                                 win_len, nb, static_cast<uint16_t*>(dqkv), lse2,
                                                 dsum));
    if (int rc = moeb::check_launch("k_attn_bwd_q_mma")) return rc;
    MOEB_FP16_SWITCH(fp16, k_attn_bwd_kv_mma, <<<grid, 128, skv, s>>>(
                                                  static_cast<const uint16_t*>(qkv),
                                                  static_cast<const uint16_t*>(dout), win_start,
                                                  win_len, nb, lse2, dsum,
                                                  static_cast<uint16_t*>(dqkv)));
    return moeb::check_launch("k_attn_bwd_kv_mma");
  }
  const size_t smq = sizeof(float) * (5 * AT * (AT + 1) + 2 * AT);
  const size_t smkv = sizeof(float) * (6 * AT * (AT + 1) + 2 * AT);
  moeb::set_smem(k_attn_bwd_q<true>, (int)smq);
  moeb::set_smem(k_attn_bwd_q<false>, (int)smq);
  moeb::set_smem(k_attn_bwd_kv<true>, (int)smkv);
  moeb::set_smem(k_attn_bwd_kv<false>, (int)smkv);
  const unsigned grid = (unsigned)((int64_t)n_windows * 8 * nb);
  MOEB_FP16_SWITCH(fp16, k_attn_bwd_q, <<<grid, 256, smq, s>>>(
                                           static_cast<const uint16_t*>(qkv),
                                           static_cast<const uint16_t*>(o),
                                           static_cast<const uint16_t*>(dout), win_start, win_len,
                                           nb, static_cast<uint16_t*>(dqkv), lse2, dsum));
  if (int rc = moeb::check_launch("k_attn_bwd_q")) return rc;
  MOEB_FP16_SWITCH(fp16, k_attn_bwd_kv, <<<grid, 256, smkv, s>>>(
                                            static_cast<const uint16_t*>(qkv),
                                            static_cast<const uint16_t*>(dout), win_start,
                                            win_len, nb, lse2, dsum,
                                            static_cast<uint16_t*>(dqkv)));
  return moeb::check_launch("k_attn_bwd_kv");
}

extern "C" int moeb_gather_inputs16(const void* tok16, const void* lay16, const int32_t* token,
                                    const int32_t* layer, int64_t M, void* F, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(tok16 && lay16 && token && layer && F && M >= 0, "bad arguments");
  if (M == 0) return MOEB_OK;
  k_gather_inputs16<<<(unsigned)M, 128, 0, moeb::as_stream(stream)>>>(
      static_cast<const uint16_t*>(tok16), static_cast<const uint16_t*>(lay16), token, layer, M,
      static_cast<uint16_t*>(F));
  return moeb::check_launch("k_gather_inputs16");
}

extern "C" int moeb_layer_emb_grad(const void* d, int ld, int64_t M, const int32_t* layer, int nl,
                                   float* dlay, int fp16, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(d && layer && dlay && M >= 0 && nl >= 1 && nl <= 64, "bad arguments");
  if (M == 0) return MOEB_OK;
  dim3 grid(512 / 32, (unsigned)std::min<int64_t>(64, (M + 255) / 256));
  MOEB_FP16_SWITCH(fp16, k_layer_emb_grad,
                   <<<grid, 256, sizeof(float) * nl * 32, moeb::as_stream(stream)>>>(
                       static_cast<const uint16_t*>(d), ld, M, layer, nl, dlay));
  return moeb::check_launch("k_layer_emb_grad");
}

extern "C" int moeb_cast_f32_to_16(const float* x, int64_t n, void* y, int fp16, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(x && y && n >= 0, "bad arguments");
  if (n == 0) return MOEB_OK;
  MOEB_FP16_SWITCH(fp16, k_cast16, <<<grid_for(n), 256, 0, moeb::as_stream(stream)>>>(
                                       x, n, static_cast<uint16_t*>(y)));
  return moeb::check_launch("k_cast16");
}

extern "C" int moeb_sumsq_f32(const float* g, int64_t n, double* out, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(g && out && n >= 0, "bad arguments");
  if (n == 0) return MOEB_OK;
  k_sumsq<<<grid_for(n), 256, 0, moeb::as_stream(stream)>>>(g, n, out);
  return moeb::check_launch("k_sumsq");
}

extern "C" int moeb_adamw_f32(float* p, const float* g, float* m, float* v, int64_t n, float lr,
                              float beta1, float beta2, float eps, float weight_decay, int step,
                              float gscale, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(p && g && m && v && n >= 0 && step >= 1, "bad arguments");
  if (n == 0) return MOEB_OK;
  const float bc1 = (float)(1.0 - std::pow((double)beta1, step));
  const float bc2 = (float)(1.0 - std::pow((double)beta2, step));
  k_adamw<<<grid_for(n), 256, 0, moeb::as_stream(stream)>>>(p, g, m, v, n, lr, beta1, beta2, eps,
                                                            weight_decay, bc1, bc2, gscale);
  return moeb::check_launch("k_adamw");
}
