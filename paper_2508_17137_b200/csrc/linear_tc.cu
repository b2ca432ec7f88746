// K3t -- learned_linear predictor with the column sums on the tensor cores
// (E = 64, L <= 32; the default path of moeb_linear_predict_counts when the
// caller provides a workspace and asks for no logits).
//
// Reference: LearnedLinearPredictor.predict (predictors.py:262-268),
// feature_vector / update_history (learner.py:52-72), top_k_experts and the
// threshold rule (learner.py:164-181).
//
// The scores obey the recurrence of linear.cu's header:
//   z_0 = b_l,  z_{t+1} = decay * z_t + G_t,
//   G_t = (1 - decay) b_l + sum_{e in x_t} W_h[:, e]   (b_l = W[:, l] + W[:, L+E])
// G_t for 128 (prompt, layer) streams at one token is a GEMM with exact 0/1
// inputs: A = [x_t | onehot(l)] (128 x (64 + 32) fp16) times B^T, B = the
// 64 x 96 table [W_h | (1 - decay) b] scaled by a power of two and split
// into two fp16 limbs stacked along N (N = 128: output columns 0..63 sum the
// hi limbs, 64..127 the lo limbs). The hi limbs are multiples of 8 below
// 2^14, so their fp32 sums are exact whatever the accumulator's rounding; the
// lo limbs are < 4 in magnitude, so their accumulation error is ~2^-30 of
// the scores. One CTA owns 128 streams for their whole
// token loop: thread r (TMEM lane r) keeps stream r's 64 scores z in fp32
// registers, selects on z_t, writes row t+2 of A (mask bits -> fp16 0/1 in
// the 128-byte-swizzled K-major layout the MMA reads), then adds G_t read
// from TMEM (tcgen05.ld) as hi + lo and one FFMA per expert. A single thread
// issues the 6 tcgen05.mma (M128 N128 K16) per token into one of two TMEM
// accumulators, so the MMA for token t+1 runs while token t is selected.
//
// Exactness. fp32 is a filter, not the answer: every stream carries a
// rigorous running bound E_t on |z_t(fp32) - z_t(exact)| (fp32 rounding of
// hi + lo and of the FFMA against the row's actual score magnitude, the limb
// split's representation error; 2^-23 per rounding, which covers truncating
// as well as round-to-nearest arithmetic). A row whose k-th and
// (k+1)-th scores are within 2 E_t (or, in threshold mode, with a score
// within E_t of 0, or with equal scores at the cut) is "ambiguous": its
// mask is recomputed by k_linear_rows_exact in fp64 exactly as the
// reference does (numpy's h *= decay; h += 1 order, then W @ f) with ties to
// the lower expert id. Every other row's top-k set provably equals the one
// the reference's fp64 scores give (their deviation from the exact scores,
// ~1e-16 relative, is inside the slack added to E_0). If more rows are
// ambiguous than the workspace list holds, the whole call is redone by the
// fp64 kernel (k_linear_predict, gated on the overflow flag).
#include <cuda_fp16.h>

#include <cstdlib>

#include "common.cuh"
#include "tc_sm100.cuh"

namespace moeb {
int launch_linear_fp64_gated(const uint64_t* truth, const int64_t* row_off, int P, int L, int E,
                             const double* W, double decay, int budget, int threshold, int warmup,
                             uint64_t* pred, int64_t* counts, const int* gate, int gate_cap,
                             cudaStream_t s);
}

namespace {

using namespace moeb::tc;

constexpr int kRows = 128;      // streams per CTA (TMEM lanes, MMA M)
// A-tile ring: token t's MMA reads stage t % 2 while the threads write
// token t + 1's rows into the other (the stage of token t - 1, whose MMA
// completed before its scores were read)
constexpr int kStages = 2;
constexpr int kThreads = 160;   // 4 score/selection warps + 1 MMA warp
constexpr int kTileA = kRows * 128;  // 128 rows x 64 fp16, SW128
constexpr int kTileB = 128 * 128;    // 128 rows (hi outputs, lo outputs) x 64 fp16, SW128
constexpr int kTileL = 128 * 64;     // 128 rows x 32 fp16 (layer one-hot / bias rows), SW64
constexpr int kTabBytes = kTileB + kTileL;  // Bx (experts, SW128), Bl (layer bias, SW64)
constexpr int kLookahead = 2;   // mask rows loaded this many tokens ahead
// One N = 128 accumulator (hi | lo limb columns), not two: token t + 1's MMA
// is issued when token t's scores have been read and runs while token t + 1
// is selected, so it needs no second buffer (128 TMEM columns per CTA)
constexpr int kTmemCols = 128;

// smem layout (69 KB per CTA)
constexpr int OFF_A = 0;
constexpr int OFF_B = OFF_A + kStages * kTileA;   // Bx (SW128) then Bl (SW64)
constexpr int OFF_AL = OFF_B + kTabBytes;         // constant one-hot tile (SW64)
constexpr int OFF_LUT = OFF_AL + kTileL;          // nibble -> 4 x fp16 {0, 1}
constexpr int kXSlots = 4;      // per-stream ring of mask rows (cp.async, kLookahead + 2 <= 4)
constexpr int OFF_XR = OFF_LUT + 16 * 8;          // [kXSlots][kRows] uint64 mask rows
constexpr int OFF_BAR = OFF_XR + kXSlots * kRows * 8;
constexpr int kSmem = OFF_BAR + 64 + 1024;        // + alignment slack

struct TcConsts {
  float lam;     // fp32(decay)
  float cmax;    // max |W_h| (scaled)
  float cbmax;   // max |(1-decay) b| (scaled)
  float eta;     // max limb representation error (scaled)
  float e0;      // initial bound (scaled)
  float inv_scale;
  int pad;
  float zr0;     // rigorous bound on |z_0| (scaled, with margin): the first key range
  int use_q15;   // the error bound's limit leaves the 15-bit keys useful
};
static_assert(sizeof(TcConsts) <= 64, "TcConsts must fit its workspace slot");

// workspace layout
constexpr size_t WS_TAB = 0;                    // B tiles (kTabBytes)
constexpr size_t WS_CONST = kTabBytes;          // TcConsts
constexpr size_t WS_Z0 = WS_CONST + 64;         // fp32 [L][64] initial scores (scaled)
inline size_t ws_counts_off(int L) { return WS_Z0 + (size_t)L * 64 * 4; }
inline size_t ws_list_n_off(int L) { return ws_counts_off(L) + 8 * (size_t)(2 + 2 * L); }
inline size_t ws_list_off(int L) { return (ws_list_n_off(L) + 8 + 15) & ~(size_t)15; }
// refine list (after the fp64 list): entries of kRefineFloats floats = the
// row's 64 fp32 scores, then {E, 0, prompt, token * L + layer}
constexpr int kRefineFloats = 68;

// 64-byte swizzle (K = 32 fp16 per row; 8-row atoms of 512 B): byte offset
// of 16-B chunk `chunk` (0..3) of row `row`
__host__ __device__ inline int sw64(int row, int chunk) {
  return (row >> 3) * 512 + (row & 7) * 64 + ((chunk ^ ((row >> 1) & 3)) << 4);
}

__host__ __device__ inline int sw128(int row, int chunk) {  // byte offset of a 16-B chunk
  return row * 128 + ((chunk ^ (row & 7)) << 4);
}

// ---------------------------------------------------------------------------
// Per-call preparation (one CTA): scaled fp16 limb tables in the MMA's smem
// layout, initial scores, error-bound constants.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_linear_tc_prep(const double* __restrict__ W, int L,
                                                        double decay, int kmax,
                                                        unsigned char* __restrict__ ws) {
  const int E = 64, F = L + E + 1;
  __shared__ double red[256];
  __shared__ double s_scale;
  __shared__ double s_zb[64];
  __shared__ double s_b0[64];
  const int tid = threadIdx.x;
  auto entry = [&](int i, int k) -> double {  // B[i][k], k < 64: W_h; 64 <= k < 96: bias
    if (k < 64) return W[(size_t)i * F + L + k];
    const int l = k - 64;
    return l < L ? (1.0 - decay) * (W[(size_t)i * F + l] + W[(size_t)i * F + L + E]) : 0.0;
  };
  // 1. max |entry|
  double m = 0.0;
  for (int j = tid; j < 64 * 96; j += 256) m = fmax(m, fabs(entry(j / 96, j % 96)));
  red[tid] = m;
  __syncthreads();
  for (int o = 128; o; o >>= 1) {
    if (tid < o) red[tid] = fmax(red[tid], red[tid + o]);
    __syncthreads();
  }
  if (tid == 0) {
    int e = 0;
    const double M = red[0];
    if (M > 0.0) frexp(M, &e);
    s_scale = M > 0.0 ? ldexp(1.0, 14 - e) : 1.0;  // M * scale in [2^13, 2^14)
  }
  __syncthreads();
  const double sc = s_scale;
  // 2. limbs in the SW128 K-major layout: tile (k >= 64), rows i (hi) and
  //    64 + i (lo). hi = w rounded to a multiple of 8 (|hi| <= 2^14: exact in
  //    fp16, and any sum of up to 2^21 of them is exact in fp32), lo = the
  //    fp16 of the remainder (|lo| <= 4)
  double eta = 0.0, cmax = 0.0, cbmax = 0.0;
  unsigned char* tab = ws + WS_TAB;
  for (int j = tid; j < 64 * 128; j += 256) {
    const int i = j / 128, k = j % 128;  // k in [96, 128): zero padding of the bias tile
    const double w = k < 96 ? entry(i, k) * sc : 0.0;
    const double hq = 8.0 * rint(w * 0.125);
    const __half hi = __double2half(hq);
    const double r = w - hq;
    const __half lo = __double2half(r);
    eta = fmax(eta, fabs(r - (double)__half2float(lo)));
    if (k < 64) cmax = fmax(cmax, fabs(w));
    else cbmax = fmax(cbmax, fabs(w));
    const int kk = k & 63;
    // output column of expert i: within each 32-column half, experts m and
    // m + 16 on columns 2m and 2m + 1, so one tcgen05.ld register pair holds
    // the score pair the main kernel keeps in one float2
    const int ci = (i & 32) + 2 * (i & 15) + ((i >> 4) & 1);
    if (k < 64) {  // Bx: SW128, K = 64
      *reinterpret_cast<__half*>(tab + sw128(ci, kk >> 3) + (kk & 7) * 2) = hi;
      *reinterpret_cast<__half*>(tab + sw128(64 + ci, kk >> 3) + (kk & 7) * 2) = lo;
    } else if (kk < 32) {  // Bl: SW64, K = 32 (layers)
      *reinterpret_cast<__half*>(tab + kTileB + sw64(ci, kk >> 3) + (kk & 7) * 2) = hi;
      *reinterpret_cast<__half*>(tab + kTileB + sw64(64 + ci, kk >> 3) + (kk & 7) * 2) = lo;
    }
  }
  // 3. initial scores z_0 = b_l (scaled, fp32)
  float* z0 = reinterpret_cast<float*>(ws + WS_Z0);
  for (int j = tid; j < L * 64; j += 256) {
    const int l = j / 64, i = j % 64;
    z0[j] = (float)((W[(size_t)i * F + l] + W[(size_t)i * F + L + E]) * sc);
  }
  // 4. |z| bound per expert: max_l |b_il| + (sum of the kmax largest |W_h[i,:]|) / (1 - decay)
  if (tid < 64) {
    const int i = tid;
    double bmax = 0.0;
    for (int l = 0; l < L; ++l)
      bmax = fmax(bmax, fabs(W[(size_t)i * F + l] + W[(size_t)i * F + L + E]));
    double smax = 0.0, last = INFINITY;
    int taken = 0;
    while (taken < kmax && taken < 64) {  // kmax largest |W_h[i, e]| (with multiplicity)
      double best = -1.0;
      int cnt = 0;
      for (int e = 0; e < 64; ++e) {
        const double v = fabs(W[(size_t)i * F + L + e]);
        if (v < last && v > best) best = v;
      }
      for (int e = 0; e < 64; ++e) cnt += fabs(W[(size_t)i * F + L + e]) == best;
      if (best < 0.0) break;
      const int use = min(cnt, kmax - taken);
      smax += use * best;
      taken += use;
      last = best;
    }
    s_zb[i] = (bmax + smax / (1.0 - decay)) * sc;
    s_b0[i] = bmax * sc;
  }
  red[tid] = eta;
  __syncthreads();
  for (int o = 128; o; o >>= 1) {
    if (tid < o) red[tid] = fmax(red[tid], red[tid + o]);
    __syncthreads();
  }
  const double eta_all = red[0];
  __syncthreads();
  red[tid] = cmax;
  __syncthreads();
  for (int o = 128; o; o >>= 1) {
    if (tid < o) red[tid] = fmax(red[tid], red[tid + o]);
    __syncthreads();
  }
  const double cmax_all = red[0];
  __syncthreads();
  red[tid] = cbmax;
  __syncthreads();
  for (int o = 128; o; o >>= 1) {
    if (tid < o) red[tid] = fmax(red[tid], red[tid + o]);
    __syncthreads();
  }
  if (tid == 0) {
    double zb = 0.0;
    for (int i = 0; i < 64; ++i) zb = fmax(zb, s_zb[i]);
    TcConsts c;
    c.lam = (float)decay;
    c.cmax = (float)(cmax_all * (1.0 + 1e-6));
    c.cbmax = (float)(red[0] * (1.0 + 1e-6));
    c.eta = (float)(eta_all * (1.0 + 1e-6));
    // rounding of z_0 to fp32, plus slack for the reference's own fp64
    // deviation from the exact scores (~1e-16 relative)
    c.e0 = (float)(ldexp(zb, -23) + 1e-12 * sc);
    c.inv_scale = (float)(1.0 / sc);
    c.pad = 0;
    double b0 = 0.0;
    for (int i = 0; i < 64; ++i) b0 = fmax(b0, s_b0[i]);
    c.zr0 = (float)(b0 * (1.0 + 1e-3) + 1.0);
    // the running bound E_t approaches 2^-23 (|z| + 2|G|) / (1 - decay) while
    // a key step is ~2 (decay |z| + |G|) / 32766: the keys decide rows only
    // while E stays well below a step
    c.use_q15 = ldexp(32766.0 * 4.0, -23) / (1.0 - decay) < 1.0 ? 1 : 0;
    *reinterpret_cast<TcConsts*>(ws + WS_CONST) = c;
  }
}

// ---------------------------------------------------------------------------
// Main kernel.
// ---------------------------------------------------------------------------
struct TcArgs {
  const uint64_t* truth;
  const int64_t* row_off;
  int P, L, budget, threshold, warmup, kmax;
  int64_t n_streams;
  int n_groups;
  const unsigned char* ws;  // tables + consts + z0
  int64_t* wcounts;         // [2 + 2L] scratch counters
  int* list_n;
  int64_t* list;
  int list_cap;
  int* refine_n;
  float* refine;
  int refine_cap;
  uint64_t* pred;
};

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ uint32_t ukey(float z) {
  const uint32_t b = __float_as_uint(z);
  return b ^ ((uint32_t)((int32_t)b >> 31) | 0x80000000u);
}
__device__ __forceinline__ float unkey(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k ^ 0x80000000u) : ~k);
}

// mask row of token j of this thread's stream -> ring slot j % kXSlots
// (zeros past the stream's end: cp.async with source size 0)
__device__ __forceinline__ void x_async(uint32_t xslot, int j, const uint64_t* xs, int L, int T) {
  const uint32_t dst = xslot + (uint32_t)(j & (kXSlots - 1)) * (kRows * 8u);
  const uint64_t* src = xs + (int64_t)(j < T ? j : 0) * L;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n"
               "cp.async.commit_group;" ::"r"(dst), "l"(src), "r"(j < T ? 8 : 0)
               : "memory");
}
template <int N>
__device__ __forceinline__ void x_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ uint64_t x_at(uint32_t xslot, int j) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];"
               : "=l"(v)
               : "r"(xslot + (uint32_t)(j & (kXSlots - 1)) * (kRows * 8u)));
  return v;
}

// refine-list slots are handed to warps in chunks; unused ones are marked
// (header offset -1) so the refine kernel skips them
constexpr int kRChunk = 64;
struct TcArgs;
__device__ __forceinline__ void refine_release(const TcArgs& a, int from, int to, int lane);

// write stream row `row`'s A entries for mask x (or zeros) into the tile at
// shared address `tile`: 16 nibbles through a 16-entry x 8-byte LUT (four fp16
// {0, 1}; entries on distinct banks, so the warp's random lookups never
// conflict), 8 shared 16-byte stores in the SW128 layout
__device__ __forceinline__ void put_row(uint32_t tile, uint32_t lut, int row, uint64_t x) {
  const uint32_t xl = (uint32_t)x, xh = (uint32_t)(x >> 32);
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const uint32_t b = c < 4 ? xl >> (8 * c) : xh >> (8 * (c - 4));
    uint32_t v0, v1, v2, v3;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v0), "=r"(v1) : "r"(lut + ((b << 3) & 0x78u)));
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v2), "=r"(v3) : "r"(lut + ((b >> 1) & 0x78u)));
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(tile + sw128(row, c)), "r"(v0),
                 "r"(v1), "r"(v2), "r"(v3)
                 : "memory");
  }
}

__device__ __forceinline__ int group_tmax(const TcArgs& a, int64_t s0) {
  const int64_t s1 = min(s0 + kRows, a.n_streams);
  int tmax = 0;
  for (int64_t p = s0 / a.L; p * a.L < s1; ++p) {
    const int T = (int)((a.row_off[p + 1] - a.row_off[p]) / a.L);
    tmax = max(tmax, T);
  }
  return tmax;
}

// Exact selection on 32-bit order-preserving keys of fp32 scores z[64]
// (natural element order) carrying the error bound E: the top-k mask, or
// the threshold mask; `amb` when the fp32 bound cannot decide the row (the
// k-th and (k+1)-th scores within 2E, ties at the cut, or in threshold mode a
// score within E of 0). zabs = max |z| (for the next bound).
template <int KT>
__device__ __forceinline__ uint64_t select_exact32(const float (&z)[64], int k_rt, int threshold,
                                                   float E, bool& amb, float& zabs) {
  uint64_t pm = 0;
  amb = false;
  zabs = 0.0f;
  if (threshold) {
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      pm |= (z[i] > 0.0f ? 1ull : 0ull) << i;
      amb |= fabsf(z[i]) <= E;
      zabs = fmaxf(zabs, fabsf(z[i]));
    }
    return pm;
  }
  const int k = KT > 0 ? KT : k_rt;
  uint32_t key[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) key[i] = ukey(z[i]);
  uint32_t bound = 0, vk = 0, vk1 = 0, vmax = 0;
  bool found = true;
#pragma unroll
  for (int it = 0; it <= (KT > 0 ? KT : 16); ++it) {
    if (KT == 0 && it > k) break;
    const uint32_t bm1 = bound - 1u;
    uint32_t m4[4] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu};
#pragma unroll
    for (int i = 0; i < 64; ++i) m4[i & 3] = min(m4[i & 3], bm1 - key[i]);
    const uint32_t tm = min(min(m4[0], m4[1]), min(m4[2], m4[3]));
    found = found && (it == 0 || (bound != 0u && tm <= bm1));
    const uint32_t v = bm1 - tm;
    if (it == 0) vmax = v;
    if (it == k - 1) vk = v;
    if (it == k) vk1 = v;
    bound = v;
  }
  {
    uint32_t n4[4] = {key[0], key[1], key[2], key[3]};
#pragma unroll
    for (int i = 4; i < 64; ++i) n4[i & 3] = min(n4[i & 3], key[i]);
    zabs = fmaxf(fabsf(unkey(vmax)), fabsf(unkey(min(min(n4[0], n4[1]), min(n4[2], n4[3])))));
  }
  // the k largest = every key above the (k+1)-th distinct one
  int cnt = 0;
#pragma unroll
  for (int i = 0; i < 64; ++i) {
    const bool sel = key[i] > vk1;
    pm |= (sel ? 1ull : 0ull) << i;
    cnt += sel;
  }
  const float gap = unkey(vk) - unkey(vk1);
  amb = !found || cnt != k || !(gap > 2.0f * E);
  return pm;
}

// select_exact32 for the top-KT rule without the key array (keys recomputed
// per pass): the main kernel's path when the 15-bit keys would leave most
// rows undecided (2 E_inf >= step / 2: decay close to 1)
template <int KT>
__device__ __forceinline__ uint64_t select_exact32_lean(const float2 (&zz)[32], float E, bool& amb,
                                                        float& zabs) {
  uint32_t bound = 0, vk = 0, vk1 = 0, vmax = 0;
  bool found = true;
#pragma unroll 1
  for (int it = 0; it <= KT; ++it) {
    const uint32_t bm1 = bound - 1u;
    uint32_t m4[4] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu};
#pragma unroll
    for (int w = 0; w < 32; ++w) {
      m4[w & 3] = min(m4[w & 3], bm1 - ukey(zz[w].x));
      m4[(w + 1) & 3] = min(m4[(w + 1) & 3], bm1 - ukey(zz[w].y));
    }
    const uint32_t tm = min(min(m4[0], m4[1]), min(m4[2], m4[3]));
    found = found && (it == 0 || (bound != 0u && tm <= bm1));
    const uint32_t v = bm1 - tm;
    if (it == 0) vmax = v;
    if (it == KT - 1) vk = v;
    if (it == KT) vk1 = v;
    bound = v;
  }
  uint32_t kmin = 0xffffffffu;
  uint64_t pm = 0;
#pragma unroll
  for (int w = 0; w < 32; ++w) {
    const int i0 = w < 16 ? w : w + 16;
    const uint32_t k0 = ukey(zz[w].x), k1 = ukey(zz[w].y);
    kmin = min(kmin, min(k0, k1));
    pm |= (k0 > vk1 ? 1ull : 0ull) << i0;
    pm |= (k1 > vk1 ? 1ull : 0ull) << (i0 + 16);
  }
  zabs = fmaxf(fabsf(unkey(vmax)), fabsf(unkey(kmin)));
  const float gap = unkey(vk) - unkey(vk1);
  amb = !found || __popcll(pm) != KT || !(gap > 2.0f * E);
  return pm;
}

// Top-KT on packed 15-bit keys (two per register, VIADDMNMX.U16x2: one
// instruction per two scores per pass). key = rint(z * qa + qb) - 2^23 is
// monotone in z. The KT + 1 passes find the KT + 1 largest distinct keys;
// the row is decided (`ok`) when exactly KT keys exceed the (KT+1)-th and the
// KT-th is at least two keys above it: then the KT-th and (KT+1)-th fp32
// scores are more than `step` apart, which exceeds 2E, so the exact scores
// (and the reference's fp64 ones) order the same way. Other rows go to the
// refine list (select_exact32 on the stored scores).
template <int KT>
__device__ __forceinline__ uint64_t select_q15(const float2 (&zz)[32], float R, float E, bool& ok,
                                               float& zabs) {
  // |z| <= R: z * qa in [-16383, 16383] (+ the rounding of qa), keys in [0, 32767]
  const float qa = __fdiv_rn(16383.0f, R);
  const float step = __frcp_ru(qa) * 1.0000005f;  // >= 1 / qa
  const float2 qa2 = make_float2(qa, qa), qb2 = make_float2(8388608.0f + 16383.5f, 8388608.0f + 16383.5f);
  uint32_t kw[32];
#pragma unroll
  for (int w = 0; w < 32; ++w) {
    const float2 q = __ffma2_rn(zz[w], qa2, qb2);
    kw[w] = __byte_perm(__float_as_uint(q.x), __float_as_uint(q.y), 0x5410);
  }
  uint32_t bound = 0x8000u, vk = 0, vk1 = 0, vmax = 0;
  bool found = true;
#pragma unroll
  for (int it = 0; it <= KT; ++it) {
    // max key below `bound`: keys < bound map to [2^16 - bound, 2^16) under
    // + (2^16 - bound) mod 2^16, keys >= bound to [0, 2^15)
    const uint32_t off2 = ((0x10000u - bound) & 0xffffu) * 0x10001u;
    uint32_t a8[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
#pragma unroll
    for (int w = 0; w < 32; ++w) a8[w & 7] = __viaddmax_u16x2(kw[w], off2, a8[w & 7]);
    const uint32_t m2 = __vmaxu2(__vmaxu2(__vmaxu2(a8[0], a8[1]), __vmaxu2(a8[2], a8[3])),
                                 __vmaxu2(__vmaxu2(a8[4], a8[5]), __vmaxu2(a8[6], a8[7])));
    const uint32_t m = max(m2 & 0xffffu, m2 >> 16);
    found = found && (m + bound >= 0x10000u);
    const uint32_t v = (m + bound) & 0xffffu;
    if (it == 0) vmax = v;
    if (it == KT - 1) vk = v;
    if (it == KT) vk1 = v;
    bound = v;
  }
  {  // |z| <= max(|vmax - 16383|, |kmin - 16384|) * step (key = rint(z qa + 16383.5))
    uint32_t n4[4] = {kw[0], kw[1], kw[2], kw[3]};
#pragma unroll
    for (int w = 4; w < 32; ++w) n4[w & 3] = __vminu2(n4[w & 3], kw[w]);
    const uint32_t n2 = __vminu2(__vminu2(n4[0], n4[1]), __vminu2(n4[2], n4[3]));
    const int kmin = (int)min(n2 & 0xffffu, n2 >> 16);
    zabs = (float)max(abs((int)vmax - 16383), abs(kmin - 16384)) * step;
  }
  // not selected <=> key <= vk1: bit 15 of (vk1 + 2^15 - key) per 16-bit lane
  // (no borrow between lanes: keys < 2^15)
  const uint32_t V2 = (vk1 + 0x8000u) * 0x10001u;
  uint32_t ns0 = 0, ns1 = 0;
#pragma unroll
  for (int w = 0; w < 16; ++w) {
    ns0 |= ((V2 - kw[w]) >> (15 - w)) & (0x10001u << w);
    ns1 |= ((V2 - kw[16 + w]) >> (15 - w)) & (0x10001u << w);
  }
  const uint64_t pm = ~(((uint64_t)ns1 << 32) | ns0);
  ok = found && __popcll(pm) == KT && vk >= vk1 + 2u && 2.0f * E < step;
  return pm;
}

__device__ __forceinline__ void refine_release(const TcArgs& a, int from, int to, int lane) {
  const int end = min(to, a.refine_cap);
  for (int sl = from + lane; sl < end; sl += 32)
    reinterpret_cast<float4*>(a.refine + (size_t)sl * kRefineFloats)[16] =
        make_float4(0.0f, 0.0f, 0.0f, __int_as_float(-1));
}

// KT > 0: two CTAs per SM (<= 204 registers; three would need <= 128 and
// spill -- measured 6.7 ms vs 4.1); the generic path keeps more
template <int KT>
__global__ void __launch_bounds__(kThreads, KT > 0 ? 2 : 1) k_linear_tc(const TcArgs a) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  unsigned char* sA = smem + OFF_A;
  unsigned char* sAL = smem + OFF_AL;
  unsigned char* sB = smem + OFF_B;
  uint4* lut = reinterpret_cast<uint4*>(smem + OFF_LUT);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* a_full = bar;          // [kStages], 128 arrivals
  uint64_t* acc_full = bar + 2;    // tcgen05.commit
  uint64_t* acc_empty = bar + 3;   // 128 arrivals
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 4);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // tables -> smem (already in the swizzled layout), byte LUT
  {
    const uint4* src = reinterpret_cast<const uint4*>(a.ws + WS_TAB);
    uint4* dst = reinterpret_cast<uint4*>(sB);
    for (int i = tid; i < kTabBytes / 16; i += kThreads) dst[i] = src[i];
    if (tid < 16) {
      uint32_t w[2];
#pragma unroll
      for (int j = 0; j < 2; ++j)
        w[j] = (((tid >> (2 * j)) & 1) ? 0x3C00u : 0u) |
               (((tid >> (2 * j + 1)) & 1) ? 0x3C000000u : 0u);
      reinterpret_cast<uint2*>(lut)[tid] = make_uint2(w[0], w[1]);
    }
  }
  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) mbar_init(&a_full[i], kRows);
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, kRows);
    fence_mbar_init();
  }
  if (warp == 4) tmem_alloc<kTmemCols>(tmem_slot);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const TcConsts cst = *reinterpret_cast<const TcConsts*>(a.ws + WS_CONST);
  const int L = a.L;

  if (warp == 4) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      constexpr uint32_t IDESC = umma_idesc_f16(128, 128, 0);
      const uint32_t b0 = smem_u32(sB);
      const uint32_t al = smem_u32(sAL);
      uint32_t u = 0;
      for (int g = blockIdx.x; g < a.n_groups; g += gridDim.x) {
        const int tmax = group_tmax(a, (int64_t)g * kRows);
        for (int t = 0; t < tmax; ++t, ++u) {
          const uint32_t st = u % kStages;
          mbar_wait_sleep(&a_full[st], (u / kStages) & 1);
          mbar_wait_sleep(acc_empty, (u & 1) ^ 1);  // token u - 1's scores read
          tc_fence_after();
          const uint32_t ax = smem_u32(sA + st * kTileA);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_f16_ss(tmem, umma_desc_sw128(ax + k * 32), umma_desc_sw128(b0 + k * 32), IDESC,
                       k != 0);
#pragma unroll
          for (int k = 0; k < 2; ++k)  // layer one-hot x bias rows, K = 32 (SW64)
            mma_f16_ss(tmem, umma_desc_sw64(al + k * 32), umma_desc_sw64(b0 + kTileB + k * 32),
                       IDESC, 1);
          mma_commit(acc_full);
        }
      }
    }
    __syncwarp();
  } else {
    // ---------------- score / selection / A-row producer (thread = stream) ----------------
    const int row = tid;  // TMEM lane
    const float* z0tab = reinterpret_cast<const float*>(a.ws + WS_Z0);
    int rc_base = -1, rc_used = kRChunk;  // this warp's refine-list chunk
    const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
    uint32_t u = 0;
    for (int g = blockIdx.x; g < a.n_groups; g += gridDim.x) {
      const int64_t s0 = (int64_t)g * kRows;
      const int tmax = group_tmax(a, s0);
      const int64_t sidx = s0 + row;
      const bool live = sidx < a.n_streams;
      const int p = live ? (int)(sidx / L) : 0;
      const int l = live ? (int)(sidx % L) : 0;
      const int64_t r0 = a.row_off[p];
      const int T = live ? (int)((a.row_off[p + 1] - r0) / L) : 0;
      const uint64_t* xs = a.truth + r0 + l;  // row t at xs[t * L]
      // one-hot layer row (bias MMA, K = 32, SW64); the previous group's
      // MMAs are complete
      {
        uint4 zero = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint4 v = zero;
          if (live && (l >> 3) == c) {
            uint32_t* w = reinterpret_cast<uint32_t*>(&v);
            w[(l & 7) >> 1] = (l & 1) ? 0x3C000000u : 0x3C00u;
          }
          *reinterpret_cast<uint4*>(sAL + sw64(row, c)) = v;
        }
      }
      // scores as pairs (element i0(w), i0(w) + 16), i0(w) = w < 16 ? w : w + 16, so
      // both elements of a pair sit in the same 32-column TMEM half and the
      // packed 15-bit keys of a pair land on mask bits w and w + 16 of a word
      float2 zz[32];
#pragma unroll
      for (int w = 0; w < 32; ++w) {
        const int i0 = w < 16 ? w : w + 16;
        zz[w] = live ? make_float2(z0tab[l * 64 + i0], z0tab[l * 64 + i0 + 16])
                     : make_float2(0.0f, 0.0f);
      }
      float E = cst.e0;
      float R = cst.zr0;  // running rigorous bound on |z_t| (fp32 scores): the key range
      bool tainted = false;
      // mask rows t .. t + kLookahead in flight: cp.async into this thread's
      // own ring slots (no register waits on the loads), one commit group per
      // token, read back with ld.shared once their group has landed
      const uint32_t xslot = smem_u32(smem + OFF_XR) + (uint32_t)row * 8u;
#pragma unroll
      for (int j = 0; j <= kLookahead; ++j) x_async(xslot, j, xs, L, T);
      x_wait<kLookahead>();  // token 0 landed
      // A rows for token 0
      if (tmax > 0) {
        put_row(smem_u32(sA + (u % kStages) * kTileA), smem_u32(lut), row, x_at(xslot, 0));
        fence_proxy_async();
        mbar_arrive(&a_full[u % kStages]);
      }
      int acc_k = 0, acc_ph = 0;
      for (int t = 0; t < tmax; ++t, ++u) {
        const bool valid = t < T;
        x_wait<kLookahead - 1>();  // tokens <= t + 1 landed
        const uint64_t x = x_at(xslot, t);
        // ---- A row for token t + 1 (its stage held token t - 1, whose MMA
        // completed before token t - 1's scores were read) ----
        if (t + 1 < tmax) {
          const uint32_t st = (u + 1) % kStages;
          put_row(smem_u32(sA + st * kTileA), smem_u32(lut), row, x_at(xslot, t + 1));
          fence_proxy_async();
          mbar_arrive(&a_full[st]);
        }
        // ---- selection on z_t ----
        uint64_t pm = 0;
        bool amb = tainted, defer = false;
        float zabs;
        if constexpr (KT > 0) {
          bool ok;
          if (cst.use_q15) {
            pm = select_q15<KT>(zz, R, E, ok, zabs);
            defer = !amb && !ok;
          } else {
            bool amb2;
            pm = select_exact32_lean<KT>(zz, E, amb2, zabs);
            amb = amb || amb2;
          }
        } else {
          float z[64];
#pragma unroll
          for (int w = 0; w < 32; ++w) {
            const int i0 = w < 16 ? w : w + 16;
            z[i0] = zz[w].x;
            z[i0 + 16] = zz[w].y;
          }
          bool amb2;
          pm = select_exact32<0>(z, a.budget, a.threshold, E, amb2, zabs);
          amb = amb || amb2;
        }
        // ---- rows the 15-bit keys cannot decide: scores to the refine list ----
        if constexpr (KT > 0) {
          const unsigned dm = __ballot_sync(0xffffffffu, defer && valid);
          if (dm) {
            // slots come from a warp-owned chunk (one atomic per kRChunk
            // deferrals instead of a round trip per event)
            const int n = __popc(dm);
            if (rc_used + n > kRChunk) {
              if (rc_base >= 0) refine_release(a, rc_base + rc_used, rc_base + kRChunk, lane);
              int nb = 0;
              if (lane == 0) nb = atomicAdd(a.refine_n, kRChunk);
              rc_base = __shfl_sync(0xffffffffu, nb, 0);
              rc_used = 0;
            }
            const int base = rc_base + rc_used;
            rc_used += n;
            if (defer && valid) {
              const int slot = base + __popc(dm & ((1u << lane) - 1u));
              if (slot < a.refine_cap) {
                float4* e = reinterpret_cast<float4*>(a.refine + (size_t)slot * kRefineFloats);
#pragma unroll
                for (int c4 = 0; c4 < 16; ++c4) {  // natural element order 4 c4 .. 4 c4 + 3
                  float v[4];
#pragma unroll
                  for (int j = 0; j < 4; ++j) {
                    const int i = 4 * c4 + j;
                    const int hi16 = (i >> 4) & 1;           // second element of its pair
                    const int w = (i & 15) + ((i >> 5) << 4);  // pair index
                    v[j] = hi16 ? zz[w].y : zz[w].x;
                  }
                  e[c4] = make_float4(v[0], v[1], v[2], v[3]);
                }
                e[16] = make_float4(E, 0.0f, __int_as_float((int)p), __int_as_float(t * L + l));
              } else {
                amb = true;  // refine list full: exact fp64 re-evaluation
              }
            }
          }
        }
        if (valid) {
          const int64_t r = r0 + (int64_t)t * L + l;
          if (amb) {
            const int slot = atomicAdd(a.list_n, 1);
            if (slot < a.list_cap) a.list[slot] = ((int64_t)p << 32) | (int64_t)(t * L + l);
          }
          if (amb || defer) pm = 0;
          a.pred[r] = pm;
          if (t >= a.warmup) {
            acc_k += __popcll(x);
            if (!amb && !defer) acc_ph += __popcll(x & pm);
          }
        }
        // ---- z_{t+1} = decay z_t + G_t ----
        mbar_wait_sleep(acc_full, u & 1);
        tc_fence_after();
        const float2 lam2 = make_float2(cst.lam, cst.lam);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t gh[32], gl[32];
          tmem_ld32(lane_base + h * 32, gh);
          tmem_ld32(lane_base + 64 + h * 32, gl);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int w = h * 16 + j;  // pair (32h + j, 32h + j + 16) = columns 2j, 2j + 1
            const float2 g = __fadd2_rn(
                make_float2(__uint_as_float(gh[2 * j]), __uint_as_float(gh[2 * j + 1])),
                make_float2(__uint_as_float(gl[2 * j]), __uint_as_float(gl[2 * j + 1])));
            zz[w] = __ffma2_rn(lam2, zz[w], g);
          }
        }
        tc_fence_before();
        mbar_arrive(acc_empty);
        // ---- error bound ----
        // per rounding 2^-23 of its operands' magnitude: the FFMA (|z_t| and
        // |z_{t+1}| <= |z_t| + |G|) incl. fp32(decay), the hi + lo add (|G|),
        // the lo-limb sums; plus the limb representation error of the row's
        // c + 1 table entries
        const int c = __popcll(x);
        tainted = tainted || c > a.kmax;
        const float gb = c * cst.cmax + cst.cbmax;
        E = (cst.lam * E + ldexpf(zabs + 2.0f * gb, -23) + (float)(c + 1) * cst.eta) * 1.000001f;
        // |z_{t+1}| <= decay |z_t| + |G_t| (+ fp32 rounding of both terms)
        R = fmaf(cst.lam, zabs, gb) * 1.0001f + 1.0f;
        // ---- load token t + kLookahead + 1 (into the slot of token t - 1) ----
        x_async(xslot, t + kLookahead + 1, xs, L, T);
      }
      x_wait<0>();
      if (live && (acc_k | acc_ph)) {
        atomicAdd(reinterpret_cast<unsigned long long*>(a.wcounts + 0), (unsigned long long)acc_k);
        atomicAdd(reinterpret_cast<unsigned long long*>(a.wcounts + 1), (unsigned long long)acc_ph);
        atomicAdd(reinterpret_cast<unsigned long long*>(a.wcounts + 2 + l), (unsigned long long)acc_k);
        atomicAdd(reinterpret_cast<unsigned long long*>(a.wcounts + 2 + L + l),
                  (unsigned long long)acc_ph);
      }
    }
    if (rc_base >= 0) refine_release(a, rc_base + rc_used, rc_base + kRChunk, lane);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
}

// ---------------------------------------------------------------------------
// Exact fp64 re-evaluation of the ambiguous rows, one warp per row.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_linear_rows_exact(
    const uint64_t* __restrict__ truth, const int64_t* __restrict__ row_off, int L,
    const double* __restrict__ W, double decay, int budget, int threshold, int warmup,
    const int* list_n, const int64_t* __restrict__ list, int list_cap, uint64_t* pred,
    int64_t* wcounts) {
  const int E = 64, F = L + E + 1;
  const int lane = threadIdx.x & 31;
  const int n = min(*list_n, list_cap);
  if (*list_n > list_cap) return;  // overflow: the gated fp64 kernel redoes everything
  const int nw = (int)(gridDim.x * blockDim.x / 32);
  for (int j = (int)((blockIdx.x * blockDim.x + threadIdx.x) / 32); j < n; j += nw) {
    const int64_t ent = list[j];
    const int p = (int)(ent >> 32);
    const int off = (int)(ent & 0xffffffff);
    const int t = off / L, l = off % L;
    const uint64_t* xs = truth + row_off[p] + l;
    // h (learner.py:62-72, numpy order: h *= decay; h[e] += 1.0), lanes own e and e + 32
    double h0 = 0.0, h1 = 0.0;
    for (int tb = 0; tb < t; tb += 32) {
      const int tt = tb + lane;
      const uint64_t xv = tt < t ? xs[(int64_t)tt * L] : 0ull;
      const int cnt = min(32, t - tb);
      for (int q = 0; q < cnt; ++q) {
        const uint64_t x = __shfl_sync(0xffffffffu, xv, q);
        h0 = __dmul_rn(h0, decay);
        h1 = __dmul_rn(h1, decay);
        if ((x >> lane) & 1ull) h0 = __dadd_rn(h0, 1.0);
        if ((x >> (lane + 32)) & 1ull) h1 = __dadd_rn(h1, 1.0);
      }
    }
    // z = W f, f = [onehot(l) | h | 1] (predictors.py:265), outputs lane and lane + 32
    double z[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int i = lane + 32 * q;
      const double* w = W + (size_t)i * F;
      double acc = w[l];
      for (int e = 0; e < 64; ++e) {
        const double he = __shfl_sync(0xffffffffu, e < 32 ? h0 : h1, e & 31);
        acc = __fma_rn(w[L + e], he, acc);
      }
      z[q] = __dadd_rn(acc, w[L + E]);
    }
    uint64_t pm = 0;
    if (threshold) {
      const unsigned b0 = __ballot_sync(0xffffffffu, z[0] > 0.0);
      const unsigned b1 = __ballot_sync(0xffffffffu, z[1] > 0.0);
      pm = (uint64_t)b0 | ((uint64_t)b1 << 32);
    } else {
      const int kk = min(budget, E);
      for (int it = 0; it < kk; ++it) {  // (-score, id) order, learner.py:164-169
        double best = -INFINITY;
        int bi = 64;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int i = lane + 32 * q;
          if (!((pm >> i) & 1ull) && (z[q] > best || (z[q] == best && i < bi) || bi == 64)) {
            best = z[q];
            bi = i;
          }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          const bool take = oi < 64 && (bi == 64 || ob > best || (ob == best && oi < bi));
          best = take ? ob : best;
          bi = take ? oi : bi;
        }
        pm |= 1ull << bi;
      }
    }
    if (lane == 0) {
      const int64_t r = row_off[p] + off;
      pred[r] = pm;
      if (t >= warmup) {
        const int ph = __popcll(truth[r] & pm);
        if (ph) {
          atomicAdd(reinterpret_cast<unsigned long long*>(wcounts + 1), (unsigned long long)ph);
          atomicAdd(reinterpret_cast<unsigned long long*>(wcounts + 2 + L + l),
                    (unsigned long long)ph);
        }
      }
    }
  }
}

// Rows the 15-bit keys left undecided: exact selection on their stored fp32
// scores (select_exact32, the same rule the fp32 path always used); rows the
// fp32 bound cannot decide either go on to the fp64 list. One thread per
// entry, prediction hits summed per block.
template <int KT>
__global__ void __launch_bounds__(256) k_linear_tc_refine(
    const uint64_t* __restrict__ truth, const int64_t* __restrict__ row_off, int L, int budget,
    int warmup, const int* refine_n, const float* __restrict__ refine, int refine_cap,
    int* list_n, int64_t* list, int list_cap, uint64_t* pred, int64_t* wcounts) {
  __shared__ unsigned long long s_ph[33];  // [0] total, [1 + l] per layer
  for (int i = threadIdx.x; i <= L; i += blockDim.x) s_ph[i] = 0ull;
  __syncthreads();
  const int n = min(*refine_n, refine_cap);
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const float4* e = reinterpret_cast<const float4*>(refine + (size_t)j * kRefineFloats);
    float z[64];
#pragma unroll
    for (int c4 = 0; c4 < 16; ++c4) {
      const float4 v = e[c4];
      z[4 * c4] = v.x;
      z[4 * c4 + 1] = v.y;
      z[4 * c4 + 2] = v.z;
      z[4 * c4 + 3] = v.w;
    }
    const float4 h = e[16];
    const int p = __float_as_int(h.z), off = __float_as_int(h.w);
    if (off < 0) continue;  // an unused slot of a warp's chunk
    bool amb;
    float zabs;
    const uint64_t pm = select_exact32<KT>(z, budget, 0, h.x, amb, zabs);
    const int t = off / L, l = off % L;
    if (amb) {
      const int slot = atomicAdd(list_n, 1);
      if (slot < list_cap) list[slot] = ((int64_t)p << 32) | (int64_t)off;
      continue;
    }
    const int64_t r = row_off[p] + off;
    pred[r] = pm;
    if (t >= warmup) {
      const int ph = __popcll(truth[r] & pm);
      if (ph) {
        atomicAdd(&s_ph[0], (unsigned long long)ph);
        atomicAdd(&s_ph[1 + l], (unsigned long long)ph);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i <= L; i += blockDim.x)
    if (s_ph[i])
      atomicAdd(reinterpret_cast<unsigned long long*>(wcounts + (i == 0 ? 1 : 2 + L + i - 1)),
                s_ph[i]);
}

// counts += scratch counts, unless the list overflowed (then the gated fp64
// kernel has added its own)
__global__ void k_linear_tc_finalize(const int* list_n, int list_cap, const int64_t* wcounts,
                                     int n, int64_t* counts) {
  if (*list_n > list_cap) return;
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (wcounts[i])
      atomicAdd(reinterpret_cast<unsigned long long*>(counts + i), (unsigned long long)wcounts[i]);
}

__global__ void k_copy_list_n(const int* list_n, int64_t* out) { *out = *list_n; }

}  // namespace

namespace moeb {

int linear_tc_ambiguous(const void* workspace, int L, int64_t* out, cudaStream_t s) {
  k_copy_list_n<<<1, 1, 0, s>>>(
      reinterpret_cast<const int*>(reinterpret_cast<const unsigned char*>(workspace) +
                                   ws_list_n_off(L)),
      out);
  return check_launch("k_copy_list_n");
}

size_t linear_tc_list_cap(int64_t rows) {
  const int64_t c = rows / 256 > 65536 ? rows / 256 : 65536;
  return (size_t)(c < (1LL << 30) ? c : (1LL << 30));
}

size_t linear_tc_min_workspace(int L) { return ws_list_off(L) + 8 * 4; }

// refine-list entries: ~1.7 % of the rows at the bench shape; 3 % + slack
static size_t refine_cap_for(int64_t rows) {
  const int64_t c = rows / 32 + 1024;
  return (size_t)(c < (1LL << 30) ? c : (1LL << 30));
}

static size_t refine_off(int L, size_t list_cap) {
  return (ws_list_off(L) + 8 * list_cap + 15) & ~(size_t)15;
}

size_t linear_tc_workspace_bytes(int64_t rows, int L) {
  return refine_off(L, linear_tc_list_cap(rows)) + 4 * kRefineFloats * refine_cap_for(rows);
}

bool linear_tc_eligible(int L, int E, int budget, const double* logits) {
  const char* env = getenv("MOEB_K3");
  if (env && env[0] == 'f') return false;  // MOEB_K3=fp64: the SIMT fp64 kernel
  return E == 64 && L >= 1 && L <= 32 && budget >= 1 && budget <= 16 && logits == nullptr;
}

int linear_tc_launch(const uint64_t* truth, const int64_t* row_off, int P, int64_t rows, int L,
                     const double* W, double decay, int budget, int threshold, int warmup,
                     int kmax, uint64_t* pred, int64_t* counts, void* workspace,
                     size_t ws_bytes, cudaStream_t s) {
  unsigned char* ws = reinterpret_cast<unsigned char*>(workspace);
  const size_t cap_fit = ws_bytes > ws_list_off(L) ? (ws_bytes - ws_list_off(L)) / 8 : 0;
  const int list_cap = (int)(cap_fit < linear_tc_list_cap(rows) ? cap_fit : linear_tc_list_cap(rows));
  int64_t* wcounts = reinterpret_cast<int64_t*>(ws + ws_counts_off(L));
  int* list_n = reinterpret_cast<int*>(ws + ws_list_n_off(L));
  int64_t* list = reinterpret_cast<int64_t*>(ws + ws_list_off(L));
  int* refine_n = list_n + 1;
  const size_t roff = refine_off(L, (size_t)list_cap);
  const size_t rfit = ws_bytes > roff ? (ws_bytes - roff) / (4 * kRefineFloats) : 0;
  const int refine_cap = (int)(rfit < refine_cap_for(rows) ? rfit : refine_cap_for(rows));
  float* refine = reinterpret_cast<float*>(ws + roff);
  if (cudaMemsetAsync(ws + ws_counts_off(L), 0, ws_list_off(L) - ws_counts_off(L), s) != cudaSuccess)
    return fail(MOEB_ECUDA, "clearing the K3t scratch");
  k_linear_tc_prep<<<1, 256, 0, s>>>(W, L, decay, kmax < 1 ? 64 : kmax, ws);
  int rc = check_launch("k_linear_tc_prep");
  if (rc) return rc;
  TcArgs a{};
  a.truth = truth;
  a.row_off = row_off;
  a.P = P;
  a.L = L;
  a.budget = budget;
  a.threshold = threshold;
  a.warmup = warmup;
  a.kmax = kmax < 1 ? 64 : kmax;
  a.n_streams = (int64_t)P * L;
  a.n_groups = (int)((a.n_streams + kRows - 1) / kRows);
  a.ws = ws;
  a.wcounts = wcounts;
  a.list_n = list_n;
  a.list = list;
  a.list_cap = list_cap;
  a.refine_n = refine_n;
  a.refine = refine;
  a.refine_cap = refine_cap;
  a.pred = pred;
  auto kern = threshold ? k_linear_tc<0> : budget == 6 ? k_linear_tc<6> : budget == 8 ? k_linear_tc<8>
                                                                                      : k_linear_tc<0>;
  set_smem(kern, kSmem);
  // persistent: 2 CTAs per SM (1 for the generic kernel), groups spread
  // evenly (every CTA gets the same count)
  const int slots = (!threshold && (budget == 6 || budget == 8) ? 2 : 1) * num_sms();
  const int per = (a.n_groups + slots - 1) / slots;
  const int grid = (a.n_groups + per - 1) / per;
  kern<<<grid, kThreads, kSmem, s>>>(a);
  rc = check_launch("k_linear_tc");
  if (rc) return rc;
  if (!threshold && (budget == 6 || budget == 8)) {
    auto rk = budget == 6 ? k_linear_tc_refine<6> : k_linear_tc_refine<8>;
    rk<<<2 * num_sms(), 256, 0, s>>>(truth, row_off, L, budget, warmup, refine_n, refine,
                                      refine_cap, list_n, list, list_cap, pred, wcounts);
    rc = check_launch("k_linear_tc_refine");
    if (rc) return rc;
  }
  k_linear_rows_exact<<<2 * num_sms(), 256, 0, s>>>(truth, row_off, L, W, decay, budget,
                                                     threshold, warmup, list_n, list, list_cap,
                                                     pred, wcounts);
  rc = check_launch("k_linear_rows_exact");
  if (rc) return rc;
  // list overflow (more ambiguous rows than the workspace holds): redo the
  // whole call with the fp64 kernel (it returns at once otherwise)
  rc = launch_linear_fp64_gated(truth, row_off, P, L, 64, W, decay, budget, threshold, warmup,
                                pred, counts, list_n, list_cap, s);
  if (rc) return rc;
  if (counts) {
    k_linear_tc_finalize<<<1, 128, 0, s>>>(list_n, list_cap, wcounts, 2 + 2 * L, counts);
    rc = check_launch("k_linear_tc_finalize");
  }
  (void)rows;
  return rc;
}

}  // namespace moeb
