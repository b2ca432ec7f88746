// K7 metrics, K2 mask head and the rule-based predictor mask tables.
//
// K7 replaces macro_f1 / position_accuracy / label_accuracy (metrics.py:12-79)
// by their integer core: per-expert TP/FP/FN, position count, exact-set
// matches and the label-correct sum. The host finishes with the reference's
// numpy expressions, so the floats are identical given identical masks.
// K2 replaces top_k_experts / predict_topk (learner.py:164-181).
// Policy masks replace OraclePredictor / LruOnlyPredictor /
// NextLayerAllPredictor / GlobalFrequencyPredictor.predict (predictors.py:57-139).
#include <cstring>

#include "common.cuh"

namespace {

// E <= 64 (one mask word): bit-sliced ("vertical") counters. Each lane owns
// four rows per iteration and adds their TP / FP / FN masks into 8 bit-planes
// each (carry-save adders); every <= 255 rows per lane the planes are
// drained into per-expert counts with ballot+popc per (expert, plane).
constexpr int kPlanes = 8;

// four rows at once: two full adders into plane 0, one into plane 1, the
// weight-4 carry rippled through planes 2.. (27 ops for 4 rows instead of 64)
__device__ __forceinline__ void vc_add4(uint64_t (&v)[kPlanes], uint64_t x1, uint64_t x2,
                                        uint64_t x3, uint64_t x4) {
  uint64_t t = v[0] ^ x1;
  const uint64_t c1 = (v[0] & x1) | (x2 & t);
  v[0] = t ^ x2;
  t = v[0] ^ x3;
  const uint64_t c2 = (v[0] & x3) | (x4 & t);
  v[0] = t ^ x4;
  t = v[1] ^ c1;
  uint64_t d = (v[1] & c1) | (c2 & t);
  v[1] = t ^ c2;
#pragma unroll
  for (int i = 2; i < kPlanes; ++i) {
    const uint64_t c = v[i] & d;
    v[i] ^= d;
    d = c;
  }
}

__device__ __forceinline__ void vc_drain(uint64_t (&va)[kPlanes], uint64_t (&vb)[kPlanes],
                                         uint64_t (&vc)[kPlanes], int lane, uint32_t (&tp)[2],
                                         uint32_t (&fp)[2], uint32_t (&fn)[2]) {
  const unsigned full = 0xffffffffu;
#pragma unroll 1
  for (int e = 0; e < 64; ++e) {
    uint32_t ca = 0, cb = 0, cc = 0;
#pragma unroll
    for (int i = 0; i < kPlanes; ++i) {
      ca += (uint32_t)__popc(__ballot_sync(full, (va[i] >> e) & 1ull)) << i;
      cb += (uint32_t)__popc(__ballot_sync(full, (vb[i] >> e) & 1ull)) << i;
      cc += (uint32_t)__popc(__ballot_sync(full, (vc[i] >> e) & 1ull)) << i;
    }
    if (lane == (e & 31)) {
      const int j = e >> 5;
      tp[j] += ca;
      fp[j] += cb;
      fn[j] += cc;
    }
  }
#pragma unroll
  for (int i = 0; i < kPlanes; ++i) va[i] = vb[i] = vc[i] = 0;
}

// Row-balanced: the trace's rows are split into equal ranges of 32-row chunks,
// one range per warp (prompt lengths do not matter), and every lane keeps
// four chunk loads in flight. A row is measured if it lies at or past its
// prompt's warm-up rows; each lane tracks its prompt boundary incrementally.
constexpr int kMetDepth = 4;
__global__ void __launch_bounds__(256) k_metrics64(const uint64_t* __restrict__ pred,
                                                   const uint64_t* __restrict__ truth,
                                                   const int64_t* __restrict__ row_off, int P,
                                                   int L, int E, int warmup, int64_t* out) {
  __shared__ unsigned long long scnt[3 * 64 + 3];
  for (int i = threadIdx.x; i < 3 * E + 3; i += blockDim.x) scnt[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t rbeg = row_off[0], rend = row_off[P];
  const int64_t chunks = (rend - rbeg + 31) >> 5;
  const int64_t c0 = chunks * w / nw, c1 = chunks * (w + 1) / nw;
  const int64_t skip = (int64_t)warmup * L;
  uint64_t va[kPlanes], vb[kPlanes], vc[kPlanes];
#pragma unroll
  for (int i = 0; i < kPlanes; ++i) va[i] = vb[i] = vc[i] = 0;
  uint32_t tp[2] = {0, 0}, fp[2] = {0, 0}, fn[2] = {0, 0};
  uint64_t npos = 0, nexact = 0, nlabel = 0;
  int pending = 0;  // rows per lane since the last drain (warp-uniform)
  // this lane's prompt: the last p with row_off[p] <= first row
  int pl = 0;
  {
    const int64_t r = rbeg + c0 * 32 + lane;
    int lo = 0, hi = P - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (row_off[mid] <= r) lo = mid; else hi = mid - 1;
    }
    pl = lo;
  }
  int64_t mstart = row_off[pl] + skip, nb = row_off[pl + 1];
  for (int64_t c = c0; c < c1; c += kMetDepth) {
    uint64_t pw[kMetDepth], tw[kMetDepth];
#pragma unroll
    for (int u = 0; u < kMetDepth; ++u) {
      const int64_t r = rbeg + (c + u) * 32 + lane;
      const bool in = c + u < c1 && r < rend;
      pw[u] = in ? __ldg(pred + r) : 0ull;
      tw[u] = in ? __ldg(truth + r) : 0ull;
    }
    static_assert(kMetDepth == 4, "vc_add4 takes the four rows of an iteration");
#pragma unroll
    for (int u = 0; u < kMetDepth; ++u) {
      const int64_t r = rbeg + (c + u) * 32 + lane;
      const bool in = c + u < c1 && r < rend;
      while (in && r >= nb) {  // crossed into the next prompt(s)
        ++pl;
        mstart = nb + skip;
        nb = row_off[pl + 1];
      }
      const bool m = in && r >= mstart;
      const uint64_t p = m ? pw[u] : 0ull, t = m ? tw[u] : 0ull;
      pw[u] = p;
      tw[u] = t;
      npos += m;
      nexact += m && p == t;
      nlabel += m ? (uint64_t)(E - __popcll(p ^ t)) : 0;
    }
    vc_add4(va, pw[0] & tw[0], pw[1] & tw[1], pw[2] & tw[2], pw[3] & tw[3]);
    vc_add4(vb, pw[0] & ~tw[0], pw[1] & ~tw[1], pw[2] & ~tw[2], pw[3] & ~tw[3]);
    vc_add4(vc, tw[0] & ~pw[0], tw[1] & ~pw[1], tw[2] & ~pw[2], tw[3] & ~pw[3]);
    pending += kMetDepth;
    if (pending > (1 << kPlanes) - 1 - kMetDepth) {  // the planes hold counts up to 255
      vc_drain(va, vb, vc, lane, tp, fp, fn);
      pending = 0;
    }
  }
  if (pending) vc_drain(va, vb, vc, lane, tp, fp, fn);
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int e = lane + 32 * j;
    if (e < E) {
      if (tp[j]) atomicAdd(&scnt[e], (unsigned long long)tp[j]);
      if (fp[j]) atomicAdd(&scnt[E + e], (unsigned long long)fp[j]);
      if (fn[j]) atomicAdd(&scnt[2 * E + e], (unsigned long long)fn[j]);
    }
  }
  atomicAdd(&scnt[3 * E], (unsigned long long)npos);
  atomicAdd(&scnt[3 * E + 1], (unsigned long long)nexact);
  atomicAdd(&scnt[3 * E + 2], (unsigned long long)nlabel);
  __syncthreads();
  for (int i = threadIdx.x; i < 3 * E + 3; i += blockDim.x)
    if (scnt[i]) atomicAdd(reinterpret_cast<unsigned long long*>(out + i), scnt[i]);
}

// One warp per prompt (grid-stride): lanes take 32 consecutive measured rows;
// per expert, ballot+popc turns the 32 rows into one count that the owning
// lane (expert % 32) accumulates. Block-level shared reduce, then one global
// atomic per counter per block.
template <int W>
__global__ void __launch_bounds__(256) k_metrics(const uint64_t* __restrict__ pred,
                                                 const uint64_t* __restrict__ truth,
                                                 const int64_t* __restrict__ row_off, int P,
                                                 int L, int E, int warmup, int64_t* out) {
  constexpr int PER_LANE = W * 2;  // experts owned per lane: lane + 32*j
  __shared__ unsigned long long scnt[3 * 256 + 3];
  for (int i = threadIdx.x; i < 3 * E + 3; i += blockDim.x) scnt[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  uint32_t tp[PER_LANE], fp[PER_LANE], fn[PER_LANE];
#pragma unroll
  for (int j = 0; j < PER_LANE; ++j) tp[j] = fp[j] = fn[j] = 0;
  uint64_t npos = 0, nexact = 0, nlabel = 0;
  for (int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < P; p += warps) {
    const int64_t r0 = row_off[p] + (int64_t)warmup * L, r1 = row_off[p + 1];
    for (int64_t base = r0; base < r1; base += 32) {
      const int64_t r = base + lane;
      const bool m = r < r1;
      uint64_t pw[W], tw[W];
      bool eq = m;
      int mism = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        pw[w] = m ? __ldg(pred + r * W + w) : 0ull;
        tw[w] = m ? __ldg(truth + r * W + w) : 0ull;
        eq = eq && pw[w] == tw[w];
        mism += __popcll(pw[w] ^ tw[w]);
      }
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const uint64_t a = pw[w] & tw[w], b = pw[w] & ~tw[w], c = tw[w] & ~pw[w];
#pragma unroll
        for (int e = 0; e < 64; ++e) {
          const uint32_t c1 = __popc(__ballot_sync(0xffffffffu, (a >> e) & 1ull));
          const uint32_t c2 = __popc(__ballot_sync(0xffffffffu, (b >> e) & 1ull));
          const uint32_t c3 = __popc(__ballot_sync(0xffffffffu, (c >> e) & 1ull));
          if (lane == (e & 31)) {
            const int j = w * 2 + (e >> 5);
            tp[j] += c1;
            fp[j] += c2;
            fn[j] += c3;
          }
        }
      }
      npos += m;
      nexact += eq;
      nlabel += m ? (uint64_t)(E - mism) : 0;
    }
  }
#pragma unroll
  for (int j = 0; j < PER_LANE; ++j) {
    const int e = lane + 32 * j;
    if (e < E) {
      if (tp[j]) atomicAdd(&scnt[e], (unsigned long long)tp[j]);
      if (fp[j]) atomicAdd(&scnt[E + e], (unsigned long long)fp[j]);
      if (fn[j]) atomicAdd(&scnt[2 * E + e], (unsigned long long)fn[j]);
    }
  }
  atomicAdd(&scnt[3 * E], (unsigned long long)npos);
  atomicAdd(&scnt[3 * E + 1], (unsigned long long)nexact);
  atomicAdd(&scnt[3 * E + 2], (unsigned long long)nlabel);
  __syncthreads();
  for (int i = threadIdx.x; i < 3 * E + 3; i += blockDim.x)
    if (scnt[i]) atomicAdd(reinterpret_cast<unsigned long long*>(out + i), scnt[i]);
}

__device__ __forceinline__ uint32_t f32_order(float x) {
  uint32_t b = __float_as_uint(x == 0.0f ? 0.0f : x);  // -0 ties +0, as in numpy
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// K2: one warp per row. Each lane holds E/32 logits; k passes of a warp-wide
// max over (order(z), -id) pick the top-k with ties to the lower id.
template <int PER_LANE>
__global__ void __launch_bounds__(256) k_mask_head(const float* __restrict__ logits,
                                                   int64_t rows, int E, int k, int threshold,
                                                   uint64_t* __restrict__ masks) {
  const int lane = threadIdx.x & 31;
  const int W = (E + 63) / 64;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += warps) {
    uint64_t key[PER_LANE];
#pragma unroll
    for (int j = 0; j < PER_LANE; ++j) {
      const int e = lane + 32 * j;
      key[j] = 0;
      if (e < E) {
        const float z = __ldg(logits + r * E + e);
        key[j] = ((uint64_t)f32_order(z) << 32) | (uint32_t)(0xFFFFFFFFu - e);
        if (threshold) key[j] = z > 0.0f ? 1ull : 0ull;
      }
    }
    uint64_t out[4] = {0, 0, 0, 0};
    if (threshold) {
#pragma unroll
      for (int j = 0; j < PER_LANE; ++j) {
        const uint32_t b = __ballot_sync(0xffffffffu, key[j] != 0);
        out[j >> 1] |= (uint64_t)b << (32 * (j & 1));
      }
    } else {
      const int kk = k < E ? k : E;
      for (int it = 0; it < kk; ++it) {
        uint64_t best = 0;
#pragma unroll
        for (int j = 0; j < PER_LANE; ++j) best = key[j] > best ? key[j] : best;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          const uint64_t other = __shfl_xor_sync(0xffffffffu, best, o);
          best = other > best ? other : best;
        }
        const int e = (int)(0xFFFFFFFFu - (uint32_t)(best & 0xFFFFFFFFu));
        out[e >> 6] |= 1ull << (e & 63);
#pragma unroll
        for (int j = 0; j < PER_LANE; ++j)
          if (key[j] == best) key[j] = 0;
      }
    }
    if (lane < W) {
      uint64_t v = out[0];
#pragma unroll
      for (int w = 1; w < 4; ++w) v = lane == w ? out[w] : v;
      masks[r * W + lane] = v;
    }
  }
}

template <int W>
__global__ void k_policy_masks(int kind, const uint64_t* __restrict__ truth, int64_t rows, int L,
                               int E, int budget, const uint64_t* __restrict__ table,
                               uint64_t* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += stride) {
    uint64_t v[W];
    if (kind == 1) {  // oracle: the `budget` lowest truth ids (predictors.py:80-81)
      int left = budget;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        uint64_t m = __ldg(truth + r * W + w), keep = 0;
        while (m && left > 0) {
          keep |= m & (~m + 1);
          m &= m - 1;
          --left;
        }
        v[w] = keep;
      }
    } else if (kind == 2) {  // next_layer_all
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const int bits = E - 64 * w;
        v[w] = bits >= 64 ? ~0ull : (bits <= 0 ? 0ull : ((1ull << bits) - 1));
      }
    } else if (kind == 3) {  // per-layer table (global_frequency); rows of
      const int l = (int)(r % L);  // a prompt start at a multiple of L
#pragma unroll
      for (int w = 0; w < W; ++w) v[w] = __ldg(table + l * W + w);
    } else {
#pragma unroll
      for (int w = 0; w < W; ++w) v[w] = 0;
    }
#pragma unroll
    for (int w = 0; w < W; ++w) out[r * W + w] = v[w];
  }
}

int grid_for(int64_t work, int threads) {
  const int64_t want = (work + threads - 1) / threads;
  const int64_t cap = (int64_t)moeb::num_sms() * 16;
  return (int)(want < cap ? (want > 0 ? want : 1) : cap);
}

}  // namespace

extern "C" int moeb_metrics(const uint64_t* pred, const uint64_t* truth,
                            const int64_t* prompt_row_off, int n_prompts, int L, int E,
                            int warmup_tokens, int64_t* metrics, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(pred && truth && prompt_row_off && metrics, "null argument");
  MOEB_REQUIRE(n_prompts >= 1 && L >= 1 && E >= 1 && E <= 256, "bad shape");
  MOEB_REQUIRE(warmup_tokens >= 0, "bad warmup");
  const int W = moeb::words_for(E);
  const int threads = 256;
  cudaStream_t s = moeb::as_stream(stream);
  if (W == 1) {  // persistent bit-sliced kernel: 4 CTAs per SM, equal row ranges per warp
    const char* kb = getenv("MOEB_K7_CTAS");  // CTAs per SM (A/B of the overlap footprint)
    const int blocks = (kb ? atoi(kb) : 4) * moeb::num_sms();
    k_metrics64<<<blocks, threads, 0, s>>>(pred, truth, prompt_row_off, n_prompts, L, E,
                                           warmup_tokens, metrics);
    return moeb::check_launch("k_metrics64");
  }
  const int blocks = grid_for((int64_t)n_prompts * 32, threads);
  switch (W) {
    case 1: k_metrics<1><<<blocks, threads, 0, s>>>(pred, truth, prompt_row_off, n_prompts, L, E, warmup_tokens, metrics); break;
    case 2: k_metrics<2><<<blocks, threads, 0, s>>>(pred, truth, prompt_row_off, n_prompts, L, E, warmup_tokens, metrics); break;
    case 3: k_metrics<3><<<blocks, threads, 0, s>>>(pred, truth, prompt_row_off, n_prompts, L, E, warmup_tokens, metrics); break;
    default: k_metrics<4><<<blocks, threads, 0, s>>>(pred, truth, prompt_row_off, n_prompts, L, E, warmup_tokens, metrics); break;
  }
  return moeb::check_launch("k_metrics");
}

extern "C" int moeb_mask_head(const float* logits, int64_t rows, int E, int k, int threshold,
                              uint64_t* masks, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(logits && masks, "null argument");
  MOEB_REQUIRE(rows >= 0 && E >= 1 && E <= 256 && k >= 1, "bad shape");
  if (rows == 0) return MOEB_OK;
  const int threads = 256;
  const int blocks = grid_for(rows * 32, threads);
  cudaStream_t s = moeb::as_stream(stream);
  const int per = (E + 31) / 32;
  if (per <= 2)
    k_mask_head<2><<<blocks, threads, 0, s>>>(logits, rows, E, k, threshold, masks);
  else if (per <= 4)
    k_mask_head<4><<<blocks, threads, 0, s>>>(logits, rows, E, k, threshold, masks);
  else
    k_mask_head<8><<<blocks, threads, 0, s>>>(logits, rows, E, k, threshold, masks);
  return moeb::check_launch("k_mask_head");
}

extern "C" int moeb_policy_masks(int kind, const uint64_t* truth, int64_t rows, int L, int E,
                                 int budget, const uint64_t* layer_table, uint64_t* out,
                                 void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(out && rows >= 0 && L >= 1 && E >= 1 && E <= 256, "bad arguments");
  MOEB_REQUIRE(kind >= 0 && kind <= 3, "unknown policy kind %d", kind);
  MOEB_REQUIRE(kind != 1 || truth, "oracle masks need truth");
  MOEB_REQUIRE(kind != 3 || layer_table, "table masks need a layer table");
  if (rows == 0) return MOEB_OK;
  const int W = moeb::words_for(E);
  const int threads = 256;
  const int blocks = grid_for(rows, threads);
  cudaStream_t s = moeb::as_stream(stream);
  switch (W) {
    case 1: k_policy_masks<1><<<blocks, threads, 0, s>>>(kind, truth, rows, L, E, budget, layer_table, out); break;
    case 2: k_policy_masks<2><<<blocks, threads, 0, s>>>(kind, truth, rows, L, E, budget, layer_table, out); break;
    case 3: k_policy_masks<3><<<blocks, threads, 0, s>>>(kind, truth, rows, L, E, budget, layer_table, out); break;
    default: k_policy_masks<4><<<blocks, threads, 0, s>>>(kind, truth, rows, L, E, budget, layer_table, out); break;
  }
  return moeb::check_launch("k_policy_masks");
}

// Compact trace rows for host->device transfer: k expert ids per row (u8,
// ascending, 0xff = none; E <= 64) <-> one-word expert masks. A row of the
// reference trace is its sorted expert-id tuple (core.py:64-90), so the ids
// are the natural wire format: k bytes per row instead of an 8-byte mask.
namespace {
__global__ void k_ids_to_masks(const uint8_t* __restrict__ ids, int64_t rows, int k, int E,
                               uint64_t* __restrict__ masks, int* __restrict__ bad) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    uint64_t m = 0;
    for (int j = 0; j < k; ++j) {
      const int e = ids[r * k + j];
      if (e == 0xff) continue;
      if (e >= E) {
        atomicExch(bad, 1);
        continue;
      }
      m |= 1ull << e;
    }
    masks[r] = m;
  }
}

__global__ void k_masks_to_ids(const uint64_t* __restrict__ masks, int64_t rows, int k,
                               uint8_t* __restrict__ ids, int* __restrict__ bad) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    uint64_t m = masks[r];
    if (__popcll(m) > k) atomicExch(bad, 1);
    for (int j = 0; j < k; ++j) {
      int e = 0xff;
      if (m) {
        e = __ffsll((long long)m) - 1;
        m &= m - 1;
      }
      ids[r * k + j] = (uint8_t)e;
    }
  }
}
}  // namespace

extern "C" int moeb_ids_to_masks(const uint8_t* ids, int64_t rows, int k, int E, uint64_t* masks,
                                 int* bad, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(ids && masks && bad && rows >= 0 && k >= 1 && k <= 64 && E >= 1 && E <= 64,
               "bad arguments");
  if (rows == 0) return MOEB_OK;
  const int blocks = (int)std::min<int64_t>((rows + 255) / 256, 8LL * moeb::num_sms());
  k_ids_to_masks<<<blocks, 256, 0, moeb::as_stream(stream)>>>(ids, rows, k, E, masks, bad);
  return moeb::check_launch("k_ids_to_masks");
}

extern "C" int moeb_masks_to_ids(const uint64_t* masks, int64_t rows, int k, uint8_t* ids, int* bad,
                                 void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(ids && masks && bad && rows >= 0 && k >= 1 && k <= 64, "bad arguments");
  if (rows == 0) return MOEB_OK;
  const int blocks = (int)std::min<int64_t>((rows + 255) / 256, 8LL * moeb::num_sms());
  k_masks_to_ids<<<blocks, 256, 0, moeb::as_stream(stream)>>>(masks, rows, k, ids, bad);
  return moeb::check_launch("k_masks_to_ids");
}

// The tightest wire format of a top-k trace row: its rank in the
// combinatorial number system (N = sum_i C(c_i, i) over the ascending ids
// c_1 < ... < c_k), one u32 per row when C(E, k) < 2^32 (C(64, 6) = 74,974,368):
// 4 bytes instead of the k-byte ids or the 8-byte mask. Every row of a
// validated reference trace has exactly k distinct ids (core.py:64-90).
namespace {
constexpr int kBinN = 65, kBinK = 9;

__device__ __forceinline__ void load_binom(uint32_t* tab) {  // tab[j * kBinN + n] = C(n, j)
  for (int i = threadIdx.x; i < kBinN * kBinK; i += blockDim.x) {
    const int j = i / kBinN, n = i % kBinN;
    uint64_t c = 1;
    for (int q = 0; q < j; ++q) c = c * (uint64_t)(n - q) / (uint64_t)(q + 1);
    tab[i] = j > n ? 0u : (c > 0xffffffffull ? 0xffffffffu : (uint32_t)c);
  }
  __syncthreads();
}

// bits == 32: one u32 per row; bits < 32: a little-endian bit stream, row r
// in bits [r bits, (r + 1) bits) (one padding word at the end)
__device__ __forceinline__ uint32_t rank_at(const uint32_t* __restrict__ w, int64_t r, int bits) {
  if (bits == 32) return w[r];
  const int64_t b = r * bits;
  const int64_t i = b >> 5;
  const int sh = (int)(b & 31);
  const uint64_t two = (uint64_t)w[i] | ((uint64_t)w[i + 1] << 32);
  return (uint32_t)(two >> sh) & ((1u << bits) - 1u);
}

__global__ void k_ranks_to_masks(const uint32_t* __restrict__ ranks, int64_t rows, int bits, int k,
                                 int E, uint64_t* __restrict__ masks, int* __restrict__ bad) {
  __shared__ uint32_t tab[kBinN * kBinK];
  load_binom(tab);
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    uint32_t N = rank_at(ranks, r, bits);
    uint64_t m = 0;
    int hi = E;  // c_i < hi
    const bool ok = N < tab[k * kBinN + E];
    for (int i = k; i >= 1; --i) {
      // largest c in [i - 1, hi) with C(c, i) <= N (C(i - 1, i) = 0): a
      // branch-free binary search of fixed length (no divergent trip counts)
      const uint32_t* t = tab + i * kBinN;
      int lo = i - 1;
#pragma unroll
      for (int step = 32; step; step >>= 1) {
        const int c = lo + step;
        lo = (c < hi && t[c] <= N) ? c : lo;
      }
      N -= t[lo];
      m |= 1ull << lo;
      hi = lo;
    }
    if (!ok) atomicExch(bad, 1);
    masks[r] = ok ? m : 0ull;
  }
}

// Table-seeded decode: digit i's candidate c comes from a byte table indexed
// by the residual's top bits (tab_i[j] = largest c with C(c, i) <= j << s_i,
// at most 4096 entries per digit), then c moves up while C(c + 1, i) <= N --
// no step for almost every row (C(c, i) grows past the bucket width for all
// but the smallest residuals). Digit 1 is the residual itself. About a
// fifth of the binary search's instructions and dependent shared loads.
constexpr int kSeedBits = 12;
struct SeedTabs {
  int shift[kBinK];
  int base[kBinK];  // byte offset of digit i's table
  int bytes;
};

__device__ __forceinline__ void seed_tabs(SeedTabs& st, const uint32_t* tab, int k, int E) {
  int off = 0;
  for (int i = 2; i <= k; ++i) {
    const uint32_t top = tab[i * kBinN + E];  // C(E, i): every residual is below it
    const int bl = 32 - __clz(top);
    st.shift[i] = bl > kSeedBits ? bl - kSeedBits : 0;
    st.base[i] = off;
    off += (int)(top >> st.shift[i]) + 1;
  }
  st.bytes = off;
}

__global__ void k_ranks_to_masks_seeded(const uint32_t* __restrict__ ranks, int64_t rows,
                                        int bits, int k, int E, uint64_t* __restrict__ masks,
                                        int* __restrict__ bad) {
  __shared__ uint32_t tab[kBinN * kBinK];
  __shared__ unsigned char seed[(kBinK - 2) * ((1 << kSeedBits) + 2)];
  load_binom(tab);
  SeedTabs st;
  seed_tabs(st, tab, k, E);
  for (int i = 2; i <= k; ++i) {
    const uint32_t* t = tab + i * kBinN;
    const int n = (int)(t[E] >> st.shift[i]) + 1;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      const uint32_t v = (uint32_t)j << st.shift[i];
      int lo = i - 1;  // largest c < E with C(c, i) <= v (C(i - 1, i) = 0)
#pragma unroll
      for (int step = 32; step; step >>= 1) {
        const int c = lo + step;
        lo = (c < E && t[c] <= v) ? c : lo;
      }
      seed[st.base[i] + j] = (unsigned char)lo;
    }
  }
  __syncthreads();
  // kRowsPT rows per thread and iteration: independent dependency chains
  constexpr int kRowsPT = 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += kRowsPT * stride) {
    uint32_t N[kRowsPT];
    bool ok[kRowsPT], in[kRowsPT];
    uint64_t m[kRowsPT];
#pragma unroll
    for (int q = 0; q < kRowsPT; ++q) {
      in[q] = r + q * stride < rows;
      N[q] = in[q] ? rank_at(ranks, r + q * stride, bits) : 0u;
      ok[q] = N[q] < tab[k * kBinN + E];
      if (!ok[q]) N[q] = 0;  // keeps the table index in range; the row is zeroed below
      m[q] = 0ull;
    }
    for (int i = k; i >= 2; --i) {
      const uint32_t* t = tab + i * kBinN;
      const unsigned char* sd = seed + st.base[i];
      const int sh = st.shift[i];
#pragma unroll
      for (int q = 0; q < kRowsPT; ++q) {
        int c = sd[N[q] >> sh];
        while (c + 1 < E && t[c + 1] <= N[q]) ++c;
        N[q] -= t[c];
        m[q] |= 1ull << c;
      }
    }
#pragma unroll
    for (int q = 0; q < kRowsPT; ++q) {
      if (!in[q]) continue;
      m[q] |= 1ull << (N[q] & 63);  // digit 1: C(c, 1) = c
      if (!ok[q]) atomicExch(bad, 1);
      masks[r + q * stride] = ok[q] ? m[q] : 0ull;
    }
  }
}

__global__ void k_masks_to_ranks(const uint64_t* __restrict__ masks, int64_t rows, int k, int bits,
                                 uint32_t* __restrict__ ranks, int* __restrict__ bad) {
  __shared__ uint32_t tab[kBinN * kBinK];
  load_binom(tab);
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    uint64_t m = masks[r];
    if (__popcll(m) != k) atomicExch(bad, 1);
    uint32_t N = 0;
    for (int i = 1; i <= k && m; ++i) {
      const int c = __ffsll((long long)m) - 1;
      m &= m - 1;
      N += tab[i * kBinN + c];
    }
    if (bits == 32) {
      ranks[r] = N;
    } else {  // OR into the zeroed bit stream (a row straddles at most two words)
      const int64_t b = r * bits;
      const int sh = (int)(b & 31);
      atomicOr(ranks + (b >> 5), N << sh);
      if (sh + bits > 32) atomicOr(ranks + (b >> 5) + 1, N >> (32 - sh));
    }
  }
}
// MOEB_RANK_DECODE=search: the fixed-length binary search (comparison)
bool rank_decode_seeded() {
  const char* e = getenv("MOEB_RANK_DECODE");
  return !(e && !strcmp(e, "search"));
}
}  // namespace

extern "C" int moeb_ranks_to_masks(const uint32_t* ranks, int64_t rows, int k, int E,
                                   uint64_t* masks, int* bad, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(ranks && masks && bad && rows >= 0 && k >= 1 && k <= 8 && E >= k && E <= 64,
               "bad arguments");
  if (rows == 0) return MOEB_OK;
  const int blocks = (int)std::min<int64_t>((rows + 255) / 256, 8LL * moeb::num_sms());
  if (rank_decode_seeded())
    k_ranks_to_masks_seeded<<<blocks, 256, 0, moeb::as_stream(stream)>>>(ranks, rows, 32, k, E,
                                                                         masks, bad);
  else
    k_ranks_to_masks<<<blocks, 256, 0, moeb::as_stream(stream)>>>(ranks, rows, 32, k, E, masks,
                                                                  bad);
  return moeb::check_launch("k_ranks_to_masks");
}

extern "C" int moeb_masks_to_ranks(const uint64_t* masks, int64_t rows, int k, int E,
                                   uint32_t* ranks, int* bad, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(ranks && masks && bad && rows >= 0 && k >= 1 && k <= 8 && E >= k && E <= 64,
               "bad arguments");
  if (rows == 0) return MOEB_OK;
  const int blocks = (int)std::min<int64_t>((rows + 255) / 256, 8LL * moeb::num_sms());
  k_masks_to_ranks<<<blocks, 256, 0, moeb::as_stream(stream)>>>(masks, rows, k, 32, ranks, bad);
  return moeb::check_launch("k_masks_to_ranks");
}

// The same ranks as a dense bit stream of `bits` per row (bits >= the
// rank's width, ceil(log2 C(E, k)) = 27 for 64 / 6: 3.4 B per row);
// `words` holds ceil(rows bits / 32) + 1 u32 (zeroed by the caller for the
// encoder).
extern "C" int moeb_packed_ranks_to_masks(const uint32_t* words, int64_t rows, int bits, int k,
                                          int E, uint64_t* masks, int* bad, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(words && masks && bad && rows >= 0 && k >= 1 && k <= 8 && E >= k && E <= 64 &&
                   bits >= 1 && bits <= 32,
               "bad arguments");
  if (rows == 0) return MOEB_OK;
  const int blocks = (int)std::min<int64_t>((rows + 255) / 256, 8LL * moeb::num_sms());
  if (rank_decode_seeded())
    k_ranks_to_masks_seeded<<<blocks, 256, 0, moeb::as_stream(stream)>>>(words, rows, bits, k, E,
                                                                         masks, bad);
  else
    k_ranks_to_masks<<<blocks, 256, 0, moeb::as_stream(stream)>>>(words, rows, bits, k, E, masks,
                                                                  bad);
  return moeb::check_launch("k_ranks_to_masks");
}

extern "C" int moeb_masks_to_packed_ranks(const uint64_t* masks, int64_t rows, int k, int E,
                                          int bits, uint32_t* words, int* bad, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(words && masks && bad && rows >= 0 && k >= 1 && k <= 8 && E >= k && E <= 64 &&
                   bits >= 1 && bits <= 32,
               "bad arguments");
  if (rows == 0) return MOEB_OK;
  const int blocks = (int)std::min<int64_t>((rows + 255) / 256, 8LL * moeb::num_sms());
  k_masks_to_ranks<<<blocks, 256, 0, moeb::as_stream(stream)>>>(masks, rows, k, bits, words, bad);
  return moeb::check_launch("k_masks_to_ranks");
}

// Packed expert ids: each row's k ascending ids at 6 bits each (E <= 64) in a
// little-endian bit stream, row r in bits [6 k r, 6 k (r + 1)) -- 4.5 B per
// row at k = 6, one more byte than the 27-bit combinatorial rank, but
// decoded with shifts instead of the rank's digit searches (`words` holds
// ceil(6 k rows / 32) + 2 u32; zeroed by the caller for the encoder).
namespace {
__device__ __forceinline__ uint64_t ids6_row(const uint32_t* __restrict__ w, int64_t r, int k) {
  const int64_t b = r * 6 * k;
  const int64_t i = b >> 5;
  const int sh = (int)(b & 31);
  const uint64_t lo = (uint64_t)__ldg(w + i) | ((uint64_t)__ldg(w + i + 1) << 32);
  uint64_t v = lo >> sh;
  if (sh + 6 * k > 64) v |= (uint64_t)__ldg(w + i + 2) << (64 - sh);  // sh > 0 here
  return v;
}

__global__ void k_ids6_to_masks(const uint32_t* __restrict__ words, int64_t rows, int k,
                                uint64_t* __restrict__ masks, int* __restrict__ bad) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t v = ids6_row(words, r, k);
    uint64_t m = 0;
    for (int j = 0; j < k; ++j) m |= 1ull << ((v >> (6 * j)) & 63u);
    if (__popcll(m) != k) atomicExch(bad, 1);  // repeated ids: not a top-k row
    masks[r] = m;
  }
}

__global__ void k_masks_to_ids6(const uint64_t* __restrict__ masks, int64_t rows, int k,
                                uint32_t* __restrict__ words, int* __restrict__ bad) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    uint64_t m = masks[r];
    if (__popcll(m) != k) atomicExch(bad, 1);
    uint64_t v = 0;
    for (int j = 0; j < k && m; ++j) {
      v |= (uint64_t)(__ffsll((long long)m) - 1) << (6 * j);
      m &= m - 1;
    }
    const int64_t b = r * 6 * k;
    const int sh = (int)(b & 31);
    uint32_t* w = words + (b >> 5);
    atomicOr(w, (uint32_t)(v << sh));
    if (sh + 6 * k > 32) atomicOr(w + 1, (uint32_t)(sh ? v >> (32 - sh) : v >> 32));
    if (sh + 6 * k > 64) atomicOr(w + 2, (uint32_t)(v >> (64 - sh)));  // sh > 0 here
  }
}
}  // namespace

extern "C" int moeb_ids6_to_masks(const uint32_t* words, int64_t rows, int k, uint64_t* masks,
                                  int* bad, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(words && masks && bad && rows >= 0 && k >= 1 && k <= 8, "bad arguments");
  if (rows == 0) return MOEB_OK;
  const int blocks = (int)std::min<int64_t>((rows + 255) / 256, 8LL * moeb::num_sms());
  k_ids6_to_masks<<<blocks, 256, 0, moeb::as_stream(stream)>>>(words, rows, k, masks, bad);
  return moeb::check_launch("k_ids6_to_masks");
}

extern "C" int moeb_masks_to_ids6(const uint64_t* masks, int64_t rows, int k, uint32_t* words,
                                  int* bad, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(words && masks && bad && rows >= 0 && k >= 1 && k <= 8, "bad arguments");
  if (rows == 0) return MOEB_OK;
  const int blocks = (int)std::min<int64_t>((rows + 255) / 256, 8LL * moeb::num_sms());
  k_masks_to_ids6<<<blocks, 256, 0, moeb::as_stream(stream)>>>(masks, rows, k, words, bad);
  return moeb::check_launch("k_masks_to_ids6");
}

// Packed id pairs: a row's k ascending ids taken two at a time, each sorted
// pair (a < b) as its rank C(b, 2) + a < 2016 in 11 bits (an odd k's last id
// in 6 bits): 33 bits = 4.125 B per row at k = 6 -- 0.75 B more than the
// 27-bit combinatorial rank, but decoded by three lookups into a 4 KB
// shared-memory table instead of six digit searches. Little-endian bit
// stream, row r in bits [bits r, bits (r + 1)), bits = 11 (k / 2) + 6 (k % 2)
// (`words`: ceil(bits rows / 32) + 2 u32, zeroed by the caller for the encoder).
namespace {
__host__ __device__ constexpr int idpair_bits(int k) { return 11 * (k / 2) + 6 * (k % 2); }

__global__ void k_idpairs_to_masks(const uint32_t* __restrict__ words, int64_t rows, int k,
                                   uint64_t* __restrict__ masks, int* __restrict__ bad) {
  __shared__ uint16_t tab[2016];  // pair rank -> a | b << 6
  for (int i = threadIdx.x; i < 2016; i += blockDim.x) {
    int b = 1;
    while ((b + 1) * b / 2 <= i) ++b;
    tab[i] = (uint16_t)((i - b * (b - 1) / 2) | (b << 6));
  }
  __syncthreads();
  const int bits = idpair_bits(k);
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b0 = r * bits;
    const int64_t i = b0 >> 5;
    const int sh = (int)(b0 & 31);
    uint64_t v = ((uint64_t)__ldg(words + i) | ((uint64_t)__ldg(words + i + 1) << 32)) >> sh;
    if (sh + bits > 64) v |= (uint64_t)__ldg(words + i + 2) << (64 - sh);  // sh > 0 here
    uint64_t m = 0;
    bool ok = true;
    for (int j = 0; j < k / 2; ++j) {
      const uint32_t pr = (uint32_t)(v >> (11 * j)) & 2047u;
      ok = ok && pr < 2016u;
      const uint32_t ab = tab[pr < 2016u ? pr : 0u];
      m |= (1ull << (ab & 63u)) | (1ull << (ab >> 6));
    }
    if (k & 1) m |= 1ull << ((v >> (11 * (k / 2))) & 63u);
    if (!ok || __popcll(m) != k) atomicExch(bad, 1);
    masks[r] = m;
  }
}

__global__ void k_masks_to_idpairs(const uint64_t* __restrict__ masks, int64_t rows, int k,
                                   uint32_t* __restrict__ words, int* __restrict__ bad) {
  const int bits = idpair_bits(k);
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    uint64_t m = masks[r];
    if (__popcll(m) != k) atomicExch(bad, 1);
    uint64_t v = 0;
    int j = 0;
    for (; j + 1 < k && m; j += 2) {
      const uint32_t a = __ffsll((long long)m) - 1;
      m &= m - 1;
      const uint32_t b = m ? __ffsll((long long)m) - 1 : a;
      m &= m - 1;
      v |= (uint64_t)(b * (b - 1) / 2 + a) << (11 * (j / 2));
    }
    if ((k & 1) && m) v |= (uint64_t)(__ffsll((long long)m) - 1) << (11 * (k / 2));
    const int64_t b0 = r * bits;
    const int sh = (int)(b0 & 31);
    uint32_t* w = words + (b0 >> 5);
    atomicOr(w, (uint32_t)(v << sh));
    if (sh + bits > 32) atomicOr(w + 1, (uint32_t)(sh ? v >> (32 - sh) : v >> 32));
    if (sh + bits > 64) atomicOr(w + 2, (uint32_t)(v >> (64 - sh)));  // sh > 0 here
  }
}
}  // namespace

extern "C" int moeb_idpairs_to_masks(const uint32_t* words, int64_t rows, int k, uint64_t* masks,
                                     int* bad, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(words && masks && bad && rows >= 0 && k >= 1 && k <= 8, "bad arguments");
  if (rows == 0) return MOEB_OK;
  const int blocks = (int)std::min<int64_t>((rows + 255) / 256, 4LL * moeb::num_sms());
  k_idpairs_to_masks<<<blocks, 256, 0, moeb::as_stream(stream)>>>(words, rows, k, masks, bad);
  return moeb::check_launch("k_idpairs_to_masks");
}

extern "C" int moeb_masks_to_idpairs(const uint64_t* masks, int64_t rows, int k, uint32_t* words,
                                     int* bad, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(words && masks && bad && rows >= 0 && k >= 1 && k <= 8, "bad arguments");
  if (rows == 0) return MOEB_OK;
  const int blocks = (int)std::min<int64_t>((rows + 255) / 256, 8LL * moeb::num_sms());
  k_masks_to_idpairs<<<blocks, 256, 0, moeb::as_stream(stream)>>>(masks, rows, k, words, bad);
  return moeb::check_launch("k_masks_to_idpairs");
}
