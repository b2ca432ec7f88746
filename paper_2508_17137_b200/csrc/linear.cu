// K3 -- learned_linear predictor over whole traces, with the K2 selection
// head and the K7 metric counters fused in.
//
// Reference: LearnedLinearPredictor.predict (predictors.py:262-268),
// feature_vector / update_history (learner.py:52-72), top_k_experts and the
// threshold rule (learner.py:164-181), metrics (metrics.py:12-79).
//
// The reference scores z = W f with f = [onehot(l) | h_l | 1], where h_l is
// the decayed activation history of layer l (h <- decay*h + x after every
// row of layer l). By linearity the score itself obeys a recurrence:
//   z_0 = b_l,   z_{t+1} = decay * z_t + (1 - decay) * b_l + sum_{e in x_t} W_h[:, e]
// with b_l = W[:, l] + W[:, L+E] and W_h = W[:, L:L+E], so each row costs one
// scaled update plus k column adds instead of a 64x91 mat-vec. All of it
// stays in fp64 (the survey measured top-6/7 logit gaps down to 3.7e-7 on
// random-init weights; fp64 keeps the selection identical to numpy's, and
// the recurrence's rounding drift stays ~1e-15 relative, tests assert 1e-12).
//
// Mapping: two threads per (prompt, layer) stream (adjacent lanes), each
// owning 32 experts: z[32] fp64 in registers (~100 registers -> 20 warps/SM),
// 16-byte column reads from shared memory. Top-k = k passes; in each pass
// every thread finds the first maximum of its unchosen half and the pair
// combines the two candidates with one shuffle (larger value, then lower id):
// exactly lexsort's (-score, id) order. Consecutive streams are consecutive
// layers of the same prompt, so mask rows are read/written contiguously.
// Metrics: ballot+popc per expert over the warp's 16 rows, then one
// shared-memory reduce and one global atomic per counter per block.
#include "common.cuh"

namespace {

constexpr int kThreads = 128;

struct LinArgs {
  const uint64_t* truth;
  const int64_t* row_off;
  int P, L, E;
  const double* Wt;  // [E][L+E+1]
  double decay;
  int budget, threshold, warmup;
  uint64_t* pred;
  double* logits;
  int64_t* metrics;
};

// Shared-memory rows of 64 doubles as two 32-double halves with a 16-byte
// gap (half h starts at double 34*h) and a row stride of 74 doubles = 37
// 16-byte units: the 16-byte chunks a quarter-warp reads (4 streams x 2
// halves, random columns) spread over all 8 bank groups.
constexpr int kES = 74;
__host__ __device__ constexpr int half_off(int h) { return 34 * h; }

template <bool FULL>  // FULL: E == 64, no per-expert bounds checks
__global__ void __launch_bounds__(kThreads) k_linear_predict(const LinArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int L = a.L, E = a.E, F = a.L + a.E + 1;
  double* colT = reinterpret_cast<double*>(smem_raw);  // [E][kES]: colT[e][j] = W[j][L+e]
  double* bias = colT + E * kES;                       // [L][kES]: b_l[j]
  double* bias2 = bias + L * kES;                      // [L][kES]: (1 - decay) b_l[j]
  unsigned long long* mcnt = reinterpret_cast<unsigned long long*>(bias2 + L * kES);  // [3E+3]
  for (int i = threadIdx.x; i < E * 64; i += blockDim.x) {
    const int e = i / 64, j = i % 64;
    colT[e * kES + half_off(j >> 5) + (j & 31)] = j < E ? a.Wt[(int64_t)j * F + L + e] : 0.0;
  }
  for (int i = threadIdx.x; i < L * 64; i += blockDim.x) {
    const int l = i / 64, j = i % 64;
    const double b = j < E ? a.Wt[(int64_t)j * F + l] + a.Wt[(int64_t)j * F + L + E] : 0.0;
    bias[l * kES + half_off(j >> 5) + (j & 31)] = b;
    bias2[l * kES + half_off(j >> 5) + (j & 31)] = (1.0 - a.decay) * b;
  }
  if (a.metrics)
    for (int i = threadIdx.x; i < 3 * E + 3; i += blockDim.x) mcnt[i] = 0;
  __syncthreads();

  const unsigned full = 0xffffffffu;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t sidx = g >> 1;  // stream
  const int h = (int)(g & 1);   // which 32 experts
  const int e0 = 32 * h;
  const bool live = sidx < (int64_t)a.L * a.P;
  const int p = live ? (int)(sidx / L) : 0;
  const int l = live ? (int)(sidx % L) : 0;
  const int64_t r0 = live ? a.row_off[p] : 0;
  const int T = live ? (int)((a.row_off[p + 1] - r0) / L) : 0;
  int Tw = T;  // warp-uniform trip count so ballots/shuffles see every lane
#pragma unroll
  for (int o = 16; o; o >>= 1) Tw = max(Tw, __shfl_xor_sync(full, Tw, o));

  double z[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) z[j] = bias[l * kES + half_off(h) + j];
  const int lane = threadIdx.x & 31;
  uint32_t tp_e = 0, fp_e = 0, fn_e = 0;  // packed counts of experts lane, lane + 32
  uint32_t npos = 0, nexact = 0;
  uint64_t nlabel = 0;
  const uint64_t emask = E == 64 ? ~0ull : ((1ull << E) - 1);
  const int k = a.budget < E ? a.budget : E;
  const double NEG = -__longlong_as_double(0x7ff0000000000000LL);

  for (int t = 0; t < Tw; ++t) {
    const bool valid = t < T;
    const int64_t r = r0 + (int64_t)t * L + l;
    const uint64_t tw = valid ? __ldg(a.truth + r) : 0ull;
    uint64_t pm = 0;
    if (a.threshold) {
      uint32_t m = 0;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if ((FULL || e0 + j < E) && z[j] > 0.0) m |= 1u << j;
      const uint32_t other = __shfl_xor_sync(full, m, 1);
      pm = h ? ((uint64_t)m << 32 | other) : ((uint64_t)other << 32 | m);
    } else {
      uint32_t chosen = 0;
      for (int it = 0; it < k; ++it) {
        double best = NEG;
        int bi = -1;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const bool ok = (FULL || e0 + j < E) && !((chosen >> j) & 1u) && z[j] > best;
          best = ok ? z[j] : best;
          bi = ok ? j : bi;
        }
        const int gi = bi < 0 ? -1 : e0 + bi;
        const double ob = __shfl_xor_sync(full, best, 1);
        const int oi = __shfl_xor_sync(full, gi, 1);
        const bool take_other = oi >= 0 && (gi < 0 || ob > best || (ob == best && oi < gi));
        const int win = take_other ? oi : gi;
        if (win >= e0 && win < e0 + 32) chosen |= 1u << (win - e0);
        pm |= 1ull << win;
      }
    }
    pm &= valid ? ~0ull : 0ull;
    if (valid) {
      if (h == 0) a.pred[r] = pm;
      if (a.logits) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (e0 + j < E) a.logits[r * E + e0 + j] = z[j];
      }
    }
    if (a.metrics) {
      // lane 2i reports experts [0, 32), lane 2i+1 experts [32, 64) of its row
      const bool m = valid && t >= a.warmup;
      const uint64_t tpm = m ? (pm & tw) : 0, fpm = m ? (pm & ~tw) : 0, fnm = m ? (tw & ~pm) : 0;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const uint32_t b1 = __ballot_sync(full, (tpm >> (e0 + j)) & 1ull);
        const uint32_t b2 = __ballot_sync(full, (fpm >> (e0 + j)) & 1ull);
        const uint32_t b3 = __ballot_sync(full, (fnm >> (e0 + j)) & 1ull);
        if (lane == j) {  // lane j owns experts j (low 16 bits) and j + 32 (high 16 bits)
          tp_e += (uint32_t)__popc(b1 & 0x55555555u) | ((uint32_t)__popc(b1 & 0xAAAAAAAAu) << 16);
          fp_e += (uint32_t)__popc(b2 & 0x55555555u) | ((uint32_t)__popc(b2 & 0xAAAAAAAAu) << 16);
          fn_e += (uint32_t)__popc(b3 & 0x55555555u) | ((uint32_t)__popc(b3 & 0xAAAAAAAAu) << 16);
        }
      }
      const bool m0 = m && h == 0;
      npos += m0;
      nexact += m0 && pm == tw;
      nlabel += m0 ? (uint64_t)(E - __popcll((pm ^ tw) & emask)) : 0;
      if ((t & 1023) == 1023) {  // flush packed 16-bit counts before they overflow
        const int j = lane;
        {
          if (j < E) {
            atomicAdd(&mcnt[j], tp_e & 0xFFFFu);
            atomicAdd(&mcnt[E + j], fp_e & 0xFFFFu);
            atomicAdd(&mcnt[2 * E + j], fn_e & 0xFFFFu);
          }
          if (j + 32 < E) {
            atomicAdd(&mcnt[j + 32], tp_e >> 16);
            atomicAdd(&mcnt[E + j + 32], fp_e >> 16);
            atomicAdd(&mcnt[2 * E + j + 32], fn_e >> 16);
          }
        }
        tp_e = fp_e = fn_e = 0;
      }
    }
    if (valid) {  // update_history (learner.py:62-72), as a logit recurrence
      const double2* b2 = reinterpret_cast<const double2*>(bias2 + l * kES + half_off(h));
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const double2 v = b2[j];
        z[2 * j] = fma(a.decay, z[2 * j], v.x);
        z[2 * j + 1] = fma(a.decay, z[2 * j + 1], v.y);
      }
      uint64_t m = tw;
      while (m) {
        const int ex = __ffsll((long long)m) - 1;
        m &= m - 1;
        const double2* col = reinterpret_cast<const double2*>(colT + ex * kES + half_off(h));
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const double2 v = col[j];
          z[2 * j] += v.x;
          z[2 * j + 1] += v.y;
        }
      }
    }
  }

  if (a.metrics) {
    const int j = lane;
    if (j < E) {
      atomicAdd(&mcnt[j], (unsigned long long)(tp_e & 0xFFFFu));
      atomicAdd(&mcnt[E + j], (unsigned long long)(fp_e & 0xFFFFu));
      atomicAdd(&mcnt[2 * E + j], (unsigned long long)(fn_e & 0xFFFFu));
    }
    if (j + 32 < E) {
      atomicAdd(&mcnt[j + 32], (unsigned long long)(tp_e >> 16));
      atomicAdd(&mcnt[E + j + 32], (unsigned long long)(fp_e >> 16));
      atomicAdd(&mcnt[2 * E + j + 32], (unsigned long long)(fn_e >> 16));
    }
    atomicAdd(&mcnt[3 * E], (unsigned long long)npos);
    atomicAdd(&mcnt[3 * E + 1], (unsigned long long)nexact);
    atomicAdd(&mcnt[3 * E + 2], (unsigned long long)nlabel);
    __syncthreads();
    for (int i = threadIdx.x; i < 3 * E + 3; i += blockDim.x)
      if (mcnt[i]) atomicAdd(reinterpret_cast<unsigned long long*>(a.metrics + i), mcnt[i]);
  }
}

}  // namespace

extern "C" int moeb_linear_predict(const uint64_t* truth, const int64_t* prompt_row_off,
                                   int n_prompts, int L, int E, const double* weights,
                                   double decay, int budget, int threshold, int warmup_tokens,
                                   uint64_t* pred, double* logits, int64_t* metrics,
                                   void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(truth && prompt_row_off && weights && pred, "null argument");
  MOEB_REQUIRE(n_prompts >= 1 && L >= 1 && E >= 1 && E <= 64,
               "learned_linear kernel supports E <= 64 (got L=%d E=%d)", L, E);
  MOEB_REQUIRE(budget >= 1 && warmup_tokens >= 0, "bad budget/warmup");
  MOEB_REQUIRE(decay >= 0.0 && decay < 1.0, "decay must be in [0, 1)");
  LinArgs a{truth, prompt_row_off, n_prompts, L, E, weights, decay, budget,
            threshold ? 1 : 0, warmup_tokens, pred, logits, metrics};
  const size_t smem = sizeof(double) * ((size_t)E * kES + 2 * (size_t)L * kES) +
                      sizeof(unsigned long long) * (3 * E + 3);
  if ((int)smem > moeb::max_smem_per_block())
    return moeb::fail(MOEB_ESMEM, "learned_linear tables need %zu B of shared memory", smem);
  auto kern = E == 64 ? k_linear_predict<true> : k_linear_predict<false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t threads = 2 * (int64_t)L * n_prompts;  // two per (prompt, layer) stream
  const int64_t blocks = (threads + kThreads - 1) / kThreads;
  kern<<<(unsigned)blocks, kThreads, smem, moeb::as_stream(stream)>>>(a);
  return moeb::check_launch("k_linear_predict");
}
