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
// Mapping: one thread per (prompt, layer) stream; consecutive threads take
// consecutive layers of the same prompt, so at every token a warp reads and
// writes ~32 contiguous mask rows (coalesced). z[64] lives in registers; W_h columns and the
// bias table live in shared memory (column-major, stride E+1 against bank
// conflicts). Metrics: each warp turns its 32 rows of pred/truth masks into
// per-expert TP/FP/FN counts with ballot+popc, then one shared-memory reduce
// and one global atomic per counter per block.
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

__global__ void __launch_bounds__(kThreads) k_linear_predict(const LinArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int L = a.L, E = a.E, F = a.L + a.E + 1;
  const int ES = E + 1;  // padded stride
  double* colT = reinterpret_cast<double*>(smem_raw);  // [E][ES]: colT[e][j] = W[j][L+e]
  double* bias = colT + E * ES;                        // [L][ES]: b_l[j]
  double* bias2 = bias + L * ES;                       // [L][ES]: (1 - decay) b_l[j]
  unsigned long long* mcnt = reinterpret_cast<unsigned long long*>(bias2 + L * ES);  // [3E+3]
  for (int i = threadIdx.x; i < E * E; i += blockDim.x) {
    const int e = i / E, j = i % E;
    colT[e * ES + j] = a.Wt[(int64_t)j * F + L + e];
  }
  for (int i = threadIdx.x; i < L * E; i += blockDim.x) {
    const int l = i / E, j = i % E;
    const double b = a.Wt[(int64_t)j * F + l] + a.Wt[(int64_t)j * F + L + E];
    bias[l * ES + j] = b;
    bias2[l * ES + j] = (1.0 - a.decay) * b;
  }
  if (a.metrics)
    for (int i = threadIdx.x; i < 3 * E + 3; i += blockDim.x) mcnt[i] = 0;
  __syncthreads();

  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = g < (int64_t)a.L * a.P;
  const int p = live ? (int)(g / L) : 0;
  const int l = live ? (int)(g % L) : 0;
  const int64_t r0 = live ? a.row_off[p] : 0;
  const int T = live ? (int)((a.row_off[p + 1] - r0) / L) : 0;
  // warp-uniform trip count so ballots see every lane
  int Tw = T;
#pragma unroll
  for (int o = 16; o; o >>= 1) Tw = max(Tw, __shfl_xor_sync(0xffffffffu, Tw, o));

  double z[64];
#pragma unroll
  for (int e = 0; e < 64; ++e) z[e] = e < E ? bias[l * ES + e] : 0.0;
  const int lane = threadIdx.x & 31;
  uint32_t tp_lo = 0, tp_hi = 0, fp_lo = 0, fp_hi = 0, fn_lo = 0, fn_hi = 0;
  uint32_t npos = 0, nexact = 0;
  uint64_t nlabel = 0;
  const uint64_t emask = E == 64 ? ~0ull : ((1ull << E) - 1);
  const int k = a.budget < E ? a.budget : E;

  for (int t = 0; t < Tw; ++t) {
    const bool valid = t < T;
    const int64_t r = r0 + (int64_t)t * L + l;
    uint64_t pm = 0, tw = 0;
    if (valid) {
      tw = __ldg(a.truth + r);
      if (a.threshold) {
#pragma unroll
        for (int e = 0; e < 64; ++e)
          if (e < E && z[e] > 0.0) pm |= 1ull << e;
      } else {
        // k passes of "first maximum among the unchosen": exactly lexsort's
        // (-score, id) order (learner.py:164-169).
        for (int j = 0; j < k; ++j) {
          double best = -__longlong_as_double(0x7ff0000000000000LL);
          int bi = -1;
#pragma unroll
          for (int e = 0; e < 64; ++e) {
            const bool ok = e < E && !((pm >> e) & 1ull) && (bi < 0 || z[e] > best);
            best = ok ? z[e] : best;
            bi = ok ? e : bi;
          }
          pm |= 1ull << bi;
        }
      }
      a.pred[r] = pm;
      if (a.logits) {
#pragma unroll
        for (int e = 0; e < 64; ++e)
          if (e < E) a.logits[r * E + e] = z[e];
      }
    }
    if (a.metrics) {
      const bool m = valid && t >= a.warmup;
      const uint64_t tpm = m ? (pm & tw) : 0, fpm = m ? (pm & ~tw) : 0,
                     fnm = m ? (tw & ~pm) : 0;
#pragma unroll
      for (int e = 0; e < 64; ++e) {
        const uint32_t c1 = __popc(__ballot_sync(0xffffffffu, (tpm >> e) & 1ull));
        const uint32_t c2 = __popc(__ballot_sync(0xffffffffu, (fpm >> e) & 1ull));
        const uint32_t c3 = __popc(__ballot_sync(0xffffffffu, (fnm >> e) & 1ull));
        if (lane == (e & 31)) {
          if (e < 32) {
            tp_lo += c1;
            fp_lo += c2;
            fn_lo += c3;
          } else {
            tp_hi += c1;
            fp_hi += c2;
            fn_hi += c3;
          }
        }
      }
      npos += m;
      nexact += m && pm == tw;
      nlabel += m ? (uint64_t)(E - __popcll((pm ^ tw) & emask)) : 0;
    }
    if (valid) {  // update_history (learner.py:62-72), as a logit recurrence
      const double* b2 = bias2 + l * ES;
#pragma unroll
      for (int e = 0; e < 64; ++e)
        if (e < E) z[e] = fma(a.decay, z[e], b2[e]);
      uint64_t m = tw;
      while (m) {
        const int ex = __ffsll((long long)m) - 1;
        m &= m - 1;
        const double* col = colT + ex * ES;
#pragma unroll
        for (int e = 0; e < 64; ++e)
          if (e < E) z[e] += col[e];
      }
    }
  }

  if (a.metrics) {
    if (lane < E) {
      atomicAdd(&mcnt[lane], tp_lo);
      atomicAdd(&mcnt[E + lane], fp_lo);
      atomicAdd(&mcnt[2 * E + lane], fn_lo);
    }
    if (lane + 32 < E) {
      atomicAdd(&mcnt[lane + 32], tp_hi);
      atomicAdd(&mcnt[E + lane + 32], fp_hi);
      atomicAdd(&mcnt[2 * E + lane + 32], fn_hi);
    }
    atomicAdd(&mcnt[3 * E], npos);
    atomicAdd(&mcnt[3 * E + 1], nexact);
    atomicAdd(&mcnt[3 * E + 2], nlabel);
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
  const size_t smem = sizeof(double) * ((size_t)E * (E + 1) + 2 * (size_t)L * (E + 1)) +
                      sizeof(unsigned long long) * (3 * E + 3);
  if ((int)smem > moeb::max_smem_per_block())
    return moeb::fail(MOEB_ESMEM, "learned_linear tables need %zu B of shared memory", smem);
  cudaFuncSetAttribute(k_linear_predict, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t streams = (int64_t)L * n_prompts;
  const int64_t blocks = (streams + kThreads - 1) / kThreads;
  k_linear_predict<<<(unsigned)blocks, kThreads, smem, moeb::as_stream(stream)>>>(a);
  return moeb::check_launch("k_linear_predict");
}
