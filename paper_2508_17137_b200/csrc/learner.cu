// learned_linear training on device: the reference's
// per-example SGD (learner.py:116-155) over training_pairs (learner.py:75-94).
//
//  * moeb_linear_features: the decayed history h_l before every trace row --
//    the feature block f[L:L+E] of training_pairs -- with numpy's operation
//    order (h *= decay, then += 1 per fired expert; no FMA contraction), so
//    the features are bit-identical to the reference's.
//  * moeb_linear_sgd_epoch: one epoch of per-example SGD in the host's
//    permutation order. SGD is a strictly sequential chain of weight updates,
//    so one CTA runs it with thread j owning weight row j (in shared memory
//    when it fits): z_j = W_j . f over the non-zero features, the example's
//    mean BCE (numpy's pairwise summation order over the E terms,
//    npy_logaddexp's branch structure), sig = 1 / (1 + exp(-z)),
//    W_j[k] -= lr * (((sig - t) / E) * f_k) with separate roundings, as
//    numpy's `weights -= lr * np.outer((sig - t) / E, f)`. The dot product's
//    summation order differs from BLAS's (ulp-level differences).
#include "common.cuh"

namespace {

// numpy pairwise_sum over a[0..n) (numpy/_core/src/umath/loops_utils.h.src)
__device__ double pairwise_sum(const double* a, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pairwise_sum(a, n2), pairwise_sum(a + n2, n - n2));
}

// npy_logaddexp(0, z)
__device__ __forceinline__ double logaddexp0(double z) {
  if (z == 0.0) return 0.69314718055994530942;  // x + LOGE2
  const double tmp = -z;                         // x - y
  if (tmp > 0) return log1p(exp(-tmp));
  if (tmp <= 0) return z + log1p(exp(tmp));
  return tmp;  // NaN
}

// warp per (prompt, layer) stream; lane handles experts lane, lane + 32, ...
__global__ void k_linear_features(const uint64_t* __restrict__ truth, const int64_t* __restrict__ row_off,
                                  int P, int L, int E, double decay, double* __restrict__ hist) {
  const int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= (int64_t)P * L) return;
  const int p = (int)(s / L), l = (int)(s % L);
  const int W = (E + 63) / 64;
  const int64_t r0 = row_off[p];
  const int T = (int)((row_off[p + 1] - r0) / L);
  double h[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) h[j] = 0.0;
  for (int t = 0; t < T; ++t) {
    const int64_t r = r0 + (int64_t)t * L + l;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int e = lane + 32 * j;
      if (e < E) hist[r * E + e] = h[j];
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int e = lane + 32 * j;
      if (e < E) {
        const uint64_t word = __ldg(truth + r * W + (e >> 6));
        h[j] = __dmul_rn(h[j], decay);  // history[layer] *= decay
        if ((word >> (e & 63)) & 1ull) h[j] = __dadd_rn(h[j], 1.0);  // += 1.0 per fired expert
      }
    }
  }
}

__global__ void k_linear_sgd_epoch(double* __restrict__ Wg, const double* __restrict__ hist,
                                   const uint64_t* __restrict__ truth,
                                   const int64_t* __restrict__ order, int64_t n, int L, int E,
                                   double lr, int w_smem, double* __restrict__ loss_total) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int F = L + E + 1;
  const int W = (E + 63) / 64;
  double* hbuf = reinterpret_cast<double*>(smem_raw);  // [2][E] features (double-buffered)
  double* terms = hbuf + 2 * E;                        // [E] loss terms
  double* Ws = terms + E;                              // [E][F] (w_smem)
  double* Wt = w_smem ? Ws : Wg;
  const int j = threadIdx.x;
  if (w_smem)
    for (int i = j; i < E * F; i += blockDim.x) Ws[i] = Wg[i];
  __syncthreads();
  double total = 0.0;
  if (j < E) hbuf[j] = hist[order[0] * E + j];
  int64_t rn = n > 1 ? order[1] : 0;
  for (int64_t it = 0; it < n; ++it) {
    const int64_t r = order[it];
    const int l = (int)(r % L);
    double* hs = hbuf + (it & 1) * E;
    // the next example's features, loaded under this example's work
    const double hn = (j < E && it + 1 < n) ? hist[rn * E + j] : 0.0;
    rn = it + 2 < n ? order[it + 2] : 0;
    __syncthreads();
    double z = 0.0, t = 0.0, term = 0.0;
    double* wr = Wt + (int64_t)j * F;
    if (j < E) {
      // z = W_j . f, f = [onehot(l) | h | 1], non-zero features in order
      z = wr[l];
      for (int e = 0; e < E; ++e) {
        const double fk = hs[e];
        if (fk != 0.0) z = fma(wr[L + e], fk, z);
      }
      z = __dadd_rn(z, wr[L + E]);
      t = ((truth[r * W + (j >> 6)] >> (j & 63)) & 1ull) ? 1.0 : 0.0;
      term = __dsub_rn(logaddexp0(z), __dmul_rn(t, z));
      terms[j] = term;
    }
    __syncthreads();
    if (j < 32) {  // numpy's pairwise mean of the E terms (same tree, warp 0)
      double part;
      if (E <= 128 && E >= 8) {
        // r[q] = a[q] + a[q+8] + ... sequentially, q < 8; tail added last
        double acc = 0.0;
        const int nb = E - (E % 8);
        if (j < 8) {
          acc = terms[j];
          for (int i = 8 + j; i < nb; i += 8) acc = __dadd_rn(acc, terms[i]);
        }
        const double s1 = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 1));  // r0+r1, ...
        const double s2 = __dadd_rn(s1, __shfl_xor_sync(0xffffffffu, s1, 2));
        double res = __dadd_rn(s2, __shfl_xor_sync(0xffffffffu, s2, 4));
        for (int i = nb; i < E; ++i) res = __dadd_rn(res, terms[i]);
        part = res;
      } else {
        part = j == 0 ? pairwise_sum(terms, E) : 0.0;
      }
      if (j == 0) total = __dadd_rn(total, part / (double)E);
    }
    if (j < E) {
      const double sig = 1.0 / (1.0 + exp(-z));
      const double g = (sig - t) / (double)E;
      // weights -= lr * outer(g, f): only non-zero features change anything
      wr[l] = __dsub_rn(wr[l], __dmul_rn(lr, __dmul_rn(g, 1.0)));
      for (int e = 0; e < E; ++e) {
        const double fk = hs[e];
        if (fk != 0.0) wr[L + e] = __dsub_rn(wr[L + e], __dmul_rn(lr, __dmul_rn(g, fk)));
      }
      wr[L + E] = __dsub_rn(wr[L + E], __dmul_rn(lr, __dmul_rn(g, 1.0)));
    }
    if (j < E) hbuf[((it + 1) & 1) * E + j] = hn;  // other buffer: no reader this round
  }
  __syncthreads();  // every row's last update lands before the copy-out
  if (w_smem)
    for (int i = j; i < E * F; i += blockDim.x) Wg[i] = Ws[i];
  if (j == 0) *loss_total = total;
}

}  // namespace

extern "C" int moeb_linear_features(const uint64_t* truth, const int64_t* prompt_row_off,
                                    int n_prompts, int L, int E, double decay, double* hist,
                                    void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(truth && prompt_row_off && hist && n_prompts >= 1, "null argument");
  MOEB_REQUIRE(L >= 1 && E >= 1 && E <= 256, "unsupported shape L=%d E=%d", L, E);
  const int64_t threads = (int64_t)n_prompts * L * 32;
  k_linear_features<<<(unsigned)((threads + 255) / 256), 256, 0, moeb::as_stream(stream)>>>(
      truth, prompt_row_off, n_prompts, L, E, decay, hist);
  return moeb::check_launch("k_linear_features");
}

extern "C" int moeb_linear_sgd_epoch(double* weights, const double* hist, const uint64_t* truth,
                                     const int64_t* order, int64_t n, int L, int E,
                                     double learning_rate, double* loss_total, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(weights && hist && truth && order && loss_total && n >= 1, "null argument");
  MOEB_REQUIRE(L >= 1 && E >= 1 && E <= 256, "unsupported shape L=%d E=%d", L, E);
  const int F = L + E + 1;
  size_t smem = sizeof(double) * (size_t)(3 * E);  // features [2][E], loss terms [E]
  const size_t wbytes = sizeof(double) * (size_t)E * F;
  const int w_smem = smem + wbytes <= (size_t)moeb::max_smem_per_block() ? 1 : 0;
  if (w_smem) smem += wbytes;
  auto k = k_linear_sgd_epoch;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int threads = ((E + 31) / 32) * 32;
  k<<<1, threads, smem, moeb::as_stream(stream)>>>(weights, hist, truth, order, n, L, E,
                                                   learning_rate, w_smem, loss_total);
  return moeb::check_launch("k_linear_sgd_epoch");
}
