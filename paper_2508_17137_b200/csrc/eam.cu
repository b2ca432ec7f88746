// K6 -- EAM cosine predictor (MoE-Infinity baseline) over whole traces.
//
// Reference: EamCosinePredictor / CosineMatchSession (predictors.py:151-219),
// SketchCollection.match_nearest / layer_block (sketches.py:145-189),
// _top_weights (predictors.py:142-148), normalize (core.py:221-231).
//
// At a measured row (t, l) the query is the partial request-level activation
// matrix (rEAM) before the row, normalised per layer. Every trace row adds
// exactly k activations, so the row sums are R = k(t+1) for layers < l and
// R = k t for layers >= l. With d_s(l') = U_s,l' . c(l')
// (c = raw counts) the cosine score is, up to the positive factor 1/(k |q|)
// that cannot change the argmax,
//     score_s(t, l) = Dlow_s / (t + 1) + Dhigh_s / t,
//     Dlow_s = sum_{l' < l} d_s(l'),  Dhigh_s = sum_{l' >= l} d_s(l')
// (a t = 0 term is zero: normalize() leaves empty rows at zero). Accumulating
// a row changes one d_s(l) by the sum of k entries of U (a coalesced gather
// from the transposed unit matrix), so each step is O(S) work instead of the
// reference session's O(S*E) or the direct form's O(S*L*E).
//
// Mapping: one CTA per prompt; thread j owns sketches j, j + blockDim, ...;
// d_s(l') lives in shared memory [L][S]; a block argmax (warp shuffles, ties
// to the lower index) picks the sketch; the prediction is a table lookup
// topw[idx][l] precomputed by moeb_eam_prepare.
#include <cfloat>
#include <cstdlib>
#include <cuda_fp16.h>

#include "common.cuh"

namespace {

constexpr int kSPT = 8;  // sketches per thread
constexpr int kMaxK = 8;  // experts per row gathered together (more: sequential loop)

__global__ void k_eam_norms(const double* __restrict__ sk, int S, int D, double* __restrict__ unit_t) {
  const int s = blockIdx.x;
  __shared__ double red[32];
  double acc = 0.0;
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    const double x = sk[(int64_t)s * D + d];
    acc = fma(x, x, acc);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  double nrm = sqrt(red[0]);
  if (!(nrm > 0.0)) nrm = 1.0;  // zero rows stay zero (sketches.py:158-160)
  for (int d = threadIdx.x; d < D; d += blockDim.x)
    unit_t[(int64_t)d * S + s] = sk[(int64_t)s * D + d] / nrm;
}

// topw[s][l] = top-`budget` strictly positive raw weights, ties to lower id.
__global__ void k_eam_topw(const double* __restrict__ sk, int S, int L, int E, int budget,
                           uint64_t* __restrict__ topw) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)S * L) return;
  const int s = (int)(i / L), l = (int)(i % L);
  const int W = (E + 63) / 64;
  const double* blk = sk + (int64_t)s * L * E + (int64_t)l * E;
  uint64_t m[4] = {0, 0, 0, 0};
  for (int j = 0; j < budget; ++j) {
    int best = -1;
    double bv = 0.0;
    for (int e = 0; e < E; ++e) {
      const double v = blk[e];
      if (!(v > 0.0) || ((m[e >> 6] >> (e & 63)) & 1ull)) continue;
      if (best < 0 || v > bv) {
        best = e;
        bv = v;
      }
    }
    if (best < 0) break;
    m[best >> 6] |= 1ull << (best & 63);
  }
  for (int w = 0; w < W; ++w) topw[i * W + w] = m[w];
}

template <int W>
__global__ void __launch_bounds__(256) k_eam_predict(
    const uint64_t* __restrict__ truth, const int64_t* __restrict__ row_off, int L, int E,
    int warmup, const double* __restrict__ unit_t, const uint64_t* __restrict__ topw, int S,
    int32_t* __restrict__ idx_out, uint64_t* __restrict__ pred) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* d = reinterpret_cast<double*>(smem_raw);  // [L][S]
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  const int p = blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
  for (int i = tid; i < L * S; i += nt) d[i] = 0.0;
  double dlo[kSPT], dhi[kSPT];
#pragma unroll
  for (int j = 0; j < kSPT; ++j) dlo[j] = dhi[j] = 0.0;
  __syncthreads();

  const int64_t r0 = row_off[p], r1 = row_off[p + 1];
  int l = 0, t = 0;
  for (int64_t r = r0; r < r1; ++r) {
    uint64_t tw[W];
#pragma unroll
    for (int w = 0; w < W; ++w) tw[w] = __ldg(truth + r * W + w);
    if (t >= warmup) {
      double best = -DBL_MAX;
      int bi = 0x7fffffff;
#pragma unroll
      for (int j = 0; j < kSPT; ++j) {
        const int s = tid + j * nt;
        if (s < S) {
          // score * t (t + 1): same argmax, no division (see k_eam_predict_tok)
          const double v = t > 0 ? fma(dlo[j], (double)t, dhi[j] * (double)(t + 1)) : dlo[j];
          if (v > best) {  // ascending s within the thread: first max wins
            best = v;
            bi = s;
          }
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) {
          best = ov;
          bi = oi;
        }
      }
      if (lane == 0) {
        red_v[wid] = best;
        red_i[wid] = bi;
      }
      __syncthreads();
      if (tid == 0) {
        double bv = red_v[0];
        int b = red_i[0];
        for (int w = 1; w < (nt >> 5); ++w)
          if (red_v[w] > bv || (red_v[w] == bv && red_i[w] < b)) {
            bv = red_v[w];
            b = red_i[w];
          }
        if (idx_out) idx_out[r] = b;
#pragma unroll
        for (int w = 0; w < W; ++w) pred[r * W + w] = topw[((int64_t)b * L + l) * W + w];
      }
      __syncthreads();
    } else if (tid == 0) {
      if (idx_out) idx_out[r] = -1;
#pragma unroll
      for (int w = 0; w < W; ++w) pred[r * W + w] = 0;
    }
    // accumulate the row into the partial rEAM (core.py:182-194). The
    // row's experts are listed first so that all gathers are in flight
    // together (one L2 round trip per row instead of one per expert); the
    // sum keeps ascending expert order.
    int exl[kMaxK];
    int nk = 0;
    if (W == 1) {  // registers: peel the lowest set bits in an unrolled sequence
      uint64_t mm = tw[0];
      nk = __popcll(mm);
#pragma unroll
      for (int i = 0; i < kMaxK; ++i) {
        exl[i] = __ffsll((long long)mm) - 1;
        mm &= mm - 1;
      }
    } else {
      MOEB_FOR_EACH_BIT(W, tw, ex, {
        if (nk < kMaxK) exl[nk] = ex;
        ++nk;
      })
    }
#pragma unroll
    for (int j = 0; j < kSPT; ++j) {
      const int s = tid + j * nt;
      if (s < S) {
        double g = 0.0;
        if (nk <= kMaxK) {
          double gv[kMaxK];
#pragma unroll
          for (int i = 0; i < kMaxK; ++i)
            gv[i] = i < nk ? __ldg(unit_t + (int64_t)(l * E + exl[i]) * S + s) : 0.0;
#pragma unroll
          for (int i = 0; i < kMaxK; ++i)
            if (i < nk) g += gv[i];
        } else {
          MOEB_FOR_EACH_BIT(W, tw, ex, { g += __ldg(unit_t + (int64_t)(l * E + ex) * S + s); })
        }
        const double dold = d[l * S + s];
        const double dnew = dold + g;
        d[l * S + s] = dnew;
        dhi[j] -= dold;
        dlo[j] += dnew;
      }
    }
    if (++l == L) {
      l = 0;
      ++t;
#pragma unroll
      for (int j = 0; j < kSPT; ++j) {
        dhi[j] = dlo[j];
        dlo[j] = 0.0;
      }
    }
  }
}

// K6 token-batched (E <= 64, S <= 128, L a template constant): thread s
// owns sketch s and keeps its per-layer partial sums d_s(l') in registers; a
// token's L rows are scored in one register pass, the L x S scores go to
// shared memory, and each warp then takes the argmax of whole rows (lane =
// 4 sketches, shuffles, ties to the lower index). Two block barriers per
// token instead of two per row. The row's expert ids are decoded once per
// token (by L threads, into shared memory), and the score is scaled by the
// positive t (t + 1) -- score' = dlo t + dhi (t + 1), same argmax, no fp64
// division (at t = 0: dlo).
template <int L, int K>
__global__ void __launch_bounds__(128) k_eam_predict_tok(
    const uint64_t* __restrict__ truth, const int64_t* __restrict__ row_off, int E, int warmup,
    const double* __restrict__ unit_t, const uint64_t* __restrict__ topw, int S,
    int32_t* __restrict__ idx_out, uint64_t* __restrict__ pred) {
  extern __shared__ __align__(16) unsigned char smem_tok[];
  auto sc = reinterpret_cast<double(*)[128]>(smem_tok);  // [L][128] scores of the token's rows
  // [L][8] element offsets (l E + ex) S of the rows' unit entries, ascending ex
  auto offs = reinterpret_cast<int(*)[8]>(smem_tok + sizeof(double) * L * 128);
  auto nks = reinterpret_cast<int*>(smem_tok + sizeof(double) * L * 128 + sizeof(int) * 8 * L);
  const int p = blockIdx.x;
  const int s = threadIdx.x, lane = s & 31, wid = s >> 5;
  const bool live = s < S;
  const double* us = unit_t + (live ? s : 0);
  double d[L];
#pragma unroll
  for (int l = 0; l < L; ++l) d[l] = 0.0;
  double dlo = 0.0, dhi = 0.0;
  const int64_t r0 = row_off[p];
  const int T = (int)((row_off[p + 1] - r0) / L);
  for (int t = 0; t < T; ++t) {
    if (s < L) {  // the row's unit-entry offsets, ascending expert id
      uint64_t mm = __ldg(truth + r0 + (int64_t)t * L + s);
      nks[s] = __popcll(mm);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int ex = mm ? __ffsll((long long)mm) - 1 : 0;
        mm &= mm - 1;
        offs[s][i] = (s * E + ex) * S;
      }
    }
    __syncthreads();  // offsets of token t in; token t-1's argmax done with sc
    const bool scored = t >= warmup;
    const double ft = (double)t, ft1 = (double)(t + 1);
    // the token's gathers in groups of kGrp layers, the next group's loads
    // issued before this group's sums and recurrence (software pipelining;
    // the loops are unrolled, so the buffer swap is register renaming)
    constexpr int kGrp = 2;
    double ga[kGrp][K], gb[kGrp][K];
    bool fa[kGrp], fb[kGrp];
    auto issue = [&](double (&gv)[kGrp][K], bool (&f)[kGrp], int l0) {
#pragma unroll
      for (int q = 0; q < kGrp; ++q) {
        const int l = l0 + q;
        f[q] = l < L && nks[l < L ? l : 0] == K;
        if (f[q]) {
          const int4 o0 = *reinterpret_cast<const int4*>(&offs[l][0]);
          const int4 o1 = *reinterpret_cast<const int4*>(&offs[l][4]);
          const int o[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
#pragma unroll
          for (int i = 0; i < K; ++i) gv[q][i] = __ldg(us + o[i]);
        }
      }
    };
    issue(ga, fa, 0);
#pragma unroll
    for (int l = 0; l < L; ++l) {
      const int q = l % kGrp;
      if (q == 0 && l + kGrp < L) issue(gb, fb, l + kGrp);
      double g;
      if (fa[q]) {  // the top-k row: summed in ascending expert order
        g = ga[q][0];
#pragma unroll
        for (int i = 1; i < K; ++i) g += ga[q][i];
      } else {  // any other expert count: in ascending order
        g = 0.0;
        uint64_t mm = __ldg(truth + r0 + (int64_t)t * L + l);
        while (mm) {
          const int ex = __ffsll((long long)mm) - 1;
          mm &= mm - 1;
          g += __ldg(us + (int64_t)(l * E + ex) * S);
        }
      }
      if (q == kGrp - 1) {
#pragma unroll
        for (int a = 0; a < kGrp; ++a) {
          fa[a] = fb[a];
#pragma unroll
          for (int i = 0; i < K; ++i) ga[a][i] = gb[a][i];
        }
      }
      if (scored) sc[l][s] = live ? (t > 0 ? fma(dlo, ft, dhi * ft1) : dlo) : -DBL_MAX;
      const double dold = d[l];
      const double dnew = dold + g;
      d[l] = dnew;
      dhi -= dold;
      dlo += dnew;
    }
    dhi = dlo;
    dlo = 0.0;
    __syncthreads();  // all scores of token t in
    const int64_t rt = r0 + (int64_t)t * L;
    if (scored) {
      for (int l = wid; l < L; l += 4) {
        double best = -DBL_MAX;
        int bi = 0x7fffffff;
#pragma unroll
        for (int j = 0; j < 4; ++j) {  // ascending s within the lane: first max wins
          const int ss = lane + 32 * j;
          const double v = sc[l][ss];
          if (ss < S && v > best) {
            best = v;
            bi = ss;
          }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ov > best || (ov == best && oi < bi)) {
            best = ov;
            bi = oi;
          }
        }
        if (lane == 0) {
          if (idx_out) idx_out[rt + l] = bi;
          pred[rt + l] = topw[(int64_t)bi * L + l];
        }
      }
    } else {
      for (int l = s; l < L; l += blockDim.x) {
        if (idx_out) idx_out[rt + l] = -1;
        pred[rt + l] = 0;
      }
    }
  }
}

}  // namespace

extern "C" int moeb_eam_prepare(const double* sketches, int S, int L, int E, int budget,
                                double* unit_t, uint64_t* topw, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(sketches && unit_t && topw, "null argument");
  MOEB_REQUIRE(S >= 1 && L >= 1 && E >= 1 && E <= 256 && budget >= 1, "bad shape");
  cudaStream_t s = moeb::as_stream(stream);
  k_eam_norms<<<S, 256, 0, s>>>(sketches, S, L * E, unit_t);
  if (int rc = moeb::check_launch("k_eam_norms")) return rc;
  const int64_t n = (int64_t)S * L;
  k_eam_topw<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(sketches, S, L, E, budget, topw);
  return moeb::check_launch("k_eam_topw");
}

extern "C" int moeb_eam_predict(const uint64_t* truth, const int64_t* prompt_row_off,
                                int n_prompts, int L, int E, int warmup_tokens,
                                const double* unit_t, const uint64_t* topw, int S,
                                int32_t* idx_out, uint64_t* pred, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(truth && prompt_row_off && unit_t && topw && pred, "null argument");
  MOEB_REQUIRE(n_prompts >= 1 && L >= 1 && E >= 1 && E <= 256 && warmup_tokens >= 0,
               "bad shape");
  MOEB_REQUIRE(S >= 1 && S <= 256 * kSPT, "eam_predict supports 1 <= S <= %d", 256 * kSPT);
  int nt = ((S + kSPT - 1) / kSPT + 31) / 32 * 32;
  nt = nt < 32 ? 32 : nt;
  while (nt < 128 && nt < ((S + 31) / 32) * 32) nt += 32;
  const size_t smem = sizeof(double) * (size_t)L * S;
  if ((int)smem > moeb::max_smem_per_block())
    return moeb::fail(MOEB_ESMEM, "eam state %zu B (L*S doubles) exceeds shared memory", smem);
  cudaStream_t s = moeb::as_stream(stream);
  const int W = moeb::words_for(E);
  const char* env = getenv("MOEB_K6");  // MOEB_K6=row: the row-by-row kernel
  if (W == 1 && S <= 128 && (L == 26 || L == 27) && !(env && env[0] == 'r')) {
    const int tsm = (int)(sizeof(double) * L * 128 + sizeof(int) * 9 * L);
#define MOEB_EAM_TOK(LL, KK)                                                                   \
  do {                                                                                         \
    moeb::set_smem(k_eam_predict_tok<LL, KK>, tsm);                                            \
    k_eam_predict_tok<LL, KK><<<n_prompts, 128, tsm, s>>>(truth, prompt_row_off, E,            \
                                                          warmup_tokens, unit_t, topw, S,       \
                                                          idx_out, pred);                       \
  } while (0)
    if (L == 26)
      MOEB_EAM_TOK(26, 6);
    else
      MOEB_EAM_TOK(27, 6);
#undef MOEB_EAM_TOK
    return moeb::check_launch("k_eam_predict_tok");
  }
#define MOEB_EAM_LAUNCH(WW)                                                                     \
  do {                                                                                         \
    cudaFuncSetAttribute(k_eam_predict<WW>, cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                         (int)smem);                                                           \
    k_eam_predict<WW><<<n_prompts, nt, smem, s>>>(truth, prompt_row_off, L, E, warmup_tokens, \
                                                  unit_t, topw, S, idx_out, pred);             \
  } while (0)
  switch (W) {
    case 1: MOEB_EAM_LAUNCH(1); break;
    case 2: MOEB_EAM_LAUNCH(2); break;
    case 3: MOEB_EAM_LAUNCH(3); break;
    default: MOEB_EAM_LAUNCH(4); break;
  }
#undef MOEB_EAM_LAUNCH
  return moeb::check_launch("k_eam_predict");
}

// ---------------------------------------------------------------------------
// K8: rEAM counts and sketch normalisation; brute-force query matcher.
// ---------------------------------------------------------------------------
namespace {

template <int W>
__global__ void k_ream_counts(const uint64_t* __restrict__ truth, const int64_t* __restrict__ row_off,
                              int L, int E, int max_tokens, int32_t* __restrict__ counts) {
  const int p = blockIdx.x;
  int32_t* c = counts + (int64_t)p * L * E;
  for (int i = threadIdx.x; i < L * E; i += blockDim.x) c[i] = 0;
  __syncthreads();
  const int64_t r0 = row_off[p];
  int64_t r1 = row_off[p + 1];
  if (max_tokens >= 0 && r0 + (int64_t)max_tokens * L < r1) r1 = r0 + (int64_t)max_tokens * L;
  for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
    const int l = (int)((r - r0) % L);
#pragma unroll
    for (int w = 0; w < W; ++w) {
      uint64_t m = __ldg(truth + r * W + w);
      while (m) {
        const int ex = w * 64 + __ffsll((long long)m) - 1;
        m &= m - 1;
        atomicAdd(c + l * E + ex, 1);
      }
    }
  }
}

__global__ void k_sketch_normalize(const int32_t* __restrict__ counts, int L, int E, int binarize,
                                   double* __restrict__ out) {
  const int p = blockIdx.x;
  for (int l = threadIdx.x >> 5; l < L; l += blockDim.x >> 5) {
    const int32_t* c = counts + ((int64_t)p * L + l) * E;
    int64_t sum = 0;
    for (int e = threadIdx.x & 31; e < E; e += 32) sum += binarize ? (c[e] > 0) : c[e];
#pragma unroll
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    double* o_ = out + ((int64_t)p * L + l) * E;
    for (int e = threadIdx.x & 31; e < E; e += 32) {
      const double v = binarize ? (double)(c[e] > 0) : (double)c[e];
      o_[e] = sum > 0 ? v / (double)sum : 0.0;
    }
  }
}

__global__ void __launch_bounds__(256) k_match_queries(const double* __restrict__ q, int D,
                                                       const double* __restrict__ unit_t, int S,
                                                       int32_t* __restrict__ idx_out,
                                                       double* __restrict__ sim_out) {
  extern __shared__ double qs[];
  __shared__ double red_v[8];
  __shared__ int red_i[8];
  const int m = blockIdx.x;
  const double* qm = q + (int64_t)m * D;
  double n2 = 0.0;
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    qs[d] = qm[d];
    n2 = fma(qm[d], qm[d], n2);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) n2 += __shfl_xor_sync(0xffffffffu, n2, o);
  if ((threadIdx.x & 31) == 0) red_v[threadIdx.x >> 5] = n2;
  __syncthreads();
  double qn2 = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) qn2 += red_v[w];
  __syncthreads();
  const double qn = sqrt(qn2);
  double best = -DBL_MAX;
  int bi = 0x7fffffff;
  for (int s = threadIdx.x; s < S; s += blockDim.x) {
    double acc = 0.0;
    for (int d = 0; d < D; ++d) acc = fma(unit_t[(int64_t)d * S + s], qs[d] / qn, acc);
    if (acc > best) {
      best = acc;
      bi = s;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) {
      best = ov;
      bi = oi;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    red_v[threadIdx.x >> 5] = best;
    red_i[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double bv = red_v[0];
    int b = red_i[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (red_v[w] > bv || (red_v[w] == bv && red_i[w] < b)) {
        bv = red_v[w];
        b = red_i[w];
      }
    if (qn2 == 0.0) {  // zero query: index 0, similarity 0 (sketches.py:179-181)
      b = 0;
      bv = 0.0;
    }
    idx_out[m] = b;
    if (sim_out) sim_out[m] = bv > 1.0 ? 1.0 : (bv < -1.0 ? -1.0 : bv);
  }
}

}  // namespace

extern "C" int moeb_ream_counts(const uint64_t* truth, const int64_t* prompt_row_off,
                                int n_prompts, int L, int E, int max_tokens, int32_t* counts,
                                void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(truth && prompt_row_off && counts, "null argument");
  MOEB_REQUIRE(n_prompts >= 1 && L >= 1 && E >= 1 && E <= 256, "bad shape");
  cudaStream_t s = moeb::as_stream(stream);
  switch (moeb::words_for(E)) {
    case 1: k_ream_counts<1><<<n_prompts, 256, 0, s>>>(truth, prompt_row_off, L, E, max_tokens, counts); break;
    case 2: k_ream_counts<2><<<n_prompts, 256, 0, s>>>(truth, prompt_row_off, L, E, max_tokens, counts); break;
    case 3: k_ream_counts<3><<<n_prompts, 256, 0, s>>>(truth, prompt_row_off, L, E, max_tokens, counts); break;
    default: k_ream_counts<4><<<n_prompts, 256, 0, s>>>(truth, prompt_row_off, L, E, max_tokens, counts); break;
  }
  return moeb::check_launch("k_ream_counts");
}

extern "C" int moeb_sketch_normalize(const int32_t* counts, int n, int L, int E, int binarize,
                                     double* sketches, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(counts && sketches && n >= 1 && L >= 1 && E >= 1, "bad arguments");
  k_sketch_normalize<<<n, 256, 0, moeb::as_stream(stream)>>>(counts, L, E, binarize, sketches);
  return moeb::check_launch("k_sketch_normalize");
}

extern "C" int moeb_match_queries(const double* queries, int M, int D, const double* unit_t,
                                  int S, int32_t* idx_out, double* sim_out, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(queries && unit_t && idx_out && M >= 0 && D >= 1 && S >= 1, "bad arguments");
  if (M == 0) return MOEB_OK;
  const size_t smem = sizeof(double) * (size_t)D;
  if ((int)smem > moeb::max_smem_per_block())
    return moeb::fail(MOEB_ESMEM, "query length %d too long", D);
  cudaFuncSetAttribute(k_match_queries, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_match_queries<<<M, 256, smem, moeb::as_stream(stream)>>>(queries, D, unit_t, S, idx_out,
                                                            sim_out);
  return moeb::check_launch("k_match_queries");
}

// ---------------------------------------------------------------------------
// K6b -- EAM matching at scale on tensor cores (BASELINE C4).
//
// scores[m][s] = C_m . U_s with C_m integer activation counts (exact in fp16
// up to 2048) and U_s the unit sketch split U = U_hi + 2^-11 U_lo' (both fp16,
// U_lo' = 2^11 (U - U_hi) kept in the normal fp16 range). The split is
// K-concatenated, so ONE tcgen05 GEMM computes
//   [C | 2^-11 C] . [U_hi | U_lo']^T = C . (U_hi + 2^-11 U_lo')
// with a fused per-(query, 256-sketch tile) max/argmax epilogue (K4
// EPI_ROWMAX). moeb_eam_rerank then re-scores, in fp64, every tile whose
// approximate maximum lies within 2 eps of the query's approximate maximum
// (eps bounds the split + fp32 accumulation error), and returns the exact
// first argmax -- SketchCollection.match_nearest semantics (sketches.py:165-184).
// ---------------------------------------------------------------------------
namespace {

__global__ void k_eam_pack_library(const double* __restrict__ sk, int S, int D,
                                   __half* __restrict__ uu, double* __restrict__ norms) {
  const int s = blockIdx.x;  // rows >= S are zero padding
  __shared__ double red[32];
  double acc = 0.0;
  if (s < S)
    for (int d = threadIdx.x; d < D; d += blockDim.x) acc = fma(sk[(int64_t)s * D + d], sk[(int64_t)s * D + d], acc);
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  double n2 = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) n2 += red[w];
  double nrm = sqrt(n2);
  if (!(nrm > 0.0)) nrm = 1.0;  // zero rows stay zero (sketches.py:158-160)
  if (threadIdx.x == 0 && s < S) norms[s] = nrm;
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    const double u = s < S ? sk[(int64_t)s * D + d] / nrm : 0.0;
    const __half hi = __double2half(u);
    const __half lo = __double2half((u - (double)__half2float(hi)) * 2048.0);
    uu[(int64_t)s * 2 * D + d] = hi;
    uu[(int64_t)s * 2 * D + D + d] = lo;
  }
}

__global__ void k_eam_pack_queries(const int32_t* __restrict__ counts, int M, int D,
                                   __half* __restrict__ cc) {
  const int64_t n = (int64_t)M * D;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / D, d = i % D;
    const float c = (float)counts[i];
    cc[m * 2 * D + d] = __float2half_rn(c);
    cc[m * 2 * D + D + d] = __float2half_rn(c * (1.0f / 2048.0f));  // exact: power-of-two scale
  }
}

__global__ void __launch_bounds__(256) k_eam_rerank(
    const float* __restrict__ pval, const int32_t* __restrict__ pidx, int ntiles,
    const int32_t* __restrict__ counts, const double* __restrict__ sk,
    const double* __restrict__ norms, int S, int D, double eps_rel, int32_t* __restrict__ idx_out,
    double* __restrict__ sim_out, int32_t* __restrict__ n_rerank) {
  extern __shared__ double cq[];  // query counts as doubles [D]
  __shared__ float red_f[8];
  __shared__ double red_v[8];
  __shared__ int red_i[8];
  const int m = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double q2 = 0.0;
  for (int d = tid; d < D; d += blockDim.x) {
    const double c = counts[(int64_t)m * D + d];
    cq[d] = c;
    q2 += c * c;
  }
  float gm = -INFINITY;
  for (int t = tid; t < ntiles; t += blockDim.x) gm = fmaxf(gm, pval[(int64_t)m * ntiles + t]);
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    gm = fmaxf(gm, __shfl_xor_sync(0xffffffffu, gm, o));
    q2 += __shfl_xor_sync(0xffffffffu, q2, o);
  }
  if (lane == 0) {
    red_f[warp] = gm;
    red_v[warp] = q2;
  }
  __syncthreads();
  gm = red_f[0];
  q2 = red_v[0];
  for (int w = 1; w < 8; ++w) {
    gm = fmaxf(gm, red_f[w]);
    q2 += red_v[w];
  }
  __syncthreads();
  if (q2 == 0.0) {  // zero query: index 0, similarity 0 (sketches.py:179-181)
    if (tid == 0) {
      idx_out[m] = 0;
      if (sim_out) sim_out[m] = 0.0;
    }
    return;
  }
  const float thr = (float)((double)gm - 2.0 * (eps_rel * fabs((double)gm) + 1e-30));
  double best = -1.0;
  int bi = 0x7fffffff, cnt = 0;
  for (int t = 0; t < ntiles; ++t) {
    if (pval[(int64_t)m * ntiles + t] < thr) continue;  // block-uniform
    ++cnt;
    // one warp per sketch, lanes over d (coalesced rows)
    for (int j = warp; j < 256; j += 8) {
      const int s = t * 256 + j;
      if (s >= S) break;
      const double* row = sk + (int64_t)s * D;
      double acc = 0.0;
      for (int d = lane; d < D; d += 32) acc = fma(row[d], cq[d], acc);
#pragma unroll
      for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      const double v = acc / norms[s];
      if (v > best || (v == best && s < bi)) {
        best = v;
        bi = s;
      }
    }
  }
  if (lane == 0) {
    red_v[warp] = best;
    red_i[warp] = bi;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < 8; ++w)
      if (red_v[w] > best || (red_v[w] == best && red_i[w] < bi)) {
        best = red_v[w];
        bi = red_i[w];
      }
    idx_out[m] = bi;
    if (sim_out) {
      const double c = best / sqrt(q2);
      sim_out[m] = c > 1.0 ? 1.0 : (c < -1.0 ? -1.0 : c);
    }
    if (n_rerank) n_rerank[m] = cnt;
  }
}

}  // namespace

extern "C" int moeb_eam_pack_library(const double* sketches, int S, int D, int S_pad,
                                     void* uu, double* norms, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(sketches && uu && norms && S >= 1 && S_pad >= S && D >= 1, "bad arguments");
  k_eam_pack_library<<<S_pad, 256, 0, moeb::as_stream(stream)>>>(
      sketches, S, D, static_cast<__half*>(uu), norms);
  return moeb::check_launch("k_eam_pack_library");
}

extern "C" int moeb_eam_pack_queries(const int32_t* counts, int M, int D, void* cc,
                                     void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(counts && cc && M >= 0 && D >= 1, "bad arguments");
  if (M == 0) return MOEB_OK;
  k_eam_pack_queries<<<148 * 8, 256, 0, moeb::as_stream(stream)>>>(counts, M, D,
                                                                   static_cast<__half*>(cc));
  return moeb::check_launch("k_eam_pack_queries");
}

extern "C" int moeb_eam_rerank(const float* pval, const int32_t* pidx, int ntiles,
                               const int32_t* counts, const double* sketches,
                               const double* norms, int M, int S, int D, double eps_rel,
                               int32_t* idx_out, double* sim_out, int32_t* n_rerank,
                               void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(pval && counts && sketches && norms && idx_out && M >= 0, "bad arguments");
  if (M == 0) return MOEB_OK;
  const size_t smem = sizeof(double) * (size_t)D;
  cudaFuncSetAttribute(k_eam_rerank, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_eam_rerank<<<M, 256, smem, moeb::as_stream(stream)>>>(pval, pidx, ntiles, counts, sketches,
                                                          norms, S, D, eps_rel, idx_out, sim_out,
                                                          n_rerank);
  return moeb::check_launch("k_eam_rerank");
}

// Per-token partial rEAM counts at layer 0 (C4 queries): for every prompt
// and token t >= warmup, the counts of all rows of tokens < t.
namespace {
template <int W>
__global__ void k_token_prefix_counts(const uint64_t* __restrict__ truth,
                                      const int64_t* __restrict__ row_off,
                                      const int64_t* __restrict__ q_off, int L, int E, int warmup,
                                      int32_t* __restrict__ out) {
  extern __shared__ int32_t cnt[];  // [L*E]
  const int p = blockIdx.x;
  const int D = L * E;
  for (int i = threadIdx.x; i < D; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  const int64_t r0 = row_off[p];
  const int T = (int)((row_off[p + 1] - r0) / L);
  int64_t q = q_off[p];
  for (int t = 0; t < T; ++t) {
    if (t >= warmup) {
      for (int i = threadIdx.x; i < D; i += blockDim.x) out[q * D + i] = cnt[i];
      ++q;
    }
    __syncthreads();
    for (int l = threadIdx.x; l < L; l += blockDim.x) {
      const uint64_t* row = truth + (r0 + (int64_t)t * L + l) * W;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        uint64_t m = row[w];
        while (m) {
          cnt[l * E + w * 64 + __ffsll((long long)m) - 1] += 1;
          m &= m - 1;
        }
      }
    }
    __syncthreads();
  }
}
}  // namespace

extern "C" int moeb_token_prefix_counts(const uint64_t* truth, const int64_t* prompt_row_off,
                                        const int64_t* query_off, int n_prompts, int L, int E,
                                        int warmup_tokens, int32_t* out, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(truth && prompt_row_off && query_off && out && n_prompts >= 1, "bad arguments");
  const size_t smem = sizeof(int32_t) * (size_t)L * E;
  cudaStream_t s = moeb::as_stream(stream);
  switch (moeb::words_for(E)) {
    case 1: k_token_prefix_counts<1><<<n_prompts, 128, smem, s>>>(truth, prompt_row_off, query_off, L, E, warmup_tokens, out); break;
    case 2: k_token_prefix_counts<2><<<n_prompts, 128, smem, s>>>(truth, prompt_row_off, query_off, L, E, warmup_tokens, out); break;
    case 3: k_token_prefix_counts<3><<<n_prompts, 128, smem, s>>>(truth, prompt_row_off, query_off, L, E, warmup_tokens, out); break;
    default: k_token_prefix_counts<4><<<n_prompts, 128, smem, s>>>(truth, prompt_row_off, query_off, L, E, warmup_tokens, out); break;
  }
  return moeb::check_launch("k_token_prefix_counts");
}
