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
// Mapping: TPS threads per (prompt, layer) stream (TPS = 2: adjacent lanes,
// part q = lane % TPS), each owning NS = 64 / TPS experts as z[NS] fp64 in
// registers, 16-byte column reads from shared memory. Consecutive streams are
// consecutive layers of the same prompt, so mask rows are read/written
// contiguously. Persistent CTAs (2 per SM) loop over groups of streams, so
// the 92 KB weight tables are staged once per CTA.
//
// Bank-conflict-free column reads: a quarter-warp (8 lanes) reads 8
// different, data-dependent columns at once. Every (column, part) is stored
// as NS 16-byte units -- its NS/2 units followed by a copy -- and a lane reads
// units [rot, rot + NS/2) with rot = lane & 7, so register pair j holds unit
// (j + rot) mod NS/2 and the 8 lanes of a quarter-warp always hit 8 distinct
// bank groups, whatever the columns. Slot s of part q thus holds expert
// NS q + ((s + 2 rot) mod NS).
//
// Selection (top-k, learner.py:164-169): 32-bit keys = order-preserving map
// of the fp64 high word with the low log2(NS) bits replaced by the register
// slot; k + 1 passes of "largest key below the last winner" (2 integer ops
// per element) pick the k largest keys, and the (k+1)-th confirms the cut: if
// the k-th and (k+1)-th truncated keys are >= 2 buckets apart, the selected
// set is exactly the fp64 top-k (the key map is monotone; equal fp64 values
// -- including +-0 -- land in equal or adjacent buckets). Otherwise the
// stream redoes the row with exact fp64 passes, ties to the lower expert id
// (lexsort's (-score, id) order). The metric counters (K7) run as a separate
// HBM-streaming pass over the predicted masks (metrics.cu).
#include <cstdlib>

#include "common.cuh"

namespace {

struct LinArgs {
  const uint64_t* truth;
  const int64_t* row_off;
  int P, L, E;
  const double* Wt;  // [E][L+E+1]
  double decay;
  int budget, threshold, warmup;
  uint64_t* pred;
  double* logits;
  int64_t* counts;  // nullable [2 + 2L]: measured accesses, prediction hits, per layer of each
  const int* gate;  // nullable: run only if *gate > gate_cap (K3t's list overflowed)
  int gate_cap;
};

template <int TPS>
struct K3Cfg {
  static constexpr int NS = 64 / TPS;                    // experts (slots) per thread
  static constexpr int kThreads = 256;  // 2 CTAs per SM (<= 128 registers, no spills)
  static constexpr int kStreams = kThreads / TPS;
  static constexpr int kUnits = NS;                      // 16-byte units per (column, part)
};

// rot as an opaque value, so per-slot expert ids are recomputed where used
// instead of being hoisted into NS live registers
__device__ __forceinline__ int opaque(int v) {
  int r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}

template <int NS>
__device__ __forceinline__ int slot_expert(int s, int q, int rot) {
  return NS * q + ((s + 2 * rot) & (NS - 1));
}

template <int NS>
__device__ __forceinline__ uint32_t order_key(double z, int s) {
  const uint32_t hi = (uint32_t)__double2hiint(z);
  const uint32_t ord = hi ^ ((uint32_t)((int32_t)hi >> 31) | 0x80000000u);
  return (ord & ~(uint32_t)(NS - 1)) | (uint32_t)s;
}

// (key, found, part) of the better of this lane's and lane ^ o's candidate:
// larger key first, equal keys -> lower part first
__device__ __forceinline__ void combine(uint32_t& k, bool& f, int& q, int o) {
  const uint32_t ok = __shfl_xor_sync(0xffffffffu, k, o);
  const bool of = __shfl_xor_sync(0xffffffffu, (int)f, o) != 0;
  const int oq = __shfl_xor_sync(0xffffffffu, q, o);
  const bool take = of && (!f || ok > k || (ok == k && oq < q));
  k = take ? ok : k;
  f = f || of;
  q = take ? oq : q;
}

// FULL: E == 64, no per-expert bounds checks. KT > 0: the budget is KT
// (compile-time: the k + 1 selection passes unroll into straight-line code)
template <int TPS, bool FULL, int KT>
__global__ void __launch_bounds__(K3Cfg<TPS>::kThreads, 2) k_linear_predict(const LinArgs a) {
  using C = K3Cfg<TPS>;
  constexpr int NS = C::NS, NU = C::kUnits, HALF = NS / 2;
  if (a.gate && *a.gate <= a.gate_cap) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int L = a.L, E = a.E, F = a.L + a.E + 1;
  double2* colT = reinterpret_cast<double2*>(smem_raw);  // [E][TPS][NU]: W[j][L+e] pairs
  double2* bias2 = colT + E * TPS * NU;                  // [L][TPS][NU]: (1 - decay) b_l
  double2* zcol = bias2 + L * TPS * NU;                  // [TPS][NU] zeros (odd pair tail)
  for (int i = threadIdx.x; i < E * TPS * NU; i += blockDim.x) {
    const int e = i / (TPS * NU), j0 = NS * ((i / NU) % TPS) + 2 * (i % HALF);
    colT[i] = make_double2(j0 < E ? a.Wt[(int64_t)j0 * F + L + e] : 0.0,
                           j0 + 1 < E ? a.Wt[(int64_t)(j0 + 1) * F + L + e] : 0.0);
  }
  for (int i = threadIdx.x; i < L * TPS * NU; i += blockDim.x) {
    const int l = i / (TPS * NU), j0 = NS * ((i / NU) % TPS) + 2 * (i % HALF);
    double b[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int j = j0 + c;
      b[c] = j < E ? (1.0 - a.decay) * (a.Wt[(int64_t)j * F + l] + a.Wt[(int64_t)j * F + L + E])
                   : 0.0;
    }
    bias2[i] = make_double2(b[0], b[1]);
  }
  for (int i = threadIdx.x; i < TPS * NU; i += blockDim.x) zcol[i] = make_double2(0.0, 0.0);
  __syncthreads();

  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int q = lane % TPS;
  const int e0 = NS * q;
  const int rot = lane & 7;
  const unsigned grp = ((1u << TPS) - 1) << (lane & ~(TPS - 1));
  const double NEG = -__longlong_as_double(0x7ff0000000000000LL);
  const int k = KT > 0 ? KT : (a.budget < E ? a.budget : E);
  const int64_t n_streams = (int64_t)a.L * a.P;

  for (int64_t gbase = (int64_t)blockIdx.x * C::kStreams; gbase < n_streams;
       gbase += (int64_t)gridDim.x * C::kStreams) {
    const int64_t sidx = gbase + threadIdx.x / TPS;
    const bool live = sidx < n_streams;
    const int p = live ? (int)(sidx / L) : 0;
    const int l = live ? (int)(sidx % L) : 0;
    const int64_t r0 = live ? a.row_off[p] : 0;
    const int T = live ? (int)((a.row_off[p + 1] - r0) / L) : 0;
    int Tw = T;  // warp-uniform trip count so shuffles see every lane
#pragma unroll
    for (int o = 16; o; o >>= 1) Tw = max(Tw, __shfl_xor_sync(full, Tw, o));

    double z[NS];  // slot s: expert slot_expert(s, q, rot); invalid experts (E < 64) = -inf
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int ex = slot_expert<NS>(s, q, rot);
      z[s] = (FULL || ex < E) ? a.Wt[(int64_t)ex * F + l] + a.Wt[(int64_t)ex * F + L + E] : NEG;
    }
    const double2* bcol = bias2 + (l * TPS + q) * NU + rot;
    int acc_k = 0, acc_ph = 0;

    for (int t = 0; t < Tw; ++t) {
      const bool valid = t < T;
      const int64_t r = r0 + (int64_t)t * L + l;
      const uint64_t tw = valid ? __ldg(a.truth + r) : 0ull;
      uint64_t pm = 0;
      if (a.threshold) {
        uint32_t m = 0;  // slot mask -> expert mask of this part: rotate by 2 rot
#pragma unroll
        for (int s = 0; s < NS; ++s)
          if (z[s] > 0.0) m |= 1u << s;
        if (NS == 32) {
          m = __funnelshift_l(m, m, 2 * rot);
        } else {
          m = ((m << (2 * rot)) | (m >> (NS - 2 * rot))) & ((1u << NS) - 1);
        }
        pm = (uint64_t)m << e0;
#pragma unroll
        for (int o = 1; o < TPS; o <<= 1) pm |= __shfl_xor_sync(full, pm, o);
      } else {
        uint32_t key[NS];
#pragma unroll
        for (int s = 0; s < NS; ++s) key[s] = order_key<NS>(z[s], s);
        uint32_t kth = 0, bound = 0;
        bool amb = false;
#pragma unroll
        for (int it = 0; it <= (KT > 0 ? KT : k); ++it) {
          uint32_t bk;
          bool found;
          // four independent partial reductions: a dependency chain of NS/4 + 2
          // instead of NS (the passes are latency-bound)
          if (it == 0) {
            uint32_t b4[4] = {key[0], key[1], key[2], key[3]};
#pragma unroll
            for (int s = 4; s < NS; ++s) b4[s & 3] = max(b4[s & 3], key[s]);
            bk = max(max(b4[0], b4[1]), max(b4[2], b4[3]));
            found = true;
          } else {  // largest key below this lane's bound
            const uint32_t bm1 = bound - 1u;
            uint32_t t4[4] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu};
#pragma unroll
            for (int s = 0; s < NS; ++s) t4[s & 3] = min(t4[s & 3], bm1 - key[s]);
            const uint32_t tm = min(min(t4[0], t4[1]), min(t4[2], t4[3]));
            found = bound != 0u && tm < bound;
            bk = bm1 - tm;
          }
          uint32_t wk = bk;
          bool wf = found;
          int wq = q;
          if (TPS == 2) {
            // one shuffle: real keys are >= 0x000fffe0 (order_key of -inf),
            // so 0 encodes "none found", and the partner's part is q ^ 1
            const uint32_t kk = found ? bk : 0u;
            const uint32_t ok = __shfl_xor_sync(0xffffffffu, kk, 1);
            const bool take = ok > kk || (ok == kk && q == 1);
            wk = take ? ok : kk;
            wq = take ? (q ^ 1) : q;
            wf = wk != 0u;
          } else {
#pragma unroll
            for (int o = 1; o < TPS; o <<= 1) combine(wk, wf, wq, o);
          }
          if (it < k) {
            const int wrot = ((lane & ~(TPS - 1)) | wq) & 7;
            pm |= 1ull << slot_expert<NS>((int)(wk & (NS - 1)), wq, wrot);
            kth = wk;
            bound = wk + (q > wq ? 1u : 0u);
          } else if (wf) {
            amb = (kth & ~(uint32_t)(NS - 1)) - (wk & ~(uint32_t)(NS - 1)) <= (uint32_t)NS;
          }
        }
        if (amb) {  // exact fp64 passes (rare): ties to the lower expert id
          pm = 0;
          for (int it = 0; it < k; ++it) {
            const int orot = opaque(rot);
            double best = NEG;
            int bi = 64;
#pragma unroll
            for (int s = 0; s < NS; ++s) {
              const int ex = slot_expert<NS>(s, q, orot);
              const bool ok = (FULL || ex < E) && !((pm >> ex) & 1ull) &&
                              (z[s] > best || (z[s] == best && ex < bi));
              best = ok ? z[s] : best;
              bi = ok ? ex : bi;
            }
#pragma unroll
            for (int o = 1; o < TPS; o <<= 1) {
              const double ob = __shfl_xor_sync(grp, best, o);
              const int oi = __shfl_xor_sync(grp, bi, o);
              const bool take = oi < 64 && (bi == 64 || ob > best || (ob == best && oi < bi));
              best = take ? ob : best;
              bi = take ? oi : bi;
            }
            pm |= 1ull << bi;
          }
        }
      }
      if (valid) {
        if (q == 0) {
          a.pred[r] = pm;
          if (t >= a.warmup) {  // the replay's access / prediction-hit counters
            acc_k += __popcll(tw);
            acc_ph += __popcll(tw & pm);
          }
        }
        if (a.logits) {
          const int orot = opaque(rot);
#pragma unroll
          for (int s = 0; s < NS; ++s) {
            const int ex = slot_expert<NS>(s, q, orot);
            if (FULL || ex < E) a.logits[r * E + ex] = z[s];
          }
        }
        // update_history (learner.py:62-72), as a logit recurrence
#pragma unroll
        for (int j = 0; j < HALF; ++j) {
          const double2 v = bcol[j];
          z[2 * j] = fma(a.decay, z[2 * j], v.x);
          z[2 * j + 1] = fma(a.decay, z[2 * j + 1], v.y);
        }
        // two fired experts per trip (ascending, so the additions round
        // exactly as one at a time); an odd last one pairs with a zero column
        uint64_t mm = tw;
        while (mm) {
          const int ex0 = __ffsll((long long)mm) - 1;
          mm &= mm - 1;
          const double2* c0 = colT + (ex0 * TPS + q) * NU + rot;
          const double2* c1 = zcol + q * NU + rot;
          if (mm) {
            const int ex1 = __ffsll((long long)mm) - 1;
            mm &= mm - 1;
            c1 = colT + (ex1 * TPS + q) * NU + rot;
          }
#pragma unroll
          for (int j = 0; j < HALF; ++j) {
            const double2 v0 = c0[j], v1 = c1[j];
            z[2 * j] = (z[2 * j] + v0.x) + v1.x;
            z[2 * j + 1] = (z[2 * j + 1] + v0.y) + v1.y;
          }
        }
      }
    }
    if (a.counts && q == 0 && live && (acc_k | acc_ph)) {
      atomicAdd(reinterpret_cast<unsigned long long*>(a.counts + 0), (unsigned long long)acc_k);
      atomicAdd(reinterpret_cast<unsigned long long*>(a.counts + 1), (unsigned long long)acc_ph);
      atomicAdd(reinterpret_cast<unsigned long long*>(a.counts + 2 + l), (unsigned long long)acc_k);
      atomicAdd(reinterpret_cast<unsigned long long*>(a.counts + 2 + L + l),
                (unsigned long long)acc_ph);
    }
  }
}

template <int TPS>
int launch_k3(const LinArgs& a, cudaStream_t s) {
  using C = K3Cfg<TPS>;
  const size_t smem = sizeof(double2) * (size_t)(a.E + a.L + 1) * TPS * C::kUnits;
  if ((int)smem > moeb::max_smem_per_block())
    return moeb::fail(MOEB_ESMEM, "learned_linear tables need %zu B of shared memory", smem);
  const int kb = a.budget < a.E ? a.budget : a.E;
  auto kern = a.E == 64 ? (kb == 6 ? k_linear_predict<TPS, true, 6>
                                   : kb == 8 ? k_linear_predict<TPS, true, 8>
                                             : k_linear_predict<TPS, true, 0>)
                        : k_linear_predict<TPS, false, 0>;
  moeb::set_smem(kern, (int)smem);
  // persistent: at most 2 CTAs per SM, each looping over groups of kStreams streams
  const int64_t groups = ((int64_t)a.L * a.P + C::kStreams - 1) / C::kStreams;
  const int64_t blocks = groups < 2LL * moeb::num_sms() ? groups : 2LL * moeb::num_sms();
  kern<<<(unsigned)blocks, C::kThreads, smem, s>>>(a);
  return moeb::check_launch("k_linear_predict");
}

// ---------------------------------------------------------------------------
// Wide K3 (64 < E <= 256, e.g. DeepSeek-V3's 256 experts): the 64-expert
// kernel's column tables would not fit shared memory, so the tables
// (moeb_linear_prepare: W_h transposed, per-layer start scores and biases)
// stay in L2 and one WARP owns one (prompt, layer) stream: lane i holds the
// scores of experts i + 32 s, column reads are 256-byte coalesced rows of the
// transposed W_h. Same fp64 recurrence; exact fp64 top-k passes (warp
// argmax, ties to the lower id) or the threshold rule.
// ---------------------------------------------------------------------------
template <int NSW>
__global__ void __launch_bounds__(256) k_linear_predict_wide(
    const uint64_t* __restrict__ truth, const int64_t* __restrict__ row_off, int P, int L, int E,
    const double* __restrict__ tab, double decay, int budget, int threshold,
    uint64_t* __restrict__ pred, double* __restrict__ logits) {
  constexpr int W = (NSW * 32 + 63) / 64;
  const int lane = threadIdx.x & 31;
  const int64_t stream = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (stream >= (int64_t)P * L) return;
  const int p = (int)(stream / L), l = (int)(stream % L);
  const double* colT = tab;                            // [E][E]
  const double* z0 = tab + (int64_t)E * E;             // [L][E]
  const double* bias = z0 + (int64_t)L * E;            // [L][E]
  const double NEG = -__longlong_as_double(0x7ff0000000000000LL);
  double z[NSW], b[NSW];
#pragma unroll
  for (int s = 0; s < NSW; ++s) {
    const int ex = lane + 32 * s;
    z[s] = ex < E ? z0[(int64_t)l * E + ex] : NEG;
    b[s] = ex < E ? bias[(int64_t)l * E + ex] : 0.0;
  }
  const int64_t r0 = row_off[p];
  const int T = (int)((row_off[p + 1] - r0) / L);
  const int k = budget < E ? budget : E;
  for (int t = 0; t < T; ++t) {
    const int64_t r = r0 + (int64_t)t * L + l;
    uint64_t pm[W];
#pragma unroll
    for (int w = 0; w < W; ++w) pm[w] = 0;
    if (threshold) {
#pragma unroll
      for (int s = 0; s < NSW; ++s) {
        const uint64_t bits = __ballot_sync(0xffffffffu, z[s] > 0.0);
        pm[s >> 1] |= bits << (32 * (s & 1));
      }
    } else {
      bool taken[NSW];
#pragma unroll
      for (int s = 0; s < NSW; ++s) taken[s] = false;
      for (int it = 0; it < k; ++it) {
        double best = NEG;
        int bi = 1 << 20;
#pragma unroll
        for (int s = 0; s < NSW; ++s) {
          const int ex = lane + 32 * s;
          const bool ok = ex < E && !taken[s] && (z[s] > best || (z[s] == best && ex < bi));
          best = ok ? z[s] : best;
          bi = ok ? ex : bi;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          const bool take = ob > best || (ob == best && oi < bi);
          best = take ? ob : best;
          bi = take ? oi : bi;
        }
        if ((bi & 31) == lane) {
#pragma unroll
          for (int s = 0; s < NSW; ++s)
            if (bi >> 5 == s) taken[s] = true;
        }
#pragma unroll
        for (int w = 0; w < W; ++w)
          if ((bi >> 6) == w) pm[w] |= 1ull << (bi & 63);
      }
    }
    if (lane < W) {
      uint64_t v = 0;
#pragma unroll
      for (int w = 0; w < W; ++w)
        if (w == lane) v = pm[w];
      pred[r * W + lane] = v;
    }
    if (logits) {
#pragma unroll
      for (int s = 0; s < NSW; ++s)
        if (lane + 32 * s < E) logits[r * E + lane + 32 * s] = z[s];
    }
    // z <- decay z + (1 - decay) b_l + sum of the truth experts' W_h columns
#pragma unroll
    for (int s = 0; s < NSW; ++s) z[s] = fma(decay, z[s], b[s]);
#pragma unroll
    for (int w = 0; w < W; ++w) {
      uint64_t mm = __ldg(truth + r * W + w);
      while (mm) {
        const int ex = w * 64 + __ffsll((long long)mm) - 1;
        mm &= mm - 1;
        const double* col = colT + (int64_t)ex * E;
#pragma unroll
        for (int s = 0; s < NSW; ++s)
          if (lane + 32 * s < E) z[s] += __ldg(col + lane + 32 * s);
      }
    }
  }
}

__global__ void k_linear_prepare(const double* __restrict__ Wt, int L, int E, double decay,
                                 double* tab) {
  const int F = L + E + 1;
  const int64_t n1 = (int64_t)E * E, n2 = (int64_t)L * E;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n1 + 2 * n2;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < n1) {
      const int e = (int)(i / E), j = (int)(i % E);
      tab[i] = Wt[(int64_t)j * F + L + e];
    } else {
      const int64_t q = (i - n1) % n2;
      const int l = (int)(q / E), j = (int)(q % E);
      const double zz = Wt[(int64_t)j * F + l] + Wt[(int64_t)j * F + L + E];
      tab[i] = i < n1 + n2 ? zz : (1.0 - decay) * zz;
    }
  }
}

}  // namespace

namespace moeb {
size_t linear_tc_workspace_bytes(int64_t rows, int L);
size_t linear_tc_min_workspace(int L);
bool linear_tc_eligible(int L, int E, int budget, const double* logits);
int linear_tc_launch(const uint64_t* truth, const int64_t* row_off, int P, int64_t rows, int L,
                     const double* W, double decay, int budget, int threshold, int warmup,
                     int kmax, uint64_t* pred, int64_t* counts, void* workspace,
                     size_t ws_bytes, cudaStream_t s);

int launch_linear_fp64_gated(const uint64_t* truth, const int64_t* row_off, int P, int L, int E,
                             const double* W, double decay, int budget, int threshold, int warmup,
                             uint64_t* pred, int64_t* counts, const int* gate, int gate_cap,
                             cudaStream_t s) {
  LinArgs a{truth, row_off, P, L, E, W, decay, budget, threshold ? 1 : 0, warmup, pred, nullptr,
            counts, gate, gate_cap};
  return launch_k3<2>(a, s);
}
}  // namespace moeb

namespace moeb {
int linear_tc_ambiguous(const void* workspace, int L, int64_t* out, cudaStream_t s);
}

extern "C" int moeb_linear_ambiguous_rows(const void* workspace, int L, int64_t* out,
                                          void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(workspace && out && L >= 1 && L <= 32, "bad argument");
  return moeb::linear_tc_ambiguous(workspace, L, out, moeb::as_stream(stream));
}

extern "C" size_t moeb_linear_workspace_bytes(int64_t rows, int L, int E) {
  if (E != 64 || L < 1 || L > 32) return 0;
  return moeb::linear_tc_workspace_bytes(rows, L);
}

extern "C" int moeb_linear_predict(const uint64_t* truth, const int64_t* prompt_row_off,
                                   int n_prompts, int L, int E, const double* weights,
                                   double decay, int budget, int threshold, int warmup_tokens,
                                   uint64_t* pred, double* logits, int64_t* metrics,
                                   void* stream) {
  return moeb_linear_predict_counts(truth, prompt_row_off, n_prompts, L, E, weights, decay,
                                    budget, threshold, warmup_tokens, 0, pred, logits, metrics,
                                    nullptr, 0, nullptr, 0, stream);
}

extern "C" int moeb_linear_predict_counts(const uint64_t* truth, const int64_t* prompt_row_off,
                                          int n_prompts, int L, int E, const double* weights,
                                          double decay, int budget, int threshold,
                                          int warmup_tokens, int top_k, uint64_t* pred,
                                          double* logits, int64_t* metrics, int64_t* counts,
                                          int64_t rows, void* workspace, size_t workspace_bytes,
                                          void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(truth && prompt_row_off && weights && pred, "null argument");
  MOEB_REQUIRE(n_prompts >= 1 && L >= 1 && E >= 1 && E <= 64,
               "moeb_linear_predict supports E <= 64 (got L=%d E=%d); use "
               "moeb_linear_prepare + moeb_linear_predict_wide", L, E);
  MOEB_REQUIRE(budget >= 1 && warmup_tokens >= 0, "bad budget/warmup");
  MOEB_REQUIRE(decay >= 0.0 && decay < 1.0, "decay must be in [0, 1)");
  cudaStream_t s = moeb::as_stream(stream);
  int rc;
  if (workspace && moeb::linear_tc_eligible(L, E, budget, logits) &&
      workspace_bytes >= moeb::linear_tc_min_workspace(L)) {
    // K3t: tensor-core column sums, fp32 scores + exact fp64 re-evaluation
    // of the rows the fp32 bound cannot decide
    rc = moeb::linear_tc_launch(truth, prompt_row_off, n_prompts, rows, L, weights, decay, budget,
                                threshold ? 1 : 0, warmup_tokens, top_k, pred, counts, workspace,
                                workspace_bytes, s);
  } else {
    LinArgs a{truth, prompt_row_off, n_prompts, L, E, weights, decay, budget,
              threshold ? 1 : 0, warmup_tokens, pred, logits, counts, nullptr, 0};
    const char* env = getenv("MOEB_K3_TPS");  // tuning knob: threads per stream (2 or 4)
    rc = (env && atoi(env) == 4) ? launch_k3<4>(a, s) : launch_k3<2>(a, s);
  }
  if (rc != 0 || metrics == nullptr) return rc;
  // K7 over the fresh masks (same stream): prediction metrics (metrics.py:12-79)
  return moeb_metrics(pred, truth, prompt_row_off, n_prompts, L, E, warmup_tokens, metrics,
                      stream);
}

extern "C" size_t moeb_linear_table_doubles(int L, int E) {
  return (size_t)E * E + 2 * (size_t)L * E;
}

extern "C" int moeb_linear_prepare(const double* weights, int L, int E, double decay,
                                   double* tables, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(weights && tables && L >= 1 && E >= 1 && E <= 256, "bad arguments");
  k_linear_prepare<<<256, 256, 0, moeb::as_stream(stream)>>>(weights, L, E, decay, tables);
  return moeb::check_launch("k_linear_prepare");
}

extern "C" int moeb_linear_predict_wide(const uint64_t* truth, const int64_t* prompt_row_off,
                                        int n_prompts, int L, int E, const double* tables,
                                        double decay, int budget, int threshold,
                                        int warmup_tokens, uint64_t* pred, double* logits,
                                        int64_t* metrics, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(truth && prompt_row_off && tables && pred, "null argument");
  MOEB_REQUIRE(n_prompts >= 1 && L >= 1 && E >= 1 && E <= 256, "bad shape L=%d E=%d", L, E);
  MOEB_REQUIRE(budget >= 1 && warmup_tokens >= 0, "bad budget/warmup");
  MOEB_REQUIRE(decay >= 0.0 && decay < 1.0, "decay must be in [0, 1)");
  cudaStream_t s = moeb::as_stream(stream);
  const int64_t threads = (int64_t)n_prompts * L * 32;
  const unsigned blocks = (unsigned)((threads + 255) / 256);
  const int nsw = (E + 31) / 32;
#define MOEB_K3W(N)                                                                        \
  case N:                                                                                  \
    k_linear_predict_wide<N><<<blocks, 256, 0, s>>>(truth, prompt_row_off, n_prompts, L, E, \
                                                    tables, decay, budget, threshold, pred, \
                                                    logits);                                \
    break;
  switch (nsw) {
    MOEB_K3W(1) MOEB_K3W(2) MOEB_K3W(3) MOEB_K3W(4) MOEB_K3W(5) MOEB_K3W(6) MOEB_K3W(7)
    default:
      k_linear_predict_wide<8><<<blocks, 256, 0, s>>>(truth, prompt_row_off, n_prompts, L, E,
                                                      tables, decay, budget, threshold, pred,
                                                      logits);
  }
#undef MOEB_K3W
  int rc = moeb::check_launch("k_linear_predict_wide");
  if (rc != 0 || metrics == nullptr) return rc;
  return moeb_metrics(pred, truth, prompt_row_off, n_prompts, L, E, warmup_tokens, metrics,
                      stream);
}
