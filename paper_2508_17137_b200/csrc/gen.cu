// Synthetic decode traces on device, bit-identical to the reference generator
// traceio._generate_prompt (traceio.py:233-283).
//
// numpy's default_rng is PCG64 (128-bit LCG, XSL-RR output; each draw steps
// the state, then outputs). random() = (next64 >> 11) * 2^-53. The reference
// draws, per prompt, in this order (traceio.py:249-253):
//   hot_keys (L*E) | token_ids (T, buffered 32-bit Lemire) | from_hot (T*L)
//   | hot_pick (T*L*h) | uni_pick (T*L*E)
// The host replays the first two blocks with numpy itself (they are small and
// the hot set's ORDER comes from np.argpartition, traceio.py:255) and hands
// over the PCG64 state after them. The device then jumps straight to each
// token's slice of the three large blocks (LCG jump-ahead: S_{n} = A^n S +
// inc * (A^n - 1)/(A - 1)) and reproduces the subsets: top-k of the h hot
// keys (mapped through the ordered hot set) or top-k of the E uniform keys.
// Draws are compared as the 53-bit integers behind the doubles, which orders
// them exactly like the doubles np.argpartition compares.
#include <vector>

#include "common.cuh"

namespace {

struct u128 {
  uint64_t lo, hi;
};

__host__ __device__ inline u128 mul128(u128 a, u128 b) {
  u128 r;
  r.lo = a.lo * b.lo;
#ifdef __CUDA_ARCH__
  r.hi = __umul64hi(a.lo, b.lo) + a.hi * b.lo + a.lo * b.hi;
#else
  r.hi = (uint64_t)(((unsigned __int128)a.lo * b.lo) >> 64) + a.hi * b.lo + a.lo * b.hi;
#endif
  return r;
}
__host__ __device__ inline u128 add128(u128 a, u128 b) {
  u128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1 : 0);
  return r;
}

// PCG_DEFAULT_MULTIPLIER_128
constexpr uint64_t kMulHi = 0x2360ED051FC65DA4ULL, kMulLo = 0x4385DF649FCCF645ULL;

__constant__ u128 c_jumpA[64];  // A^(2^i)
__constant__ u128 c_jumpG[64];  // (A^(2^i) - 1) / (A - 1)

struct Pcg {
  u128 s, inc;
  __device__ __forceinline__ uint64_t next() {
    s = add128(mul128(s, u128{kMulLo, kMulHi}), inc);
    const uint64_t x = s.hi ^ s.lo;
    const unsigned rot = (unsigned)(s.hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  __device__ __forceinline__ void jump(uint64_t n) {
    for (int i = 0; n; ++i, n >>= 1)
      if (n & 1) s = add128(mul128(c_jumpA[i], s), mul128(inc, c_jumpG[i]));
  }
  __device__ __forceinline__ void jump_by(u128 A, u128 G) { s = add128(mul128(A, s), mul128(inc, G)); }
};

constexpr int KMAX = 16;

// Positions (in draw order) of the k largest of n consecutive draws.
__device__ __forceinline__ void topk_positions(Pcg& g, int n, int k, int (&pos)[KMAX]) {
  uint64_t val[KMAX];
#pragma unroll
  for (int q = 0; q < KMAX; ++q) {
    val[q] = 0;
    pos[q] = -1;
  }
  int filled = 0, mi = 0;
  uint64_t minv = 0;
  for (int j = 0; j < n; ++j) {
    const uint64_t v = (g.next() >> 11) + 1;  // +1 keeps 0 as "empty"
    if (filled < k) {
#pragma unroll
      for (int q = 0; q < KMAX; ++q)
        if (q == filled) {
          val[q] = v;
          pos[q] = j;
        }
      ++filled;
      if (filled == k) {
        minv = ~0ull;
#pragma unroll
        for (int q = 0; q < KMAX; ++q)
          if (q < k && val[q] < minv) {
            minv = val[q];
            mi = q;
          }
      }
    } else if (v > minv) {
#pragma unroll
      for (int q = 0; q < KMAX; ++q)
        if (q == mi) {
          val[q] = v;
          pos[q] = j;
        }
      minv = ~0ull;
#pragma unroll
      for (int q = 0; q < KMAX; ++q)
        if (q < k && val[q] < minv) {
          minv = val[q];
          mi = q;
        }
    }
  }
}

template <int W>
__global__ void __launch_bounds__(128) k_gen_traces(const uint64_t* __restrict__ st,
                                                    const uint8_t* __restrict__ hot, int P, int T,
                                                    int L, int E, int k, int h, double skew,
                                                    u128 Ah, u128 Gh, u128 Ae, u128 Ge,
                                                    uint64_t* __restrict__ truth) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (int64_t)P * T) return;
  const int p = (int)(gid / T), t = (int)(gid % T);
  Pcg base;
  base.s = u128{st[4 * (int64_t)p + 1], st[4 * (int64_t)p + 0]};
  base.inc = u128{st[4 * (int64_t)p + 3], st[4 * (int64_t)p + 2]};
  const uint64_t TL = (uint64_t)T * L;
  Pcg gf = base, gh = base, gu = base;
  gf.jump((uint64_t)t * L);                         // from_hot[t, 0]
  gh.jump(TL + (uint64_t)t * L * h);                // hot_pick[t, 0, 0]
  gu.jump(TL + TL * h + (uint64_t)t * L * E);       // uni_pick[t, 0, 0]
  const uint8_t* hp = hot + (int64_t)p * L * h;
  uint64_t* out = truth + ((int64_t)p * T + t) * L * W;
  for (int l = 0; l < L; ++l) {
    const double x = (double)(gf.next() >> 11) * (1.0 / 9007199254740992.0);
    uint64_t m[W];
#pragma unroll
    for (int w = 0; w < W; ++w) m[w] = 0;
    int pos[KMAX];
    if (x < skew) {
      topk_positions(gh, h, k, pos);
      gu.jump_by(Ae, Ge);
#pragma unroll
      for (int q = 0; q < KMAX; ++q)
        if (q < k) {
          const int e = hp[l * h + pos[q]];
#pragma unroll
          for (int w = 0; w < W; ++w)
            if ((e >> 6) == w) m[w] |= 1ull << (e & 63);
        }
    } else {
      gh.jump_by(Ah, Gh);
      topk_positions(gu, E, k, pos);
#pragma unroll
      for (int q = 0; q < KMAX; ++q)
        if (q < k) {
          const int e = pos[q];
#pragma unroll
          for (int w = 0; w < W; ++w)
            if ((e >> 6) == w) m[w] |= 1ull << (e & 63);
        }
    }
#pragma unroll
    for (int w = 0; w < W; ++w) out[l * W + w] = m[w];
  }
}

void host_jump(uint64_t n, u128& A, u128& G) {
  // (A, G) for n steps: S_n = A S + inc G.
  u128 a{kMulLo, kMulHi}, g{1, 0};  // one step
  A = u128{1, 0};
  G = u128{0, 0};
  while (n) {
    if (n & 1) {  // compose (A,G) then (a,g): A' = a A, G' = a G + g
      G = add128(mul128(a, G), g);
      A = mul128(a, A);
    }
    g = mul128(g, add128(a, u128{1, 0}));  // doubling: g2 = g (a + 1)
    a = mul128(a, a);
    n >>= 1;
  }
}

bool g_tables_ready = false;
int upload_tables() {
  if (g_tables_ready) return MOEB_OK;
  u128 A[64], G[64];
  for (int i = 0; i < 64; ++i) host_jump(1ull << i, A[i], G[i]);
  if (cudaMemcpyToSymbol(c_jumpA, A, sizeof(A)) != cudaSuccess ||
      cudaMemcpyToSymbol(c_jumpG, G, sizeof(G)) != cudaSuccess)
    return moeb::fail(MOEB_ECUDA, "uploading PCG64 jump tables");
  g_tables_ready = true;
  return MOEB_OK;
}

}  // namespace

extern "C" int moeb_gen_traces(const uint64_t* pcg_state, const uint8_t* hot, int n_prompts,
                               int T, int L, int E, int k, int h, double skew, uint64_t* truth,
                               void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(pcg_state && hot && truth, "null argument");
  MOEB_REQUIRE(n_prompts >= 1 && T >= 1 && L >= 1 && E >= 1 && E <= 256, "bad shape");
  MOEB_REQUIRE(k >= 1 && k <= KMAX && k <= h && h <= E, "need 1 <= k <= min(h, %d), h <= E",
               KMAX);
  if (int rc = upload_tables()) return rc;
  u128 Ah, Gh, Ae, Ge;
  host_jump((uint64_t)h, Ah, Gh);
  host_jump((uint64_t)E, Ae, Ge);
  const int64_t n = (int64_t)n_prompts * T;
  const int threads = 128;
  const unsigned blocks = (unsigned)((n + threads - 1) / threads);
  cudaStream_t s = moeb::as_stream(stream);
  switch (moeb::words_for(E)) {
    case 1: k_gen_traces<1><<<blocks, threads, 0, s>>>(pcg_state, hot, n_prompts, T, L, E, k, h, skew, Ah, Gh, Ae, Ge, truth); break;
    case 2: k_gen_traces<2><<<blocks, threads, 0, s>>>(pcg_state, hot, n_prompts, T, L, E, k, h, skew, Ah, Gh, Ae, Ge, truth); break;
    case 3: k_gen_traces<3><<<blocks, threads, 0, s>>>(pcg_state, hot, n_prompts, T, L, E, k, h, skew, Ah, Gh, Ae, Ge, truth); break;
    default: k_gen_traces<4><<<blocks, threads, 0, s>>>(pcg_state, hot, n_prompts, T, L, E, k, h, skew, Ah, Gh, Ae, Ge, truth); break;
  }
  return moeb::check_launch("k_gen_traces");
}
