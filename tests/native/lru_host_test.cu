// Host-side unit test of the sequential cache state machines in
// paper_2508_17137_b200/csrc/cache_sim.cu (compiled __host__ __device__),
// checked against the C oracle (oracle/moeb_oracle.c). Runs without a GPU:
//   make -C tests/native && tests/native/lru_host_test
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "../../paper_2508_17137_b200/csrc/cache_sim.cu"

extern "C" int orc_cache_ops(const int32_t*, const int32_t*, int64_t, int, int, int64_t, int,
                             uint8_t*);
extern "C" int orc_cache_sim(const uint64_t*, const uint64_t*, const uint8_t*, const int64_t*, int,
                             int, int, int, int64_t, int, int, int, int64_t*, int64_t*,
                             uint64_t*);

template <int W, class State>
static void host_ops(SimArgs a, const std::vector<int>& ops, const std::vector<int>& keys,
                     std::vector<uint8_t>& res) {
  std::vector<unsigned char> mem(a.sim_bytes + 64, 0xAB);
  State st;
  st.init(mem.data(), a, a.L);
  for (size_t i = 0; i < ops.size(); ++i) {
    uint8_t r = 0;
    if (ops[i] == 0) {
      st.begin_step(st.cur);
    } else {
      st.focus(keys[i] / a.E);
      const int ex = keys[i] % a.E;
      r = ops[i] == 1 ? (uint8_t)st.touch(ex) : (uint8_t)st.prefetch(ex);
    }
    res[i] = r;
  }
}

// sequential trace replay with the trace-mode state machine (what the warp
// kernel's fallback runs per row)
template <int W, class State>
static void host_trace(SimArgs a, const std::vector<uint64_t>& truth,
                       const std::vector<uint64_t>& pred, const std::vector<int64_t>& off,
                       int limit, std::vector<int64_t>& cnt, std::vector<uint64_t>& hits) {
  const int L = a.L;
  for (int p = 0; p + 1 < (int)off.size(); ++p) {
    std::vector<unsigned char> mem(a.sim_bytes + 64, 0xCD);
    State st;
    st.init(mem.data(), a, L);
    int l = 0, t = 0;
    for (int64_t r = off[p]; r < off[p + 1]; ++r) {
      uint64_t tw[W], pw[W];
      for (int w = 0; w < W; ++w) {
        tw[w] = truth[r * W + w];
        pw[w] = pred[r * W + w];
      }
      uint64_t hw[W] = {};
      if (t < a.warmup) {
        st.focus(l);
        for (int w = 0; w < W; ++w)
          for (uint64_t m = tw[w]; m; m &= m - 1) {
            const int ex = w * 64 + moeb_ffs64(m) - 1;
            if (st.touch(ex)) hw[w] |= 1ull << (ex & 63);
          }
      } else {
        st.begin_step(l);
        int taken = 0;
        for (int w = 0; w < W; ++w)
          for (uint64_t m = pw[w]; m && taken < limit; m &= m - 1, ++taken)
            st.prefetch(w * 64 + moeb_ffs64(m) - 1);
        int k = 0, ch = 0, ph = 0;
        for (int w = 0; w < W; ++w) {
          k += moeb_popc64(tw[w]);
          ph += moeb_popc64(tw[w] & pw[w]);
          for (uint64_t m = tw[w]; m; m &= m - 1) {
            const int ex = w * 64 + moeb_ffs64(m) - 1;
            if (st.touch(ex)) {
              ++ch;
              hw[w] |= 1ull << (ex & 63);
            }
          }
        }
        cnt[0] += k;
        cnt[1] += ch;
        cnt[2] += ph;
        cnt[4 + l] += k;
        cnt[4 + L + l] += ch;
        cnt[4 + 2 * L + l] += ph;
      }
      for (int w = 0; w < W; ++w) hits[r * W + w] = hw[w];
      if (++l == L) {
        l = 0;
        ++t;
      }
    }
  }
}

static int failures = 0;

template <int W>
static void run_case(int L, int E, int k, int P, int T, int warmup, int cap, int budget,
                     int npred, bool unbounded, int policy, unsigned seed) {
  std::mt19937_64 rng(seed);
  const int64_t rows = (int64_t)P * T * L;
  std::vector<uint64_t> truth(rows * W, 0), pred(rows * W, 0);
  std::vector<int64_t> off(P + 1);
  for (int p = 0; p <= P; ++p) off[p] = (int64_t)p * T * L;
  for (int64_t r = 0; r < rows; ++r) {
    const int l = (int)(r % L);
    for (int j = 0; j < k;) {  // skewed: half the draws from a small hot set
      const int e = (rng() % 2) ? (int)((l * 7 + rng() % (k + 2)) % E) : (int)(rng() % E);
      uint64_t& wd = truth[r * W + e / 64];
      if (!(wd >> (e % 64) & 1)) {
        wd |= 1ull << (e % 64);
        ++j;
      }
    }
    for (int j = 0; j < npred; ++j) {
      const int e = (rng() % 2) ? (int)((l * 7 + rng() % (k + 2)) % E) : (int)(rng() % E);
      pred[r * W + e / 64] |= 1ull << (e % 64);
    }
  }
  SimArgs a{};
  a.L = L;
  a.E = E;
  a.cap = cap;
  a.warmup = warmup;
  a.budget = budget;
  layout(a, policy, false);
  std::vector<int64_t> got(4 + 3 * L, 0), want(4 + 3 * L, 0), pp(P * 4);
  std::vector<uint64_t> hg(rows * W), hw(rows * W);
  const int limit = unbounded ? E : budget;
  if (policy == MOEB_POLICY_LRU)
    host_trace<W, LruState<W, -1, false>>(a, truth, pred, off, limit, got, hg);
  else
    host_trace<W, LfuState<W, false>>(a, truth, pred, off, limit, got, hg);
  orc_cache_sim(truth.data(), pred.data(), nullptr, off.data(), P, L, E, warmup, cap, budget,
                unbounded, policy, want.data(), pp.data(), hw.data());
  bool ok = got == want && hg == hw;
  if (!ok) {
    ++failures;
    printf("FAIL trace L=%d E=%d cap=%d budget=%d npred=%d unb=%d pol=%d: hits %lld vs %lld\n", L,
           E, cap, budget, npred, (int)unbounded, policy, (long long)got[1], (long long)want[1]);
  }
  // op stream
  std::vector<int> ops, keys;
  for (int i = 0; i < 4000; ++i) {
    const int o = (int)(rng() % 4);
    ops.push_back(o == 3 ? 1 : o);
    keys.push_back((int)(rng() % (L * E)));
  }
  SimArgs b{};
  b.L = L;
  b.E = E;
  b.cap = cap;
  layout(b, policy, true);
  std::vector<uint8_t> rg(ops.size()), rw(ops.size());
  if (policy == MOEB_POLICY_LRU)
    host_ops<W, LruState<W, -1, true>>(b, ops, keys, rg);
  else
    host_ops<W, LfuState<W, true>>(b, ops, keys, rg);
  orc_cache_ops(ops.data(), keys.data(), (int64_t)ops.size(), L, E, cap, policy, rw.data());
  if (rg != rw) {
    ++failures;
    printf("FAIL ops L=%d E=%d cap=%d pol=%d\n", L, E, cap, policy);
  }
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  for (int policy = 0; policy < 2; ++policy)
    for (int cap : {1, 2, 3, 5, 8, 17, 40, 100, 300})
      for (int budget : {1, 2, 6})
        for (int npred : {0, 2, 6, 9}) {
          run_case<1>(3, 8, 2, 3, 40, 2, cap > 24 ? 24 : cap, budget, npred > 8 ? 8 : npred,
                      false, policy, cap * 131 + budget * 7 + npred);
          run_case<1>(5, 64, 6, 2, 60, 4, cap, budget, npred, npred == 9, policy,
                      cap * 17 + budget + npred * 3);
          run_case<2>(3, 100, 4, 2, 30, 2, cap, budget, npred, false, policy, cap + budget + npred);
        }
  printf("%s (%d failures)\n", failures ? "FAILED" : "ok", failures);
  return failures ? 1 : 0;
}
