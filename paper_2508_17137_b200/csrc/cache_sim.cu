// K1 -- prediction-guided expert-cache replay on device.
//
// Replaces engine.replay_prompt / replay_traces (engine.py:113-238) and the
// ExpertCache protocol (cache.py:58-154). One CUDA thread owns one
// simulation = (prediction stream, capacity, prompt); its whole cache state
// lives in a private slice of shared memory, and the thread walks the
// prompt's rows in (token, layer) order exactly as the reference loop does.
// Every step touches only keys of ONE layer, so that layer's resident and
// pinned bitmasks stay in registers for the step (written back on layer
// change), and set-membership / prediction-hit tests are register bit ops
// (popc(truth & pred) for prediction hits).
//
// LRU state (bit-exact with the reference OrderedDict, cache.py:68-124):
//   stamp[key]  u16 recency stamp of each resident key (0 = not resident)
//   q[]         ring deque of (stamp << 16 | layer << 8 | expert) entries in
//               push order. A "move to end" pushes a fresh entry and leaves a
//               stale one behind (lazy deletion): entry valid iff
//               stamp[key] == entry stamp. The LRU key is the first valid
//               entry from the head; eviction skips pinned ones in place
//               (`_evict_one`, cache.py:93-100). When the ring is full or the
//               16-bit clock is exhausted, the ring is compacted in order and
//               stamps renumbered 1..n (order preserved).
// LFU state (builder-defined; parity unpinned): slot array
//   vals[slot] = pin << 63 | freq << 32 | clock, evict = argmin over slots.
#include <algorithm>

#include "common.cuh"

namespace {

constexpr uint64_t kPin = 1ull << 63;

// The sequential state machines are __host__ __device__ so that
// tests/native/lru_host_test.cu can run them on the CPU against the oracle.
#define MOEB_HD __host__ __device__
#ifdef __CUDA_ARCH__
#define MOEB_ANY(x) __any_sync(__activemask(), (x))
#define MOEB_GROUP_SYNC() __syncwarp(__activemask())
__device__ __forceinline__ int moeb_ffs64(uint64_t x) { return __ffsll((long long)x); }
__device__ __forceinline__ int moeb_popc64(uint64_t x) { return __popcll(x); }
#else
#define MOEB_ANY(x) (x)
#define MOEB_GROUP_SYNC() ((void)0)
inline int moeb_ffs64(uint64_t x) { return __builtin_ffsll((long long)x); }
inline int moeb_popc64(uint64_t x) { return __builtin_popcountll(x); }
#endif

struct SimArgs {
  const uint64_t* truth;
  const uint64_t* preds[MOEB_MAX_PREDS];
  const uint8_t* covered[MOEB_MAX_PREDS];
  uint32_t unbounded_bits;
  int n_preds;
  int any_cov;
  const int64_t* row_off;
  int P, L, E, warmup, budget;
  int64_t cap;
  int64_t rows;
  int64_t* counters;  // this capacity: + pred * pred_stride
  int64_t counters_stride;
  int64_t* per_prompt;
  int64_t per_prompt_stride;
  uint64_t* hits;
  int64_t hits_stride;
  // nullable [n_preds][2 + 2L]: measured accesses / prediction hits (total,
  // per layer) computed upstream; used by the fast LRU kernel only
  const int64_t* given;
  // nullable: the fast LRU kernel replays only prompts plist[pi * P + i],
  // i < plist_n[pi] (the stack-distance replay's undecided prompts)
  const int32_t* plist;
  const int32_t* plist_n;
  // caller workspace (moeb_cache_sim_workspace_bytes), host-side use only
  void* ws;
  size_t ws_bytes;
  // nullable: LRU key -> queue-position tables in global memory, [n_preds][P]
  // [L*E] u16 (from the caller's workspace, moeb_cache_sim_workspace_bytes_shape)
  // instead of shared memory, for shapes whose table would cap the resident
  // simulations per SM (V3: 29.7 KB of a 39.6 KB state)
  uint16_t* pos_g;
  // per-simulation shared-memory layout (bytes)
  int off_r, off_q, off_k, off_c, sim_bytes;
  uint32_t magic;  // layer_of(key) = (key * magic) >> 22
  uint32_t qmask;  // LRU queue size - 1
};

template <int W>
MOEB_HD __forceinline__ uint64_t word_get(const uint64_t (&a)[W], int w) {
  uint64_t v = a[0];
#pragma unroll
  for (int j = 1; j < W; ++j) v = (w == j) ? a[j] : v;
  return v;
}
template <int W>
MOEB_HD __forceinline__ void word_or(uint64_t (&a)[W], int w, uint64_t bit) {
#pragma unroll
  for (int j = 0; j < W; ++j)
    if (w == j) a[j] |= bit;
}
template <int W>
MOEB_HD __forceinline__ void word_clear(uint64_t (&a)[W], int w, uint64_t bit) {
#pragma unroll
  for (int j = 0; j < W; ++j)
    if (w == j) a[j] &= ~bit;
}

// ---------------------------------------------------------------------------
// LRU: lazy-deletion recency queue, exactly the reference's OrderedDict order
// (cache.py:68). Every access (touch hit/miss, prefetch insert/refresh)
// appends the key at the queue tail and records pos_of[key] = its queue
// index (mod 2^16); an entry q[i] is valid iff pos_of[q[i]] == i, so moving a
// key to the MRU end is two stores and its old entry simply goes stale. The
// LRU key is the first valid entry from the head: `_evict_one`
// (cache.py:93-100) pops stale entries, skips pinned ones in place, and
// invalidates the victim (pos_of set outside the live window). The head
// entry and its validity are kept pre-loaded in registers, so a miss usually
// has no shared-memory load on its critical path. When the queue is full it
// is compacted in place, order preserved.
// ---------------------------------------------------------------------------
template <int W, int ES, bool GENERAL>
struct LruState {
  uint16_t* pos_of;  // [NK] queue index (mod 2^16) of the key's latest entry
  uint16_t* q;       // [qn] keys in access order
  uint64_t* R;       // [L*W] resident masks (stale for the current layer)
  uint64_t* Psm;     // GENERAL only: [L*W] pin masks
  uint32_t head, tail, qmask;
  int count, cap, npins, cur, E, L;
  uint32_t mE;
  int hk;    // q[head] (pre-loaded)
  bool hv;   // entry at head is valid (pre-loaded)
  uint64_t Rl[W], Pm[W];

  MOEB_HD void init(unsigned char* base, const SimArgs& a, int L_) {
    L = L_;
    E = a.E;
    cap = (int)a.cap;
    mE = a.magic;
    qmask = a.qmask;
    pos_of = reinterpret_cast<uint16_t*>(base);
    R = reinterpret_cast<uint64_t*>(base + a.off_r);
    Psm = GENERAL ? R + L * W : nullptr;
    q = reinterpret_cast<uint16_t*>(base + a.off_q);
    head = tail = 0;
    count = 0;
    npins = 0;
    cur = 0;
    hk = 0;
    hv = false;
#pragma unroll
    for (int j = 0; j < W; ++j) Rl[j] = Pm[j] = 0;
    for (int j = 0; j < L * W * (GENERAL ? 2 : 1); ++j) R[j] = 0;
  }

  MOEB_HD __forceinline__ int layer_of(int k) const {
    return ES >= 0 ? (k >> ES) : (int)(((uint32_t)k * mE) >> 22);
  }
  MOEB_HD __forceinline__ int expert_of(int k, int l) const {
    return ES >= 0 ? (k & ((1 << (ES >= 0 ? ES : 0)) - 1)) : k - l * E;
  }
  MOEB_HD __forceinline__ int key_of(int l, int ex) const {
    return ES >= 0 ? ((l << ES) | ex) : l * E + ex;
  }

  MOEB_HD __forceinline__ void focus(int l) {
    if (l == cur) return;
#pragma unroll
    for (int j = 0; j < W; ++j) {
      R[cur * W + j] = Rl[j];
      Rl[j] = R[l * W + j];
      if (GENERAL) {
        Psm[cur * W + j] = Pm[j];
        Pm[j] = Psm[l * W + j];
      }
    }
    cur = l;
  }

  MOEB_HD __forceinline__ bool is_pinned(int k) const {
    const int l = layer_of(k), ex = expert_of(k, l);
    const uint64_t bit = 1ull << (ex & 63);
    if (l == cur) return (word_get<W>(Pm, ex >> 6) & bit) != 0;
    if (GENERAL) return (Psm[l * W + (ex >> 6)] & bit) != 0;
    return false;  // trace mode: pins only ever exist in the current layer
  }

  MOEB_HD __forceinline__ void load_head() {
    hk = q[head & qmask];
    hv = head != tail && pos_of[hk] == (uint16_t)head;
  }

  MOEB_HD __forceinline__ void compact() {
    // every lane of the group runs this replicated loop over the shared queue:
    // all lanes read an entry before any lane rewrites the queue
    uint32_t n = head;
    for (uint32_t i = head; i != tail; ++i) {
      const int k = q[i & qmask];
      const bool live = pos_of[k] == (uint16_t)i;
      MOEB_GROUP_SYNC();
      if (live) {
        q[n & qmask] = (uint16_t)k;
        pos_of[k] = (uint16_t)n;
        ++n;
      }
      MOEB_GROUP_SYNC();
    }
    tail = n;
  }

  MOEB_HD __forceinline__ void clear_resident(int v) {
    const int l = layer_of(v), ex = expert_of(v, l);
    const uint64_t bit = 1ull << (ex & 63);
    if (l == cur)
      word_clear<W>(Rl, ex >> 6, bit);
    else
      R[l * W + (ex >> 6)] &= ~bit;
  }

  // One access of expert ex of the current layer: touch (cache.py:106-124)
  // or, with pin, one key of prefetch (cache.py:141-153). Returns whether
  // the key was resident. Straight-line except the stale-entry pops and the
  // warp-uniform rare paths.
  MOEB_HD __forceinline__ bool access(int ex, bool pin, bool active) {
    const int k = key_of(cur, ex);
    const int w = ex >> 6;
    const uint64_t bit = 1ull << (ex & 63);
    const bool hit = (word_get<W>(Rl, w) & bit) != 0;
    const bool full = count >= cap;
    const bool reject = !active || (!hit && full && count <= npins);
    const bool ev = !hit && full && !reject;
    if (MOEB_ANY(ev)) {
      if (ev) {
        while (!hv && head != tail) {  // pop stale entries (bounded by the live window)
          ++head;
          load_head();
        }
      }
      // `_evict_one` (cache.py:93-100) skips pinned keys in place; pins only
      // reach the LRU end in tiny caches.
      if (MOEB_ANY(ev && is_pinned(hk))) {
        if (ev && is_pinned(hk)) {
          uint32_t i = head + 1;
          int v = q[i & qmask];
          while (pos_of[v] != (uint16_t)i || is_pinned(v)) {
            ++i;
            v = q[i & qmask];
          }
          pos_of[v] = (uint16_t)(i + 0x8000u);  // invalidate in place
          clear_resident(v);
          hv = true;  // head entry unchanged and still valid
        } else if (ev) {
          pos_of[hk] = (uint16_t)(head + 0x8000u);
          clear_resident(hk);
          ++head;
          hv = false;
        }
      } else if (ev) {
        pos_of[hk] = (uint16_t)(head + 0x8000u);
        clear_resident(hk);
        ++head;
        hv = false;  // reloaded after the push below
      }
    }
    const bool ins = !hit && !reject;
    if (ins) {
      word_or<W>(Rl, w, bit);
      count += full ? 0 : 1;
    }
    // append at the MRU end
    if (MOEB_ANY(!reject && tail - head > qmask)) {
      if (!reject && tail - head > qmask) {
        compact();
        load_head();
      }
    }
    if (!reject) {
      const bool empty = tail == head;
      q[tail & qmask] = (uint16_t)k;
      pos_of[k] = (uint16_t)tail;
      hv = empty || (hv && hk != k);  // k's old entry (if at the head) just went stale
      hk = empty ? k : hk;
      ++tail;
    }
    if (ev && !hv) load_head();
    if (pin && !reject && !(word_get<W>(Pm, w) & bit)) {
      word_or<W>(Pm, w, bit);
      ++npins;
    }
    return hit;
  }

  MOEB_HD void begin_step(int l) {
    if (GENERAL) {
      for (int j = 0; j < L * W; ++j) Psm[j] = 0;
    }
#pragma unroll
    for (int j = 0; j < W; ++j) Pm[j] = 0;
    npins = 0;
    focus(l);
  }

  MOEB_HD __forceinline__ bool touch(int ex) { return access(ex, false, true); }
  MOEB_HD __forceinline__ bool prefetch(int ex) {
    const bool was = (word_get<W>(Rl, ex >> 6) & (1ull << (ex & 63))) != 0;
    access(ex, true, true);
    return !was && (word_get<W>(Rl, ex >> 6) & (1ull << (ex & 63))) != 0;
  }
};

// ---------------------------------------------------------------------------
// LFU (builder-defined): evict the non-pinned resident key with the fewest
// demand touches since insertion, least-recently-used among ties. Touch
// insert -> freq 1, prefetch insert -> freq 0, touch hit -> freq + 1,
// prefetch refresh -> recency only.
// ---------------------------------------------------------------------------
template <int W, bool GENERAL>
struct LfuState {
  uint16_t* slot_of;  // [L*E] valid for resident keys only
  uint64_t* R;        // [L*W]
  uint64_t* vals;     // [cap]
  uint16_t* skeys;    // [cap] (layer << 8 | expert)
  int64_t count, cap;
  uint32_t clock;
  int npins, E, L, cur;
  uint64_t Rl[W], Pm[W];

  MOEB_HD void init(unsigned char* base, const SimArgs& a, int L_) {
    L = L_;
    E = a.E;
    cap = a.cap;
    slot_of = reinterpret_cast<uint16_t*>(base);
    R = reinterpret_cast<uint64_t*>(base + a.off_r);
    vals = reinterpret_cast<uint64_t*>(base + a.off_q);
    skeys = reinterpret_cast<uint16_t*>(base + a.off_q + 8 * a.cap);
    count = 0;
    clock = 1;
    npins = 0;
    cur = 0;
#pragma unroll
    for (int j = 0; j < W; ++j) Rl[j] = Pm[j] = 0;
    for (int j = 0; j < L * W; ++j) R[j] = 0;
  }

  MOEB_HD __forceinline__ void focus(int l) {
    if (l == cur) return;
#pragma unroll
    for (int j = 0; j < W; ++j) {
      R[cur * W + j] = Rl[j];
      Rl[j] = R[l * W + j];
    }
    cur = l;
  }
  MOEB_HD __forceinline__ void writeback() {
#pragma unroll
    for (int j = 0; j < W; ++j) R[cur * W + j] = Rl[j];
  }

  MOEB_HD int victim_slot() const {
    uint64_t best = ~0ull;
    int bs = 0;
    for (int s = 0; s < (int)count; ++s) {
      const uint64_t v = vals[s];
      if (v < best) {
        best = v;
        bs = s;
      }
    }
    return bs;
  }

  // Returns the slot to fill: a fresh one, or the evicted victim's.
  MOEB_HD int make_room() {
    if (count < cap) return (int)count++;
    const int s = victim_slot();
    const uint32_t vk = skeys[s];
    const int l = (int)(vk >> 8), ex = (int)(vk & 0xFFu);
    const uint64_t bit = 1ull << (ex & 63);
    if (l == cur)
      word_clear<W>(Rl, ex >> 6, bit);
    else
      R[l * W + (ex >> 6)] &= ~bit;
    return s;
  }

  MOEB_HD void begin_step(int l) {
    if (GENERAL) {
      for (int s = 0; s < (int)count; ++s) vals[s] &= ~kPin;
    } else {
      for (int w = 0; w < W; ++w) {
        uint64_t m = Pm[w];
        while (m) {
          const int ex = w * 64 + moeb_ffs64(m) - 1;
          m &= m - 1;
          vals[slot_of[cur * E + ex]] &= ~kPin;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < W; ++j) Pm[j] = 0;
    npins = 0;
    focus(l);
  }

  MOEB_HD __forceinline__ bool touch(int ex) {
    const uint64_t bit = 1ull << (ex & 63);
    const int key = cur * E + ex;
    if (word_get<W>(Rl, ex >> 6) & bit) {
      const int s = slot_of[key];
      const uint64_t v = vals[s];
      const uint64_t freq = ((v & ~kPin) >> 32) + 1;
      vals[s] = (v & kPin) | (freq << 32) | clock++;
      return true;
    }
    if (count >= cap && count <= npins) return false;
    const int s = make_room();
    vals[s] = (1ull << 32) | clock++;
    skeys[s] = (uint16_t)((cur << 8) | ex);
    slot_of[key] = (uint16_t)s;
    word_or<W>(Rl, ex >> 6, bit);
    return false;
  }

  MOEB_HD __forceinline__ bool access(int ex, bool pin, bool active) {
    if (!active) return false;
    const bool was = (word_get<W>(Rl, ex >> 6) & (1ull << (ex & 63))) != 0;
    if (pin) {
      prefetch(ex);
      return was;
    }
    return touch(ex);
  }

  MOEB_HD __forceinline__ bool prefetch(int ex) {
    const int w = ex >> 6;
    const uint64_t bit = 1ull << (ex & 63);
    const int key = cur * E + ex;
    if (word_get<W>(Rl, w) & bit) {
      const int s = slot_of[key];
      const uint64_t v = vals[s];
      vals[s] = kPin | (v & 0x7FFFFFFF00000000ull) | clock++;
      if (!(v & kPin)) {
        word_or<W>(Pm, w, bit);
        ++npins;
      }
      return false;
    }
    if (count >= cap && count <= npins) return false;
    const int s = make_room();
    vals[s] = kPin | clock++;
    skeys[s] = (uint16_t)((cur << 8) | ex);
    slot_of[key] = (uint16_t)s;
    word_or<W>(Rl, w, bit);
    word_or<W>(Pm, w, bit);
    ++npins;
    return true;
  }
};

// ---------------------------------------------------------------------------
// Trace replay driver (engine.py:157-206), shared by both policies.
// One thread = one simulation; a warp = 32 simulations stepping in lockstep
// over row index i of their own prompts. Every prompt starts at layer 0, so
// all lanes are always at the same layer and the same warm-up phase: only
// the cache operations themselves differ per lane. Per-layer counters are
// warp-reduced each measured row into block-level shared counters.
// ---------------------------------------------------------------------------
constexpr int kPrefetchRows = 4;

template <int W, class State>
__global__ void __launch_bounds__(32) k_cache_sim(const SimArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int L = a.L;
  unsigned int* bcnt = reinterpret_cast<unsigned int*>(smem);  // [3L] block counters
  for (int j = threadIdx.x; j < 3 * L; j += blockDim.x) bcnt[j] = 0;
  __syncthreads();
  const int pi = blockIdx.y;  // prediction stream: never mixed within a block
  const int64_t pg = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = pg < a.P;
  const int p = live ? (int)pg : 0;
  unsigned char* base = smem + a.off_c + (size_t)threadIdx.x * a.sim_bytes;
  const int64_t r0 = live ? a.row_off[p] : 0;
  const int64_t nrows = live ? a.row_off[p + 1] - r0 : 0;
  const unsigned full = 0xffffffffu;
  int64_t nmax = nrows;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const int64_t other = __shfl_xor_sync(full, nmax, o);
    nmax = other > nmax ? other : nmax;
  }

  State st;
  if (live) st.init(base, a, L);

  const uint64_t* __restrict__ pred = a.preds[pi];
  const uint8_t* __restrict__ cov = a.covered[pi];
  const bool unbounded = (a.unbounded_bits >> pi) & 1u;
  const int limit = unbounded ? a.E : a.budget;
  uint64_t* hits = a.hits ? a.hits + pi * a.hits_stride : nullptr;
  const uint64_t* __restrict__ tr = a.truth + r0 * W;
  const uint64_t* __restrict__ pr = pred ? pred + r0 * W : nullptr;

  int64_t tot_k = 0, tot_ch = 0, tot_ph = 0, tot_unc = 0;
  // software-pipelined row reads: rows i .. i+kPrefetchRows-1 in registers
  uint64_t tbuf[kPrefetchRows][W], pbuf[kPrefetchRows][W];
#pragma unroll
  for (int d = 0; d < kPrefetchRows; ++d)
#pragma unroll
    for (int w = 0; w < W; ++w) {
      tbuf[d][w] = d < nrows ? __ldg(tr + d * W + w) : 0ull;
      pbuf[d][w] = (pr && d < nrows) ? __ldg(pr + d * W + w) : 0ull;
    }
  int l = 0, t = 0;
  for (int64_t i0 = 0; i0 < nmax; i0 += kPrefetchRows) {
#pragma unroll
    for (int d = 0; d < kPrefetchRows; ++d) {
      const int64_t i = i0 + d;
      if (i >= nmax) break;  // warp-uniform
      const bool valid = i < nrows;
      uint64_t tw[W], pw[W], hw[W];
#pragma unroll
      for (int w = 0; w < W; ++w) {
        tw[w] = tbuf[d][w];
        pw[w] = pbuf[d][w];
        hw[w] = 0;
        const int64_t j = i + kPrefetchRows;  // refill this slot
        tbuf[d][w] = j < nrows ? __ldg(tr + j * W + w) : 0ull;
        pbuf[d][w] = (pr && j < nrows) ? __ldg(pr + j * W + w) : 0ull;
      }
      // One flat op stream per row: prefetch(sorted(pred)[:limit]) then touch
      // every truth expert ascending (engine.py:160-184). Warm-up rows only
      // touch (no begin_step, no counters).
      const bool measured = t >= a.warmup;
      uint64_t mk[W], mt[W];
#pragma unroll
      for (int w = 0; w < W; ++w) {
        mk[w] = (valid && measured) ? pw[w] : 0ull;
        mt[w] = valid ? tw[w] : 0ull;
      }
      if (valid && measured) st.begin_step(l);  // engine.py:172
      else if (valid) st.focus(l);
      int k = 0, ph = 0, ch = 0, taken = 0;
      if (valid && measured) {
#pragma unroll
        for (int w = 0; w < W; ++w) {
          k += __popcll(tw[w]);
          ph += __popcll(tw[w] & pw[w]);  // FULL predicted set (engine.py:181-182)
        }
        if (cov && !cov[r0 + i]) ++tot_unc;  // engine.py:175-176
      }
      if (limit <= 0) {
#pragma unroll
        for (int w = 0; w < W; ++w) mk[w] = 0;
      }
      for (;;) {
        bool any_k = false, any_t = false;
#pragma unroll
        for (int w = 0; w < W; ++w) {
          any_k |= mk[w] != 0;
          any_t |= mt[w] != 0;
        }
        const bool act = any_k || any_t;
        if (!__any_sync(full, act)) break;
        const bool pf = any_k;
        int ex = 0;
        bool found = false;
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const uint64_t m = pf ? mk[w] : mt[w];
          if (!found && m) {
            ex = w * 64 + __ffsll((long long)m) - 1;
            found = true;
            if (pf) mk[w] = m & (m - 1); else mt[w] = m & (m - 1);
          }
        }
        const bool hit = st.access(ex, pf, act);
        if (act && !pf && hit) {
          ++ch;
          word_or<W>(hw, ex >> 6, 1ull << (ex & 63));
        }
        if (act && pf && ++taken >= limit) {
#pragma unroll
          for (int w = 0; w < W; ++w) mk[w] = 0;
        }
      }
      if (measured) {
        if (!valid) ch = 0;
        if (!measured) ch = 0;
        tot_k += k;
        tot_ch += ch;
        tot_ph += ph;
        const unsigned sk = __reduce_add_sync(full, (unsigned)k);
        const unsigned sc = __reduce_add_sync(full, (unsigned)ch);
        const unsigned sp = __reduce_add_sync(full, (unsigned)ph);
        if ((threadIdx.x & 31) == 0) {
          atomicAdd(&bcnt[l], sk);
          atomicAdd(&bcnt[L + l], sc);
          atomicAdd(&bcnt[2 * L + l], sp);
        }
      }
      if (hits && valid) {
#pragma unroll
        for (int w = 0; w < W; ++w) hits[(r0 + i) * W + w] = hw[w];
      }
      if (++l == L) {
        l = 0;
        ++t;
      }
    }
  }

  __syncthreads();
  int64_t* c = a.counters + pi * a.counters_stride;
  if (live) {
    atomicAdd(reinterpret_cast<unsigned long long*>(c + 0), (unsigned long long)tot_k);
    atomicAdd(reinterpret_cast<unsigned long long*>(c + 1), (unsigned long long)tot_ch);
    atomicAdd(reinterpret_cast<unsigned long long*>(c + 2), (unsigned long long)tot_ph);
    if (tot_unc) atomicAdd(reinterpret_cast<unsigned long long*>(c + 3), (unsigned long long)tot_unc);
    if (a.per_prompt) {
      int64_t* pp = a.per_prompt + pi * a.per_prompt_stride + 4 * (int64_t)p;
      pp[0] += tot_k;
      pp[1] += tot_ch;
      pp[2] += tot_ph;
      pp[3] += tot_unc;
    }
  }
  for (int j = threadIdx.x; j < 3 * L; j += blockDim.x)
    if (bcnt[j]) atomicAdd(reinterpret_cast<unsigned long long*>(c + 4 + j), (unsigned long long)bcnt[j]);
}

// Op-stream interpreter (one cache): the reference's per-call API.
template <int W, class State>
__global__ void k_cache_ops(const SimArgs a, const int32_t* ops, const int32_t* keys, int64_t n,
                            uint8_t* results) {
  extern __shared__ __align__(16) unsigned char smem[];
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  State st;
  st.init(smem, a, a.L);
  for (int64_t i = 0; i < n; ++i) {
    uint8_t res = 0;
    if (ops[i] == 0) {
      st.begin_step(st.cur);
    } else {
      const int key = keys[i];
      st.focus(key / a.E);
      const int ex = key % a.E;
      res = ops[i] == 1 ? (uint8_t)st.touch(ex) : (uint8_t)st.prefetch(ex);
    }
    results[i] = res;
  }
}

inline int align16(int64_t x) { return (int)((x + 15) / 16 * 16); }

uint32_t layer_magic(int L, int E) {
  const uint32_t m = (uint32_t)(((1u << 22) + E - 1) / E);
  for (int v = 0; v <= L * E; ++v)
    if ((int)(((uint64_t)v * m) >> 22) != v / E) return 0;
  return m;
}

// Shared-memory layout of one simulation (LRU: slot map, masks, ring links,
// slot keys; LFU: slot map, masks, slot values/keys).
void layout(SimArgs& a, int policy, bool general) {
  const int W = moeb::words_for(a.E);
  const int64_t NK = (int64_t)a.L * a.E;
  const int64_t rbytes = 8LL * a.L * W * (general ? 2 : 1);
  if (policy == MOEB_POLICY_LRU) {
    uint32_t qn = 64;  // >= 2 * cap: compaction at most every cap pushes
    while (qn < 2 * a.cap + 32) qn <<= 1;
    a.qmask = qn - 1;
    a.off_r = (a.pos_g && !general) ? 0 : align16(2 * NK);  // pos_of (unless in global memory)
    a.off_q = align16(a.off_r + rbytes);
    a.off_k = 0;
    a.sim_bytes = align16(a.off_q + 2LL * qn) + 16;  // +16 B skews smem banks
  } else {
    a.qmask = 0;
    a.off_r = (a.pos_g && !general) ? 0 : align16(2 * NK);  // slot_of (unless in global memory)
    a.off_q = align16(a.off_r + rbytes);  // vals [cap] u64, skeys [cap] u16
    a.off_k = 0;
    a.sim_bytes = align16(a.off_q + 10LL * a.cap) + 16;
  }
  a.magic = layer_magic(a.L, a.E);
}

// ---------------------------------------------------------------------------
// K1 LRU, warp-per-simulation, row-batched. One warp owns one (stream,
// prompt) simulation and resolves a whole trace row at once:
//   accesses A = [K = sorted(pred)[:limit]] ++ [T = truth], all in layer l;
//   with R_l the layer's resident mask at row start and no interplay,
//     touch hits   = T & (R_l | K)
//     inserts m    = |K \ R_l| + |T \ (R_l | K)|
//     evictions e  = max(0, count + m - cap), the first e VALID queue entries
//   (found with one 32-wide ballot per queue chunk), and the row's keys are
//   appended in access order ((K \ T) ascending, then T ascending -- the
//   order the reference's OrderedDict ends in; the superseded first push of
//   a K&T key is stale anyway). "Interplay" -- a victim that the same row
//   accesses, or a cache so small that pins/rejections can matter -- makes
//   that warp replay the row with the exact sequential state machine
//   (LruState::access), executed by all lanes in lockstep.
// Trace rows are read as coalesced 32-row windows (one row per lane,
// double-buffered) and broadcast with shuffles.
// ---------------------------------------------------------------------------
template <int W>
__device__ __forceinline__ void keep_lowest(uint64_t (&m)[W], int n) {
#pragma unroll
  for (int w = 0; w < W; ++w) {
    int c = __popcll(m[w]);
    if (n <= 0) {
      m[w] = 0;
    } else if (c > n) {
      uint64_t x = m[w], keep = 0;
      for (int i = 0; i < n; ++i) {
        keep |= x & (~x + 1);
        x &= x - 1;
      }
      m[w] = keep;
      c = n;
    }
    n -= c;
  }
}

template <int W>
__device__ __forceinline__ int popc_w(const uint64_t (&m)[W]) {
  int c = 0;
#pragma unroll
  for (int w = 0; w < W; ++w) c += __popcll(m[w]);
  return c;
}

// number of set bits of m below expert e
template <int W>
__device__ __forceinline__ int rank_below(const uint64_t (&m)[W], int e) {
  int c = 0;
#pragma unroll
  for (int w = 0; w < W; ++w) {
    const int lo = w * 64;
    if (e >= lo + 64)
      c += __popcll(m[w]);
    else if (e > lo)
      c += __popcll(m[w] & ((1ull << (e - lo)) - 1));
  }
  return c;
}

// position of the n-th (0-based) set bit of a 64-bit word, n < popc(m):
// halving steps with popcounts, branch-free
__device__ __forceinline__ int nth_bit64(uint64_t m, int n) {
  const uint32_t lo = (uint32_t)m;
  const int cl = __popc(lo);
  const bool up = n >= cl;
  uint32_t x = up ? (uint32_t)(m >> 32) : lo;
  int base = up ? 32 : 0;
  n -= up ? cl : 0;
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
    const int c = __popc(x & ((1u << w) - 1u));
    const bool hi = n >= c;
    x = hi ? x >> w : x;
    base += hi ? w : 0;
    n -= hi ? c : 0;
  }
  return base;
}

// n-th set bit (ascending expert order) of a W-word mask, n < popc
template <int W>
__device__ __forceinline__ int nth_bit(const uint64_t (&m)[W], int n) {
  if (W == 1) return nth_bit64(m[0], n);
  int w = 0;
  uint64_t sel = m[0];
#pragma unroll
  for (int j = 0; j < W; ++j) {
    const int c = __popcll(m[j]);
    if (w == j) {
      if (n < c) {
        sel = m[j];
      } else {
        n -= c;
        ++w;
      }
    }
  }
  return w * 64 + nth_bit64(sel, n);
}

// KPH = false: the measured-access / prediction-hit counters are not
// computed here (they do not depend on the cache); block 0 adds a.given
template <int W, int ES, int G, bool EXTRA, bool KPH = true>
__global__ void __launch_bounds__(128) k_cache_sim_warp(const SimArgs a) {
  // G lanes per simulation (32: one per warp; 16: two per warp). All
  // collectives below are restricted to the group's lanes (gmask), so the
  // two groups of a warp may diverge (fallback rows, different row counts).
  static_assert(G == 8 || G == 16 || G == 32, "G must be 8, 16 or 32");
  extern __shared__ __align__(16) unsigned char smem[];
  const int L = a.L, E = a.E;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int hl = lane & (G - 1), gbase = lane - hl;
  const unsigned glow = G == 32 ? 0xffffffffu : ((1u << G) - 1u);
  const unsigned gmask = glow << gbase;
  unsigned int* bcnt = reinterpret_cast<unsigned int*>(smem);  // [3L] block counters
  for (int j = threadIdx.x; j < 3 * L; j += blockDim.x) bcnt[j] = 0;
  __syncthreads();
  const int pi = blockIdx.y;
  const int sims_per_block = nw * (32 / G);
  const int sl = wib * (32 / G) + lane / G;  // simulation within the block
  const int sidx = blockIdx.x * sims_per_block + sl;
  const bool live = a.plist ? sidx < a.plist_n[pi] : sidx < a.P;
  const int p = a.plist ? (live ? a.plist[(int64_t)pi * a.P + sidx] : 0) : sidx;
  constexpr unsigned FULL = 0xffffffffu;
  // The whole warp runs the row loop to the longer of its groups' prompts
  // (missing rows are all-zero no-op rows), so the common path's warp
  // collectives can use the full mask: a dead or shorter group still takes
  // part. Rare paths (scan, fallback, compaction) keep the group mask.
  if (__any_sync(FULL, live)) {
    unsigned char* base = smem + a.off_c + (size_t)sl * a.sim_bytes;
    LruState<W, ES, false> st;
    st.init(base, a, L);  // every lane of the group holds the same state
    // the key-position table of this (stream, prompt) in global memory: no
    // initialisation needed (an entry is read only for a key pushed by this
    // simulation, and every push writes it)
    if (a.pos_g) st.pos_of = a.pos_g + ((int64_t)pi * a.P + p) * ((int64_t)L * E);
    uint16_t* pos_of = st.pos_of;
    uint16_t* q = st.q;
    uint64_t* R = st.R;
    const uint32_t qmask = st.qmask;
    const uint64_t* __restrict__ pred = a.preds[pi];
    const uint8_t* __restrict__ cov = EXTRA ? a.covered[pi] : nullptr;
    const bool unbounded = (a.unbounded_bits >> pi) & 1u;
    const int limit = unbounded ? E : a.budget;
    uint64_t* hits = (EXTRA && a.hits) ? a.hits + pi * a.hits_stride : nullptr;
    const int64_t r0 = live ? a.row_off[p] : 0;
    // rows per prompt < 2^31 - 64 (checked by the host wrapper): 32-bit row loop
    const int nrows = live ? (int)(a.row_off[p + 1] - r0) : 0;
    int nmax = nrows;
#pragma unroll
    for (int o = G; o < 32; o <<= 1) nmax = max(nmax, __shfl_xor_sync(FULL, nmax, o));
    const uint64_t* __restrict__ tr = a.truth + r0 * W;
    const uint64_t* __restrict__ pr = pred ? pred + r0 * W : nullptr;
    int tot_k = 0, tot_ch = 0, tot_ph = 0, tot_unc = 0;
    __syncwarp(gmask);

    uint64_t wt[W], wp[W], nt[W], np[W];  // current / next G-row windows
#pragma unroll
    for (int w = 0; w < W; ++w) {
      wt[w] = hl < nrows ? __ldg(tr + (int64_t)hl * W + w) : 0ull;
      wp[w] = (pr && hl < nrows) ? __ldg(pr + (int64_t)hl * W + w) : 0ull;
    }
    int l = 0, t = 0;
    for (int i = 0; i < nmax; ++i) {
      const int slot = i & (G - 1);
      if (slot == 0) {  // prefetch the next window
        const int j = i + G + hl;
#pragma unroll
        for (int w = 0; w < W; ++w) {
          nt[w] = j < nrows ? __ldg(tr + (int64_t)j * W + w) : 0ull;
          np[w] = (pr && j < nrows) ? __ldg(pr + (int64_t)j * W + w) : 0ull;
        }
      }
      uint64_t T[W], P[W], K[W];
#pragma unroll
      for (int w = 0; w < W; ++w) {
        T[w] = __shfl_sync(FULL, wt[w], slot, G);
        P[w] = __shfl_sync(FULL, wp[w], slot, G);
      }
      if (slot == G - 1) {
#pragma unroll
        for (int w = 0; w < W; ++w) {
          wt[w] = nt[w];
          wp[w] = np[w];
        }
      }
      const bool measured = t >= a.warmup;
      int npk = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        K[w] = measured ? P[w] : 0ull;
        npk += __popcll(K[w]);
      }
      if (npk > limit) {
        keep_lowest<W>(K, limit);
        npk = limit;  // = popc(K)
      }
      uint64_t Rl[W], S[W], Hm[W];
#pragma unroll
      for (int w = 0; w < W; ++w) {
        Rl[w] = R[l * W + w];
        S[w] = K[w] | T[w];
      }
      // inserts m = |K \ R| + |T \ (R | K)| = |S \ R|; refreshed = |S & R| = ns - m
      int m = 0, ns = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        m += __popcll(S[w] & ~Rl[w]);
        ns += __popcll(S[w]);
        Hm[w] = T[w] & (Rl[w] | K[w]);
      }
      const int refresh = ns - m;
      const int e = st.count + m - st.cap > 0 ? st.count + m - st.cap : 0;
      bool fallback = (st.cap <= npk) || (e > st.count - refresh);
      // first victim window: all lanes of the warp, converged (full-mask votes)
      uint32_t newhead = st.head;
      bool applied = false;
      {
        // branch-free (bitwise &, unconditional key decode): the vote chain
        // below is the row's critical path
        const bool want = !fallback & (e > 0);
        const uint32_t idx = st.head + hl;
        const bool inr = (uint32_t)hl < st.tail - st.head;
        const int key = q[idx & qmask];
        const bool valid = inr && pos_of[key] == (uint16_t)idx;
        const unsigned vb = (__ballot_sync(FULL, valid) >> gbase) & glow;
        const bool ok1 = want & (__popc(vb) >= e);
        const bool victim = ok1 & valid & (__popc(vb & ((1u << hl) - 1)) < e);
        int vl = 0, ve = 0;
        bool bad = false;
        if (W == 1) {  // one mask word: decode unconditionally
          vl = st.layer_of(key);
          ve = st.expert_of(key, vl);
          bad = victim & (vl == l) & (((S[0] >> (ve & 63)) & 1ull) != 0);
        } else if (victim) {
          vl = st.layer_of(key);
          ve = st.expert_of(key, vl);
          bad = vl == l && ((word_get<W>(S, ve >> 6) >> (ve & 63)) & 1ull);
        }
        const bool anybad = ((__ballot_sync(FULL, bad) >> gbase) & glow) != 0u;
        if (ok1 & anybad) fallback = true;
        applied = ok1 & !anybad;
        if (applied && victim) {
          pos_of[key] = (uint16_t)(idx + 0x8000u);
          atomicAnd(reinterpret_cast<unsigned int*>(R + vl * W + (ve >> 6)) + ((ve >> 5) & 1),
                    ~(1u << (ve & 31)));
        }
        const unsigned vict = (__ballot_sync(FULL, applied && victim) >> gbase) & glow;
        if (applied) newhead = st.head + (32 - __clz(vict));
      }
      if (!fallback && e > 0 && !applied) {  // scan: find the e-th valid entry, check interplay
        int found = 0;
        uint32_t pos = st.head;
        while (found < e) {
          if (pos - st.head >= st.tail - st.head) {  // cannot happen; never spin
            fallback = true;
            break;
          }
          const uint32_t idx = pos + hl;
          const bool inr = idx - st.head < st.tail - st.head;
          const int key = q[idx & qmask];
          const bool valid = inr && pos_of[key] == (uint16_t)idx;
          const unsigned vb = (__ballot_sync(gmask, valid) >> gbase) & glow;
          const int need = e - found;
          const int rank = __popc(vb & ((1u << hl) - 1));
          const bool victim = valid && rank < need;
          bool bad = false;
          if (victim) {
            const int vl = st.layer_of(key), ve = st.expert_of(key, vl);
            bad = vl == l && ((word_get<W>(S, ve >> 6) >> (ve & 63)) & 1ull);
          }
          if (__any_sync(gmask, bad)) {
            fallback = true;
            break;
          }
          const int nv = __popc(vb);
          if (nv >= need) {
            const unsigned vict = (__ballot_sync(gmask, victim) >> gbase) & glow;
            newhead = pos + (32 - __clz(vict));  // after the e-th victim
            found = e;
          } else {
            found += nv;
            pos += G;
          }
        }
      }
      int ch;
      if (!fallback) {
        // evict: every valid entry in [head, newhead) is a victim
        for (uint32_t pos = st.head; !applied && pos != newhead; pos += G) {
          const uint32_t idx = pos + hl;
          if (idx - pos < newhead - pos) {
            const int key = q[idx & qmask];
            if (pos_of[key] == (uint16_t)idx) {
              pos_of[key] = (uint16_t)(idx + 0x8000u);
              const int vl = st.layer_of(key), ve = st.expert_of(key, vl);
              atomicAnd(reinterpret_cast<unsigned int*>(R + vl * W + (ve >> 6)) + ((ve >> 5) & 1),
                        ~(1u << (ve & 31)));
            }
          }
          if (newhead - pos <= (uint32_t)G) break;
        }
        st.head = newhead;
        st.count += m - e;
        if (st.tail - st.head + (uint32_t)ns > qmask + 1) {  // group compaction
          __syncwarp(gmask);
          uint32_t n = st.head;
          for (uint32_t pos = st.head; pos != st.tail; pos += G) {
            const uint32_t idx = pos + hl;
            const bool inr = idx - pos < st.tail - pos;
            const int key = q[idx & qmask];
            const bool valid = inr && pos_of[key] == (uint16_t)idx;
            const unsigned vb = (__ballot_sync(gmask, valid) >> gbase) & glow;
            __syncwarp(gmask);
            if (valid) {
              const uint32_t dst = n + __popc(vb & ((1u << hl) - 1));
              q[dst & qmask] = (uint16_t)key;
              pos_of[key] = (uint16_t)dst;
            }
            __syncwarp(gmask);
            n += __popc(vb);
            if (st.tail - pos <= (uint32_t)G) break;
          }
          st.tail = n;
        }
        // append the row's keys: (K \ T) ascending, then T ascending -- lane
        // i < ns writes the i-th key of that order (ns <= budget + top_k)
        uint64_t A[W];
#pragma unroll
        for (int w = 0; w < W; ++w) A[w] = K[w] & ~T[w];
        const int na = popc_w<W>(A);
        for (int i0 = 0; i0 < ns; i0 += G) {
          const int i = i0 + hl;
          if (i < ns) {
            const bool in_a = i < na;  // select the mask first: one n-th-bit search
            uint64_t M[W];
#pragma unroll
            for (int w = 0; w < W; ++w) M[w] = in_a ? A[w] : T[w];
            const int ex = nth_bit<W>(M, in_a ? i : i - na);
            const uint32_t dst = st.tail + (uint32_t)i;
            const int key = st.key_of(l, ex);
            q[dst & qmask] = (uint16_t)key;
            pos_of[key] = (uint16_t)dst;
          }
        }
        st.tail += ns;
        if (W == 1) {
          // R_l |= S as shared atomics: on this path no victim is in S, so the
          // victims' atomicAnd and this OR commute and need no barrier between
          if (hl == 0) {
            unsigned int* rw = reinterpret_cast<unsigned int*>(R + l);
            if ((uint32_t)S[0]) atomicOr(rw, (uint32_t)S[0]);
            if ((uint32_t)(S[0] >> 32)) atomicOr(rw + 1, (uint32_t)(S[0] >> 32));
          }
        } else {
          __syncwarp(gmask);
          if (hl < W) {
            uint64_t v = 0;
#pragma unroll
            for (int w = 0; w < W; ++w)
              if (w == hl) v = R[l * W + w] | S[w];
            R[l * W + hl] = v;
          }
        }
        __syncwarp(gmask);
        ch = popc_w<W>(Hm);
      } else {
        // exact sequential replay of this row (all lanes of the group in lockstep)
        st.cur = l;
#pragma unroll
        for (int w = 0; w < W; ++w) {
          st.Rl[w] = R[l * W + w];
          st.Pm[w] = 0;
          Hm[w] = 0;
        }
        st.npins = 0;
        st.load_head();
        MOEB_FOR_EACH_BIT(W, K, ex, { st.access(ex, true, true); })
        ch = 0;
        MOEB_FOR_EACH_BIT(W, T, ex, {
          if (st.access(ex, false, true)) {
            ++ch;
            word_or<W>(Hm, ex >> 6, 1ull << (ex & 63));
          }
        })
        __syncwarp(gmask);
        if (hl < W) {
          uint64_t v = 0;
#pragma unroll
          for (int w = 0; w < W; ++w)
            if (w == hl) v = st.Rl[w];
          R[l * W + hl] = v;
        }
        __syncwarp(gmask);
      }
      if (EXTRA && hits && hl < W && i < nrows) {
        uint64_t v = 0;
#pragma unroll
        for (int w = 0; w < W; ++w)
          if (w == hl) v = Hm[w];
        hits[(r0 + i) * W + hl] = v;
      }
      if (measured) {
        int k = 0, ph = 0;
        if (KPH) {
          k = popc_w<W>(T);
#pragma unroll
          for (int w = 0; w < W; ++w) ph += __popcll(T[w] & P[w]);  // FULL predicted set
        }
        if (EXTRA && cov && i < nrows && cov[r0 + i] == 0) ++tot_unc;  // engine.py:175-176
        tot_k += k;
        tot_ch += ch;
        tot_ph += ph;
        if (hl == 0) {  // per-layer counters: fire-and-forget shared-memory reductions
          if (KPH) atomicAdd(&bcnt[l], (unsigned)k);  // native 32-bit shared atomics (a
          atomicAdd(&bcnt[L + l], (unsigned)ch);      // 64-bit one is a CAS loop)
          if (KPH) atomicAdd(&bcnt[2 * L + l], (unsigned)ph);
        }
      }
      if (++l == L) {
        l = 0;
        ++t;
      }
    }
    int64_t* c = a.counters + pi * a.counters_stride;
    if (hl == 0 && live) {
      atomicAdd(reinterpret_cast<unsigned long long*>(c + 0), (unsigned long long)tot_k);
      atomicAdd(reinterpret_cast<unsigned long long*>(c + 1), (unsigned long long)tot_ch);
      atomicAdd(reinterpret_cast<unsigned long long*>(c + 2), (unsigned long long)tot_ph);
      if (tot_unc) atomicAdd(reinterpret_cast<unsigned long long*>(c + 3), (unsigned long long)tot_unc);
      if (a.per_prompt) {
        int64_t* pp = a.per_prompt + pi * a.per_prompt_stride + 4 * (int64_t)p;
        pp[0] += tot_k;
        pp[1] += tot_ch;
        pp[2] += tot_ph;
        pp[3] += tot_unc;
      }
    }
  }
  __syncthreads();
  int64_t* c = a.counters + pi * a.counters_stride;
  for (int j = threadIdx.x; j < 3 * L; j += blockDim.x)
    if (bcnt[j]) atomicAdd(reinterpret_cast<unsigned long long*>(c + 4 + j), (unsigned long long)bcnt[j]);
  if (!KPH && a.given && blockIdx.x == 0) {  // the upstream counts, once per prediction stream
    const int64_t* g = a.given + (int64_t)pi * (2 + 2 * L);
    for (int j = threadIdx.x; j < 2 + 2 * L; j += blockDim.x) {
      const int idx = j == 0 ? 0 : j == 1 ? 2 : j < 2 + L ? 4 + (j - 2) : 4 + 2 * L + (j - 2 - L);
      if (g[j]) atomicAdd(reinterpret_cast<unsigned long long*>(c + idx), (unsigned long long)g[j]);
    }
  }
}

// ---------------------------------------------------------------------------
// K1 LFU, warp per simulation. Same semantics and op stream as LfuState (one
// access at a time, bit-exact with the thread-per-simulation kernel and its
// oracle), but the eviction argmin is warp-parallel: lane i owns the slots
// i, i + 32, ... of the slot array and keeps the minimum (value, slot) of
// its slots in registers; a victim is a 5-step shuffle argmin over the 32
// lane minima, and only the lane owning a changed slot rescans its slots.
// Values are pin << 63 | freq << 32 | clock (unique clock: no ties).
// ---------------------------------------------------------------------------
template <int W, bool EXTRA>
__global__ void __launch_bounds__(128) k_cache_sim_lfu_warp(const SimArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr unsigned FULL = 0xffffffffu;
  const int L = a.L, E = a.E;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nw = blockDim.x >> 5;
  unsigned int* bcnt = reinterpret_cast<unsigned int*>(smem);  // [3L] block counters
  for (int j = threadIdx.x; j < 3 * L; j += blockDim.x) bcnt[j] = 0;
  __syncthreads();
  const int pi = blockIdx.y;
  const int p = blockIdx.x * nw + wib;
  if (p < a.P) {
    unsigned char* base = smem + a.off_c + (size_t)wib * a.sim_bytes;
    // key -> slot: shared memory, or this simulation's table in global memory
    // (read only for resident keys, written at their insert: no initialisation)
    uint16_t* slot_of = a.pos_g ? a.pos_g + ((int64_t)pi * a.P + p) * ((int64_t)L * E)
                                : reinterpret_cast<uint16_t*>(base);
    uint64_t* Rs = reinterpret_cast<uint64_t*>(base + a.off_r);
    uint64_t* vals = reinterpret_cast<uint64_t*>(base + a.off_q);
    uint16_t* skeys = reinterpret_cast<uint16_t*>(base + a.off_q + 8 * a.cap);
    for (int j = lane; j < L * W; j += 32) Rs[j] = 0;
    const int cap = (int)a.cap;
    int count = 0, npins = 0, cur = 0;
    uint32_t clock = 1;
    uint64_t Rl[W], Pm[W];
#pragma unroll
    for (int w = 0; w < W; ++w) Rl[w] = Pm[w] = 0;
    uint64_t mv = ~0ull;  // this lane's minimum slot value, and its slot
    int ms = -1;
    __syncwarp();

    auto rescan = [&]() {  // owner lane: minimum over its slots < count
      uint64_t best = ~0ull;
      int bs = -1;
      for (int sl = lane; sl < count; sl += 32) {
        const uint64_t v = vals[sl];
        if (v < best) {
          best = v;
          bs = sl;
        }
      }
      mv = best;
      ms = bs;
    };
    auto focus = [&](int l) {
      if (l == cur) return;
      __syncwarp();
      if (lane < W) {
        uint64_t v = 0;
#pragma unroll
        for (int w = 0; w < W; ++w)
          if (w == lane) v = Rl[w];
        Rs[cur * W + lane] = v;
      }
      __syncwarp();
#pragma unroll
      for (int w = 0; w < W; ++w) Rl[w] = Rs[l * W + w];
      cur = l;
    };
    // slot for a new key: a fresh one or the evicted victim's (make_room)
    auto make_room = [&]() -> int {
      if (count < cap) return count++;
      uint64_t bv = mv;
      int bsl = ms;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const uint64_t ov = __shfl_xor_sync(FULL, bv, o);
        const int os = __shfl_xor_sync(FULL, bsl, o);
        if (ov < bv) {
          bv = ov;
          bsl = os;
        }
      }
      const uint32_t vk = skeys[bsl];
      const int vl = (int)(vk >> 8), vex = (int)(vk & 0xFFu);
      const uint64_t bit = 1ull << (vex & 63);
      if (vl == cur) {
        word_clear<W>(Rl, vex >> 6, bit);
      } else if (lane == 0) {
        Rs[vl * W + (vex >> 6)] &= ~bit;
      }
      return bsl;
    };
    auto place = [&](int sl, uint64_t v, int key, int ex) {  // write a slot (owner lane)
      if ((sl & 31) == lane) {
        vals[sl] = v;
        skeys[sl] = (uint16_t)((cur << 8) | ex);
        if (sl == ms) {
          __threadfence_block();
          rescan();
        } else if (v < mv) {
          mv = v;
          ms = sl;
        }
      }
      if (lane == 0) slot_of[key] = (uint16_t)sl;
    };
    auto update = [&](int sl, uint64_t v) {  // change a resident slot's value
      if ((sl & 31) == lane) {
        vals[sl] = v;
        if (sl == ms) rescan();
        else if (v < mv) {
          mv = v;
          ms = sl;
        }
      }
    };

    const uint64_t* __restrict__ pred = a.preds[pi];
    const uint8_t* __restrict__ cov = EXTRA ? a.covered[pi] : nullptr;
    const bool unbounded = (a.unbounded_bits >> pi) & 1u;
    const int limit = unbounded ? E : a.budget;
    uint64_t* hits = (EXTRA && a.hits) ? a.hits + pi * a.hits_stride : nullptr;
    const int64_t r0 = a.row_off[p];
    const int64_t nrows = a.row_off[p + 1] - r0;
    int64_t tot_k = 0, tot_ch = 0, tot_ph = 0, tot_unc = 0;
    int l = 0, t = 0;
    uint64_t tw = 0, pw = 0;  // row words held by lane w (coalesced reads)
    for (int64_t i = 0; i < nrows; ++i) {
      if (lane < W) {
        tw = __ldg(a.truth + (r0 + i) * W + lane);
        pw = pred ? __ldg(pred + (r0 + i) * W + lane) : 0ull;
      }
      uint64_t T[W], P[W], K[W], Hm[W];
#pragma unroll
      for (int w = 0; w < W; ++w) {
        T[w] = __shfl_sync(FULL, tw, w);
        P[w] = __shfl_sync(FULL, pw, w);
        Hm[w] = 0;
      }
      const bool measured = t >= a.warmup;
      if (measured) {
        // begin_step (cache.py:102-104): unpin the previous step's keys
        MOEB_FOR_EACH_BIT(W, Pm, ex, {
          const int sl = slot_of[cur * E + ex];
          __syncwarp();
          if ((sl & 31) == lane) {
            const uint64_t v = vals[sl] & ~kPin;
            vals[sl] = v;
            if (v < mv) {
              mv = v;
              ms = sl;
            }
          }
        })
#pragma unroll
        for (int w = 0; w < W; ++w) Pm[w] = 0;
        npins = 0;
      }
      focus(l);
      int npk = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        K[w] = measured ? P[w] : 0ull;
        npk += __popcll(K[w]);
      }
      if (limit <= 0) {
#pragma unroll
        for (int w = 0; w < W; ++w) K[w] = 0;
      } else if (npk > limit) {
        keep_lowest<W>(K, limit);
      }
      // prefetch(sorted(pred)[:limit]) (cache.py:126-154)
      MOEB_FOR_EACH_BIT(W, K, ex, {
        const int key = l * E + ex;
        const uint64_t bit = 1ull << (ex & 63);
        __syncwarp();
        if (word_get<W>(Rl, ex >> 6) & bit) {
          const int sl = slot_of[key];
          const uint64_t v = vals[sl];
          __syncwarp();
          update(sl, kPin | (v & 0x7FFFFFFF00000000ull) | clock++);
          if (!(v & kPin)) {
            word_or<W>(Pm, ex >> 6, bit);
            ++npins;
          }
        } else if (!(count >= cap && count <= npins)) {
          const int sl = make_room();
          __syncwarp();
          place(sl, kPin | clock++, key, ex);
          word_or<W>(Rl, ex >> 6, bit);
          word_or<W>(Pm, ex >> 6, bit);
          ++npins;
        }
      })
      // touch every truth expert ascending (cache.py:106-124)
      int ch = 0;
      MOEB_FOR_EACH_BIT(W, T, ex, {
        const int key = l * E + ex;
        const uint64_t bit = 1ull << (ex & 63);
        __syncwarp();
        if (word_get<W>(Rl, ex >> 6) & bit) {
          const int sl = slot_of[key];
          const uint64_t v = vals[sl];
          __syncwarp();
          const uint64_t freq = ((v & ~kPin) >> 32) + 1;
          update(sl, (v & kPin) | (freq << 32) | clock++);
          ++ch;
          word_or<W>(Hm, ex >> 6, bit);
        } else if (!(count >= cap && count <= npins)) {
          const int sl = make_room();
          __syncwarp();
          place(sl, (1ull << 32) | clock++, key, ex);
          word_or<W>(Rl, ex >> 6, bit);
        }
      })
      if (EXTRA && hits && lane < W) {
        uint64_t v = 0;
#pragma unroll
        for (int w = 0; w < W; ++w)
          if (w == lane) v = Hm[w];
        hits[(r0 + i) * W + lane] = v;
      }
      if (measured) {
        const int k = popc_w<W>(T);
        int ph = 0;
#pragma unroll
        for (int w = 0; w < W; ++w) ph += __popcll(T[w] & P[w]);
        if (EXTRA && cov && cov[r0 + i] == 0) ++tot_unc;
        tot_k += k;
        tot_ch += ch;
        tot_ph += ph;
        if (lane == 0) {
          atomicAdd(&bcnt[l], (unsigned)k);
          atomicAdd(&bcnt[L + l], (unsigned)ch);
          atomicAdd(&bcnt[2 * L + l], (unsigned)ph);
        }
      }
      if (++l == L) {
        l = 0;
        ++t;
      }
    }
    int64_t* c = a.counters + pi * a.counters_stride;
    if (lane == 0) {
      atomicAdd(reinterpret_cast<unsigned long long*>(c + 0), (unsigned long long)tot_k);
      atomicAdd(reinterpret_cast<unsigned long long*>(c + 1), (unsigned long long)tot_ch);
      atomicAdd(reinterpret_cast<unsigned long long*>(c + 2), (unsigned long long)tot_ph);
      if (tot_unc) atomicAdd(reinterpret_cast<unsigned long long*>(c + 3), (unsigned long long)tot_unc);
      if (a.per_prompt) {
        int64_t* pp = a.per_prompt + pi * a.per_prompt_stride + 4 * (int64_t)p;
        pp[0] += tot_k;
        pp[1] += tot_ch;
        pp[2] += tot_ph;
        pp[3] += tot_unc;
      }
    }
  }
  __syncthreads();
  int64_t* c = a.counters + pi * a.counters_stride;
  for (int j = threadIdx.x; j < 3 * L; j += blockDim.x)
    if (bcnt[j]) atomicAdd(reinterpret_cast<unsigned long long*>(c + 4 + j), (unsigned long long)bcnt[j]);
}

template <int W>
int launch_lfu_warp(SimArgs a, cudaStream_t s) {
  const int max_block = moeb::max_smem_per_block();
  const int head = align16(4LL * 3 * a.L);
  a.off_c = head;
  int nw = 4;
  while (nw > 1 && head + (int64_t)nw * a.sim_bytes > max_block) --nw;
  if (head + (int64_t)nw * a.sim_bytes > max_block)
    return moeb::fail(MOEB_ESMEM, "cache state %d B/sim exceeds %d B of shared memory",
                      a.sim_bytes, max_block);
  {  // the block size that keeps the most simulations resident per SM
    const int64_t sm = moeb::max_smem_per_sm();
    int best = nw, best_sims = 0;
    for (int w = nw; w >= 1; --w) {
      const int64_t blocks =
          std::min<int64_t>(sm / (head + (int64_t)w * a.sim_bytes + 1024), 64 / w);
      if (blocks * w > best_sims) {
        best_sims = (int)(blocks * w);
        best = w;
      }
    }
    nw = best;
  }
  const size_t smem = head + (size_t)nw * a.sim_bytes;
  auto k = (a.hits || a.any_cov) ? k_cache_sim_lfu_warp<W, true> : k_cache_sim_lfu_warp<W, false>;
  moeb::set_smem(k, (int)smem);
  const dim3 blocks((unsigned)((a.P + nw - 1) / nw), (unsigned)a.n_preds);
  k<<<blocks, 32 * nw, smem, s>>>(a);
  return moeb::check_launch("k_cache_sim_lfu_warp");
}

template <class K>
int launch_kernel(K k, const SimArgs& a, int tpb, size_t smem, cudaStream_t s) {
  moeb::set_smem(k, (int)smem);
  const dim3 blocks((unsigned)((a.P + tpb - 1) / tpb), (unsigned)a.n_preds);
  k<<<blocks, tpb, smem, s>>>(a);
  return moeb::check_launch("k_cache_sim");
}


// ---------------------------------------------------------------------------
// K1s -- stack-distance replay (E <= 64, LRU, no coverage / hit-mask /
// per-prompt outputs). When no pin can bind (capacity C > every row's
// distinct-key count, so the LRU victim is never a key prefetched in the
// same row and nothing is rejected) the reference's cache is a pure LRU over
// the access sequence (row order; in a row: sorted(pred)[:limit], then the
// truth keys ascending), and a touch of key x hits iff fewer than C distinct
// other keys were accessed since x's previous access (Mattson's stack
// distance). Keys of different layers are distinct and every row is one
// layer, so with S_q the row key sets and n_q = |S_q|:
//  * x prefetched in the same row: hit;
//  * x in S_{r-L} (previous token): D = sum of n over rows r-L+1..r-1 (prefix
//    sums) + |after(x in row r-L) | before(x in row r)| -- O(1);
//  * otherwise D >= sum of n over rows r-L..r-1; if that is >= C: miss;
//    else x's previous access is searched up to dmax tokens back and D is
//    the exact per-layer union over the span; beyond that the prompt is
//    undecided and goes to the exact kernel (plist).
// One warp per prompt, 32 rows per step (lane = row), the last H rows' masks
// and prefix sums in a shared-memory ring. Cache-hit counters only (the
// cache-independent ones come from a.given). Undecided prompts contribute
// nothing here and are replayed by k_cache_sim_warp over plist.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t above_bits(int x) { return x >= 63 ? 0ull : ~((2ull << x) - 1ull); }
__device__ __forceinline__ uint64_t below_bits(int x) { return (1ull << x) - 1ull; }
// keys of row (k, t) accessed after x's last access in that row
__device__ __forceinline__ uint64_t after_last(uint64_t k, uint64_t t, int x) {
  return ((t >> x) & 1ull) ? (t & above_bits(x)) : ((k & above_bits(x)) | t);
}

template <bool KPH>  // KPH: also the cache-independent counters (else a.given is added)
// (128, 10): at most 48 registers, so ten blocks (40 warps) fit an SM -- the
// shared-memory limit -- and C2's 6,994 prompt warps take 1.2 resident rounds
// instead of 1.5 (step 5.14 -> 5.04 ms, profiles/r02_k1s_launch_bounds_ab.log)
__global__ void __launch_bounds__(128, 10) k_stack_replay(const SimArgs a, int H, int dmax,
                                                      int32_t* plist, int32_t* plist_n) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr unsigned FULL = 0xffffffffu;
  const int L = a.L;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const size_t lb = (size_t)((12 * L + 15) / 16) * 16;
  unsigned int* bch = reinterpret_cast<unsigned int*>(smem);  // [3L] block: k, ch, ph per layer
  unsigned char* wbase = smem + lb + (size_t)wib * ((size_t)H * 20 + lb);
  uint64_t* rK = reinterpret_cast<uint64_t*>(wbase);  // [H] prefetched keys of row q
  uint64_t* rT = rK + H;                               // [H] touched keys
  uint32_t* rP = reinterpret_cast<uint32_t*>(rT + H);  // [H] inclusive prefix of n (mod 2^32)
  unsigned int* wch = reinterpret_cast<unsigned int*>(rP + H);  // [3L] this prompt's k, ch, ph
  for (int j = threadIdx.x; j < 3 * L; j += blockDim.x) bch[j] = 0;
  for (int j = lane; j < 3 * L; j += 32) wch[j] = 0;
  __syncthreads();
  const int pi = blockIdx.y;
  const int p = blockIdx.x * (blockDim.x >> 5) + wib;
  const uint32_t cap = (uint32_t)a.cap;
  const int hm = H - 1;
  if (p < a.P) {
    const uint64_t* __restrict__ pred = a.preds[pi];
    const bool unbounded = (a.unbounded_bits >> pi) & 1u;
    const int limit = unbounded ? a.E : a.budget;
    const int64_t r0 = a.row_off[p];
    const int nrows = (int)(a.row_off[p + 1] - r0);
    const uint64_t* __restrict__ tr = a.truth + r0;
    const uint64_t* __restrict__ pr = pred ? pred + r0 : nullptr;
    bool undecided = false;
    int unions = 0;  // span-union evaluations by this lane (bounded: see below)
    uint32_t carry = 0;
    long long tot = 0, tk = 0, tph = 0;
    auto pn = [&](int q) -> uint32_t { return q < 0 ? 0u : rP[q & hm]; };
    for (int base = 0; base < nrows; base += 32) {
      const int i = base + lane;
      const bool in = i < nrows;
      const uint64_t T = in ? __ldg(tr + i) : 0ull;
      const uint64_t Pf = (in && pr) ? __ldg(pr + i) : 0ull;  // full predicted set
      uint64_t K = Pf;
      const int t = i / L, l = i - t * L;
      const bool measured = in && t >= a.warmup;
      if (!measured) K = 0ull;
      if (__popcll(K) > limit) {
        uint64_t k1[1] = {K};
        keep_lowest<1>(k1, limit);
        K = k1[0];
      }
      const uint32_t n = (uint32_t)__popcll(K | T);
      if (in && n >= cap) undecided = true;  // a pin could bind: exact kernel
      uint32_t v = n;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, v, o);
        if (lane >= o) v += y;
      }
      const uint32_t pfx = carry + v;
      carry = __shfl_sync(FULL, pfx, 31);
      rK[i & hm] = K;
      rT[i & hm] = T;
      rP[i & hm] = pfx;
      __syncwarp();
      if (measured) {
        int ch = __popcll(T & K);  // prefetched in this row, then touched: hits
        // every other touch misses when even the L-1 rows since the previous
        // token of this layer hold >= C keys (D >= that sum for d = 1 and for
        // d >= 2), or when there is no previous token: skip the per-key work
        uint64_t tm = (i < L || pn(i - 1) - pn(i - L) >= cap) ? 0ull : (T & ~K);
        while (tm) {
          const int x = __ffsll((long long)tm) - 1;
          tm &= tm - 1;
          const uint64_t before = K | (T & below_bits(x));
          bool hit = false;
          const int q1 = i - L;
          if (q1 >= 0 && (((rK[q1 & hm] | rT[q1 & hm]) >> x) & 1ull)) {
            const uint32_t D = (pn(i - 1) - pn(i - L)) +
                               (uint32_t)__popcll(after_last(rK[q1 & hm], rT[q1 & hm], x) | before);
            hit = D < cap;
          } else if (i - 2 * L >= 0 && pn(i - 1) - pn(i - L - 1) < cap) {
            // the full previous token (distinct layers) does not decide it
            int jf = 0;
            bool none = false;
            for (int j = 2; j <= dmax; ++j) {
              const int q = i - j * L;
              if (q < 0) {
                none = true;  // no earlier access of x at all: miss
                break;
              }
              if (((rK[q & hm] | rT[q & hm]) >> x) & 1ull) {
                jf = j;
                break;
              }
            }
            // a prompt that keeps needing span unions (large capacities) is
            // cheaper in the exact kernel: give up on it after a few
            if (!none && ++unions > 8) {
              undecided = true;
              none = true;
            }
            if (!none) {
              const int j = jf ? jf : dmax;  // exact union over the span (a lower bound if !jf)
              uint32_t D = 0;
              for (int o = 1; o < L && D < cap; ++o) {
                uint64_t u = 0;
                for (int q = i - j * L + o; q < i; q += L) u |= rK[q & hm] | rT[q & hm];
                D += (uint32_t)__popcll(u);
              }
              uint64_t u = before;
              for (int m = 1; m < j; ++m) u |= rK[(i - m * L) & hm] | rT[(i - m * L) & hm];
              if (jf) u |= after_last(rK[(i - j * L) & hm], rT[(i - j * L) & hm], x);
              D += (uint32_t)__popcll(u);
              if (jf) {
                hit = D < cap;
              } else if (D < cap) {
                if (i - (dmax + 1) * L >= 0) undecided = true;  // x may be older than dmax tokens
              }
            }
          }
          ch += hit ? 1 : 0;
        }
        if (ch) atomicAdd(&wch[L + l], (unsigned)ch);
        tot += ch;
        if (KPH) {
          const int kk = __popcll(T), ph = __popcll(T & Pf);
          if (kk) atomicAdd(&wch[l], (unsigned)kk);
          if (ph) atomicAdd(&wch[2 * L + l], (unsigned)ph);
          tk += kk;
          tph += ph;
        }
      }
      // an undecided prompt goes to the exact kernel anyway: stop here
      if (__any_sync(FULL, undecided)) break;
      __syncwarp();
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      tot += __shfl_xor_sync(FULL, tot, o);
      if (KPH) {
        tk += __shfl_xor_sync(FULL, tk, o);
        tph += __shfl_xor_sync(FULL, tph, o);
      }
    }
    if (__any_sync(FULL, undecided)) {
      if (lane == 0) {
        const int k = atomicAdd(plist_n + pi, 1);
        plist[(int64_t)pi * a.P + k] = p;
      }
    } else {
      for (int j = lane; j < 3 * L; j += 32)
        if (wch[j]) atomicAdd(&bch[j], wch[j]);
      if (lane == 0) {
        int64_t* c = a.counters + pi * a.counters_stride;
        if (KPH && tk) atomicAdd(reinterpret_cast<unsigned long long*>(c + 0), (unsigned long long)tk);
        if (tot) atomicAdd(reinterpret_cast<unsigned long long*>(c + 1), (unsigned long long)tot);
        if (KPH && tph) atomicAdd(reinterpret_cast<unsigned long long*>(c + 2), (unsigned long long)tph);
        if (a.per_prompt) {
          int64_t* pp = a.per_prompt + pi * a.per_prompt_stride + 4 * (int64_t)p;
          pp[0] += tk;
          pp[1] += tot;
          pp[2] += tph;
        }
      }
    }
  }
  __syncthreads();
  int64_t* c = a.counters + pi * a.counters_stride;
  for (int j = threadIdx.x; j < 3 * L; j += blockDim.x)
    if (bch[j]) atomicAdd(reinterpret_cast<unsigned long long*>(c + 4 + j), (unsigned long long)bch[j]);
  if (!KPH && a.given && blockIdx.x == 0) {  // the upstream counts, once per prediction stream
    const int64_t* g = a.given + (int64_t)pi * (2 + 2 * L);
    for (int j = threadIdx.x; j < 2 + 2 * L; j += blockDim.x) {
      const int idx = j == 0 ? 0 : j == 1 ? 2 : j < 2 + L ? 4 + (j - 2) : 4 + 2 * L + (j - 2 - L);
      if (g[j]) atomicAdd(reinterpret_cast<unsigned long long*>(c + idx), (unsigned long long)g[j]);
    }
  }
}

// MOEB_K1_STACK=0 disables the stack-distance replay (every prompt through
// the exact kernel)
inline bool stack_mode() {
  const char* env = getenv("MOEB_K1_STACK");
  return !(env && env[0] == '0');
}

template <int W, int ES, int G>
int launch_lru_g(SimArgs a, cudaStream_t s, int head, int max_block);

// LRU: warp-per-simulation kernel; E = 64 / 256 get shift-based key math.
template <int W, int ES>
int launch_lru(SimArgs a, cudaStream_t s) {
  const int max_block = moeb::max_smem_per_block();
  const int head = align16(4LL * 3 * a.L);
  a.off_c = head;
  // Two simulations per warp (16 lanes each) unless the state is so large
  // that only one or two simulations fit a block. MOEB_K1_G (tuning knob):
  // lanes per simulation, 8 / 16 / 32.
  const char* env = getenv("MOEB_K1_G");
  const int g = env ? atoi(env) : 16;
  if (g == 8) return launch_lru_g<W, ES, 8>(a, s, head, max_block);
  if (g == 32) return launch_lru_g<W, ES, 32>(a, s, head, max_block);
  return launch_lru_g<W, ES, 16>(a, s, head, max_block);
}

template <int W, int ES, int G>
int launch_lru_g(SimArgs a, cudaStream_t s, int head, int max_block) {
  int nw = 4;  // warps per block
  while (nw > 1 && head + (int64_t)nw * (32 / G) * a.sim_bytes > max_block) --nw;
  {
    // small states (the key-position table in global memory): the block size
    // that keeps the most simulations resident per SM (blocks of 4 warps
    // would strand up to a block's worth of shared memory)
    const int64_t sm = moeb::max_smem_per_sm();
    int best = nw, best_sims = 0;
    for (int w = nw; w >= 1; --w) {
      const int64_t per_block = head + (int64_t)w * (32 / G) * a.sim_bytes + 1024;
      const int64_t blocks = std::min<int64_t>(sm / per_block, 64 / w);
      if (blocks * w * (32 / G) > best_sims) {
        best_sims = (int)(blocks * w * (32 / G));
        best = w;
      }
    }
    nw = best;
  }
  if (head + (int64_t)nw * (32 / G) * a.sim_bytes > max_block) {
    if (head + (int64_t)a.sim_bytes > max_block)
      return moeb::fail(MOEB_ESMEM, "cache state %d B/sim exceeds %d B of shared memory",
                        a.sim_bytes, max_block);
    const size_t smem1 = head + (size_t)a.sim_bytes;
    auto k1 = (a.hits || a.any_cov) ? k_cache_sim_warp<W, ES, 32, true>
                                    : k_cache_sim_warp<W, ES, 32, false>;
    moeb::set_smem(k1, (int)smem1);
    k1<<<dim3((unsigned)a.P, (unsigned)a.n_preds), 32, smem1, s>>>(a);
    return moeb::check_launch("k_cache_sim_warp");
  }
  const size_t smem = head + (size_t)nw * (32 / G) * a.sim_bytes;
  // K1s pays off when rows carry predictions: without them (lru_only) a row
  // is just the top-k truth keys, one token's keys (L * k) can stay below
  // the capacity, and too many touches need the span unions; the exact
  // kernel is cheap for those rows anyway.
  bool all_pred = true;
  for (int i = 0; i < a.n_preds; ++i) all_pred = all_pred && a.preds[i] != nullptr;
  if (W == 1 && G == 16 && !a.hits && !a.any_cov && all_pred && stack_mode()) {
    // K1s over every prompt, then the exact kernel over the undecided ones
    const int dmax = 4;
    int H = 64;
    while (H < (dmax + 1) * a.L + 64) H <<= 1;
    const size_t lbytes = (size_t)((12 * a.L + 15) / 16) * 16;
    const size_t ssmem = lbytes + 4 * ((size_t)H * 20 + lbytes);
    // the undecided-prompt list lives in the caller's workspace
    // (moeb_cache_sim_workspace_bytes); without one every prompt takes the
    // exact kernel below
    const size_t plbytes = sizeof(int32_t) * ((size_t)a.n_preds * a.P + a.n_preds);
    if ((int)ssmem <= max_block && a.ws && a.ws_bytes >= plbytes) {
      int32_t* pl = reinterpret_cast<int32_t*>(a.ws);
      int32_t* pln = pl + (size_t)a.n_preds * a.P;
      if (cudaMemsetAsync(pln, 0, sizeof(int32_t) * a.n_preds, s) != cudaSuccess)
        return moeb::fail(MOEB_ECUDA, "clearing the undecided-prompt count");
      // with upstream counts (and no per-prompt output) neither kernel computes them
      const bool given = a.given && !a.per_prompt;
      auto ks = given ? k_stack_replay<false> : k_stack_replay<true>;
      moeb::set_smem(ks, (int)ssmem);
      ks<<<dim3((unsigned)((a.P + 3) / 4), (unsigned)a.n_preds), 128, ssmem, s>>>(
          a, H, dmax, pl, pln);
      int rc = moeb::check_launch("k_stack_replay");
      if (rc == 0) {
        SimArgs b = a;
        b.given = nullptr;  // added by k_stack_replay
        b.plist = pl;
        b.plist_n = pln;
        auto k = given ? k_cache_sim_warp<W, ES, G, false, false> : k_cache_sim_warp<W, ES, G, false>;
        moeb::set_smem(k, (int)smem);
        const int spb = nw * (32 / G);
        k<<<dim3((unsigned)((a.P + spb - 1) / spb), (unsigned)a.n_preds), 32 * nw, smem, s>>>(b);
        rc = moeb::check_launch("k_cache_sim_warp");
      }
      return rc;
    }
  }
  auto k = (a.hits || a.any_cov) ? k_cache_sim_warp<W, ES, G, true>
           : (a.given && !a.per_prompt) ? k_cache_sim_warp<W, ES, G, false, false>
                                        : k_cache_sim_warp<W, ES, G, false>;
  moeb::set_smem(k, (int)smem);
  const int spb = nw * (32 / G);
  const dim3 blocks((unsigned)((a.P + spb - 1) / spb), (unsigned)a.n_preds);
  k<<<blocks, 32 * nw, smem, s>>>(a);
  return moeb::check_launch("k_cache_sim_warp");
}

template <int W>
int launch_sim(SimArgs a, int policy, cudaStream_t s) {
  const int max_block = moeb::max_smem_per_block();
  if (policy == MOEB_POLICY_LFU && a.pos_g) {
    const char* env = getenv("MOEB_LFU_KERNEL");
    if (env && env[0] == 't') {  // the thread-per-simulation kernel keeps its tables in shared memory
      a.pos_g = nullptr;
      layout(a, policy, false);
    }
  }
  const int head = align16(4LL * 3 * a.L);  // block counters
  a.off_c = head;
  if (a.magic == 0) return moeb::fail(MOEB_EINVAL, "layer magic failed for E=%d", a.E);
  // One lockstep warp of simulations per block (fewer if the state is large).
  int tpb = 32;
  while (tpb > 1 && head + (int64_t)tpb * a.sim_bytes > max_block) --tpb;
  if (head + (int64_t)tpb * a.sim_bytes > max_block)
    return moeb::fail(MOEB_ESMEM, "cache state %d B/sim exceeds %d B of shared memory",
                      a.sim_bytes, max_block);
  const size_t smem = head + (size_t)tpb * a.sim_bytes;
  if (policy == MOEB_POLICY_LFU) {
    const char* env = getenv("MOEB_LFU_KERNEL");  // "thread": the thread-per-simulation kernel
    if (!(env && env[0] == 't')) return launch_lfu_warp<W>(a, s);
    return launch_kernel(k_cache_sim<W, LfuState<W, false>>, a, tpb, smem, s);
  }
  if (W == 1 && a.E == 64) return launch_lru<1, 6>(a, s);
  if (W == 4 && a.E == 256) return launch_lru<4, 8>(a, s);
  return launch_lru<W, -1>(a, s);
}

}  // namespace

extern "C" size_t moeb_cache_sim_workspace_bytes(int n_preds, int n_prompts) {
  if (n_preds < 1 || n_prompts < 1) return 0;
  return sizeof(int32_t) * ((size_t)n_preds * n_prompts + n_preds);
}

namespace {
// keys above which the LRU key-position table goes to global memory: its
// 2 B per key would otherwise leave fewer than ~8 simulations per SM
constexpr int kGlobalPosKeys = 8192;
size_t list_bytes_aligned(int n_preds, int n_prompts) {
  return (moeb_cache_sim_workspace_bytes(n_preds, n_prompts) + 255) / 256 * 256;
}
size_t pos_table_bytes(int n_preds, int n_prompts, int L, int E) {
  if ((int64_t)L * E <= kGlobalPosKeys) return 0;
  return sizeof(uint16_t) * (size_t)n_preds * n_prompts * (size_t)L * E;
}
}  // namespace

extern "C" size_t moeb_cache_sim_workspace_bytes_shape(int n_preds, int n_prompts, int L, int E) {
  if (n_preds < 1 || n_prompts < 1 || L < 1 || E < 1) return 0;
  return list_bytes_aligned(n_preds, n_prompts) + pos_table_bytes(n_preds, n_prompts, L, E);
}

extern "C" int moeb_cache_sim(const uint64_t* truth, const uint64_t* const* preds,
                              const uint8_t* const* covered, const int32_t* unbounded,
                              int n_preds, const int64_t* prompt_row_off, int n_prompts, int L,
                              int E, int warmup_tokens, const int64_t* capacities, int n_caps,
                              int budget, int policy, int64_t* counters, int64_t* per_prompt,
                              uint64_t* hit_masks, int64_t rows, void* workspace,
                              size_t workspace_bytes, void* stream) {
  return moeb_cache_sim_counted(truth, preds, covered, unbounded, n_preds, prompt_row_off,
                                n_prompts, L, E, warmup_tokens, capacities, n_caps, budget,
                                policy, counters, per_prompt, hit_masks, nullptr, rows,
                                workspace, workspace_bytes, stream);
}

extern "C" int moeb_cache_sim_counted(const uint64_t* truth, const uint64_t* const* preds,
                                      const uint8_t* const* covered, const int32_t* unbounded,
                                      int n_preds, const int64_t* prompt_row_off, int n_prompts,
                                      int L, int E, int warmup_tokens, const int64_t* capacities,
                                      int n_caps, int budget, int policy, int64_t* counters,
                                      int64_t* per_prompt, uint64_t* hit_masks,
                                      const int64_t* given_counts, int64_t rows, void* workspace,
                                      size_t workspace_bytes, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(truth && prompt_row_off && counters && capacities, "null argument");
  MOEB_REQUIRE(n_preds >= 1 && n_preds <= MOEB_MAX_PREDS, "n_preds must be in [1, %d]",
               MOEB_MAX_PREDS);
  MOEB_REQUIRE(n_prompts >= 1 && L >= 1 && E >= 1 && E <= 256 && L <= 255 && L * E <= 65536,
               "unsupported shape L=%d E=%d", L, E);
  MOEB_REQUIRE(warmup_tokens >= 0 && budget >= 1, "bad warmup/budget");
  MOEB_REQUIRE(policy == MOEB_POLICY_LRU || policy == MOEB_POLICY_LFU, "unknown policy %d",
               policy);
  MOEB_REQUIRE(rows >= 0, "rows must be >= 0");
  const int W = moeb::words_for(E);
  SimArgs a{};
  a.truth = truth;
  a.n_preds = n_preds;
  for (int i = 0; i < n_preds; ++i) {
    a.preds[i] = preds ? preds[i] : nullptr;
    a.covered[i] = covered ? covered[i] : nullptr;
    if (a.covered[i]) a.any_cov = 1;
    if (unbounded && unbounded[i]) a.unbounded_bits |= 1u << i;
  }
  a.row_off = prompt_row_off;
  a.P = n_prompts;
  a.L = L;
  a.E = E;
  a.warmup = warmup_tokens;
  a.budget = budget;
  a.rows = rows;
  a.given = given_counts;
  a.ws = workspace;
  a.ws_bytes = workspace ? workspace_bytes : 0;
  {
    const size_t tb = pos_table_bytes(n_preds, n_prompts, L, E);
    const size_t lb = list_bytes_aligned(n_preds, n_prompts);
    const char* env = getenv("MOEB_K1_POS");  // "smem": keep the table in shared memory
    if (tb && a.ws_bytes >= lb + tb && !(env && env[0] == 's'))
      a.pos_g = reinterpret_cast<uint16_t*>(static_cast<unsigned char*>(workspace) + lb);
  }
  const int nc = 4 + 3 * L;
  cudaStream_t s = moeb::as_stream(stream);
  for (int c = 0; c < n_caps; ++c) {
    MOEB_REQUIRE(capacities[c] >= 1 && capacities[c] <= (int64_t)L * E,
                 "capacity %lld out of range [1, %d]", (long long)capacities[c], L * E);
    a.cap = capacities[c];
    a.counters = counters + (int64_t)c * nc;
    a.counters_stride = (int64_t)n_caps * nc;
    a.per_prompt = per_prompt ? per_prompt + (int64_t)c * n_prompts * 4 : nullptr;
    a.per_prompt_stride = (int64_t)n_caps * n_prompts * 4;
    a.hits = hit_masks ? hit_masks + (int64_t)c * rows * W : nullptr;
    a.hits_stride = (int64_t)n_caps * rows * W;
    layout(a, policy, false);
    int rc = W == 1 ? launch_sim<1>(a, policy, s)
             : W == 2 ? launch_sim<2>(a, policy, s)
             : W == 3 ? launch_sim<3>(a, policy, s)
                      : launch_sim<4>(a, policy, s);
    if (rc) return rc;
  }
  return MOEB_OK;
}

template <int W>
static int launch_ops(SimArgs& a, int policy, const int32_t* ops, const int32_t* keys, int64_t n,
                      uint8_t* results, cudaStream_t s) {
  layout(a, policy, true);
  const size_t smem = a.sim_bytes;
  if ((int)smem > moeb::max_smem_per_block())
    return moeb::fail(MOEB_ESMEM, "cache state %zu B exceeds shared memory", smem);
  if (policy == MOEB_POLICY_LRU) {
    auto k = k_cache_ops<W, LruState<W, -1, true>>;
    moeb::set_smem(k, (int)smem);
    k<<<1, 32, smem, s>>>(a, ops, keys, n, results);
  } else {
    auto k = k_cache_ops<W, LfuState<W, true>>;
    moeb::set_smem(k, (int)smem);
    k<<<1, 32, smem, s>>>(a, ops, keys, n, results);
  }
  return moeb::check_launch("k_cache_ops");
}

extern "C" int moeb_cache_ops(const int32_t* ops, const int32_t* keys, int64_t n, int L, int E,
                              int64_t capacity, int policy, uint8_t* results, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(ops && keys && results, "null argument");
  MOEB_REQUIRE(L >= 1 && E >= 1 && E <= 256 && L <= 255 && L * E <= 65536,
               "unsupported shape L=%d E=%d", L, E);
  MOEB_REQUIRE(capacity >= 1 && capacity <= (int64_t)L * E, "capacity out of range");
  MOEB_REQUIRE(policy == MOEB_POLICY_LRU || policy == MOEB_POLICY_LFU, "unknown policy");
  SimArgs a{};
  a.L = L;
  a.E = E;
  a.cap = capacity;
  const int W = moeb::words_for(E);
  cudaStream_t s = moeb::as_stream(stream);
  return W == 1 ? launch_ops<1>(a, policy, ops, keys, n, results, s)
         : W == 2 ? launch_ops<2>(a, policy, ops, keys, n, results, s)
         : W == 3 ? launch_ops<3>(a, policy, ops, keys, n, results, s)
                  : launch_ops<4>(a, policy, ops, keys, n, results, s);
}

// ---------------------------------------------------------------------------
// K1m: exact multi-capacity LRU replay by stack distances (E <= 64).
//
// When every capacity C exceeds the number of keys prefetched in any row,
// no pin can bind and nothing is rejected (cache.py:93-154), so the cache is
// a pure LRU over each prompt's access sequence -- per row, sorted(pred)[:
// budget] then the truth keys ascending (engine.py:172-184) -- and a touch of
// key x hits iff it was prefetched in the same row or fewer than C distinct
// keys were accessed since its previous access (Mattson's stack distance D).
// D does not depend on C, so one pass decides every capacity at once.
//
// One warp per (prompt, prediction stream), state in shared memory:
//   lr[L][64]   last access of each key: (row << 7) | pos, pos = expert id +
//               64 if it was a truth key there (the row's access order)
//   cnt[row]    number of keys whose last access is that row (u8), with
//               32-row block sums blk[] and 1024-row super sums sup[]
// For a touch of x (not prefetched in this row) whose last access is at
// row rx (same layer) and position px:
//   D = #{keys, last access row > rx}            (cnt suffix: blocked sum)
//     + #{layer-l keys, last access row == rx, position > px}
//     + #{keys accessed in this row before x not counted above}
// then the row's keys move to this row in the structure.
// ---------------------------------------------------------------------------
namespace {

constexpr int kMaxMultiCaps = 16;
constexpr uint32_t kNever = 0xffffffffu;

struct MultiArgs {
  const uint64_t* truth;
  const uint64_t* preds[MOEB_MAX_PREDS];
  uint32_t unbounded_bits;
  const int64_t* row_off;
  int P, L, E, warmup, budget, n_caps;
  int64_t caps[kMaxMultiCaps];
  int rmax;                 // max rows of one prompt (shared-memory sizing)
  int off_cnt, off_blk, off_sup, off_ctr, warp_bytes;
  int64_t* counters;        // [n_preds][n_caps][4 + 3L]
  int64_t* per_prompt;      // nullable [n_preds][n_caps][P][4]
  uint32_t* lr_g;           // nullable: lr tables [n_preds][P][L * 64] in global memory
};

// NIB: per-row counts as 4-bit fields (rows touch at most 15 keys: budget +
// top-k <= 15, no unbounded stream), half the shared memory of u8 counts
template <bool NIB>
__global__ void __launch_bounds__(128) k_stack_multi(const MultiArgs a) {
  extern __shared__ __align__(16) unsigned char smem_m[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int si = blockIdx.y;
  unsigned char* base = smem_m + (size_t)warp * a.warp_bytes;
  uint32_t* lr = reinterpret_cast<uint32_t*>(base);  // or per prompt in global memory
  uint32_t* cnt32 = reinterpret_cast<uint32_t*>(base + a.off_cnt);
  uint32_t* blk32 = reinterpret_cast<uint32_t*>(base + a.off_blk);  // u16 block sums
  const uint16_t* blk = reinterpret_cast<const uint16_t*>(blk32);
  uint32_t* sup = reinterpret_cast<uint32_t*>(base + a.off_sup);
  uint32_t* ctr = reinterpret_cast<uint32_t*>(base + a.off_ctr);  // flushed as int64
  const int L = a.L, C = a.n_caps;
  // ctr: [0, L) accesses, [L, 2L) prediction hits, then per layer a
  // histogram over h = the number of capacities <= D ([2L + l (C+1) + h));
  // touches with D below every capacity (and prefetched ones) land in h = 0.
  // A capacity c hits exactly the touches with h <= c. Per prompt the same
  // histogram (last C + 1 entries) gives the per-prompt counters.
  const int nctr = 2 * L + L * (C + 1);
  uint32_t* pph = ctr + nctr;
  for (int i = lane; i < nctr; i += 32) ctr[i] = 0u;
  // hlut[D] = #capacities <= D (block-shared, D in [0, L * 64])
  unsigned char* hlut = smem_m + (size_t)(blockDim.x >> 5) * a.warp_bytes;
  for (int d = threadIdx.x; d <= L * 64; d += blockDim.x) {
    int h = 0;
    for (int c = 0; c < C; ++c) h += a.caps[c] <= d;
    hlut[d] = (unsigned char)h;
  }
  __syncthreads();
  const uint64_t* pred = a.preds[si];
  const bool unbounded = (a.unbounded_bits >> si) & 1u;
  const uint64_t emask = a.E >= 64 ? ~0ull : ((1ull << a.E) - 1ull);
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  for (int p = blockIdx.x * (blockDim.x >> 5) + warp; p < a.P; p += nwarps) {
    const int64_t r0 = a.row_off[p];
    const int R = (int)(a.row_off[p + 1] - r0);
    const int nblk = (R + 31) >> 5, nsup = (R + 1023) >> 10;
    if (a.lr_g) lr = a.lr_g + ((int64_t)si * a.P + p) * (L * 64);
    for (int i = lane; i < L * 64; i += 32) lr[i] = kNever;
    // zeroed over whole 32-row blocks / 1024-row super blocks: the suffix
    // sums read those spans without bounds tests
    for (int i = lane; i < nblk * (NIB ? 4 : 8); i += 32) cnt32[i] = 0u;
    for (int i = lane; i < nsup * 16; i += 32) blk32[i] = 0u;
    for (int i = lane; i < nsup; i += 32) sup[i] = 0u;
    for (int i = lane; i <= C; i += 32) pph[i] = 0u;
    __syncwarp();
    const unsigned char* cnt = reinterpret_cast<const unsigned char*>(cnt32);
    int64_t pp_acc = 0, pp_ph = 0;
    // the next row's layer entries, loaded one row ahead (with L > 1 a row
    // never changes another layer's entries; L == 1 reloads after the update)
    uint32_t nv0 = lr[lane], nv1 = lr[32 + lane];
    for (int rb = 0; rb < R; rb += 32) {
      // this batch's rows, one per lane
      const int rl = rb + lane;
      const uint64_t xt = rl < R ? a.truth[r0 + rl] : 0ull;
      const uint64_t xp = (rl < R && pred) ? pred[r0 + rl] : 0ull;
      const int nb = min(32, R - rb);
      for (int i = 0; i < nb; ++i) {
        const int rr = rb + i;
        const int l = rr % L, t = rr / L;
        const uint64_t x = __shfl_sync(0xffffffffu, xt, i) & emask;
        const uint64_t pm = __shfl_sync(0xffffffffu, xp, i) & emask;
        const bool measured = t >= a.warmup;
        // warm-up rows only touch their truth keys (engine.py:160-167): no
        // prediction, no prefetch
        uint64_t K = measured ? pm : 0ull;
        if (!unbounded && measured) {  // sorted(pred)[:budget]: the lowest `budget` ids
          uint64_t rest = pm;
          for (int j = 0; j < a.budget && rest; ++j) rest &= rest - 1;
          K = pm & ~rest;
        }
        const uint64_t A = K | x;
        const uint32_t v0 = nv0, v1 = nv1;
        if (L > 1) {
          const int ln = l + 1 == L ? 0 : l + 1;
          nv0 = lr[ln * 64 + lane];
          nv1 = lr[ln * 64 + 32 + lane];
        }
        // touches not prefetched in this row
        uint64_t miss = x & ~K;
        uint32_t hist0 = (uint32_t)__popcll(x & K);  // h = 0: hit at every capacity
        while (miss) {
          const int e = __ffsll((long long)miss) - 1;
          miss &= miss - 1;
          const uint32_t vx = __shfl_sync(0xffffffffu, e < 32 ? v0 : v1, e & 31);
          int h = C;  // first access: a miss at every capacity
          if (vx != kNever) {
            const int rx = (int)(vx >> 7);
            const uint32_t px = vx & 127u;
            // rows after rx: partial 32-row block, the blocks of its
            // 1024-row super block, the super blocks after it (entries past
            // the current row are still zero)
            const int rho = (rx & ~31) + lane;
            const int b = ((rx >> 10) << 5) + lane;
            const int sidx = (rx >> 10) + 1 + lane;
            uint32_t part = rho > rx ? (NIB ? (cnt32[rho >> 3] >> (4 * (rho & 7))) & 15u
                                            : (uint32_t)cnt[rho])
                                     : 0u;
            part += b > (rx >> 5) ? (uint32_t)blk[b] : 0u;
            part += sidx < nsup ? sup[sidx] : 0u;
            // layer-l keys: counted in the suffix (row > rx) / after x in row rx
            // (never-accessed keys hold 0xffffffff: row field larger than any rx,
            // so they are excluded by the explicit test)
            const uint32_t rx7 = (uint32_t)rx << 7;
            const bool g0 = v0 != kNever && v0 >= rx7 + 128u;
            const bool g1 = v1 != kNever && v1 >= rx7 + 128u;
            const bool f0 = v0 > vx && v0 < rx7 + 128u;
            const bool f1 = v1 > vx && v1 < rx7 + 128u;
            const uint64_t gt = (uint64_t)__ballot_sync(0xffffffffu, g0) |
                                ((uint64_t)__ballot_sync(0xffffffffu, g1) << 32);
            const uint64_t af = (uint64_t)__ballot_sync(0xffffffffu, f0) |
                                ((uint64_t)__ballot_sync(0xffffffffu, f1) << 32);
            const uint64_t xb = 1ull << e;
            const uint64_t before = K | (x & (xb - 1ull));
            const int D = (int)__reduce_add_sync(0xffffffffu, part) + __popcll(af) +
                          __popcll(before & ~(gt | af) & ~xb);
            h = hlut[min(D, a.L * 64)];  // #capacities <= D
          }
          if (h == 0) ++hist0;
          else if (measured && lane == 0) {
            ctr[2 * L + l * (C + 1) + h] += 1u;
            pph[h] += 1u;
          }
        }
        if (measured) {
          const int acc = __popcll(x), ph = __popcll(x & pm);
          if (lane == 0) {
            ctr[l] += (uint32_t)acc;
            ctr[L + l] += (uint32_t)ph;
            ctr[2 * L + l * (C + 1)] += hist0;
            pph[0] += hist0;
          }
          pp_acc += acc;
          pp_ph += ph;
        }
        // the row's keys move to this row: (rr << 7) | position in the row
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int e = lane + 32 * hh;
          if ((A >> e) & 1ull) {
            const uint32_t old = hh ? v1 : v0;
            if (old != kNever) {
              const int ro = (int)(old >> 7);
              if (NIB)
                atomicSub(&cnt32[ro >> 3], 1u << (4 * (ro & 7)));
              else
                atomicSub(&cnt32[ro >> 2], 1u << (8 * (ro & 3)));
              atomicSub(&blk32[ro >> 6], 1u << (16 * ((ro >> 5) & 1)));
              atomicSub(&sup[ro >> 10], 1u);
            }
            lr[l * 64 + e] = ((uint32_t)rr << 7) | (uint32_t)(e + (((x >> e) & 1ull) ? 64 : 0));
          }
        }
        if (lane == 0) {
          const uint32_t n = (uint32_t)__popcll(A);
          if (NIB)
            atomicAdd(&cnt32[rr >> 3], n << (4 * (rr & 7)));
          else
            atomicAdd(&cnt32[rr >> 2], n << (8 * (rr & 3)));
          atomicAdd(&blk32[rr >> 6], n << (16 * ((rr >> 5) & 1)));
          atomicAdd(&sup[rr >> 10], n);
        }
        __syncwarp();
        if (L == 1) {
          nv0 = lr[lane];
          nv1 = lr[32 + lane];
        }
      }
    }
    if (a.per_prompt && lane == 0) {
      int64_t cum = 0;
      for (int c = 0; c < C; ++c) {
        cum += (int64_t)pph[c];
        int64_t* o = a.per_prompt + (((int64_t)si * C + c) * a.P + p) * 4;
        o[0] += pp_acc;
        o[1] += cum;
        o[2] += pp_ph;
      }
    }
    __syncwarp();
  }
  // flush this warp's counters (capacity c hits = histogram prefix up to c)
  const int nc = 4 + 3 * L;
  for (int l = lane; l < L; l += 32) {
    const unsigned long long acc = ctr[l], ph = ctr[L + l];  // u32 -> u64
    unsigned long long cum = 0;
    for (int c = 0; c < C; ++c) {
      cum += (unsigned long long)ctr[2 * L + l * (C + 1) + c];
      unsigned long long* o =
          reinterpret_cast<unsigned long long*>(a.counters + ((int64_t)si * C + c) * nc);
      if (acc) {
        atomicAdd(o + 0, acc);
        atomicAdd(o + 4 + l, acc);
      }
      if (ph) {
        atomicAdd(o + 2, ph);
        atomicAdd(o + 4 + 2 * L + l, ph);
      }
      if (cum) {
        atomicAdd(o + 1, cum);
        atomicAdd(o + 4 + L + l, cum);
      }
    }
  }
}

}  // namespace

extern "C" size_t moeb_cache_replay_stack_workspace_bytes(int n_preds, int n_prompts, int L) {
  if (n_preds < 1 || n_prompts < 1 || L < 1) return 0;
  return sizeof(uint32_t) * (size_t)n_preds * n_prompts * (size_t)L * 64;
}

extern "C" int moeb_cache_replay_stack(const uint64_t* truth, const uint64_t* const* preds,
                                       const int32_t* unbounded, int n_preds,
                                       const int64_t* prompt_row_off, int n_prompts, int L, int E,
                                       int warmup_tokens, const int64_t* capacities, int n_caps,
                                       int budget, int64_t max_prompt_rows, int max_row_keys,
                                       int64_t* counters, int64_t* per_prompt, void* workspace,
                                       size_t workspace_bytes, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(truth && prompt_row_off && counters && capacities, "null argument");
  MOEB_REQUIRE(n_preds >= 1 && n_preds <= MOEB_MAX_PREDS, "n_preds must be in [1, %d]",
               MOEB_MAX_PREDS);
  MOEB_REQUIRE(n_prompts >= 1 && L >= 1 && L <= 255 && E >= 1 && E <= 64, "unsupported shape");
  MOEB_REQUIRE(n_caps >= 1 && n_caps <= kMaxMultiCaps, "n_caps must be in [1, %d]",
               kMaxMultiCaps);
  MOEB_REQUIRE(max_prompt_rows >= 0 && max_prompt_rows <= 32768,
               "the stack replay takes prompts of up to 32768 rows");
  MOEB_REQUIRE(warmup_tokens >= 0 && budget >= 1, "bad warmup/budget");
  MultiArgs a{};
  a.truth = truth;
  int kmax = budget;
  for (int i = 0; i < n_preds; ++i) {
    a.preds[i] = preds ? preds[i] : nullptr;
    if (unbounded && unbounded[i]) {
      a.unbounded_bits |= 1u << i;
      kmax = E;
    }
  }
  for (int c = 0; c < n_caps; ++c) {
    // exact only while no pin can bind: C > the keys prefetched in any row
    MOEB_REQUIRE(capacities[c] > kmax && capacities[c] <= (int64_t)L * E,
                 "capacity %lld: the stack replay needs %d < C <= L*E",
                 (long long)capacities[c], kmax);
    MOEB_REQUIRE(c == 0 || capacities[c] >= capacities[c - 1],
                 "the stack replay takes capacities in ascending order");
    a.caps[c] = capacities[c];
  }
  a.row_off = prompt_row_off;
  a.P = n_prompts;
  a.L = L;
  a.E = E;
  a.warmup = warmup_tokens;
  a.budget = budget;
  a.n_caps = n_caps;
  a.rmax = (int)max_prompt_rows;
  const int R = a.rmax + 1;
  const char* env = getenv("MOEB_K1M_LR");  // "smem": keep the lr tables in shared memory
  if (workspace && workspace_bytes >= moeb_cache_replay_stack_workspace_bytes(n_preds, n_prompts, L) &&
      !(env && env[0] == 's'))
    a.lr_g = static_cast<uint32_t*>(workspace);
  a.off_cnt = a.lr_g ? 0 : align16(4LL * L * 64);
  // 4-bit row counts when no row can touch more than 15 keys: opt-in
  // (MOEB_K1M_NIB=1; measured no faster than u8 counts, and a truth row with
  // more than max_row_keys experts would overflow its field)
  const char* nenv = getenv("MOEB_K1M_NIB");
  const bool nib = max_row_keys > 0 && kmax + max_row_keys <= 15 && nenv && nenv[0] == '1';
  a.off_blk = a.off_cnt + align16((R + 31) / 32 * (nib ? 16 : 32));
  a.off_sup = a.off_blk + align16(2LL * 32 * ((R + 1023) / 1024));
  a.off_ctr = a.off_sup + align16(4LL * ((R + 1023) / 1024 + 1));
  a.warp_bytes = a.off_ctr + align16(4LL * (2 * L + L * (n_caps + 1) + n_caps + 1));
  a.counters = counters;
  a.per_prompt = per_prompt;
  const int max_block = moeb::max_smem_per_block();
  int nw = 4;
  const int lut = align16(L * 64 + 1);
  while (nw > 1 && (int64_t)nw * a.warp_bytes + lut > max_block) --nw;
  if ((int64_t)nw * a.warp_bytes + lut > max_block)
    return moeb::fail(MOEB_ESMEM, "stack replay state %d B/prompt exceeds shared memory",
                      a.warp_bytes);
  const size_t smem = (size_t)nw * a.warp_bytes + align16(L * 64 + 1);
  auto kern = nib ? k_stack_multi<true> : k_stack_multi<false>;
  moeb::set_smem(kern, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * nw, smem);
  const int64_t want = (n_prompts + nw - 1) / nw;
  const int64_t cap = (int64_t)(per_sm > 0 ? per_sm : 1) * moeb::num_sms();
  const unsigned gx = (unsigned)(want < cap ? want : cap);
  kern<<<dim3(gx, (unsigned)n_preds), 32 * nw, smem, moeb::as_stream(stream)>>>(a);
  return moeb::check_launch("k_stack_multi");
}
