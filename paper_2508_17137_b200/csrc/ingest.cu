// Trace ingestion on device: the reference's trace CSV and
// predictions JSONL formats (traceio.py:47-186) parsed and written by CUDA
// kernels, so a 66 M-row trace goes from file bytes in HBM to packed expert
// masks without a Python loop per line.
//
// Pipeline (paper_2508_17137_b200/traceio.py drives it):
//   1. moeb_count_bytes / moeb_find_bytes: ordered newline positions. Each
//      block owns MOEB_SCAN_CHUNK bytes read as coalesced 16-byte vectors in
//      16 rounds of 256 x 16 B; a block-wide scan per round ranks the matches
//      in file order (HBM-bound: the file is read twice).
//   2. moeb_parse_trace_csv / moeb_parse_predictions: one thread per line,
//      bytes through a 16-byte register window; the Python int()/float()
//      grammar and the reference's validation order reproduced exactly for
//      ASCII input. Lines outside the device grammar are flagged HOST and the
//      host parses just those lines with the reference's own expressions.
//   3. moeb_keys_check / moeb_prompt_flags / moeb_check_grid: duplicate keys
//      and the PromptTrace grid invariants; the host formats the message of
//      the first failing line / prompt only.
//   4. moeb_predictions_join: external predictions onto trace rows (binary
//      search per row in the key-sorted table).
//   5. writers: per-line lengths -> exclusive scan -> formatted bytes.
#include "common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kRounds = MOEB_SCAN_CHUNK / (kThreads * 16);  // 16 rounds of 4 KiB
static_assert(kRounds * kThreads * 16 == MOEB_SCAN_CHUNK, "chunk geometry");

// ---------------------------------------------------------------------------
// Block-wide exclusive scan of one int64 per thread (256 threads).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t* sh /*[9]*/,
                                                   int64_t* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();  // sh may still be read by the previous call
  if (lane == 31) sh[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int64_t s = lane < kThreads / 32 ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < kThreads / 32) sh[lane] = s;
  }
  __syncthreads();
  *total = sh[kThreads / 32 - 1];
  return x - v + (wid > 0 ? sh[wid - 1] : 0);
}

__device__ __forceinline__ uint32_t byte_eq_mask(uint32_t w, uint32_t pat4) {
  // 0x80 in every byte equal to the pattern byte
  const uint32_t x = w ^ pat4;
  return ~(((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) | x | 0x7f7f7f7fu);
}

__device__ __forceinline__ uint4 load_vec(const uint8_t* buf, int64_t n, int64_t off) {
  // off is 16-aligned; bytes at or beyond n read as 0 (never match '\n')
  if (off + 16 <= n) return __ldg(reinterpret_cast<const uint4*>(buf + off));
  uint32_t w[4] = {0, 0, 0, 0};
  for (int k = 0; k < 16 && off + k < n; ++k) w[k >> 2] |= (uint32_t)buf[off + k] << ((k & 3) * 8);
  return make_uint4(w[0], w[1], w[2], w[3]);
}

__global__ void __launch_bounds__(kThreads) k_count_bytes(const uint8_t* buf, int64_t n,
                                                          uint32_t pat4, int64_t* counts) {
  __shared__ int64_t sh[9];
  const int64_t base = (int64_t)blockIdx.x * MOEB_SCAN_CHUNK;
  int c = 0;
#pragma unroll 4
  for (int r = 0; r < kRounds; ++r) {
    const int64_t off = base + ((int64_t)r * kThreads + threadIdx.x) * 16;
    if (off < n) {
      const uint4 v = load_vec(buf, n, off);
      c += __popc(byte_eq_mask(v.x, pat4)) + __popc(byte_eq_mask(v.y, pat4)) +
           __popc(byte_eq_mask(v.z, pat4)) + __popc(byte_eq_mask(v.w, pat4));
    }
  }
  int64_t tot;
  block_excl_scan(c, sh, &tot);
  if (threadIdx.x == 0) counts[blockIdx.x] = tot;
}

// Single-block exclusive scan of `n` int64 in place; data[n] = *total = sum.
__global__ void __launch_bounds__(kThreads) k_scan_inplace(int64_t* data, int64_t n,
                                                           int64_t* total) {
  __shared__ int64_t sh[9];
  constexpr int kPer = 16;
  int64_t carry = 0;
  for (int64_t t0 = 0; t0 < n; t0 += (int64_t)kThreads * kPer) {
    const int64_t i0 = t0 + (int64_t)threadIdx.x * kPer;
    int64_t v[kPer], s = 0;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      v[k] = i0 + k < n ? data[i0 + k] : 0;
      s += v[k];
    }
    int64_t tile;
    int64_t run = carry + block_excl_scan(s, sh, &tile);
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      if (i0 + k < n) data[i0 + k] = run;
      run += v[k];
    }
    carry += tile;
  }
  if (threadIdx.x == 0) {
    data[n] = carry;
    if (total) *total = carry;
  }
}

__global__ void __launch_bounds__(kThreads) k_find_bytes(const uint8_t* buf, int64_t n,
                                                         uint32_t pat4, const int64_t* offs,
                                                         int64_t* pos) {
  __shared__ int64_t sh[9];
  const int64_t base = (int64_t)blockIdx.x * MOEB_SCAN_CHUNK;
  int64_t carry = offs[blockIdx.x];
  for (int r = 0; r < kRounds; ++r) {
    const int64_t off = base + ((int64_t)r * kThreads + threadIdx.x) * 16;
    uint32_t m[4] = {0, 0, 0, 0};
    if (off < n) {
      const uint4 v = load_vec(buf, n, off);
      m[0] = byte_eq_mask(v.x, pat4);
      m[1] = byte_eq_mask(v.y, pat4);
      m[2] = byte_eq_mask(v.z, pat4);
      m[3] = byte_eq_mask(v.w, pat4);
    }
    const int c = __popc(m[0]) + __popc(m[1]) + __popc(m[2]) + __popc(m[3]);
    int64_t tot;
    int64_t dst = carry + block_excl_scan(c, sh, &tot);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t x = m[q];
      while (x) {
        const int bit = __ffs(x) - 1;  // 7, 15, 23 or 31
        x &= x - 1;
        pos[dst++] = off + q * 4 + (bit >> 3);
      }
    }
    carry += tot;
    if (base + (int64_t)(r + 1) * kThreads * 16 >= n) break;  // block-uniform
  }
}

// ---------------------------------------------------------------------------
// Line access and the Python literal grammars.
// ---------------------------------------------------------------------------
struct ByteReader {
  const uint4* v;
  int64_t cur;
  uint4 w;
  __device__ explicit ByteReader(const uint8_t* b)
      : v(reinterpret_cast<const uint4*>(b)), cur(-1), w(make_uint4(0, 0, 0, 0)) {}
  __device__ __forceinline__ uint32_t at(int64_t i) {
    const int64_t vi = i >> 4;
    if (vi != cur) {
      w = __ldg(v + vi);
      cur = vi;
    }
    const int k = (int)(i & 15);
    const uint32_t word = k < 4 ? w.x : k < 8 ? w.y : k < 12 ? w.z : w.w;
    return (word >> ((k & 3) * 8)) & 0xffu;
  }
};

__device__ __forceinline__ void segment(const int64_t* nl, int64_t n_nl, int64_t n, int64_t j,
                                        int64_t* s, int64_t* e) {
  *s = j == 0 ? 0 : nl[j - 1] + 1;
  *e = j < n_nl ? nl[j] : n;
}

// int()/float() strip " \t\n\v\f\r" (ASCII; other code points are HOST lines)
__device__ __forceinline__ bool py_space(uint32_t c) { return c == 32 || (c >= 9 && c <= 13); }
__device__ __forceinline__ bool is_digit(uint32_t c) { return c - '0' < 10u; }

enum { kIntOk = 0, kIntBad = 1, kIntBig = 2 };

// Python int(text) for base 10 on ASCII: strip, [+-], digit ( [_] digit )*.
__device__ int py_int(ByteReader& rd, int64_t a, int64_t b, int64_t* out) {
  while (a < b && py_space(rd.at(a))) ++a;
  while (b > a && py_space(rd.at(b - 1))) --b;
  if (a >= b) return kIntBad;
  bool neg = false;
  uint32_t c = rd.at(a);
  if (c == '+' || c == '-') {
    neg = c == '-';
    ++a;
  }
  if (a >= b || !is_digit(rd.at(a))) return kIntBad;
  unsigned long long v = 0;
  bool big = false, prev_us = false;
  for (int64_t i = a; i < b; ++i) {
    c = rd.at(i);
    if (c == '_') {
      if (prev_us) return kIntBad;
      prev_us = true;
      continue;
    }
    if (!is_digit(c)) return kIntBad;
    prev_us = false;
    const unsigned d = c - '0';
    if (v > (9223372036854775807ull - d) / 10ull) big = true;
    else v = v * 10ull + d;
  }
  if (prev_us) return kIntBad;
  if (big) return kIntBig;
  *out = neg ? -(int64_t)v : (int64_t)v;
  return kIntOk;
}

__device__ __forceinline__ uint32_t lower(uint32_t c) { return (c >= 'A' && c <= 'Z') ? c + 32 : c; }

// digitpart = digit ( [_] digit )*, starting at *i; returns digits consumed
__device__ int digitpart(ByteReader& rd, int64_t* i, int64_t b, bool* bad) {
  int nd = 0;
  bool prev_us = false;
  while (*i < b) {
    const uint32_t c = rd.at(*i);
    if (is_digit(c)) {
      ++nd;
      prev_us = false;
    } else if (c == '_' && nd > 0 && !prev_us) {
      prev_us = true;
    } else {
      break;
    }
    ++*i;
  }
  if (prev_us) *bad = true;
  return nd;
}

// Python float(text) acceptance on ASCII.
__device__ bool py_float_ok(ByteReader& rd, int64_t a, int64_t b) {
  while (a < b && py_space(rd.at(a))) ++a;
  while (b > a && py_space(rd.at(b - 1))) --b;
  if (a >= b) return false;
  uint32_t c = rd.at(a);
  if (c == '+' || c == '-') ++a;
  if (a >= b) return false;
  // inf / infinity / nan, case-insensitive
  const int64_t len = b - a;
  if (len == 3 || len == 8) {
    const char* words[3] = {"inf", "nan", "infinity"};
    for (int w = 0; w < 3; ++w) {
      const char* s = words[w];
      int sl = w == 2 ? 8 : 3;
      if (sl != len) continue;
      bool eq = true;
      for (int k = 0; k < sl; ++k) eq = eq && lower(rd.at(a + k)) == (uint32_t)s[k];
      if (eq) return true;
    }
  }
  bool bad = false;
  int64_t i = a;
  const int ni = digitpart(rd, &i, b, &bad);
  if (bad) return false;
  int nf = 0;
  if (i < b && rd.at(i) == '.') {
    ++i;
    if (i < b && is_digit(rd.at(i))) {
      nf = digitpart(rd, &i, b, &bad);
      if (bad) return false;
    }
  }
  if (ni + nf == 0) return false;
  if (i < b && lower(rd.at(i)) == 'e') {
    ++i;
    if (i < b && (rd.at(i) == '+' || rd.at(i) == '-')) ++i;
    if (i >= b || !is_digit(rd.at(i))) return false;
    digitpart(rd, &i, b, &bad);
    if (bad) return false;
  }
  return i == b;
}

constexpr int kMaxParts = 32;

// ---------------------------------------------------------------------------
// Trace CSV lines (traceio.py:64-103 + TokenRecord.validate, core.py:84-105).
// ---------------------------------------------------------------------------

// Fast path for canonical lines -- unsigned decimal fields of <= 18 digits,
// '|' only inside expert_ids, in-range expert ids, empty embedding -- in one
// pass over the line's 16-byte vectors. Returns false when the line needs
// the general path (which then decides the status); otherwise sets the
// status (OK or the TokenRecord.validate error) and the record.
template <int W>
__device__ __forceinline__ bool fast_csv_line(const uint8_t* buf, int64_t s, int64_t e, int L,
                                              int E, int top_k, int64_t* out_vals /*pid,tok,lay,tid*/,
                                              uint64_t (&m)[W], uint8_t* st) {
  uint64_t v = 0;
  int nd = 0, f = 0, np = 0;
  bool ok = true, dup = false;
  uint64_t vals[5] = {0, 0, 0, 0, 0};
  const uint4* vp = reinterpret_cast<const uint4*>(buf);
  for (int64_t base = s & ~(int64_t)15; base < e && ok; base += 16) {
    const uint4 q = __ldg(vp + (base >> 4));
    const uint32_t words[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int64_t pos = base + k;
      const uint32_t c = (words[k >> 2] >> ((k & 3) * 8)) & 0xffu;
      const uint32_t d = c - '0';
      const bool in = pos >= s && pos < e;
      if (in && d < 10u) {
        v = v * 10u + d;
        ++nd;
      } else if (in) {
        // a separator: ',' ends field f, '|' ends one expert part (f == 3)
        const bool sep_ok = (c == ',' && f < 5) || (c == '|' && f == 3);
        ok = ok && sep_ok && nd > 0 && nd <= 18;
        if (f == 3) {
          ok = ok && v < (uint64_t)E;
          const int ex = (int)(v & 255);
#pragma unroll
          for (int w = 0; w < W; ++w) {
            const uint64_t bit = (ex >> 6) == w ? (1ull << (ex & 63)) : 0ull;
            dup |= (m[w] & bit) != 0;
            m[w] |= bit;
          }
          ++np;
        } else {
          vals[f < 5 ? f : 4] = v;
        }
        f += c == ',' ? 1 : 0;
        v = 0;
        nd = 0;
      }
    }
  }
  // the line must end inside an empty embedding field
  ok = ok && f == 5 && nd == 0;
  if (!ok) return false;
  out_vals[0] = (int64_t)vals[0];
  out_vals[1] = (int64_t)vals[1];
  out_vals[2] = (int64_t)vals[2];
  out_vals[3] = (int64_t)vals[4];
  if (vals[2] >= (uint64_t)L) *st = MOEB_LINE_RANGE_LAYER;
  else if (dup) *st = MOEB_LINE_RANGE_DUPEXP;
  else if (np != top_k) *st = MOEB_LINE_RANGE_COUNT;
  else *st = MOEB_LINE_OK;
  return true;
}
template <int W>
__global__ void __launch_bounds__(kThreads) k_parse_trace_csv(
    const uint8_t* buf, int64_t n, const int64_t* nl, int64_t n_nl, int64_t first_seg,
    int64_t n_lines, int L, int E, int top_k, uint8_t* status, int64_t* prompt_id,
    int64_t* token_index, int32_t* layer_id, uint64_t* masks, int64_t* token_id,
    uint8_t* has_emb, int32_t* flags) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_lines) return;
  int64_t s, e;
  segment(nl, n_nl, n, first_seg + i, &s, &e);
  {
    uint64_t fm[W];
#pragma unroll
    for (int w = 0; w < W; ++w) fm[w] = 0;
    int64_t vals[4];
    uint8_t fst;
    if (fast_csv_line<W>(buf, s, e, L, E, top_k, vals, fm, &fst)) {
      status[i] = fst;
      prompt_id[i] = vals[0];
      token_index[i] = vals[1];
      layer_id[i] = (int32_t)vals[2];
      token_id[i] = vals[3];
      has_emb[i] = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) masks[i * W + w] = fst == MOEB_LINE_OK ? fm[w] : 0ull;
      return;
    }
  }
  ByteReader rd(buf);
  // general path: field boundaries, non-ASCII
  int64_t fb[7];
  fb[0] = s;
  int ncomma = 0;
  bool nonascii = false;
  for (int64_t k = s; k < e; ++k) {
    const uint32_t c = rd.at(k);
    nonascii |= c >= 0x80;
    if (c == ',') {
      if (ncomma < 5) fb[ncomma + 1] = k + 1;
      ++ncomma;
    }
  }
  fb[6] = e + 1;  // field f spans [fb[f], fb[f+1] - 1)
  uint8_t st = MOEB_LINE_OK;
  int64_t pid = 0, tok = 0, tid = 0, lay = 0;
  uint64_t m[W];
#pragma unroll
  for (int w = 0; w < W; ++w) m[w] = 0;
  uint8_t emb = 0;
  if (nonascii) {
    atomicOr(flags, 1);
    st = MOEB_LINE_HOST;
  } else if (ncomma != 5) {
    st = MOEB_LINE_COLS;
  } else {
    int r = py_int(rd, fb[0], fb[1] - 1, &pid);
    if (r) st = r == kIntBig ? MOEB_LINE_HOST : MOEB_LINE_INT_PROMPT;
    if (!st) {
      r = py_int(rd, fb[1], fb[2] - 1, &tok);
      if (r) st = r == kIntBig ? MOEB_LINE_HOST : MOEB_LINE_INT_TOKEN;
    }
    if (!st) {
      r = py_int(rd, fb[2], fb[3] - 1, &lay);
      if (r) st = r == kIntBig ? MOEB_LINE_HOST : MOEB_LINE_INT_LAYER;
    }
    int64_t parts[kMaxParts];
    int np = 0;
    if (!st) {
      const int64_t a = fb[3], b = fb[4] - 1;
      if (a >= b) {
        st = MOEB_LINE_EMPTY_EXPERTS;
      } else {
        int64_t p0 = a;
        for (int64_t k = a; k <= b && !st; ++k) {
          if (k == b || rd.at(k) == '|') {
            if (np == kMaxParts) {
              st = MOEB_LINE_HOST;
              break;
            }
            int64_t v = 0;
            r = py_int(rd, p0, k, &v);
            if (r) st = r == kIntBig ? MOEB_LINE_HOST : MOEB_LINE_INT_EXPERT;
            parts[np++] = v;
            p0 = k + 1;
          }
        }
      }
    }
    if (!st) {
      r = py_int(rd, fb[4], fb[5] - 1, &tid);
      if (r) st = r == kIntBig ? MOEB_LINE_HOST : MOEB_LINE_INT_TOKID;
    }
    if (!st) {
      const int64_t a = fb[5], b = fb[6] - 1;
      if (a < b) {
        emb = 1;
        int64_t p0 = a;
        for (int64_t k = a; k <= b; ++k) {
          if (k == b || rd.at(k) == '|') {
            if (!py_float_ok(rd, p0, k)) {
              st = MOEB_LINE_EMBED;
              break;
            }
            p0 = k + 1;
          }
        }
      }
    }
    // TokenRecord.validate, in order
    if (!st && (pid < 0 || tok < 0)) st = MOEB_LINE_RANGE_NEG;
    if (!st && !(lay >= 0 && lay < L)) st = MOEB_LINE_RANGE_LAYER;
    if (!st) {
      bool dup = false;
      for (int a = 0; a < np && !dup; ++a)
        for (int b = a + 1; b < np; ++b) dup |= parts[a] == parts[b];
      if (dup) st = MOEB_LINE_RANGE_DUPEXP;
    }
    if (!st && np != top_k) st = MOEB_LINE_RANGE_COUNT;
    if (!st) {
      for (int a = 0; a < np; ++a) {
        if (parts[a] < 0 || parts[a] >= E) {
          st = MOEB_LINE_RANGE_EXPERT;
          break;
        }
        const int ex = (int)parts[a];
#pragma unroll
        for (int w = 0; w < W; ++w)
          if ((ex >> 6) == w) m[w] |= 1ull << (ex & 63);
      }
    }
  }
  status[i] = st;
  prompt_id[i] = pid;
  token_index[i] = tok;
  layer_id[i] = (int32_t)lay;
  token_id[i] = tid;
  has_emb[i] = emb;
#pragma unroll
  for (int w = 0; w < W; ++w) masks[i * W + w] = m[w];
  if (emb) atomicOr(flags, 2);
}

// ---------------------------------------------------------------------------
// Predictions JSONL lines (traceio.py:142-169). Device grammar: one JSON
// object of the four known keys with integer values / an integer array,
// JSON whitespace anywhere between tokens. Anything else -> HOST.
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool json_ws(uint32_t c) { return c == 32 || c == 9 || c == 10 || c == 13; }
// str.strip() whitespace (blank-line test) on ASCII
__device__ __forceinline__ bool str_space(uint32_t c) {
  return c == 32 || (c >= 9 && c <= 13) || (c >= 28 && c <= 31);
}

// JSON integer: -?(0|[1-9][0-9]*) not followed by . e E
__device__ int json_int(ByteReader& rd, int64_t* i, int64_t e, int64_t* out) {
  int64_t k = *i;
  bool neg = false;
  if (k < e && rd.at(k) == '-') {
    neg = true;
    ++k;
  }
  if (k >= e || !is_digit(rd.at(k))) return kIntBad;
  unsigned long long v = 0;
  bool big = false;
  if (rd.at(k) == '0') {
    ++k;
  } else {
    while (k < e && is_digit(rd.at(k))) {
      const unsigned d = rd.at(k) - '0';
      if (v > (9223372036854775807ull - d) / 10ull) big = true;
      else v = v * 10ull + d;
      ++k;
    }
  }
  if (k < e) {
    const uint32_t c = rd.at(k);
    if (c == '.' || c == 'e' || c == 'E' || is_digit(c)) return kIntBad;
  }
  if (big) return kIntBig;
  *out = neg ? -(int64_t)v : (int64_t)v;
  *i = k;
  return kIntOk;
}

template <int W>
__global__ void __launch_bounds__(kThreads) k_parse_predictions(
    const uint8_t* buf, int64_t n, const int64_t* nl, int64_t n_nl, int64_t n_lines, int L,
    int E, uint8_t* status, int64_t* prompt_id, int64_t* token_index, int32_t* layer_id,
    uint64_t* masks, int32_t* flags) {
  const int64_t li = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (li >= n_lines) return;
  int64_t s, e;
  segment(nl, n_nl, n, li, &s, &e);
  ByteReader rd(buf);
  bool blank = true, nonascii = false;
  for (int64_t k = s; k < e; ++k) {
    const uint32_t c = rd.at(k);
    nonascii |= c >= 0x80;
    blank &= str_space(c);
  }
  uint8_t st = MOEB_LINE_HOST;
  int64_t v[3] = {0, 0, 0};
  uint64_t m[W];
#pragma unroll
  for (int w = 0; w < W; ++w) m[w] = 0;
  int64_t first_bad_expert = 0;
  bool expert_bad = false;
  if (nonascii) {
    atomicOr(flags, 1);
  } else if (blank) {
    st = MOEB_LINE_SKIP;
  } else {
    // ws { ws "key" ws : ws value ( ws , ws "key" ... )* ws } ws
    int64_t i = s;
    bool ok = true;
    int seen = 0;  // bits: prompt_id, token_index, layer_id, experts
    while (i < e && json_ws(rd.at(i))) ++i;
    ok = i < e && rd.at(i) == '{';
    ++i;
    bool first = true;
    while (ok) {
      while (i < e && json_ws(rd.at(i))) ++i;
      if (i < e && rd.at(i) == '}' && first) {
        ++i;
        break;
      }
      if (!first) {
        if (i < e && rd.at(i) == '}') {
          ++i;
          break;
        }
        if (!(i < e && rd.at(i) == ',')) {
          ok = false;
          break;
        }
        ++i;
        while (i < e && json_ws(rd.at(i))) ++i;
      }
      first = false;
      // key: one of the four names, no escapes
      if (!(i < e && rd.at(i) == '"')) {
        ok = false;
        break;
      }
      ++i;
      const int64_t k0 = i;
      while (i < e && rd.at(i) != '"' && rd.at(i) != '\\') ++i;
      if (!(i < e && rd.at(i) == '"')) {
        ok = false;
        break;
      }
      const int64_t klen = i - k0;
      ++i;
      int which = -1;
      {
        const char* names[4] = {"prompt_id", "token_index", "layer_id", "experts"};
        const int lens[4] = {9, 11, 8, 7};
        for (int w = 0; w < 4 && which < 0; ++w) {
          if (lens[w] != klen) continue;
          bool eq = true;
          for (int c = 0; c < lens[w]; ++c) eq = eq && rd.at(k0 + c) == (uint32_t)names[w][c];
          if (eq) which = w;
        }
      }
      if (which < 0 || (seen >> which) & 1) {  // unknown or repeated key: host json
        ok = false;
        break;
      }
      seen |= 1 << which;
      while (i < e && json_ws(rd.at(i))) ++i;
      if (!(i < e && rd.at(i) == ':')) {
        ok = false;
        break;
      }
      ++i;
      while (i < e && json_ws(rd.at(i))) ++i;
      if (which < 3) {
        int64_t x = 0;
        if (json_int(rd, &i, e, &x) != kIntOk) {
          ok = false;
          break;
        }
        v[which] = x;
      } else {
        if (!(i < e && rd.at(i) == '[')) {
          ok = false;
          break;
        }
        ++i;
        while (i < e && json_ws(rd.at(i))) ++i;
        if (i < e && rd.at(i) == ']') {
          ++i;
        } else {
          for (;;) {
            int64_t x = 0;
            if (json_int(rd, &i, e, &x) != kIntOk) {
              ok = false;
              break;
            }
            if (x < 0 || x >= E) {
              if (!expert_bad) first_bad_expert = x;
              expert_bad = true;
            } else {
#pragma unroll
              for (int w = 0; w < W; ++w)
                if ((x >> 6) == w) m[w] |= 1ull << (x & 63);
            }
            while (i < e && json_ws(rd.at(i))) ++i;
            if (i < e && rd.at(i) == ',') {
              ++i;
              while (i < e && json_ws(rd.at(i))) ++i;
              continue;
            }
            if (i < e && rd.at(i) == ']') {
              ++i;
              break;
            }
            ok = false;
            break;
          }
          if (!ok) break;
        }
      }
    }
    while (ok && i < e && json_ws(rd.at(i))) ++i;
    if (ok && i == e && seen == 15) {
      if (expert_bad) st = MOEB_LINE_RANGE_EXPERT;
      else if (!(v[2] >= 0 && v[2] < L)) st = MOEB_LINE_RANGE_LAYER;
      else st = MOEB_LINE_OK;
    }
  }
  (void)first_bad_expert;
  status[li] = st;
  prompt_id[li] = v[0];
  token_index[li] = v[1];
  layer_id[li] = (int32_t)v[2];
#pragma unroll
  for (int w = 0; w < W; ++w) masks[li * W + w] = m[w];
}

// ---------------------------------------------------------------------------
// Reductions over parsed lines.
// ---------------------------------------------------------------------------
// out[0] = v0, out[1] = v1 (n = 1 or 2): a stream-ordered initialisation
// (instead of an async copy from a host stack variable)
__global__ void k_fill_i64(int64_t* out, int n, int64_t v0, int64_t v1) {
  if (threadIdx.x < n) out[threadIdx.x] = threadIdx.x == 0 ? v0 : v1;
}

__global__ void k_first_status(const uint8_t* status, int64_t n, int skip, int64_t* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int st = status[i];
  if (st != 0 && st != skip) atomicMin(reinterpret_cast<unsigned long long*>(out), (unsigned long long)i);
}

__device__ __forceinline__ int key_cmp(int64_t a0, int64_t b0, int32_t c0, int64_t a1, int64_t b1,
                                       int32_t c1) {
  if (a0 != a1) return a0 < a1 ? -1 : 1;
  if (b0 != b1) return b0 < b1 ? -1 : 1;
  if (c0 != c1) return c0 < c1 ? -1 : 1;
  return 0;
}

// Rows with status 0 only; "previous" = nearest earlier counted row, found by
// a short backwards walk (skipped rows are rare blank lines).
__global__ void k_keys_check(const int64_t* a, const int64_t* b, const int32_t* c,
                             const uint8_t* status, int skip, int64_t n, int64_t* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (status && status[i] != 0) return;
  int64_t j = i - 1;
  while (j >= 0 && status && status[j] != 0) --j;
  if (j < 0) return;
  const int r = key_cmp(a[j], b[j], c[j], a[i], b[i], c[i]);
  if (r > 0) atomicAdd(reinterpret_cast<unsigned long long*>(out), 1ull);
  if (r == 0) atomicMin(reinterpret_cast<unsigned long long*>(out + 1), (unsigned long long)i);
}

__global__ void k_prompt_flags(const int64_t* pid, int64_t n, uint8_t* flags) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  flags[i] = (i == 0 || pid[i] != pid[i - 1]) ? '\n' : 0;  // counted by moeb_count_bytes('\n')
}

__global__ void k_check_grid(const int64_t* starts, int64_t P, int64_t rows, const int64_t* tok,
                             const int32_t* lay, int L, int64_t* bad) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  int64_t lo = 0, hi = P - 1;  // last start <= r
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (starts[mid] <= r) lo = mid;
    else hi = mid - 1;
  }
  const int64_t j = r - starts[lo];
  const int64_t end = lo + 1 < P ? starts[lo + 1] : rows;
  bool ok = tok[r] == j / L && lay[r] == (int32_t)(j % L);
  if (r == end - 1) ok = ok && (end - starts[lo]) % L == 0;
  if (!ok) atomicMin(reinterpret_cast<unsigned long long*>(bad), (unsigned long long)lo);
}

template <int W>
__global__ void k_predictions_join(const int64_t* tp, const int64_t* tt, const int32_t* tl,
                                   const uint64_t* tm, int64_t nt, const int64_t* pids,
                                   const int64_t* row_off, int P, int L, uint64_t* pred,
                                   uint8_t* cov) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t rows = row_off[P];
  if (r >= rows) return;
  int lo = 0, hi = P - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (row_off[mid] <= r) lo = mid;
    else hi = mid - 1;
  }
  const int64_t j = r - row_off[lo];
  const int64_t pid = pids[lo], t = j / L;
  const int32_t l = (int32_t)(j % L);
  int64_t a = 0, b = nt;  // first table row >= key
  while (a < b) {
    const int64_t mid = (a + b) >> 1;
    if (key_cmp(tp[mid], tt[mid], tl[mid], pid, t, l) < 0) a = mid + 1;
    else b = mid;
  }
  const bool hit = a < nt && key_cmp(tp[a], tt[a], tl[a], pid, t, l) == 0;
#pragma unroll
  for (int w = 0; w < W; ++w) pred[r * W + w] = hit ? tm[a * W + w] : 0ull;
  cov[r] = hit ? 1 : 0;
}

// ---------------------------------------------------------------------------
// Writers.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int dec_len(int64_t v) {
  int n = v < 0 ? 2 : 1;
  unsigned long long u = v < 0 ? (unsigned long long)(-(v + 1)) + 1ull : (unsigned long long)v;
  while (u >= 10) {
    u /= 10;
    ++n;
  }
  return n;
}

__device__ __forceinline__ int64_t put_dec(uint8_t* out, int64_t p, int64_t v) {
  const int len = dec_len(v);
  unsigned long long u = v < 0 ? (unsigned long long)(-(v + 1)) + 1ull : (unsigned long long)v;
  if (v < 0) out[p] = '-';
  int64_t q = p + len - 1;
  do {
    out[q--] = (uint8_t)('0' + u % 10);
    u /= 10;
  } while (u);
  return p + len;
}

__device__ __forceinline__ int64_t put_str(uint8_t* out, int64_t p, const char* s) {
  while (*s) out[p++] = (uint8_t)*s++;
  return p;
}

template <int W>
__device__ __forceinline__ int mask_list_len(const uint64_t* m, int E) {
  int len = 0, cnt = 0;
#pragma unroll
  for (int w = 0; w < W; ++w) {
    uint64_t x = m[w];
    while (x) {
      const int ex = w * 64 + __ffsll((long long)x) - 1;
      x &= x - 1;
      if (ex < E) {
        len += dec_len(ex);
        ++cnt;
      }
    }
  }
  return len + (cnt > 0 ? cnt - 1 : 0);
}

template <int W>
__device__ __forceinline__ int64_t put_mask_list(uint8_t* out, int64_t p, const uint64_t* m, int E,
                                                 uint8_t sep) {
  bool first = true;
#pragma unroll
  for (int w = 0; w < W; ++w) {
    uint64_t x = m[w];
    while (x) {
      const int ex = w * 64 + __ffsll((long long)x) - 1;
      x &= x - 1;
      if (ex < E) {
        if (!first) out[p++] = sep;
        first = false;
        p = put_dec(out, p, ex);
      }
    }
  }
  return p;
}

__device__ __forceinline__ int row_prompt(const int64_t* row_off, int P, int64_t r) {
  int lo = 0, hi = P - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (row_off[mid] <= r) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

template <int W, bool WRITE>
__global__ void k_trace_csv(const uint64_t* truth, const int64_t* pids, const int64_t* row_off,
                            int P, int L, int E, const int32_t* tokid, int64_t* lens,
                            const int64_t* offs, uint8_t* out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= row_off[P]) return;
  const int p = row_prompt(row_off, P, r);
  const int64_t j = r - row_off[p];
  const int64_t pid = pids[p], t = j / L, l = j % L;
  const int64_t tid = tokid ? tokid[r / L] : 0;
  const uint64_t* m = truth + r * W;
  if (!WRITE) {
    lens[r] = dec_len(pid) + dec_len(t) + dec_len(l) + mask_list_len<W>(m, E) + dec_len(tid) + 6;
    return;
  }
  int64_t q = offs[r];
  q = put_dec(out, q, pid);
  out[q++] = ',';
  q = put_dec(out, q, t);
  out[q++] = ',';
  q = put_dec(out, q, l);
  out[q++] = ',';
  q = put_mask_list<W>(out, q, m, E, '|');
  out[q++] = ',';
  q = put_dec(out, q, tid);
  out[q++] = ',';
  out[q++] = '\n';
}

template <int W, bool WRITE>
__global__ void k_predictions_jsonl(const int64_t* tp, const int64_t* tt, const int32_t* tl,
                                    const uint64_t* tm, int64_t n, int E, int64_t* lens,
                                    const int64_t* offs, uint8_t* out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const uint64_t* m = tm + r * W;
  // {"prompt_id":,"token_index":,"layer_id":,"experts":[]}\n = 55 bytes
  if (!WRITE) {
    lens[r] = 55 + dec_len(tp[r]) + dec_len(tt[r]) + dec_len(tl[r]) + mask_list_len<W>(m, E);
    return;
  }
  int64_t q = offs[r];
  q = put_str(out, q, "{\"prompt_id\":");
  q = put_dec(out, q, tp[r]);
  q = put_str(out, q, ",\"token_index\":");
  q = put_dec(out, q, tt[r]);
  q = put_str(out, q, ",\"layer_id\":");
  q = put_dec(out, q, tl[r]);
  q = put_str(out, q, ",\"experts\":[");
  q = put_mask_list<W>(out, q, m, E, ',');
  q = put_str(out, q, "]}\n");
}

// Generic exclusive scan: per-4096 block sums, scan of the sums, block scans.
__global__ void __launch_bounds__(kThreads) k_block_sums(const int64_t* in, int64_t n,
                                                         int64_t* sums) {
  __shared__ int64_t sh[9];
  const int64_t base = (int64_t)blockIdx.x * kThreads * 16;
  int64_t s = 0;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const int64_t i = base + (int64_t)r * kThreads + threadIdx.x;
    if (i < n) s += in[i];
  }
  int64_t tot;
  block_excl_scan(s, sh, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kThreads) k_block_scan(const int64_t* in, int64_t n,
                                                         const int64_t* sums, int64_t* out) {
  __shared__ int64_t sh[9];
  const int64_t base = (int64_t)blockIdx.x * kThreads * 16;
  int64_t carry = sums[blockIdx.x];
  for (int r = 0; r < 16; ++r) {
    const int64_t i = base + (int64_t)r * kThreads + threadIdx.x;
    const int64_t v = i < n ? in[i] : 0;
    int64_t tot;
    const int64_t x = block_excl_scan(v, sh, &tot);
    if (i < n) out[i] = carry + x;
    carry += tot;
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = carry;
}

inline unsigned blocks_for(int64_t n, int t = kThreads) { return (unsigned)((n + t - 1) / t); }
inline uint32_t pat4_of(int v) { return 0x01010101u * (uint32_t)(v & 0xff); }

#define MOEB_DISPATCH_W(W_, call_)                        \
  switch (W_) {                                           \
    case 1: { constexpr int kW = 1; call_; } break;       \
    case 2: { constexpr int kW = 2; call_; } break;       \
    case 3: { constexpr int kW = 3; call_; } break;       \
    default: { constexpr int kW = 4; call_; } break;      \
  }

}  // namespace

extern "C" {

int moeb_count_bytes(const uint8_t* buf, int64_t n, int value, int64_t* block_offsets,
                     int64_t* total, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(block_offsets && (n == 0 || buf), "null argument");
  MOEB_REQUIRE(n >= 0 && (reinterpret_cast<uintptr_t>(buf) & 15) == 0, "buffer must be 16-byte aligned");
  cudaStream_t s = moeb::as_stream(stream);
  const int64_t nb = (n + MOEB_SCAN_CHUNK - 1) / MOEB_SCAN_CHUNK;
  if (nb > 0) k_count_bytes<<<(unsigned)nb, kThreads, 0, s>>>(buf, n, pat4_of(value), block_offsets);
  k_scan_inplace<<<1, kThreads, 0, s>>>(block_offsets, nb, total);
  return moeb::check_launch("k_count_bytes");
}

int moeb_find_bytes(const uint8_t* buf, int64_t n, int value, const int64_t* block_offsets,
                    int64_t* positions, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(block_offsets && positions && (n == 0 || buf), "null argument");
  MOEB_REQUIRE((reinterpret_cast<uintptr_t>(buf) & 15) == 0, "buffer must be 16-byte aligned");
  const int64_t nb = (n + MOEB_SCAN_CHUNK - 1) / MOEB_SCAN_CHUNK;
  if (nb > 0)
    k_find_bytes<<<(unsigned)nb, kThreads, 0, moeb::as_stream(stream)>>>(buf, n, pat4_of(value),
                                                                         block_offsets, positions);
  return moeb::check_launch("k_find_bytes");
}

int moeb_parse_trace_csv(const uint8_t* buf, int64_t n, const int64_t* nl, int64_t n_nl,
                         int64_t first_segment, int64_t n_lines, int L, int E, int top_k,
                         uint8_t* status, int64_t* prompt_id, int64_t* token_index,
                         int32_t* layer_id, uint64_t* masks, int64_t* token_id,
                         uint8_t* has_embedding, int32_t* flags, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(L >= 1 && E >= 1 && E <= 256, "unsupported shape L=%d E=%d", L, E);
  MOEB_REQUIRE((reinterpret_cast<uintptr_t>(buf) & 15) == 0, "buffer must be 16-byte aligned");
  if (n_lines <= 0) return MOEB_OK;
  MOEB_REQUIRE(status && prompt_id && token_index && layer_id && masks && token_id &&
                   has_embedding && flags && buf, "null argument");
  cudaStream_t s = moeb::as_stream(stream);
  const int W = moeb::words_for(E);
  MOEB_DISPATCH_W(W, (k_parse_trace_csv<kW><<<blocks_for(n_lines), kThreads, 0, s>>>(
                          buf, n, nl, n_nl, first_segment, n_lines, L, E, top_k, status,
                          prompt_id, token_index, layer_id, masks, token_id, has_embedding,
                          flags)));
  return moeb::check_launch("k_parse_trace_csv");
}

int moeb_parse_predictions(const uint8_t* buf, int64_t n, const int64_t* nl, int64_t n_nl,
                           int64_t n_lines, int L, int E, uint8_t* status, int64_t* prompt_id,
                           int64_t* token_index, int32_t* layer_id, uint64_t* masks,
                           int32_t* flags, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(L >= 1 && E >= 1 && E <= 256, "unsupported shape L=%d E=%d", L, E);
  MOEB_REQUIRE((reinterpret_cast<uintptr_t>(buf) & 15) == 0, "buffer must be 16-byte aligned");
  if (n_lines <= 0) return MOEB_OK;
  MOEB_REQUIRE(status && prompt_id && token_index && layer_id && masks && flags && buf,
               "null argument");
  cudaStream_t s = moeb::as_stream(stream);
  const int W = moeb::words_for(E);
  MOEB_DISPATCH_W(W, (k_parse_predictions<kW><<<blocks_for(n_lines), kThreads, 0, s>>>(
                          buf, n, nl, n_nl, n_lines, L, E, status, prompt_id, token_index,
                          layer_id, masks, flags)));
  return moeb::check_launch("k_parse_predictions");
}

int moeb_first_status(const uint8_t* status, int64_t n, int skip_code, int64_t* out,
                      void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(out && (n == 0 || status), "null argument");
  cudaStream_t s = moeb::as_stream(stream);
  k_fill_i64<<<1, 32, 0, s>>>(out, 1, n, 0);
  if (n > 0) k_first_status<<<blocks_for(n), kThreads, 0, s>>>(status, n, skip_code, out);
  return moeb::check_launch("k_first_status");
}

int moeb_keys_check(const int64_t* a, const int64_t* b, const int32_t* c, const uint8_t* status,
                    int skip_code, int64_t n, int64_t* out, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(out && (n == 0 || (a && b && c)), "null argument");
  (void)skip_code;
  cudaStream_t s = moeb::as_stream(stream);
  k_fill_i64<<<1, 32, 0, s>>>(out, 2, 0, n);
  if (n > 0) k_keys_check<<<blocks_for(n), kThreads, 0, s>>>(a, b, c, status, skip_code, n, out);
  return moeb::check_launch("k_keys_check");
}

int moeb_prompt_flags(const int64_t* prompt_id, int64_t n, uint8_t* flags, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(n == 0 || (prompt_id && flags), "null argument");
  if (n > 0) k_prompt_flags<<<blocks_for(n), kThreads, 0, moeb::as_stream(stream)>>>(prompt_id, n, flags);
  return moeb::check_launch("k_prompt_flags");
}

int moeb_check_grid(const int64_t* starts, int64_t n_prompts, int64_t n_rows,
                    const int64_t* token_index, const int32_t* layer_id, int L,
                    int64_t* bad_prompt, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(bad_prompt && L >= 1, "bad argument");
  cudaStream_t s = moeb::as_stream(stream);
  k_fill_i64<<<1, 32, 0, s>>>(bad_prompt, 1, n_prompts, 0);
  if (n_rows > 0 && n_prompts > 0)
    k_check_grid<<<blocks_for(n_rows), kThreads, 0, s>>>(starts, n_prompts, n_rows, token_index,
                                                         layer_id, L, bad_prompt);
  return moeb::check_launch("k_check_grid");
}

int moeb_predictions_join(const int64_t* t_prompt, const int64_t* t_token, const int32_t* t_layer,
                          const uint64_t* t_masks, int64_t n_table, const int64_t* prompt_ids,
                          const int64_t* prompt_row_off, int n_prompts, int64_t rows, int L,
                          int E, uint64_t* pred, uint8_t* covered, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(prompt_ids && prompt_row_off && pred && covered && n_prompts >= 1, "null argument");
  MOEB_REQUIRE(L >= 1 && E >= 1 && E <= 256 && rows >= 0, "unsupported shape");
  if (rows == 0) return MOEB_OK;
  cudaStream_t s = moeb::as_stream(stream);
  const int W = moeb::words_for(E);
  MOEB_DISPATCH_W(W, (k_predictions_join<kW><<<blocks_for(rows), kThreads, 0, s>>>(
                          t_prompt, t_token, t_layer, t_masks, n_table, prompt_ids,
                          prompt_row_off, n_prompts, L, pred, covered)));
  return moeb::check_launch("k_predictions_join");
}

static int trace_csv(const uint64_t* truth, const int64_t* pids, const int64_t* row_off, int P,
                     int64_t rows, int L, int E, const int32_t* tokid, int64_t* lens,
                     const int64_t* offs, uint8_t* out, bool write, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(truth && pids && row_off && P >= 1 && (write ? (offs && out) : lens != nullptr),
               "null argument");
  MOEB_REQUIRE(L >= 1 && E >= 1 && E <= 256 && rows >= 0, "unsupported shape");
  if (rows == 0) return MOEB_OK;
  cudaStream_t s = moeb::as_stream(stream);
  const int W = moeb::words_for(E);
  if (write) {
    MOEB_DISPATCH_W(W, (k_trace_csv<kW, true><<<blocks_for(rows), kThreads, 0, s>>>(
                            truth, pids, row_off, P, L, E, tokid, lens, offs, out)));
  } else {
    MOEB_DISPATCH_W(W, (k_trace_csv<kW, false><<<blocks_for(rows), kThreads, 0, s>>>(
                            truth, pids, row_off, P, L, E, tokid, lens, offs, out)));
  }
  return moeb::check_launch("k_trace_csv");
}

int moeb_trace_csv_lengths(const uint64_t* truth, const int64_t* prompt_ids,
                           const int64_t* prompt_row_off, int n_prompts, int64_t rows, int L,
                           int E, const int32_t* token_ids, int64_t* lens, void* stream) {
  return trace_csv(truth, prompt_ids, prompt_row_off, n_prompts, rows, L, E, token_ids, lens,
                   nullptr, nullptr, false, stream);
}

int moeb_trace_csv_write(const uint64_t* truth, const int64_t* prompt_ids,
                         const int64_t* prompt_row_off, int n_prompts, int64_t rows, int L,
                         int E, const int32_t* token_ids, const int64_t* offsets, uint8_t* out,
                         void* stream) {
  return trace_csv(truth, prompt_ids, prompt_row_off, n_prompts, rows, L, E, token_ids, nullptr,
                   offsets, out, true, stream);
}

static int predictions_jsonl(const int64_t* tp, const int64_t* tt, const int32_t* tl,
                             const uint64_t* tm, int64_t n, int E, int64_t* lens,
                             const int64_t* offs, uint8_t* out, bool write, void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(E >= 1 && E <= 256, "unsupported E");
  if (n <= 0) return MOEB_OK;
  MOEB_REQUIRE(tp && tt && tl && tm && (write ? (offs && out) : lens != nullptr), "null argument");
  cudaStream_t s = moeb::as_stream(stream);
  const int W = moeb::words_for(E);
  if (write) {
    MOEB_DISPATCH_W(W, (k_predictions_jsonl<kW, true><<<blocks_for(n), kThreads, 0, s>>>(
                            tp, tt, tl, tm, n, E, lens, offs, out)));
  } else {
    MOEB_DISPATCH_W(W, (k_predictions_jsonl<kW, false><<<blocks_for(n), kThreads, 0, s>>>(
                            tp, tt, tl, tm, n, E, lens, offs, out)));
  }
  return moeb::check_launch("k_predictions_jsonl");
}

int moeb_predictions_jsonl_lengths(const int64_t* t_prompt, const int64_t* t_token,
                                   const int32_t* t_layer, const uint64_t* t_masks, int64_t n,
                                   int E, int64_t* lens, void* stream) {
  return predictions_jsonl(t_prompt, t_token, t_layer, t_masks, n, E, lens, nullptr, nullptr,
                           false, stream);
}

int moeb_predictions_jsonl_write(const int64_t* t_prompt, const int64_t* t_token,
                                 const int32_t* t_layer, const uint64_t* t_masks, int64_t n,
                                 int E, const int64_t* offsets, uint8_t* out, void* stream) {
  return predictions_jsonl(t_prompt, t_token, t_layer, t_masks, n, E, nullptr, offsets, out, true,
                           stream);
}

int moeb_exclusive_scan_i64(const int64_t* in, int64_t n, int64_t* out, int64_t* ws,
                            void* stream) {
  moeb::clear_error();
  MOEB_REQUIRE(out && ws && (n == 0 || in), "null argument");
  cudaStream_t s = moeb::as_stream(stream);
  const int64_t nb = (n + kThreads * 16 - 1) / (kThreads * 16);
  if (nb == 0) {
    k_fill_i64<<<1, 32, 0, s>>>(out, 1, 0, 0);
    return moeb::check_launch("k_fill_i64");
  }
  k_block_sums<<<(unsigned)nb, kThreads, 0, s>>>(in, n, ws);
  k_scan_inplace<<<1, kThreads, 0, s>>>(ws, nb, nullptr);
  k_block_scan<<<(unsigned)nb, kThreads, 0, s>>>(in, n, ws, out);
  return moeb::check_launch("k_exclusive_scan");
}

}  // extern "C"
