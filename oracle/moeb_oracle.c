/*
 * moeb_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, deliberately naive CPU restatement of the MoE-Beyond reference
 * hot path (package `moesim`, mounted read-only at /root/reference). It is the
 * checker that the CUDA product path in paper_2508_17137_b200/csrc is compared
 * against; nothing in the product links or calls it. Only tests/, the
 * __graft_entry__.smoke() check and bench.py's cpu_baseline leg may load it.
 *
 * Every function cites the reference code it restates. The restatement is
 * pinned against the reference itself through tests/golden/ fixtures that
 * tests/golden/make_golden.py produced by importing the reference.
 *
 * Data conventions (shared with the product ABI, include/moeb.h):
 *   - A trace row is one (prompt, token, layer) step; rows of a prompt are in
 *     (token, layer) order, prompt p owns rows [row_off[p], row_off[p+1]).
 *   - An expert set is a bitmask of W = ceil(E/64) uint64 words per row,
 *     bit e of word e/64 = expert e.
 *   - A cache key (layer, expert) is the integer layer*E + expert.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EINVAL 1
#define ORC_ENOMEM 2

static inline int words_for(int E) { return (E + 63) / 64; }
static inline int bit_get(const uint64_t* m, int e) { return (int)((m[e >> 6] >> (e & 63)) & 1u); }
static inline void bit_set(uint64_t* m, int e) { m[e >> 6] |= (uint64_t)1 << (e & 63); }

/* ------------------------------------------------------------------------ */
/* Expert cache: LRU (reference) and LFU (builder-defined, parity unpinned). */
/* ------------------------------------------------------------------------ */

/* The resident set is an array ordered least- to most-recently used, the
 * same order as the reference's OrderedDict (cache.py:68, `resident` :79-82).
 * All operations are O(capacity) scans: slow, but obviously equal to the
 * reference's semantics. */
typedef struct {
  int64_t cap;
  int policy; /* 0 = LRU (cache.py:58-154), 1 = LFU */
  int64_t n;
  int32_t* keys;   /* [cap] LRU-first */
  int64_t* freq;   /* [cap] LFU demand counts, parallel to keys */
  uint8_t* pinned; /* [num_keys] current-step pins (cache.py:69, :102-104) */
  int32_t* pin_list;
  int64_t npins;
} orc_cache;

static int cache_init(orc_cache* c, int64_t cap, int policy, int64_t num_keys) {
  c->cap = cap;
  c->policy = policy;
  c->n = 0;
  c->npins = 0;
  c->keys = (int32_t*)malloc(sizeof(int32_t) * (size_t)cap);
  c->freq = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap);
  c->pinned = (uint8_t*)calloc((size_t)num_keys, 1);
  c->pin_list = (int32_t*)malloc(sizeof(int32_t) * (size_t)num_keys);
  if (!c->keys || !c->freq || !c->pinned || !c->pin_list) return ORC_ENOMEM;
  return ORC_OK;
}

static void cache_free(orc_cache* c) {
  free(c->keys);
  free(c->freq);
  free(c->pinned);
  free(c->pin_list);
}

static int64_t cache_find(const orc_cache* c, int32_t key) {
  for (int64_t i = 0; i < c->n; ++i)
    if (c->keys[i] == key) return i;
  return -1;
}

static void cache_remove_at(orc_cache* c, int64_t i) {
  memmove(c->keys + i, c->keys + i + 1, sizeof(int32_t) * (size_t)(c->n - i - 1));
  memmove(c->freq + i, c->freq + i + 1, sizeof(int64_t) * (size_t)(c->n - i - 1));
  c->n--;
}

static void cache_append(orc_cache* c, int32_t key, int64_t freq) {
  c->keys[c->n] = key;
  c->freq[c->n] = freq;
  c->n++;
}

/* move_to_end (cache.py:119, :146) */
static void cache_move_to_end(orc_cache* c, int64_t i) {
  int32_t key = c->keys[i];
  int64_t f = c->freq[i];
  cache_remove_at(c, i);
  cache_append(c, key, f);
}

/* _evict_one (cache.py:93-100): first non-pinned key from the LRU end.
 * LFU: the non-pinned key with the smallest demand count, LRU-most on ties. */
static int cache_evict_one(orc_cache* c) {
  int64_t victim = -1;
  for (int64_t i = 0; i < c->n; ++i) {
    if (c->pinned[c->keys[i]]) continue;
    if (c->policy == 0) {
      victim = i;
      break;
    }
    if (victim < 0 || c->freq[i] < c->freq[victim]) victim = i;
  }
  if (victim < 0) return 0;
  cache_remove_at(c, victim);
  return 1;
}

/* begin_step (cache.py:102-104) */
static void cache_begin_step(orc_cache* c) {
  for (int64_t i = 0; i < c->npins; ++i) c->pinned[c->pin_list[i]] = 0;
  c->npins = 0;
}

static void cache_pin(orc_cache* c, int32_t key) {
  if (!c->pinned[key]) {
    c->pinned[key] = 1;
    c->pin_list[c->npins++] = key;
  }
}

/* touch (cache.py:106-124). Returns 1 on hit. */
static int cache_touch(orc_cache* c, int32_t key) {
  int64_t i = cache_find(c, key);
  if (i >= 0) {
    c->freq[i] += 1;
    cache_move_to_end(c, i);
    return 1;
  }
  if (c->n >= c->cap && !cache_evict_one(c)) return 0;
  cache_append(c, key, 1);
  return 0;
}

/* one key of prefetch (cache.py:141-153). Returns 1 if newly inserted. */
static int cache_prefetch_one(orc_cache* c, int32_t key) {
  int64_t i = cache_find(c, key);
  if (i >= 0) {
    cache_move_to_end(c, i);
    cache_pin(c, key);
    return 0;
  }
  if (c->n >= c->cap && !cache_evict_one(c)) return 0;
  cache_append(c, key, 0);
  cache_pin(c, key);
  return 1;
}

/*
 * Op-stream interface over one cache (the reference's per-call ExpertCache
 * API, cache.py:58-154): op 0 = begin_step, 1 = touch(key), 2 = prefetch(key).
 * results[i] = touch hit / prefetch inserted (0 for begin_step).
 */
int orc_cache_ops(const int32_t* ops, const int32_t* keys, int64_t n, int L, int E,
                  int64_t cap, int policy, uint8_t* results) {
  if (cap < 1 || L < 1 || E < 1) return ORC_EINVAL;
  orc_cache c;
  if (cache_init(&c, cap, policy, (int64_t)L * E) != ORC_OK) return ORC_ENOMEM;
  for (int64_t i = 0; i < n; ++i) {
    uint8_t r = 0;
    if (ops[i] == 0) {
      cache_begin_step(&c);
    } else {
      if (keys[i] < 0 || keys[i] >= L * E) {
        cache_free(&c);
        return ORC_EINVAL;
      }
      r = (uint8_t)(ops[i] == 1 ? cache_touch(&c, keys[i]) : cache_prefetch_one(&c, keys[i]));
    }
    results[i] = r;
  }
  cache_free(&c);
  return ORC_OK;
}

/*
 * Trace replay of every prompt under one capacity: engine.replay_prompt
 * (engine.py:113-207) with the cache protocol of Appendix A in SURVEY.md.
 *   pred      predicted masks per row (NULL = empty prediction, lru_only)
 *   covered   per-row coverage flags for the external predictor (NULL = all)
 * counters  [4 + 3L] = measured_accesses, cache_hits, prediction_hits,
 *           uncovered_queries, layer_accesses[L], layer_cache_hits[L],
 *           layer_prediction_hits[L]   (engine.py:62-110, :185-206)
 * per_prompt [P][4] = measured_accesses, cache_hits, prediction_hits,
 *           uncovered (nullable)
 * hit_masks [rows][W] bit e set iff the touch of truth expert e hit
 *           (warm-up rows included; nullable)
 */
int orc_cache_sim(const uint64_t* truth, const uint64_t* pred, const uint8_t* covered,
                  const int64_t* row_off, int P, int L, int E, int warmup, int64_t cap,
                  int budget, int unbounded, int policy, int64_t* counters,
                  int64_t* per_prompt, uint64_t* hit_masks) {
  if (cap < 1 || L < 1 || E < 1 || budget < 1 || warmup < 0) return ORC_EINVAL;
  const int W = words_for(E);
  memset(counters, 0, sizeof(int64_t) * (size_t)(4 + 3 * L));
  for (int p = 0; p < P; ++p) {
    orc_cache c;
    if (cache_init(&c, cap, policy, (int64_t)L * E) != ORC_OK) return ORC_ENOMEM;
    int64_t pc[4] = {0, 0, 0, 0};
    for (int64_t r = row_off[p]; r < row_off[p + 1]; ++r) {
      const int64_t local = r - row_off[p];
      const int t = (int)(local / L), l = (int)(local % L);
      const uint64_t* tm = truth + r * W;
      uint64_t* hm = hit_masks ? hit_masks + r * W : NULL;
      if (hm) memset(hm, 0, sizeof(uint64_t) * (size_t)W);
      if (t < warmup) { /* engine.py:160-167 */
        for (int e = 0; e < E; ++e)
          if (bit_get(tm, e) && cache_touch(&c, l * E + e) && hm) bit_set(hm, e);
        continue;
      }
      const uint64_t* pm = pred ? pred + r * W : NULL;
      cache_begin_step(&c); /* engine.py:172 */
      int taken = 0;        /* sorted(predicted)[:budget] (engine.py:173-174) */
      if (pm)
        for (int e = 0; e < E; ++e) {
          if (!bit_get(pm, e)) continue;
          if (!unbounded && taken >= budget) break;
          cache_prefetch_one(&c, l * E + e);
          taken++;
        }
      if (covered && !covered[r]) { /* engine.py:175-176 */
        counters[3]++;
        pc[3]++;
      }
      int64_t k = 0, ch = 0, ph = 0; /* engine.py:178-191 */
      for (int e = 0; e < E; ++e) {
        if (!bit_get(tm, e)) continue;
        k++;
        if (pm && bit_get(pm, e)) ph++;
        if (cache_touch(&c, l * E + e)) {
          ch++;
          if (hm) bit_set(hm, e);
        }
      }
      counters[0] += k;
      counters[1] += ch;
      counters[2] += ph;
      counters[4 + l] += k;
      counters[4 + L + l] += ch;
      counters[4 + 2 * L + l] += ph;
      pc[0] += k;
      pc[1] += ch;
      pc[2] += ph;
    }
    if (per_prompt) memcpy(per_prompt + 4 * (int64_t)p, pc, sizeof(pc));
    cache_free(&c);
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Selection: top_k_experts (learner.py:164-169), threshold (:177-181).      */
/* ------------------------------------------------------------------------ */

/* k highest scores, ties to the lower expert id; written as a selection loop
 * over the reference's lexsort order. */
static void select_topk(const double* z, int E, int k, uint64_t* out) {
  const int W = words_for(E);
  memset(out, 0, sizeof(uint64_t) * (size_t)W);
  if (k > E) k = E;
  for (int j = 0; j < k; ++j) {
    int best = -1;
    for (int e = 0; e < E; ++e) {
      if (bit_get(out, e)) continue;
      if (best < 0 || z[e] > z[best]) best = e;
    }
    bit_set(out, best);
  }
}

static void select_threshold(const double* z, int E, uint64_t* out) {
  const int W = words_for(E);
  memset(out, 0, sizeof(uint64_t) * (size_t)W);
  for (int e = 0; e < E; ++e)
    if (z[e] > 0.0) bit_set(out, e);
}

/* Mask head on a logits table (fp32 or fp64 input widened to fp64). */
int orc_mask_head_f32(const float* logits, int64_t rows, int E, int k, int threshold,
                      uint64_t* masks) {
  const int W = words_for(E);
  double* z = (double*)malloc(sizeof(double) * (size_t)E);
  if (!z) return ORC_ENOMEM;
  for (int64_t r = 0; r < rows; ++r) {
    for (int e = 0; e < E; ++e) z[e] = (double)logits[r * E + e];
    if (threshold)
      select_threshold(z, E, masks + r * W);
    else
      select_topk(z, E, k, masks + r * W);
  }
  free(z);
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* learned_linear (predictors.py:245-268, learner.py:52-72).                */
/* ------------------------------------------------------------------------ */

/* For every row: f = [onehot_L(l) | history[l] | 1] (learner.py:52-59),
 * z = W f (predictors.py:265) as a plain left-to-right fp64 dot, then top-k
 * (budget) or z > 0. After the row, history[l] = decay*history[l] + x
 * (learner.py:62-72). W is [E][L+E+1] row-major fp64 (LinearModel.weights).
 * logits [rows][E] fp64 nullable. */
int orc_linear_predict(const uint64_t* truth, const int64_t* row_off, int P, int L, int E,
                       const double* Wt, double decay, int budget, int threshold,
                       uint64_t* pred, double* logits) {
  const int W = words_for(E);
  const int F = L + E + 1;
  double* hist = (double*)malloc(sizeof(double) * (size_t)L * E);
  double* f = (double*)malloc(sizeof(double) * (size_t)F);
  double* z = (double*)malloc(sizeof(double) * (size_t)E);
  if (!hist || !f || !z) return ORC_ENOMEM;
  for (int p = 0; p < P; ++p) {
    memset(hist, 0, sizeof(double) * (size_t)L * E);
    for (int64_t r = row_off[p]; r < row_off[p + 1]; ++r) {
      const int l = (int)((r - row_off[p]) % L);
      memset(f, 0, sizeof(double) * (size_t)F);
      f[l] = 1.0;
      memcpy(f + L, hist + (int64_t)l * E, sizeof(double) * (size_t)E);
      f[F - 1] = 1.0;
      for (int e = 0; e < E; ++e) {
        double acc = 0.0;
        for (int j = 0; j < F; ++j) acc += Wt[(int64_t)e * F + j] * f[j];
        z[e] = acc;
      }
      if (logits) memcpy(logits + r * E, z, sizeof(double) * (size_t)E);
      if (threshold)
        select_threshold(z, E, pred + r * W);
      else
        select_topk(z, E, budget, pred + r * W);
      /* update_history: multiply first, then add 1.0 per fired expert */
      double* h = hist + (int64_t)l * E;
      for (int e = 0; e < E; ++e) h[e] = h[e] * decay;
      for (int e = 0; e < E; ++e)
        if (bit_get(truth + r * W, e)) h[e] = h[e] + 1.0;
    }
  }
  free(hist);
  free(f);
  free(z);
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Metrics (metrics.py:12-79) over the measured rows of every prompt.        */
/* out[3E + 3] = TP[E], FP[E], FN[E], n_positions, exact_matches,            */
/*               label_correct                                               */
/* ------------------------------------------------------------------------ */
int orc_metrics(const uint64_t* pred, const uint64_t* truth, const int64_t* row_off, int P,
                int L, int E, int warmup, int64_t* out) {
  const int W = words_for(E);
  memset(out, 0, sizeof(int64_t) * (size_t)(3 * E + 3));
  for (int p = 0; p < P; ++p) {
    for (int64_t r = row_off[p] + (int64_t)warmup * L; r < row_off[p + 1]; ++r) {
      const uint64_t* pm = pred + r * W;
      const uint64_t* tm = truth + r * W;
      int equal = 1, mismatches = 0;
      for (int e = 0; e < E; ++e) {
        int a = bit_get(pm, e), b = bit_get(tm, e);
        if (a && b) out[e]++;
        if (a && !b) out[E + e]++;
        if (!a && b) out[2 * E + e]++;
        if (a != b) {
          equal = 0;
          mismatches++;
        }
      }
      out[3 * E] += 1;
      out[3 * E + 1] += equal;
      out[3 * E + 2] += E - mismatches;
    }
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* EAM cosine matcher (sketches.py:165-184, predictors.py:142-174).          */
/* ------------------------------------------------------------------------ */

/* Per measured row: query = normalize(partial rEAM) (core.py:221-231) over all
 * rows of the prompt before this one; idx = argmax_s U_s . q (first max; zero
 * query -> 0); prediction = top-`budget` strictly positive weights of the RAW
 * sketch block at the row's layer, ties to the lower id (_top_weights,
 * predictors.py:142-148). The scan is maintained incrementally per changed
 * layer row exactly as CosineMatchSession does (predictors.py:177-219), which
 * is the form replay_prompt and collect_prediction_sets use.
 * U = sketches / ||sketch|| with zero rows left at zero (sketches.py:157-160).
 * sketches [S][L*E] fp64. idx_out [rows] (nullable; -1 on warm-up rows),
 * pred [rows][W]. */
int orc_eam_predict(const uint64_t* truth, const int64_t* row_off, int P, int L, int E,
                    int warmup, const double* sketches, int S, int budget, int32_t* idx_out,
                    uint64_t* pred) {
  const int W = words_for(E);
  const int64_t D = (int64_t)L * E;
  double* unit = (double*)malloc(sizeof(double) * (size_t)(S * D));
  int64_t* counts = (int64_t*)malloc(sizeof(int64_t) * (size_t)D);
  double* query = (double*)malloc(sizeof(double) * (size_t)D);
  double* dots = (double*)malloc(sizeof(double) * (size_t)S);
  double* delta = (double*)malloc(sizeof(double) * (size_t)E);
  int64_t* sums = (int64_t*)malloc(sizeof(int64_t) * (size_t)L);
  int64_t* seen = (int64_t*)malloc(sizeof(int64_t) * (size_t)L);
  if (!unit || !counts || !query || !dots || !delta || !sums || !seen) return ORC_ENOMEM;
  for (int s = 0; s < S; ++s) {
    double n2 = 0.0;
    for (int64_t d = 0; d < D; ++d) n2 += sketches[s * D + d] * sketches[s * D + d];
    double nrm = sqrt(n2);
    if (!(nrm > 0)) nrm = 1.0;
    for (int64_t d = 0; d < D; ++d) unit[s * D + d] = sketches[s * D + d] / nrm;
  }
  for (int p = 0; p < P; ++p) {
    memset(counts, 0, sizeof(int64_t) * (size_t)D);
    memset(query, 0, sizeof(double) * (size_t)D);
    memset(dots, 0, sizeof(double) * (size_t)S);
    memset(sums, 0, sizeof(int64_t) * (size_t)L);
    memset(seen, 0, sizeof(int64_t) * (size_t)L);
    double qsq = 0.0;
    for (int64_t r = row_off[p]; r < row_off[p + 1]; ++r) {
      const int64_t local = r - row_off[p];
      const int t = (int)(local / L), l = (int)(local % L);
      if (t >= warmup) {
        for (int ll = 0; ll < L; ++ll) { /* _refresh (predictors.py:202-210) */
          if (sums[ll] == seen[ll]) continue;
          double nn = 0.0, oo = 0.0;
          for (int e = 0; e < E; ++e) {
            double nv = (double)counts[ll * E + e] / (double)sums[ll];
            double ov = query[ll * E + e];
            delta[e] = nv - ov;
            nn += nv * nv;
            oo += ov * ov;
            query[ll * E + e] = nv;
          }
          for (int s = 0; s < S; ++s) {
            double acc = 0.0;
            for (int e = 0; e < E; ++e) acc += unit[s * D + ll * E + e] * delta[e];
            dots[s] += acc;
          }
          qsq += nn - oo;
          seen[ll] = sums[ll];
        }
        int idx = 0; /* predictors.py:214-217 */
        if (qsq > 0.0)
          for (int s = 1; s < S; ++s)
            if (dots[s] > dots[idx]) idx = s;
        if (idx_out) idx_out[r] = idx;
        const double* blk = sketches + (int64_t)idx * D + (int64_t)l * E;
        uint64_t* out = pred + r * W;
        memset(out, 0, sizeof(uint64_t) * (size_t)W);
        for (int j = 0; j < budget; ++j) { /* _top_weights on the raw block */
          int best = -1;
          for (int e = 0; e < E; ++e) {
            if (bit_get(out, e) || !(blk[e] > 0.0)) continue;
            if (best < 0 || blk[e] > blk[best]) best = e;
          }
          if (best < 0) break;
          bit_set(out, best);
        }
      } else {
        if (idx_out) idx_out[r] = -1;
        memset(pred + r * W, 0, sizeof(uint64_t) * (size_t)W);
      }
      for (int e = 0; e < E; ++e) /* ActivationMatrix.accumulate (core.py:182-194) */
        if (bit_get(truth + r * W, e)) {
          counts[(int64_t)l * E + e]++;
          sums[l]++;
        }
    }
  }
  free(unit);
  free(counts);
  free(query);
  free(dots);
  free(delta);
  free(sums);
  free(seen);
  return ORC_OK;
}
