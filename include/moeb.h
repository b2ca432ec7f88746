/*
 * moeb.h -- C ABI of the B200-native MoE-Beyond hot path (libmoeb.so).
 *
 * The reference (`moesim`, pure Python/numpy) has no native FFI: its hot path
 * is a per-step Python callback protocol (predictor.predict(ctx) ->
 * frozenset, ExpertCache.touch/prefetch). A per-step callback cannot be made
 * GPU-native, so this ABI moves the boundary to BATCH granularity: every entry
 * point processes whole packed traces. Each function names the reference
 * interface it replaces (file:line under /root/reference/pkg/src/moesim/).
 * INTEGRATION.md shows the ctypes binding the reference package would add.
 *
 * Conventions
 *  - All array pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors)
 *    unless the parameter says "host". The caller owns all memory: the
 *    library allocates no device or host memory. Scratch space comes from a
 *    caller-provided workspace sized by the matching *_workspace_bytes()
 *    query. Process-wide state is limited to idempotent caches (per-(device,
 *    kernel) function attributes already set, the cuTensorMapEncodeTiled
 *    entry point) and constant tables uploaded once (the generator's PCG64
 *    jump tables); no call's result depends on another call.
 *  - `stream` is a cudaStream_t passed as void*. Calls are stream-ordered and
 *    asynchronous; they return after enqueueing.
 *  - Return 0 on success, a nonzero MOEB_E* code on failure; a thread-local
 *    message is available from moeb_last_error(). Exceptions never cross.
 *  - A trace row is one (prompt, token, layer) step. Rows of prompt p are the
 *    half-open range [prompt_row_off[p], prompt_row_off[p+1]) in (token,
 *    layer) order; every offset is therefore a multiple of L.
 *  - An expert set is a bitmask of W = ceil(E/64) uint64 words per row (bit e
 *    of word e/64 = expert e). E <= 256, L*E <= 65536.
 *  - Counters are int64 and ACCUMULATED (+=) into the output, so results of
 *    several launches (or several GPUs after an all-reduce) simply add.
 */
#ifndef MOEB_H_
#define MOEB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MOEB_OK 0
#define MOEB_EINVAL 1   /* bad argument (shape, range, null pointer) */
#define MOEB_ECUDA 2    /* CUDA launch / runtime error */
#define MOEB_ESMEM 3    /* per-simulation state does not fit in shared memory */
#define MOEB_EDEVICE 4  /* device is not sm_100 (B200) */

#define MOEB_MAX_PREDS 16

/* Cache policies. LRU is the reference's ExpertCache (cache.py:58-154);
 * LFU is builder-defined, parity unpinned. */
#define MOEB_POLICY_LRU 0
#define MOEB_POLICY_LFU 1

const char* moeb_last_error(void);
int moeb_version(void);
/* 0 if the current device is sm_100 and the kernels are loadable. */
int moeb_device_check(void);

/*
 * K1 -- prediction-guided cache replay.
 * Replaces engine.replay_prompt / replay_traces (engine.py:113-238) with the
 * ExpertCache protocol (cache.py:93-154): per prompt, warm-up rows touch the
 * truth experts; measured rows run begin_step, prefetch(sorted(pred)[:budget]
 * or all when unbounded), then touch every truth expert in ascending order.
 * One simulation per (pred stream, capacity, prompt); all run concurrently.
 *
 *  truth            [rows][W]
 *  preds            host array [n_preds] of device pointers [rows][W];
 *                   a NULL entry means the empty prediction (lru_only)
 *  covered          host array [n_preds] of device pointers [rows] uint8 or
 *                   NULL (external predictor coverage, engine.py:175-176)
 *  unbounded        host array [n_preds] (predictor.unbounded_prefetch)
 *  capacities       host array [n_caps] of resolved entry counts
 *                   (CacheConfig.resolve_capacity, cache.py:52-55)
 *  counters         [n_preds][n_caps][4 + 3L] += measured_accesses,
 *                   cache_hits, prediction_hits, uncovered_queries,
 *                   layer_accesses[L], layer_cache_hits[L],
 *                   layer_prediction_hits[L]          (engine.py:62-110)
 *  per_prompt       [n_preds][n_caps][n_prompts][4] (nullable) +=
 *                   measured_accesses, cache_hits, prediction_hits, uncovered
 *  hit_masks        [n_preds][n_caps][rows][W] (nullable): bit e set iff the
 *                   touch of truth expert e hit (warm-up rows included)
 *  rows             host: prompt_row_off[n_prompts] (total trace rows)
 *  workspace        [workspace_bytes] scratch, >= moeb_cache_sim_workspace_bytes
 *                   (n_preds, n_prompts) for the stack-distance replay K1s (its
 *                   undecided-prompt list); NULL / smaller -> every prompt is
 *                   replayed by the exact kernel (same results, slower).
 *                   >= moeb_cache_sim_workspace_bytes_shape(n_preds, n_prompts,
 *                   L, E): also the LRU key -> queue-position tables of shapes
 *                   with more than 8192 keys (V3: 58 x 256) in global memory,
 *                   so that more simulations fit each SM (same results)
 *  Limit: every prompt has fewer than 2^31 - 64 rows (the caller checks).
 */
size_t moeb_cache_sim_workspace_bytes(int n_preds, int n_prompts);
size_t moeb_cache_sim_workspace_bytes_shape(int n_preds, int n_prompts, int L, int E);
int moeb_cache_sim(const uint64_t* truth, const uint64_t* const* preds,
                   const uint8_t* const* covered, const int32_t* unbounded, int n_preds,
                   const int64_t* prompt_row_off, int n_prompts, int L, int E,
                   int warmup_tokens, const int64_t* capacities, int n_caps, int budget,
                   int policy, int64_t* counters, int64_t* per_prompt, uint64_t* hit_masks,
                   int64_t rows, void* workspace, size_t workspace_bytes, void* stream);

/*
 * moeb_cache_sim with the cache-independent counters supplied by the caller:
 * given_counts [n_preds][2 + 2L] = measured accesses, prediction hits, then
 * per layer of each (e.g. from moeb_linear_predict_counts over the same rows
 * and warm-up). The fast LRU kernel then skips computing them and adds these
 * instead; every other kernel (LFU, coverage / hit-mask outputs, per-prompt
 * counters) ignores them. Results are identical to moeb_cache_sim's.
 */
int moeb_cache_sim_counted(const uint64_t* truth, const uint64_t* const* preds,
                           const uint8_t* const* covered, const int32_t* unbounded, int n_preds,
                           const int64_t* prompt_row_off, int n_prompts, int L, int E,
                           int warmup_tokens, const int64_t* capacities, int n_caps, int budget,
                           int policy, int64_t* counters, int64_t* per_prompt,
                           uint64_t* hit_masks, const int64_t* given_counts, int64_t rows,
                           void* workspace, size_t workspace_bytes, void* stream);

/*
 * K1m -- exact LRU replay of every capacity in one pass by stack distances
 * (E <= 64, prompts of <= 32768 rows, no coverage / hit-mask output). Valid
 * when every capacity exceeds the keys prefetched in any row (C > budget, or
 * C > E for an unbounded stream): then no pin binds and nothing is rejected
 * (cache.py:93-154), and a touch hits iff it was prefetched in its row or
 * fewer than C distinct keys were accessed since its previous access.
 * Counters as moeb_cache_sim (+=), for n_caps <= 16 capacities in ascending order;
 * max_prompt_rows sizes the per-prompt shared-memory state. max_row_keys: an
 * upper bound on the experts of any truth row (ModelShape.top_k for validated
 * traces; 0 = unknown): with budget + max_row_keys <= 15 and MOEB_K1M_NIB=1
 * the per-row key counts are kept as 4-bit fields (half the shared memory,
 * same results).
 * workspace (nullable, >= moeb_cache_replay_stack_workspace_bytes(n_preds,
 * n_prompts, L) bytes): the per-key last-access tables live there instead of
 * in shared memory, so more prompts are replayed per SM (same results).
 */
size_t moeb_cache_replay_stack_workspace_bytes(int n_preds, int n_prompts, int L);
int moeb_cache_replay_stack(const uint64_t* truth, const uint64_t* const* preds,
                            const int32_t* unbounded, int n_preds, const int64_t* prompt_row_off,
                            int n_prompts, int L, int E, int warmup_tokens,
                            const int64_t* capacities, int n_caps, int budget,
                            int64_t max_prompt_rows, int max_row_keys, int64_t* counters,
                            int64_t* per_prompt, void* workspace, size_t workspace_bytes,
                            void* stream);

/*
 * ExpertCache op stream (cache.py:58-154) for one cache, executed on device:
 * ops[i] = 0 begin_step, 1 touch(keys[i]), 2 prefetch([keys[i]]).
 * results[i] = touch hit / prefetch inserted. keys = layer*E + expert.
 * Used for the reference's per-call API and its known-answer tests.
 */
int moeb_cache_ops(const int32_t* ops, const int32_t* keys, int64_t n, int L, int E,
                   int64_t capacity, int policy, uint8_t* results, void* stream);

/*
 * K3 (+K2 +K7 fused) -- learned_linear predictor over whole traces.
 * Replaces LearnedLinearPredictor.predict (predictors.py:262-268) with
 * feature_vector / update_history (learner.py:52-72) and top_k_experts /
 * threshold selection (learner.py:164-181). E <= 64.
 *  weights     [E][L+E+1] fp64 (LinearModel.weights)
 *  pred        [rows][W] predicted masks (every row; warm-up rows included)
 *  logits      [rows][E] fp64 (nullable)
 *  metrics     [3E+3] (nullable) += TP[E], FP[E], FN[E], positions,
 *              exact matches, label-correct over rows with token >= warmup
 *              (metrics.py:12-79)
 */
int moeb_linear_predict(const uint64_t* truth, const int64_t* prompt_row_off, int n_prompts,
                        int L, int E, const double* weights, double decay, int budget,
                        int threshold, int warmup_tokens, uint64_t* pred, double* logits,
                        int64_t* metrics, void* stream);
/* moeb_linear_predict that also accumulates, over rows with token >= warmup,
 * counts [2 + 2L] (nullable) += sum |truth|, sum |truth & pred|, then the
 * same per layer (the replay's measured accesses and prediction hits,
 * engine.py:175-200).
 *  top_k       experts per trace row (ModelShape.top_k; rows are validated
 *              to hold exactly top_k, core.py:84-104). Only sizes the fast
 *              path's error bound; a row with more ids is still exact (its
 *              stream falls back to fp64). 0 = unknown (bound for E).
 *  rows        host: prompt_row_off[n_prompts]
 *  workspace   >= moeb_linear_workspace_bytes(rows, L, E) enables K3t (E =
 *              64, L <= 32, budget <= 16, logits == NULL): tensor-core
 *              column sums and fp32 scores with a rigorous error bound, the
 *              rows it cannot decide re-evaluated in fp64 -- masks identical
 *              to the fp64 kernel's. NULL -> the fp64 kernel. */
size_t moeb_linear_workspace_bytes(int64_t rows, int L, int E);
/* Diagnostics: out[0] (device int64) = the number of rows the last K3t call
 * on this workspace re-evaluated in fp64 (> list capacity: the whole call
 * was redone by the fp64 kernel). */
int moeb_linear_ambiguous_rows(const void* workspace, int L, int64_t* out, void* stream);
int moeb_linear_predict_counts(const uint64_t* truth, const int64_t* prompt_row_off,
                               int n_prompts, int L, int E, const double* weights, double decay,
                               int budget, int threshold, int warmup_tokens, int top_k,
                               uint64_t* pred, double* logits, int64_t* metrics, int64_t* counts,
                               int64_t rows, void* workspace, size_t workspace_bytes,
                               void* stream);

/*
 * Wide K3 for 64 < E <= 256 (DeepSeek-V3: 256 experts), same semantics as
 * moeb_linear_predict. moeb_linear_prepare builds the fp64 tables once per
 * (weights, decay): tables [moeb_linear_table_doubles(L, E)] = W_h transposed
 * [E][E], start scores [L][E] (W[:, l] + bias), (1 - decay) * start [L][E].
 */
size_t moeb_linear_table_doubles(int L, int E);
int moeb_linear_prepare(const double* weights, int L, int E, double decay, double* tables,
                        void* stream);
int moeb_linear_predict_wide(const uint64_t* truth, const int64_t* prompt_row_off,
                             int n_prompts, int L, int E, const double* tables, double decay,
                             int budget, int threshold, int warmup_tokens, uint64_t* pred,
                             double* logits, int64_t* metrics, void* stream);

/*
 * learned_linear training (learner.train, learner.py:75-155).
 * moeb_linear_features: hist [rows][E] fp64 = the decayed history of the
 *   row's layer before the row (training_pairs' feature block), bit-identical.
 * moeb_linear_sgd_epoch: per-example SGD over the rows in `order` (the
 *   host's rng.permutation), weights [E][L+E+1] fp64 updated in place;
 *   *loss_total = sum over examples of the example's mean BCE.
 */
int moeb_linear_features(const uint64_t* truth, const int64_t* prompt_row_off, int n_prompts,
                         int L, int E, double decay, double* hist, void* stream);
int moeb_linear_sgd_epoch(double* weights, const double* hist, const uint64_t* truth,
                          const int64_t* order, int64_t n, int L, int E, double learning_rate,
                          double* loss_total, void* stream);

/*
 * K2 -- mask head: logits -> top-k (ties to lower id) or logit > 0 masks.
 * Replaces top_k_experts / predict_topk (learner.py:164-181). fp32 logits.
 */
int moeb_mask_head(const float* logits, int64_t rows, int E, int k, int threshold,
                   uint64_t* masks, void* stream);

/*
 * K7 -- prediction-quality counters over rows with token >= warmup_tokens.
 * Replaces macro_f1 / position_accuracy / label_accuracy (metrics.py:12-79);
 * the host finishes F1 with the reference's numpy expression.
 *  metrics [3E+3] += TP[E], FP[E], FN[E], positions, exact, label_correct
 */
int moeb_metrics(const uint64_t* pred, const uint64_t* truth, const int64_t* prompt_row_off,
                 int n_prompts, int L, int E, int warmup_tokens, int64_t* metrics,
                 void* stream);

/*
 * Compact trace rows (the host->device wire format of StreamingReplay): k
 * expert ids per row, u8, ascending, 0xff = none, E <= 64 (a row of the
 * reference trace is its sorted expert-id tuple, core.py:64-90).
 *  moeb_ids_to_masks: ids [rows][k] -> masks [rows]; *bad = 1 if an id >= E
 *  moeb_masks_to_ids: masks [rows] -> ids [rows][k]; *bad = 1 if a row has > k
 */
int moeb_ids_to_masks(const uint8_t* ids, int64_t rows, int k, int E, uint64_t* masks, int* bad,
                      void* stream);
int moeb_masks_to_ids(const uint64_t* masks, int64_t rows, int k, uint8_t* ids, int* bad,
                      void* stream);

/*
 * The 4-byte wire format of top-k rows: each row's rank in the combinatorial
 * number system, N = sum_i C(c_i, i) over its ascending expert ids c_1 < ... <
 * c_k (k <= 8, E <= 64, C(E, k) < 2^32; every validated reference row has
 * exactly k ids, core.py:64-90).
 *  moeb_ranks_to_masks: ranks [rows] -> masks [rows]; *bad = 1 if N >= C(E, k)
 *  moeb_masks_to_ranks: masks [rows] -> ranks [rows]; *bad = 1 if a row's
 *                       popcount != k
 */
int moeb_ranks_to_masks(const uint32_t* ranks, int64_t rows, int k, int E, uint64_t* masks,
                        int* bad, void* stream);
int moeb_masks_to_ranks(const uint64_t* masks, int64_t rows, int k, int E, uint32_t* ranks,
                        int* bad, void* stream);
/* The ranks as a bit stream of `bits` (>= ceil(log2 C(E, k))) per row, row r
 * in bits [r bits, (r + 1) bits) of little-endian u32 words: 27 bits = 3.4 B
 * per row for 64 / 6. `words` = ceil(rows bits / 32) + 1 u32; the encoder
 * ORs into it (zero it first). */
int moeb_packed_ranks_to_masks(const uint32_t* words, int64_t rows, int bits, int k, int E,
                               uint64_t* masks, int* bad, void* stream);
int moeb_masks_to_packed_ranks(const uint64_t* masks, int64_t rows, int k, int E, int bits,
                               uint32_t* words, int* bad, void* stream);
/* Packed expert ids: each row's k ascending ids at 6 bits (E <= 64) in a
 * little-endian bit stream, row r in bits [6 k r, 6 k (r + 1)): 4.5 B per row
 * at k = 6, decoded with shifts (`words`: ceil(6 k rows / 32) + 2 u32, zeroed
 * by the caller for the encoder). *bad = 1 if a row does not hold exactly k
 * distinct experts. Host wire format of the end-to-end replay (no reference
 * counterpart: the reference reads rows from CSV, traceio.py:47-106). */
int moeb_ids6_to_masks(const uint32_t* words, int64_t rows, int k, uint64_t* masks, int* bad,
                       void* stream);
int moeb_masks_to_ids6(const uint64_t* masks, int64_t rows, int k, uint32_t* words, int* bad,
                       void* stream);
/* Packed id pairs: the k ascending ids two at a time, each sorted pair
 * (a < b) as C(b, 2) + a in 11 bits (an odd k's last id in 6 bits): 33 bits
 * per row at k = 6, decoded by table lookups. Same stream layout and error
 * behaviour as the packed ids above (bits per row = 11 (k / 2) + 6 (k % 2)). */
int moeb_idpairs_to_masks(const uint32_t* words, int64_t rows, int k, uint64_t* masks, int* bad,
                          void* stream);
int moeb_masks_to_idpairs(const uint64_t* masks, int64_t rows, int k, uint32_t* words, int* bad,
                          void* stream);

/*
 * Rule-based predictors as mask tables (predictors.py:57-139).
 *  kind 0 lru_only (empty), 1 oracle (truth truncated to the `budget` lowest
 *  ids, :80-81), 2 next_layer_all (all E), 3 per-layer table
 *  (global_frequency: table [L][W], :137-139).
 */
int moeb_policy_masks(int kind, const uint64_t* truth, int64_t rows, int L, int E, int budget,
                      const uint64_t* layer_table, uint64_t* out, void* stream);

/*
 * Synthetic traces on device, bit-identical to traceio._generate_prompt
 * (traceio.py:233-283). The host supplies, per prompt, the PCG64 state after
 * the hot-key and token-id draws (state hi/lo, inc hi/lo) and the ordered hot
 * set hot[p][L][h] (from np.argpartition on the host, traceio.py:255); the
 * device replays the remaining draws (from_hot, hot_pick, uni_pick) with
 * PCG64 jump-ahead and writes truth [P*T*L][W].
 */
int moeb_gen_traces(const uint64_t* pcg_state /*[P][4]*/, const uint8_t* hot /*[P][L][h]*/,
                    int n_prompts, int T, int L, int E, int k, int h, double skew,
                    uint64_t* truth, void* stream);

/*
 * K6 -- EAM cosine predictor (MoE-Infinity baseline) over whole traces.
 * Replaces EamCosinePredictor / CosineMatchSession (predictors.py:151-219)
 * and SketchCollection.match_nearest (sketches.py:165-184).
 *
 * moeb_eam_prepare: from raw sketches [S][L*E] fp64 (SketchCollection
 *   .sketches) compute the unit-norm matrix TRANSPOSED, unit_t [L*E][S]
 *   (sketches / ||row||, zero rows stay zero, sketches.py:157-160), and the
 *   per-(sketch, layer) prediction table topw [S][L][W] = top-`budget`
 *   strictly positive raw weights, ties to the lower id (_top_weights,
 *   predictors.py:142-148, on the raw block sketches.py:186-189).
 * moeb_eam_predict: for every row with token >= warmup: idx = argmax_s
 *   U_s . normalize(partial rEAM before the row) (first max; zero query -> 0,
 *   predictors.py:212-217); pred[row] = topw[idx][layer]; idx_out[row] = idx
 *   (nullable; -1 on warm-up rows, whose pred is 0). S <= 8192.
 */
int moeb_eam_prepare(const double* sketches, int S, int L, int E, int budget, double* unit_t,
                     uint64_t* topw, void* stream);
int moeb_eam_predict(const uint64_t* truth, const int64_t* prompt_row_off, int n_prompts,
                     int L, int E, int warmup_tokens, const double* unit_t,
                     const uint64_t* topw, int S, int32_t* idx_out, uint64_t* pred,
                     void* stream);

/*
 * K8 -- request-level activation matrices (rEAMs) from packed traces.
 * moeb_ream_counts: counts[p][l*E+e] = activations of expert e at layer l in
 *   prompt p over its first `max_tokens` tokens (all if max_tokens < 0);
 *   ActivationMatrix.from_trace (core.py:196-205).
 * moeb_sketch_normalize: sketches[p] = normalize(counts[p]) (core.py:221-231),
 *   optionally binarized first (sketches._sketch_from_matrix, sketches.py:192-197).
 */
int moeb_ream_counts(const uint64_t* truth, const int64_t* prompt_row_off, int n_prompts, int L,
                     int E, int max_tokens, int32_t* counts, void* stream);
int moeb_sketch_normalize(const int32_t* counts, int n, int L, int E, int binarize,
                          double* sketches, void* stream);

/*
 * Brute-force fp64 nearest-sketch scan for explicit query vectors:
 * SketchCollection.match_nearest (sketches.py:165-184) for M queries at once.
 *  queries [M][D] fp64, unit_t [D][S] (from moeb_eam_prepare).
 *  idx_out [M] = argmax_s unit_s . q/|q| (first max; zero query -> 0),
 *  sim_out [M] = that cosine clipped to [-1, 1] (0 for a zero query).
 */
int moeb_match_queries(const double* queries, int M, int D, const double* unit_t, int S,
                       int32_t* idx_out, double* sim_out, void* stream);

/*
 * K4 -- tcgen05 GEMM (TMA + tensor memory), transformer predictor building
 * block: C[M][N] = A[M][K] . B[N][K]^T, A/B 16-bit (fp16 if `fp16` else
 * bf16), row strides lda/ldb elements, fp32 accumulation, fused epilogue:
 *  0 F32: out32 = C + bias (bias nullable)       1 BIAS: out16 = C + bias
 *  2 BIAS_RELU: out16 = relu(C + bias)             3 BIAS_GELU: gelu (erf)
 *  4 RESID_LN (N == 512): out32 = LayerNorm(out32 + C + bias; ln_w, ln_b,
 *    ln_eps) in place, out16 = 16-bit copy (post-norm encoder sublayer)
 *  5 ROW-MAX (N % 256 == 0): out32 [M][N/256] = max of each 256-column tile
 *    of each row, out16 (as int32) = its first argmax column (m-fastest raster)
 *  6 RESID_ADD: out32 += C + bias (fp32 residual stream, in place; the
 *    post-norm LayerNorm then runs as moeb_layernorm_rows)
 *  7 RESID_ADD16: out16 += C + bias (16-bit residual stream, row stride ld16,
 *    in place; then moeb_layernorm_rows16)
 * K % 64 == 0, N % 64 == 0.
 */
int moeb_gemm(const void* A, int lda, const void* B, int ldb, int M, int N, int K, int fp16,
              int epi, const float* bias, float* out32, void* out16, int ld16,
              const float* ln_w, const float* ln_b, float ln_eps, void* stream);

/*
 * K5 -- windowed multi-head attention of the transformer predictor: qkv
 * [rows][1536] 16-bit (q | k | v, 8 heads x 64), windows (start row, length
 * <= max_len) of consecutive rows, bidirectional with key padding;
 * out [rows][512] 16-bit; rows = the valid rows of qkv (TMA bounds: key
 * chunks past a window's end read the following rows, which must be finite,
 * or zeros past `rows`).
 */
int moeb_window_attention(const void* qkv, void* out, const int64_t* win_start,
                          const int32_t* win_len, int n_windows, int max_len, int64_t rows,
                          int fp16, void* stream);

/* Transformer input rows: out32[r] = ptok[token_ids[r / L]] + play[r % L]
 * (factorised input projection), out16 = 16-bit copy. Rows of 512. out32
 * may be null (the 16-bit residual stream needs only out16). */
int moeb_embed_rows(const float* ptok, const float* play, const int32_t* token_ids, int L,
                    int64_t rows, float* out32, void* out16, int fp16, void* stream);
/* Post-norm LayerNorm of 512-wide rows: x32 = LN(x32; w, b, eps) in place,
 * out16 = 16-bit copy (the next GEMM's operand). */
int moeb_layernorm_rows(float* x32, void* out16, const float* w, const float* b, int64_t rows,
                        float eps, int fp16, void* stream);
/* The 16-bit residual stream's LayerNorm (512 columns, in place): x16 =
 * LayerNorm(x16) with fp32 statistics; pairs with the GEMM epilogue
 * EPI_RESID_ADD16 (out16 += A B^T + bias). */
int moeb_layernorm_rows16(void* x16, const float* w, const float* b, int64_t rows, float eps,
                          int fp16, void* stream);
/* fp32 -> 16-bit (fp16 or bf16) conversion (weight packing). */
int moeb_to16(const float* x, void* y, int64_t n, int fp16, void* stream);

/*
 * K6b -- EAM matching at scale on tensor cores (BASELINE C4): queries are
 * integer activation-count vectors (exact in fp16 up to 2048), sketches are
 * unit-normalised and split U = U_hi + 2^-11 U_lo' into fp16.
 *  moeb_eam_pack_library: sketches [S][D] fp64 -> uu [S_pad][2D] fp16
 *    (rows >= S zero), norms [S] fp64 (sketches.py:157-160)
 *  moeb_eam_pack_queries: counts [M][D] int32 -> cc [M][2D] fp16 [C | C/2048]
 *  then moeb_gemm(cc, uu, M, S_pad, 2D, fp16=1, epi=5 ROW-MAX) writes per
 *    (query, 256-sketch tile) max (pval [M][S_pad/256] fp32) and first argmax
 *  moeb_eam_rerank: exact fp64 re-score of every tile within 2*eps_rel of the
 *    query's approximate max; idx_out [M] = first argmax of unit . q
 *    (zero query -> 0), sim_out [M] cosine (nullable), n_rerank [M] tiles
 *    re-scored (nullable). SketchCollection.match_nearest (sketches.py:165-184).
 */
int moeb_eam_pack_library(const double* sketches, int S, int D, int S_pad, void* uu,
                          double* norms, void* stream);
int moeb_eam_pack_queries(const int32_t* counts, int M, int D, void* cc, void* stream);
int moeb_eam_rerank(const float* pval, const int32_t* pidx, int ntiles, const int32_t* counts,
                    const double* sketches, const double* norms, int M, int S, int D,
                    double eps_rel, int32_t* idx_out, double* sim_out, int32_t* n_rerank,
                    void* stream);

/* C4 queries: for every prompt and token t >= warmup, the partial rEAM counts
 * at layer 0 (all rows of tokens < t); out [sum_p (T_p - warmup)][L*E] int32,
 * prompt p's rows start at query_off[p]. */
int moeb_token_prefix_counts(const uint64_t* truth, const int64_t* prompt_row_off,
                             const int64_t* query_off, int n_prompts, int L, int E,
                             int warmup_tokens, int32_t* out, void* stream);

/*
 * Trace ingestion: the reference's file formats parsed and
 * emitted on device. Byte buffers are device copies of the file; they must be
 * 16-byte aligned and readable up to the next multiple of 16 bytes.
 *
 * moeb_count_bytes / moeb_find_bytes -- ordered positions of every byte equal
 *   to `value` (text.split("\n") in parse_trace_csv / parse_predictions,
 *   traceio.py:58-61, :142). Blocks of MOEB_SCAN_CHUNK bytes;
 *   block_offsets has ceil(n / MOEB_SCAN_CHUNK) + 1 entries: count_bytes
 *   writes the exclusive block offsets and the total (also to *total), and
 *   find_bytes writes positions[0 .. total).
 */
#define MOEB_SCAN_CHUNK 65536
int moeb_count_bytes(const uint8_t* buf, int64_t n, int value, int64_t* block_offsets,
                     int64_t* total, void* stream);
int moeb_find_bytes(const uint8_t* buf, int64_t n, int value, const int64_t* block_offsets,
                    int64_t* positions, void* stream);

/* Line status codes of the device parsers (0 = record OK). */
#define MOEB_LINE_OK 0
#define MOEB_LINE_COLS 1          /* trace csv: not 6 columns */
#define MOEB_LINE_INT_PROMPT 2    /* column prompt_id not an integer */
#define MOEB_LINE_INT_TOKEN 3     /* column token_index not an integer */
#define MOEB_LINE_INT_LAYER 4     /* column layer_id not an integer */
#define MOEB_LINE_EMPTY_EXPERTS 5 /* empty expert_ids */
#define MOEB_LINE_INT_EXPERT 6    /* an expert_ids part not an integer */
#define MOEB_LINE_INT_TOKID 7     /* column token_id not an integer */
#define MOEB_LINE_EMBED 8         /* bad embedding */
#define MOEB_LINE_RANGE_NEG 16    /* TokenRecord.validate: negative prompt/token */
#define MOEB_LINE_RANGE_LAYER 17  /* layer out of range */
#define MOEB_LINE_RANGE_DUPEXP 18 /* duplicate expert ids */
#define MOEB_LINE_RANGE_COUNT 19  /* not top_k expert ids */
#define MOEB_LINE_RANGE_EXPERT 20 /* expert out of range */
#define MOEB_LINE_SKIP 30         /* predictions: blank line (skipped) */
#define MOEB_LINE_HOST 32         /* outside the device grammar (non-ASCII,
                                     > int64, > 32 expert parts, general JSON):
                                     the host parses this line itself */

/*
 * moeb_parse_trace_csv -- parse_trace_csv's per-line loop (traceio.py:64-103):
 * data line i (0-based, file line i + 2) is segment first_segment + i of the
 * newline split (segment j = [nl[j-1]+1, nl[j]) with nl[-1] = -1, the last
 * one ending at n). Python int()/float() grammar (ASCII whitespace, sign,
 * digit underscores; float inf/nan) and TokenRecord.validate (core.py:84-105)
 * in the reference's check order. Per line: status (MOEB_LINE_*), key
 * (prompt_id, token_index, layer_id), expert mask [W], token_id and
 * has_embedding. flags |= 1 if any byte >= 0x80 (UTF-8 check on the host).
 */
int moeb_parse_trace_csv(const uint8_t* buf, int64_t n, const int64_t* nl, int64_t n_nl,
                         int64_t first_segment, int64_t n_lines, int L, int E, int top_k,
                         uint8_t* status, int64_t* prompt_id, int64_t* token_index,
                         int32_t* layer_id, uint64_t* masks, int64_t* token_id,
                         uint8_t* has_embedding, int32_t* flags, void* stream);

/*
 * moeb_parse_predictions -- parse_predictions' per-line loop
 * (traceio.py:142-169) for lines 1..n_lines (segments 0..n_lines-1): blank
 * lines -> MOEB_LINE_SKIP; objects of integer fields prompt_id, token_index,
 * layer_id and an integer array experts (any key order, JSON whitespace) are
 * parsed on device; the expert range check (list order) reports
 * MOEB_LINE_RANGE_EXPERT, then the layer range check MOEB_LINE_RANGE_LAYER.
 * Everything else is MOEB_LINE_HOST (json.loads on the host for that line).
 */
int moeb_parse_predictions(const uint8_t* buf, int64_t n, const int64_t* nl, int64_t n_nl,
                           int64_t n_lines, int L, int E, uint8_t* status, int64_t* prompt_id,
                           int64_t* token_index, int32_t* layer_id, uint64_t* masks,
                           int32_t* flags, void* stream);

/* First index i in [0, n) with status[i] != 0 and != skip_code (n if none) ->
 * *out (device). */
int moeb_first_status(const uint8_t* status, int64_t n, int skip_code, int64_t* out,
                      void* stream);

/* Key order check over rows [0, n) of (a, b, c) int64/int64/int32 keys whose
 * status is 0 (other rows ignored, `status` nullable): out[0] = number of
 * adjacent descents, out[1] = first index i whose key equals the previous
 * counted key (n if none). Sorted input => out[1] is the first duplicate. */
int moeb_keys_check(const int64_t* a, const int64_t* b, const int32_t* c, const uint8_t* status,
                    int skip_code, int64_t n, int64_t* out, void* stream);

/*
 * Prompt grid of sorted, duplicate-free trace rows (PromptTrace.validate,
 * core.py:128-149): starts[p] = first row of prompt p (rows where prompt_id
 * changes; moeb_count_bytes/find_bytes over `flags` from moeb_prompt_flags),
 * then moeb_check_grid: every prompt's rows must be exactly (t, l) for
 * t < T_p, l < L; *bad_prompt = first failing prompt index (P if none).
 */
int moeb_prompt_flags(const int64_t* prompt_id, int64_t n, uint8_t* flags, void* stream);
int moeb_check_grid(const int64_t* starts, int64_t n_prompts, int64_t n_rows,
                    const int64_t* token_index, const int32_t* layer_id, int L,
                    int64_t* bad_prompt, void* stream);

/*
 * External predictions joined onto packed traces (ExternalPredictor,
 * predictors.py:222-242; engine.py:175-176): table rows sorted by (prompt_id,
 * token_index, layer_id); for every trace row, pred = the table's mask and
 * covered = 1, or pred = 0 and covered = 0 when the step is absent.
 */
int moeb_predictions_join(const int64_t* t_prompt, const int64_t* t_token, const int32_t* t_layer,
                          const uint64_t* t_masks, int64_t n_table, const int64_t* prompt_ids,
                          const int64_t* prompt_row_off, int n_prompts, int64_t rows, int L,
                          int E, uint64_t* pred, uint8_t* covered, void* stream);

/*
 * Canonical writers on device. Both first size every line (lens), then the
 * caller runs moeb_exclusive_scan_i64 over lens (offsets, total), then writes.
 * moeb_trace_csv_*: write_trace_csv (traceio.py:113-128) of packed traces
 *   without embeddings: "prompt_id,token_index,layer_id,e1|e2|..,token_id,\n"
 *   (token_ids per trace token, nullable -> 0); header by the caller.
 * moeb_predictions_jsonl_*: write_predictions_jsonl (traceio.py:172-186) of a
 *   table sorted by key: {"prompt_id":p,"token_index":t,"layer_id":l,
 *   "experts":[...]}\n.
 * moeb_exclusive_scan_i64: out[i] = sum(in[0..i)), out[n] = total; ws holds
 *   ceil(n / 4096) + 1 int64.
 */
int moeb_trace_csv_lengths(const uint64_t* truth, const int64_t* prompt_ids,
                           const int64_t* prompt_row_off, int n_prompts, int64_t rows, int L,
                           int E, const int32_t* token_ids, int64_t* lens, void* stream);
int moeb_trace_csv_write(const uint64_t* truth, const int64_t* prompt_ids,
                         const int64_t* prompt_row_off, int n_prompts, int64_t rows, int L,
                         int E, const int32_t* token_ids, const int64_t* offsets, uint8_t* out,
                         void* stream);
int moeb_predictions_jsonl_lengths(const int64_t* t_prompt, const int64_t* t_token,
                                   const int32_t* t_layer, const uint64_t* t_masks, int64_t n,
                                   int E, int64_t* lens, void* stream);
int moeb_predictions_jsonl_write(const int64_t* t_prompt, const int64_t* t_token,
                                 const int32_t* t_layer, const uint64_t* t_masks, int64_t n,
                                 int E, const int64_t* offsets, uint8_t* out, void* stream);
int moeb_exclusive_scan_i64(const int64_t* in, int64_t n, int64_t* out, int64_t* ws,
                            void* stream);

/*
 * EAMC k-means on device (sketches.kmeans, sketches.py:62-139).
 *  moeb_row_sqnorms    out[i] = (X[i] * X[i]).sum() with numpy's pairwise
 *                      summation (bit-identical)
 *  moeb_sqdist_argmin  per vector: first centroid minimising
 *                      max((xn - 2 x.c) + cn, 0) (_squared_distances,
 *                      sketches.py:62-69) and that distance (out_d2 nullable)
 *  moeb_sqdist_update  k-means++: d2 = dist(x, c) (init) or minimum(d2, dist)
 *                      for one centroid c with squared norm *cn (device)
 *  moeb_cluster_means  centroids[j] = mean of the members of cluster j, members
 *                      listed cluster by cluster in index order (members,
 *                      offs [k+1]); empty clusters keep their centroid
 * X [n][D], C [k][D] fp64 row-major.
 */
int moeb_row_sqnorms(const double* X, int64_t n, int64_t D, double* out, void* stream);
int moeb_sqdist_argmin(const double* X, const double* xn, const double* C, const double* cn,
                       int64_t n, int k, int64_t D, int64_t* out_idx, double* out_d2,
                       void* stream);
int moeb_sqdist_update(const double* X, const double* xn, const double* c, const double* cn,
                       int64_t n, int64_t D, int init, double* d2, void* stream);
int moeb_cluster_means(const double* X, const int64_t* members, const int64_t* offs, int k,
                       int64_t D, double* centroids, void* stream);

/*
 * Transformer predictor training: the
 * backward pass and AdamW around the forward kernels. The backward GEMMs are
 * moeb_gemm calls on transposed 16-bit operands (dX = dY W with W^T, dW =
 * dY^T X with the transposed activations); these are the rest. All 16-bit
 * tensors are fp16 when `fp16`, else bf16; gradients of activations carry
 * the loss scale; fp32 outputs accumulate (+=).
 *  moeb_transpose16: out[C][ld_out] = in[R][ld_in]^T
 *  moeb_colsum16: out[N] += sum over rows of in[M][ld] (bias gradients)
 *  moeb_layernorm_bwd16: 512-wide post-norm LayerNorm backward from the
 *    pre-norm rows x16 (statistics recomputed): dx16 = LN'(dy16); dw, db +=
 *  moeb_relu_bwd16: d[i] = 0 where act[i] <= 0
 *  moeb_gelu_fwd16 / moeb_gelu_bwd16: g = gelu(u) (erf); d *= gelu'(u)
 *  moeb_bce_logits_grad: BCEWithLogits(z, bits of truth rows), mean over
 *    M x E: *loss_sum += sum of the element losses, dz16 = (sigmoid(z) - y)
 *    * scale / (M E)
 *  moeb_attention_bwd: windowed attention backward (K5's layout: qkv
 *    [rows][1536], o / dout [rows][512]) -> dqkv [rows][1536]; lse2, dsum
 *    [rows][8] scratch (softmax log2-normaliser, rowsum(dO * O))
 *  moeb_gather_inputs16: F[M][2560] = [tok16[token] | lay16[layer]]
 *  moeb_layer_emb_grad: dlay[layer[r]][c] += d[r][c] (512 columns)
 *  moeb_cast_f32_to_16: y = 16-bit(x)
 *  moeb_sumsq_f32: *out += sum g^2 (fp64)
 *  moeb_adamw_f32: one torch.optim.AdamW step on n parameters, gradient
 *    multiplied by gscale (loss-scale removal x clipping factor)
 */
int moeb_transpose16(const void* in, int64_t R, int C, int ld_in, void* out, int ld_out,
                     void* stream);
int moeb_colsum16(const void* in, int64_t M, int N, int ld, float* out, int fp16, void* stream);
int moeb_layernorm_bwd16(const void* dy16, const void* x16, const float* w, int64_t M, float eps,
                         void* dx16, float* dw, float* db, int fp16, void* stream);
int moeb_relu_bwd16(void* d, const void* act, int64_t n, int fp16, void* stream);
int moeb_gelu_fwd16(const void* u, void* g, int64_t n, int fp16, void* stream);
int moeb_gelu_bwd16(void* d, const void* u, int64_t n, int fp16, void* stream);
int moeb_bce_logits_grad(const float* z, const uint64_t* truth, int64_t M, int E, float scale,
                         void* dz16, double* loss_sum, int fp16, void* stream);
int moeb_attention_bwd(const void* qkv, const void* o, const void* dout, const int64_t* win_start,
                       const int32_t* win_len, int n_windows, int max_len, void* dqkv,
                       float* lse2, float* dsum, int fp16, void* stream);
int moeb_gather_inputs16(const void* tok16, const void* lay16, const int32_t* token,
                         const int32_t* layer, int64_t M, void* F, void* stream);
int moeb_layer_emb_grad(const void* d, int ld, int64_t M, const int32_t* layer, int nl,
                        float* dlay, int fp16, void* stream);
int moeb_cast_f32_to_16(const float* x, int64_t n, void* y, int fp16, void* stream);
int moeb_sumsq_f32(const float* g, int64_t n, double* out, void* stream);
int moeb_adamw_f32(float* p, const float* g, float* m, float* v, int64_t n, float lr, float beta1,
                   float beta2, float eps, float weight_decay, int step, float gscale,
                   void* stream);

#ifdef __cplusplus
}
#endif

#endif /* MOEB_H_ */
