"""Generate golden fixtures by running the REFERENCE (`moesim`) itself.

Run here (the reference is mounted read-only at /root/reference and imports
with plain numpy); the outputs are committed as small .npz files next to this
script so that tests on the GPU box (where /root/reference does not exist)
can check both the CPU oracle and the CUDA path against the reference.

    python tests/golden/make_golden.py

Each case stores, for synthetic traces from the reference generator
(traceio.generate_synthetic):
  truth / row_off / token_ids        packed traces (bitmask rows, W words/row)
  pred_<policy>                      predicted masks from collect_prediction_sets
                                     (engine.py:241-272), zero on warm-up rows
  logits_learned_linear              model.weights @ feature_vector (fp64)
  eamidx                             argmax index per measured row (session form)
  hits_<policy>_c<cap>               per-row cache-hit masks recorded by an
                                     instrumented ExpertCache (every touch,
                                     warm-up included; cache.py:106-124)
  counters_<policy>_c<cap>           SimReport counters (engine.py:62-110)
  perprompt_<policy>_c<cap>          per-prompt counters
  metrics_<policy>                   [macro_f1, macro_f1(include_all),
                                      position_accuracy, label_accuracy]
The predictor policies follow make_predictor (predictors.py:271-303).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _import_ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import moesim  # noqa: F401
    return moesim


def pack(traces, shape):
    L, E = shape.num_layers, shape.num_experts
    W = (E + 63) // 64
    rows, offs, toks = [], [0], []
    for tr in traces:
        for rec in tr.records:
            m = np.zeros(W, dtype=np.uint64)
            for e in rec.expert_ids:
                m[e >> 6] |= np.uint64(1) << np.uint64(e & 63)
            rows.append(m)
        offs.append(offs[-1] + len(tr.records))
        toks.append([tr.records[t * L].token_id for t in range(tr.num_tokens)])
    return (np.array(rows, dtype=np.uint64).reshape(-1, W), np.array(offs, dtype=np.int64),
            np.array(toks, dtype=np.int32))


def sets_to_rows(sets, W):
    out = np.zeros((len(sets), W), dtype=np.uint64)
    for i, s in enumerate(sets):
        for e in s:
            out[i, e >> 6] |= np.uint64(1) << np.uint64(e & 63)
    return out


def measured_rows(traces, shape, warmup):
    idx, base = [], 0
    for tr in traces:
        for j, rec in enumerate(tr.records):
            if rec.token_index >= warmup:
                idx.append(base + j)
        base += len(tr.records)
    return np.array(idx, dtype=np.int64)


def make_case(name, shape_args, gen_args, warmup, budget, capacities, train_gen, eamc_gen,
              eamc_cap, policies, external_prompts=None, decay=0.9, seed_model=0):
    moesim = _import_ref()
    from moesim import engine as eng
    from moesim.cache import CacheConfig, ExpertCache
    from moesim.core import ActivationMatrix, ModelShape
    from moesim.engine import ReplayConfig, collect_prediction_sets, replay_traces
    from moesim.learner import LearnerConfig, LinearModel, feature_vector, update_history
    from moesim.metrics import label_accuracy, macro_f1, position_accuracy
    from moesim.predictors import make_predictor
    from moesim.sketches import EamcConfig, build_eamc
    from moesim.traceio import GeneratorConfig, generate_synthetic

    shape = ModelShape(*shape_args)
    L, E = shape.num_layers, shape.num_experts
    W = (E + 63) // 64
    traces = generate_synthetic(GeneratorConfig(*gen_args[:2], shape, *gen_args[2:]))
    truth, row_off, toks = pack(traces, shape)
    out = dict(truth=truth, row_off=row_off, token_ids=toks,
               shape=np.array([L, E, shape.top_k]), warmup=np.array(warmup),
               budget=np.array(budget), gen=np.array(gen_args, dtype=np.float64),
               decay=np.array(decay))
    mrows = measured_rows(traces, shape, warmup)
    out["measured_rows"] = mrows

    train = generate_synthetic(GeneratorConfig(*train_gen[:2], shape, *train_gen[2:]))
    out["train_gen"] = np.array(train_gen, dtype=np.float64)
    # global_frequency counts (predictors.py:120-135) are recomputed by tests
    # from these packed training traces.
    out["train_truth"], out["train_row_off"], _ = pack(train, shape)
    eamc_traces = generate_synthetic(GeneratorConfig(*eamc_gen[:2], shape, *eamc_gen[2:]))
    mats = [ActivationMatrix.from_trace(t, shape) for t in eamc_traces]
    eamc = build_eamc(mats, EamcConfig(mode="recent", capacity=eamc_cap))
    out["sketches"] = eamc.sketches.copy()

    weights = np.random.default_rng(seed_model).normal(0.0, 0.01, size=(E, L + E + 1))
    model = LinearModel(shape, LearnerConfig(epochs=0, decay=decay, seed=seed_model), weights,
                        trained=True)
    out["weights"] = weights

    table = None
    if external_prompts is not None:
        table = {}
        for tr in traces:
            if tr.prompt_id in external_prompts:
                for rec in tr.records:
                    # a deterministic, imperfect external prediction: truth
                    # shifted by one expert id
                    table[(rec.prompt_id, rec.token_index, rec.layer_id)] = frozenset(
                        (e + 1) % E for e in rec.expert_ids)
        covered = np.zeros(len(truth), dtype=np.uint8)
        base = 0
        for tr in traces:
            for j, rec in enumerate(tr.records):
                covered[base + j] = (rec.prompt_id, rec.token_index, rec.layer_id) in table
            base += len(tr.records)
        out["covered"] = covered
        ext_rows = np.zeros_like(truth)
        base = 0
        for tr in traces:
            for j, rec in enumerate(tr.records):
                s = table.get((rec.prompt_id, rec.token_index, rec.layer_id), frozenset())
                ext_rows[base + j] = sets_to_rows([s], W)[0]
            base += len(tr.records)
        out["external_table"] = ext_rows

    def factory(kind):
        if kind == "oracle":
            return make_predictor("oracle", shape, traces=traces)
        if kind == "lru_only":
            return make_predictor("lru_only", shape)
        if kind == "next_layer_all":
            return make_predictor("next_layer_all", shape)
        if kind == "global_frequency":
            return make_predictor("global_frequency", shape, train_traces=train)
        if kind == "eam_cosine":
            return make_predictor("eam_cosine", shape, eamc=eamc)
        if kind == "learned_linear":
            return make_predictor("learned_linear", shape, model=model)
        if kind == "learned_linear_thr":
            return make_predictor("learned_linear", shape, model=model, threshold=True)
        if kind == "external":
            return make_predictor("external", shape, predictions=table)
        raise ValueError(kind)

    # Per-row logits of the learned model, restated with the reference's own
    # helpers (learner.py:52-72, predictors.py:262-265).
    logits = np.zeros((len(truth), E), dtype=np.float64)
    base = 0
    for tr in traces:
        hist = np.zeros((L, E), dtype=np.float64)
        for j, rec in enumerate(tr.records):
            f = feature_vector(rec.layer_id, hist[rec.layer_id], shape)
            logits[base + j] = model.weights @ f
            update_history(hist, rec.layer_id, rec.expert_ids, decay)
        base += len(tr.records)
    out["logits_learned_linear"] = logits

    # Session argmax per measured row (predictors.py:212-217), via a wrapper
    # around the reference's own session object.
    if "eam_cosine" in policies:
        pred = make_predictor("eam_cosine", shape, eamc=eamc)
        idx_rows = np.full(len(truth), -1, dtype=np.int32)
        base = 0
        for tr in traces:
            sess = pred.new_session()
            ream = ActivationMatrix(shape)
            for j, rec in enumerate(tr.records):
                if rec.token_index >= warmup:
                    sess._refresh(ream)
                    idx_rows[base + j] = 0 if sess._qsq <= 0.0 else int(np.argmax(sess._dots))
                ream.accumulate(rec.layer_id, rec.expert_ids)
            base += len(tr.records)
        out["eamidx"] = idx_rows

    for kind in policies:
        cfg0 = ReplayConfig(shape, CacheConfig(capacity_entries=1, prefetch_budget=budget),
                            warmup_tokens=warmup, history_decay=decay)
        ps, ts, ls = collect_prediction_sets(traces, factory(kind), cfg0)
        prow = np.zeros_like(truth)
        prow[mrows] = sets_to_rows(ps, W)
        out[f"pred_{kind}"] = prow
        out[f"metrics_{kind}"] = np.array([
            macro_f1(ps, ts, E), macro_f1(ps, ts, E, include_all=True),
            position_accuracy(ps, ts), label_accuracy(ps, ts, E)], dtype=np.float64)

        for cap in capacities:
            log = []

            class LoggingCache(ExpertCache):
                def touch(self, key):
                    r = super().touch(key)
                    log.append(r)
                    return r

            saved = eng.ExpertCache
            eng.ExpertCache = LoggingCache
            try:
                cfg = ReplayConfig(shape, CacheConfig(capacity_entries=cap,
                                                      prefetch_budget=budget),
                                   warmup_tokens=warmup, history_decay=decay)
                rep = replay_traces(traces, factory(kind), cfg, jobs=1)
            finally:
                eng.ExpertCache = saved
            hits = np.zeros_like(truth)
            it = iter(log)
            base = 0
            for tr in traces:
                for j, rec in enumerate(tr.records):
                    for e in rec.expert_ids:  # touched in ascending id order
                        if next(it):
                            hits[base + j, e >> 6] |= np.uint64(1) << np.uint64(e & 63)
                base += len(tr.records)
            assert next(it, None) is None
            out[f"hits_{kind}_c{cap}"] = hits
            out[f"counters_{kind}_c{cap}"] = np.concatenate([
                np.array([rep.measured_accesses, rep.cache_hits, rep.prediction_hits,
                          rep.uncovered_queries], dtype=np.int64),
                rep.layer_accesses, rep.layer_cache_hits, rep.layer_prediction_hits])
            assert rep.prediction_opportunities == rep.measured_accesses
            out[f"perprompt_{kind}_c{cap}"] = np.array(
                [[rep.per_prompt[t.prompt_id].measured_accesses,
                  rep.per_prompt[t.prompt_id].cache_hits,
                  rep.per_prompt[t.prompt_id].prediction_hits] for t in traces],
                dtype=np.int64)
    out["policies"] = np.array(policies)
    out["capacities"] = np.array(capacities, dtype=np.int64)
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(truth)} rows, {len(policies)} policies, caps {capacities}")


ALL = ["lru_only", "oracle", "next_layer_all", "global_frequency", "eam_cosine",
       "learned_linear", "learned_linear_thr", "external"]


def main():
    # (3, 8, 2) is the reference test-suite shape (test_engine.py:18).
    make_case("tiny_e8", (3, 8, 2), (5, 14, 3, 0.7, 2), warmup=1, budget=2,
              capacities=[1, 2, 3, 6, 24], train_gen=(4, 10, 3, 0.7, 2, 1000),
              eamc_gen=(6, 10, 3, 0.7, 5, 500), eamc_cap=6, policies=ALL,
              external_prompts={0, 2})
    # DeepSeek-V2-Lite shape (26 MoE layers x 64 experts, top-6), BASELINE C1
    # generator settings (hot 8, skew 0.9, seed 7) on a small prompt set.
    make_case("v2lite_small", (26, 64, 6), (6, 40, 8, 0.9, 7), warmup=8, budget=6,
              capacities=[6, 16, 83, 166, 832, 1664], train_gen=(8, 24, 8, 0.9, 7, 1000),
              eamc_gen=(24, 32, 8, 0.9, 11, 1000000), eamc_cap=24, policies=ALL,
              external_prompts={1, 4})
    # DeepSeek-V3 shape (58 x 256, top-8): 4 mask words per row.
    make_case("v3_small", (58, 256, 8), (2, 14, 16, 0.9, 7), warmup=4, budget=8,
              capacities=[8, 1484], train_gen=(2, 10, 16, 0.9, 7, 1000),
              eamc_gen=(4, 10, 16, 0.9, 11, 1000000), eamc_cap=4,
              policies=["lru_only", "oracle", "next_layer_all", "learned_linear",
                        "learned_linear_thr", "eam_cosine"])


if __name__ == "__main__":
    main()
