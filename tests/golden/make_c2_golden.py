"""Golden counters for the HEADLINE configuration, produced by the reference.

BASELINE configs[1] / bench.py's workload (C2): DeepSeek-V2-Lite shape
26 x 64 top-6, the reference generator (hot set 8, skew 0.9, seed 7) at 363
decode tokens per prompt, learned_linear with the random-init weights
np.random.default_rng(0).normal(0, 0.01, (64, 91)) (learner.py:128-129),
prefetch budget 6, warm-up 8. The sample is the reference arm's own bounded
sample (bench.py --impl reference): prompts 0..255. For every capacity
fraction of the C3 sweep this records what moesim.replay_traces reports
(engine.py:62-110, 222-238) for learned_linear and for lru_only --
aggregate counters, per-layer counters, per-prompt counters -- plus the
integer prediction metrics (TP/FP/FN per expert, exact matches,
label-correct count, positions) behind macro_f1 / position_accuracy /
label_accuracy (metrics.py:12-79) and the reference's own float results.

    python tests/golden/make_c2_golden.py      # ~5 min on 8 cores

Writes tests/golden/c2_sample256.npz (the truth masks are NOT stored: the
test regenerates them with the device generator and checks their sha256).
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import _import_ref, pack  # noqa: E402

FRACTIONS = [0.05, 0.10, 0.15, 0.20, 0.25, 0.30, 0.40, 0.50]
P, T, SEED = 256, 363, 7


def main():
    moesim = _import_ref()
    from moesim.learner import LearnerConfig, LinearModel
    from moesim.metrics import label_accuracy, macro_f1, position_accuracy
    shape = moesim.ModelShape(26, 64, 6)
    traces = moesim.generate_synthetic(moesim.GeneratorConfig(P, T, shape, 8, 0.9, SEED))
    truth, off, _ = pack(traces, shape)
    w = np.random.default_rng(0).normal(0.0, 0.01, (64, 91))
    model = LinearModel(shape, LearnerConfig(epochs=0), w, trained=True)
    jobs = os.cpu_count() or 1
    out = {"fractions": np.array(FRACTIONS), "truth_sha256": np.frombuffer(
        hashlib.sha256(np.ascontiguousarray(truth).tobytes()).digest(), dtype=np.uint8)}
    L = shape.num_layers
    for kind in ("learned_linear", "lru_only"):
        cnt, pp, caps = [], [], []
        for f in FRACTIONS:
            pred = (moesim.make_predictor(kind, shape, model=model) if kind == "learned_linear"
                    else moesim.make_predictor(kind, shape))
            cfg = moesim.ReplayConfig(shape, moesim.CacheConfig(capacity_fraction=f,
                                                                prefetch_budget=6),
                                      warmup_tokens=8)
            t0 = time.perf_counter()
            rep = moesim.replay_traces(traces, pred, cfg, jobs=jobs)
            print(kind, f, rep.cache_hits, rep.measured_accesses, f"{time.perf_counter() - t0:.1f}s",
                  flush=True)
            caps.append(cfg.cache.resolve_capacity(shape))
            cnt.append(np.concatenate([[rep.measured_accesses, rep.cache_hits,
                                        rep.prediction_hits, rep.uncovered_queries],
                                       rep.layer_accesses, rep.layer_cache_hits,
                                       rep.layer_prediction_hits]).astype(np.int64))
            pids = sorted(rep.per_prompt)
            assert pids == list(range(P))
            pp.append(np.array([[rep.per_prompt[p].measured_accesses, rep.per_prompt[p].cache_hits,
                                 rep.per_prompt[p].prediction_hits, 0] for p in pids],
                               dtype=np.int64))
        out[f"counters_{kind}"] = np.stack(cnt)
        out[f"perprompt_{kind}"] = np.stack(pp)
        out["capacities"] = np.array(caps, dtype=np.int64)
    # prediction metrics over every measured step (engine.py:241-272)
    t0 = time.perf_counter()
    cfg = moesim.ReplayConfig(shape, moesim.CacheConfig(capacity_fraction=0.1, prefetch_budget=6),
                              warmup_tokens=8)
    from moesim.engine import collect_prediction_sets
    ps, ts, ls = collect_prediction_sets(
        traces, moesim.make_predictor("learned_linear", shape, model=model), cfg)
    E = shape.num_experts
    tp, fp, fn = np.zeros(E, np.int64), np.zeros(E, np.int64), np.zeros(E, np.int64)
    exact = label = 0
    for p_, t_ in zip(ps, ts):
        for e in p_ & t_:
            tp[e] += 1
        for e in p_ - t_:
            fp[e] += 1
        for e in t_ - p_:
            fn[e] += 1
        exact += p_ == t_
        label += E - len(p_ ^ t_)
    out["metrics_ints"] = np.concatenate([tp, fp, fn, [len(ps), exact, label]]).astype(np.int64)
    out["metrics_floats"] = np.array([macro_f1(ps, ts, E), macro_f1(ps, ts, E, include_all=True),
                                      position_accuracy(ps, ts), label_accuracy(ps, ts, E)])
    print("metrics", out["metrics_floats"], f"{time.perf_counter() - t0:.1f}s")
    np.savez_compressed(os.path.join(HERE, "c2_sample256.npz"), **out)


if __name__ == "__main__":
    main()
