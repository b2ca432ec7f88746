"""Golden learned_linear training runs from the REFERENCE (moesim.learner.train,
read-only at /root/reference).

    python tests/golden/make_train_golden.py   -> tests/golden/train_cases.npz

Cases: the reference test suite's layer-rule traces (SHAPE 4x8 top-2, default
10 epochs with seed 5 -- early stopping territory -- and 5 epochs seed 1),
and generated synthetic traces (26x64 top-6, 3 epochs; 3x100 top-3, 4
epochs). Stored: packed truth (bit rows), row offsets, final weights, the
epoch loss history, and the training_pairs features of the first case.
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def pack(traces, shape):
    W = (shape.num_experts + 63) // 64
    rows, off = [], [0]
    for tr in traces:
        for rec in tr.records:
            m = np.zeros(W, dtype=np.uint64)
            for e in rec.expert_ids:
                m[e >> 6] |= np.uint64(1) << np.uint64(e & 63)
            rows.append(m)
        off.append(len(rows))
    return np.array(rows, dtype=np.uint64).reshape(-1, W), np.array(off, dtype=np.int64)


def main():
    sys.path.insert(0, REF)
    from moesim import traceio
    from moesim.core import ModelShape, PromptTrace, TokenRecord
    from moesim.learner import LearnerConfig, train, training_pairs

    def layer_rule(shape, P, T):
        out = []
        for p in range(P):
            tr = PromptTrace(p)
            for t in range(T):
                for l in range(shape.num_layers):
                    tr.records.append(TokenRecord(
                        p, t, l, tuple((l + i) % shape.num_experts for i in range(shape.top_k))))
            out.append(tr)
        return out

    small = ModelShape(4, 8, 2)
    cases = [
        ("rule10", small, layer_rule(small, 4, 16), LearnerConfig(seed=5)),
        ("rule5", small, layer_rule(small, 3, 12), LearnerConfig(epochs=5, seed=1)),
        ("v2lite", ModelShape(26, 64, 6), traceio.generate_synthetic(
            traceio.GeneratorConfig(3, 12, ModelShape(26, 64, 6), 8, 0.9, 7)),
         LearnerConfig(epochs=3, seed=7)),
        ("e100", ModelShape(3, 100, 3), traceio.generate_synthetic(
            traceio.GeneratorConfig(4, 10, ModelShape(3, 100, 3), 6, 0.8, 2)),
         LearnerConfig(epochs=4, seed=3, learning_rate=0.2, decay=0.5)),
        ("stop", ModelShape(2, 8, 2), traceio.generate_synthetic(
            traceio.GeneratorConfig(2, 6, ModelShape(2, 8, 2), 3, 0.9, 1)),
         LearnerConfig(epochs=60, seed=2, learning_rate=2.0)),  # early stop after 13 epochs
    ]
    out = {}
    for name, shape, traces, cfg in cases:
        model = train(traces, shape, cfg)
        truth, off = pack(traces, shape)
        out[f"{name}_shape"] = np.array([shape.num_layers, shape.num_experts, shape.top_k])
        out[f"{name}_cfg"] = np.array([cfg.learning_rate, cfg.epochs, cfg.decay, cfg.seed])
        out[f"{name}_truth"] = truth
        out[f"{name}_off"] = off
        out[f"{name}_weights"] = model.weights
        out[f"{name}_loss"] = np.array(model.loss_history)
        if name == "v2lite":
            x, _ = training_pairs(traces, shape, cfg.decay)
            out[f"{name}_hist"] = x[:, shape.num_layers:shape.num_layers + shape.num_experts]
        print(name, len(model.loss_history), model.loss_history[-1])
    np.savez_compressed(os.path.join(HERE, "train_cases.npz"), **out)


if __name__ == "__main__":
    main()
