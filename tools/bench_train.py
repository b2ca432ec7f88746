"""learned_linear training: device SGD vs the reference's train() on the C1
traces (16 prompts x 128 tokens, 26x64 top-6, 53,248 examples per epoch).
    python tools/bench_train.py [--epochs 3]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--epochs", type=int, default=3)
    args = ap.parse_args()
    import numpy as np
    import torch
    import paper_2508_17137_b200 as m
    m.load_library()
    shape = m.ModelShape(26, 64, 6)
    packed = m.generate_packed(m.GeneratorConfig(16, 128, shape, 8, 0.9, 7))
    cfg = m.LearnerConfig(epochs=args.epochs, seed=0)
    m.train(packed.select(0, 1), shape, m.LearnerConfig(epochs=1))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    model = m.train(packed, shape, cfg)
    torch.cuda.synchronize()
    dev_s = time.perf_counter() - t0
    res = {"examples_per_epoch": packed.rows, "epochs": len(model.loss_history),
           "device_s": dev_s, "device_examples_per_s": packed.rows * len(model.loss_history) / dev_s}
    sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
    try:
        import moesim
        from moesim.learner import LearnerConfig, train
        traces = moesim.generate_synthetic(moesim.GeneratorConfig(
            16, 128, moesim.ModelShape(26, 64, 6), 8, 0.9, 7))
        t0 = time.perf_counter()
        ref = train(traces, moesim.ModelShape(26, 64, 6), LearnerConfig(epochs=args.epochs, seed=0))
        ref_s = time.perf_counter() - t0
        res.update(reference_s=ref_s, reference_examples_per_s=packed.rows * args.epochs / ref_s,
                   max_weight_diff=float(np.abs(ref.weights - model.weights).max()),
                   loss_history=model.loss_history, reference_loss_history=ref.loss_history)
    except Exception as exc:  # noqa: BLE001
        res["reference"] = f"unavailable: {exc}"
    print(json.dumps(res))


if __name__ == "__main__":
    main()
