"""Diagnosis: the bench's device-timed phase (PipelinedReplay over C2 with
metrics and per-prompt counters) with per-step K3 times and K3t's list
counters (rows sent to fp64 re-evaluation / to the refine list)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_17137_b200 as m  # noqa: E402


def main():
    m.load_library()
    shape = m.ModelShape(26, 64, 6)
    packed = m.generate_packed(m.GeneratorConfig(6994, 363, shape, 8, 0.9, 7))
    w = np.random.default_rng(0).normal(0.0, 0.01, (64, 91))
    model = m.LinearModel(shape, m.LearnerConfig(epochs=0), w, trained=True)
    pred = m.make_predictor("learned_linear", shape, model=model)
    pipe = m.PipelinedReplay(packed, 1)

    def step(timing=None):
        vec = m.metrics.metric_vector(64, packed.device)
        return pipe.run(pred, [166], 8, 6, metrics=vec, timing=timing, per_prompt=True)

    t0 = time.time()
    n = 0
    while time.time() - t0 < 2.0:
        step()
        n += 1
    torch.cuda.synchronize()
    k3 = []
    lists = []
    for _ in range(20):
        timing = []
        step(timing)
        torch.cuda.synchronize()
        k3.append(round(timing[0][1].elapsed_time(timing[0][2]), 3))
        ws = pred.last_workspace
        lists.append(pred.ambiguous_rows())
    print("warmup", n, "K3 ms", k3[:6], "median", float(np.median(k3)), "lists", lists[:3],
          "ptr truth", hex(packed.truth.data_ptr()), "ws", hex(pred.last_workspace.data_ptr()))


if __name__ == "__main__":
    main()
