"""K3 (fp64 SIMT) vs K3t (tensor cores) on the C2 bench workload: per-call
device time (CUDA events, after warm-up), ambiguous rows, mask equality."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_17137_b200 as m  # noqa: E402


def main():
    P = int(sys.argv[1]) if len(sys.argv) > 1 else 6994
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 363
    m.load_library()
    shape = m.ModelShape(26, 64, 6)
    packed = m.generate_packed(m.GeneratorConfig(P, T, shape, 8, 0.9, 7))
    w = np.random.default_rng(0).normal(0.0, 0.01, (64, 91))
    model = m.LinearModel(shape, m.LearnerConfig(epochs=0), w, trained=True)
    pred = m.make_predictor("learned_linear", shape, model=model)
    res = {}
    for mode in ("tc", "fp64"):
        if mode == "fp64":
            os.environ["MOEB_K3"] = "fp64"
        else:
            os.environ.pop("MOEB_K3", None)
        cnt = torch.zeros(2 + 2 * 26, dtype=torch.int64, device="cuda")
        for _ in range(3):
            masks = pred.predict_masks(packed, 6, 8, counts=cnt)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            masks = pred.predict_masks(packed, 6, 8, counts=cnt)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        amb = pred.ambiguous_rows() if mode == "tc" else None
        res[mode] = (masks.clone(), float(np.median(ts)), amb)
        print(mode, "ms median", round(float(np.median(ts)), 3), "min", round(min(ts), 3),
              "ambiguous", amb, flush=True)
    print("masks equal:", torch.equal(res["tc"][0], res["fp64"][0]))


if __name__ == "__main__":
    main()
