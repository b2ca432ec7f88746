"""K1 time per capacity on the C2 traces (learned_linear masks), K1s vs the
exact kernel, and how many prompts K1s leaves undecided."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_17137_b200 as m  # noqa: E402

shape = m.ModelShape(26, 64, 6)
packed = m.generate_packed(m.GeneratorConfig(6994, 363, shape, 8, 0.9, 7))
w = np.random.default_rng(0).normal(0.0, 0.01, (64, 91))
pred = m.make_predictor("learned_linear", shape,
                        model=m.LinearModel(shape, m.LearnerConfig(epochs=0), w, trained=True))
gc = torch.zeros((1, 2 + 2 * 26), dtype=torch.int64, device="cuda")
masks = pred.predict_masks(packed, 6, 8, counts=gc[0])
for frac in (0.05, 0.1, 0.15, 0.2, 0.25, 0.3, 0.4, 0.5):
    cap = m.CacheConfig(capacity_fraction=frac).resolve_capacity(shape)
    res = {}
    for mode in ("1", "0"):
        os.environ["MOEB_K1_STACK"] = mode
        for _ in range(2):
            m.cache_replay(packed, [(masks, None, False)], [cap], 8, 6, want_per_prompt=False,
                           given_counts=gc)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        c, _, _ = m.cache_replay(packed, [(masks, None, False)], [cap], 8, 6,
                                 want_per_prompt=False, given_counts=gc)
        e.record()
        torch.cuda.synchronize()
        res[mode] = (s.elapsed_time(e), c[0, 0, 1].item())
    assert res["1"][1] == res["0"][1]
    print(f"cap {cap:4d}: K1s path {res['1'][0]:7.2f} ms   exact {res['0'][0]:7.2f} ms   hits {res['1'][1]}")
