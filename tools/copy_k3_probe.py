"""Which side slows down when the e2e leg's H2D copy runs beside K3t: each
stream timed with its own events."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_17137_b200 as m  # noqa: E402

m.load_library()
shape = m.ModelShape(26, 64, 6)
packed = m.generate_packed(m.GeneratorConfig(6994, 363, shape, 8, 0.9, 7))
ranks = m.masks_to_ranks(packed.truth, 6, 64, packed=True)
host = ranks.cpu().pin_memory()
dev = torch.empty_like(ranks)
w = np.random.default_rng(0).normal(0.0, 0.01, (64, 91))
model = m.LinearModel(shape, m.LearnerConfig(epochs=0), w, trained=True)
pred = m.make_predictor("learned_linear", shape, model=model)
cnt = torch.zeros(54, dtype=torch.int64, device="cuda")
out = torch.empty_like(packed.truth)
sc, sk = torch.cuda.Stream(), torch.cuda.Stream()
pred.predict_masks(packed, 6, 8, counts=cnt, out=out)
torch.cuda.synchronize()
for rep in range(4):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    torch.cuda.synchronize()
    with torch.cuda.stream(sc):
        ev[0].record(sc)
        dev.copy_(host, non_blocking=True)
        ev[1].record(sc)
    with torch.cuda.stream(sk):
        ev[2].record(sk)
        pred.predict_masks(packed, 6, 8, counts=cnt, out=out)
        ev[3].record(sk)
    torch.cuda.synchronize()
    print(f"together: copy {ev[0].elapsed_time(ev[1]):.3f} ms, K3t {ev[2].elapsed_time(ev[3]):.3f} ms")
    for name, fn, s in (("copy alone", lambda: dev.copy_(host, non_blocking=True), sc),
                        ("K3t alone", lambda: pred.predict_masks(packed, 6, 8, counts=cnt, out=out), sk)):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            a.record(s)
            fn()
            b.record(s)
        torch.cuda.synchronize()
        print(f"  {name} {a.elapsed_time(b):.3f} ms")
