"""Can K3 (learned_linear predict) and K1 (cache replay) share the SMs?

Times, on the C2 workload: K3 / K1 over all prompts; over half of them; and
K1 on half A (high-priority stream, launched first) beside K3 on half B
(low-priority stream). If the pair takes about max(K1(half), K3(half)) the
two kernels' bottlenecks (K1: issue / latency, K3: shared-memory bandwidth)
overlap and a half-batch pipeline pays."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_17137_b200 as m  # noqa: E402
from paper_2508_17137_b200.engine import cache_replay  # noqa: E402

dev = torch.device("cuda", 0)
shape = m.ModelShape(26, 64, 6)
P = int(os.environ.get("P", "6994"))
packed = m.generate_packed(m.GeneratorConfig(P, 363, shape, 8, 0.9, 7), dev)
cap = m.CacheConfig(capacity_fraction=0.1).resolve_capacity(shape)
w = np.random.default_rng(0).normal(0.0, 0.01, (64, 26 + 64 + 1))
pred = m.make_predictor("learned_linear", shape,
                        model=m.LinearModel(shape, m.LearnerConfig(epochs=0), w, trained=True))
halves = [packed.select(0, P // 2), packed.select(P // 2, P)]
hi = torch.cuda.Stream(dev, priority=-1)
lo = torch.cuda.Stream(dev, priority=0)


def k3(pk):
    return pred.predict_masks(pk, 6, 8)


def k1(pk, masks):
    cache_replay(pk, [(masks, None, False)], [cap], 8, 6, "lru", want_per_prompt=False)


def timed(fn, n=3):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


full_m = k3(packed)
hm = [k3(h) for h in halves]
torch.cuda.synchronize()
print(f"K3 all {timed(lambda: k3(packed)):.2f} ms   K1 all {timed(lambda: k1(packed, full_m)):.2f} ms")
print(f"K3 half {timed(lambda: k3(halves[1])):.2f} ms   K1 half {timed(lambda: k1(halves[0], hm[0])):.2f} ms")


def pair():
    main = torch.cuda.current_stream()
    hi.wait_stream(main)
    lo.wait_stream(main)
    with torch.cuda.stream(hi):
        k1(halves[0], hm[0])
    with torch.cuda.stream(lo):
        k3(halves[1])
    main.wait_stream(hi)
    main.wait_stream(lo)


print(f"K1 half A || K3 half B {timed(pair):.2f} ms")


def pair_rev():
    main = torch.cuda.current_stream()
    hi.wait_stream(main)
    lo.wait_stream(main)
    with torch.cuda.stream(hi):
        k3(halves[1])
    with torch.cuda.stream(lo):
        k1(halves[0], hm[0])
    main.wait_stream(hi)
    main.wait_stream(lo)


print(f"K3 half B (high prio) || K1 half A {timed(pair_rev):.2f} ms")
