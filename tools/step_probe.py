import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2508_17137_b200 as m
shape = m.ModelShape(26, 64, 6)
packed = m.generate_packed(m.GeneratorConfig(6994, 363, shape, 8, 0.9, 7))
w = np.random.default_rng(0).normal(0.0, 0.01, (64, 91))
pred = m.make_predictor("learned_linear", shape, model=m.LinearModel(shape, m.LearnerConfig(epochs=0), w, trained=True))
pipe = m.PipelinedReplay(packed, 1)
for met in (True, False):
    def step():
        vec = m.metrics.metric_vector(64, "cuda") if met else None
        return pipe.run(pred, [166], 8, 6, metrics=vec)
    for _ in range(3): step()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20): step()
    e.record(); torch.cuda.synchronize()
    print("metrics" if met else "no metrics", s.elapsed_time(e) / 20)
# K3 alone and K1 alone back to back
gc = torch.zeros((1, 54), dtype=torch.int64, device="cuda")
def k3(): return pred.predict_masks(packed, 6, 8, counts=gc[0])
masks = k3()
def k1(): m.cache_replay(packed, [(masks, None, False)], [166], 8, 6, want_per_prompt=False, given_counts=gc)
for f, name in ((k3, "K3"), (k1, "K1")):
    for _ in range(3): f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20): f()
    e.record(); torch.cuda.synchronize()
    print(name, s.elapsed_time(e) / 20)
