"""StreamingReplay (double-buffered host batches) gives exactly the counters
and metrics of a direct replay of each batch."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_streaming_equals_direct():
    import paper_2508_17137_b200 as m
    m.load_library()
    shape = m.ModelShape(26, 64, 6)
    cfgs = [m.GeneratorConfig(40, 30, shape, 8, 0.9, s) for s in (1, 2, 3)]
    batches = [m.generate_packed(c) for c in cfgs]
    w = np.random.default_rng(0).normal(0.0, 0.01, (64, 91))
    model = m.LinearModel(shape, m.LearnerConfig(epochs=0), w, trained=True)
    pred = m.make_predictor("learned_linear", shape, model=model)
    caps = [83, 166]
    sr = m.StreamingReplay(shape, batches[0].row_off_host, batches[0].prompt_ids)
    hosts = [b.truth.cpu().pin_memory() for b in batches]
    res = sr.run(pred, caps, 8, 6, hosts + hosts[:1], metrics=True)
    torch.cuda.synchronize()
    for i, (c_h, v_h) in enumerate(res):
        b = batches[i % 3]
        vec = torch.zeros(3 * 64 + 3, dtype=torch.int64, device="cuda")
        masks = pred.predict_masks(b, 6, 8, metrics=vec)
        want, _, _ = m.cache_replay(b, [(masks, None, False)], caps, 8, 6, want_per_prompt=False)
        assert torch.equal(c_h, want[0].cpu())
        assert torch.equal(v_h, vec.cpu())
