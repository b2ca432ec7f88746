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


def test_streaming_compact_ids_equals_masks():
    """Host batches as u8 expert ids (decoded on device) give the counters and
    metrics of the mask batches; ids <-> masks round trip."""
    import paper_2508_17137_b200 as m
    m.load_library()
    shape = m.ModelShape(26, 64, 6)
    b = m.generate_packed(m.GeneratorConfig(50, 30, shape, 8, 0.9, 4))
    ids = m.masks_to_ids(b.truth, 6)
    assert ids.shape == (b.rows, 6) and ids.dtype == torch.uint8
    back = torch.empty_like(b.truth)
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    m.ids_to_masks(ids, 64, back, bad)
    torch.cuda.synchronize()
    assert torch.equal(back, b.truth) and int(bad.item()) == 0
    w = np.random.default_rng(2).normal(0.0, 0.01, (64, 91))
    model = m.LinearModel(shape, m.LearnerConfig(epochs=0), w, trained=True)
    pred = m.make_predictor("learned_linear", shape, model=model)
    sr = m.StreamingReplay(shape, b.row_off_host, b.prompt_ids)
    mask_host = b.truth.cpu().pin_memory()
    id_host = ids.cpu().pin_memory()
    r1 = sr.run(pred, [83, 166], 8, 6, [mask_host, mask_host, mask_host], metrics=True)
    r2 = sr.run(pred, [83, 166], 8, 6, [id_host, id_host, id_host], metrics=True)
    torch.cuda.synchronize()
    assert int(sr.ids_bad.item()) == 0
    for (c1, v1), (c2, v2) in zip(r1, r2):
        assert torch.equal(c1, c2) and torch.equal(v1, v2)
    bad_ids = ids.clone()
    bad_ids[3, 2] = 70
    m.ids_to_masks(bad_ids, 64, back, bad)
    torch.cuda.synchronize()
    assert int(bad.item()) == 1
