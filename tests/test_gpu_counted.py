"""The replay's cache-independent counters fused into K3
(moeb_linear_predict_counts) and consumed by K1 (moeb_cache_sim_counted) give
exactly the counters of the plain replay, for every kernel variant the
replay dispatches to (fast LRU, tiny capacities, per-prompt counters, LFU)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _setup(prompts, tokens, seed, ragged=False):
    import paper_2508_17137_b200 as m
    m.load_library()
    shape = m.ModelShape(26, 64, 6)
    packed = m.generate_packed(m.GeneratorConfig(prompts, tokens, shape, 8, 0.9, seed))
    if ragged:  # prompts of different lengths (9..39 tokens)
        L = shape.num_layers
        truth_all = packed.truth.reshape(-1)
        rows, off = [], [0]
        for p in range(packed.num_prompts):
            T = 9 + (p * 7) % 31
            r0 = int(packed.row_off_host[p])
            rows.append(truth_all[r0:r0 + T * L])
            off.append(off[-1] + T * L)
        off = np.array(off, dtype=np.int64)
        packed = m.PackedTraces(shape, torch.cat(rows).reshape(-1, 1).contiguous(),
                                torch.from_numpy(off).cuda(), off,
                                np.arange(packed.num_prompts, dtype=np.int64))
    w = np.random.default_rng(seed).normal(0.0, 0.01, (64, 91))
    model = m.LinearModel(shape, m.LearnerConfig(epochs=0), w, trained=True)
    return m, shape, packed, m.make_predictor("learned_linear", shape, model=model)


@pytest.mark.parametrize("ragged", [False, True])
@pytest.mark.parametrize("policy", ["lru", "lfu"])
def test_counted_replay_equals_plain(ragged, policy):
    m, shape, packed, pred = _setup(48, 40, 11, ragged)
    L = shape.num_layers
    warmup, budget = 8, 6
    gc = torch.zeros((1, 2 + 2 * L), dtype=torch.int64, device="cuda")
    masks = pred.predict_masks(packed, budget, warmup, counts=gc[0])
    caps = [1, 3, 12, 83, 166, 832]
    want, pp_want, _ = m.cache_replay(packed, [(masks, None, False)], caps, warmup, budget,
                                      policy, want_per_prompt=True)
    got, _, _ = m.cache_replay(packed, [(masks, None, False)], caps, warmup, budget, policy,
                               want_per_prompt=False, given_counts=gc)
    assert torch.equal(got, want)
    # per-prompt counters requested: the counted call falls back to counting itself
    got2, pp2, _ = m.cache_replay(packed, [(masks, None, False)], caps, warmup, budget,
                                  policy, want_per_prompt=True, given_counts=gc)
    assert torch.equal(got2, want) and torch.equal(pp2, pp_want)
    c = want[0, 0].cpu()
    g = gc[0].cpu()
    assert int(g[0]) == int(c[0]) and int(g[1]) == int(c[2])
    assert torch.equal(g[2:2 + L], c[4:4 + L])
    assert torch.equal(g[2 + L:], c[4 + 2 * L:])


def test_pipelines_use_fused_counts():
    """PipelinedReplay / StreamingReplay (which pass the fused counts) match a
    plain replay."""
    m, shape, packed, pred = _setup(60, 30, 5)
    caps = [166]
    plain_masks = pred.predict_masks(packed, 6, 8)
    want, _, _ = m.cache_replay(packed, [(plain_masks, None, False)], caps, 8, 6,
                                want_per_prompt=False)
    vec = torch.zeros(3 * 64 + 3, dtype=torch.int64, device="cuda")
    got = m.PipelinedReplay(packed, 3).run(pred, caps, 8, 6, metrics=vec)
    torch.cuda.synchronize()
    assert torch.equal(got, want)
    sr = m.StreamingReplay(shape, packed.row_off_host, packed.prompt_ids)
    host = packed.truth.cpu().pin_memory()
    res = sr.run(pred, caps, 8, 6, [host, host, host], metrics=True)
    torch.cuda.synchronize()
    for c_h, _ in res:
        assert torch.equal(c_h, want[0].cpu())
