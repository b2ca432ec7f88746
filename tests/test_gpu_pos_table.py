"""The exact LRU kernel with its key -> queue-position table in global memory
(the caller's workspace, `moeb_cache_sim_workspace_bytes_shape`; used for
shapes with more than 8192 keys such as DeepSeek-V3's 58 x 256) gives exactly
the counters, per-prompt counters and hit masks of the shared-memory table
(`MOEB_K1_POS=smem`) and of the C oracle, for LRU and for LFU (its key ->
slot table): lru_only, budgeted and unbounded
prediction streams, capacities from 1 to all keys, ragged prompts, warm-up 0
and 8."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _packed(m, shape, prompts, tokens, seed, ragged):
    packed = m.generate_packed(m.GeneratorConfig(prompts, tokens, shape, 16, 0.9, seed))
    if not ragged:
        return packed
    L, W = shape.num_layers, shape.mask_words
    truth_all = packed.truth.reshape(-1, W)
    rows, off = [], [0]
    for p in range(packed.num_prompts):
        T = 1 + (p * 7) % tokens
        r0 = int(packed.row_off_host[p])
        rows.append(truth_all[r0:r0 + T * L])
        off.append(off[-1] + T * L)
    off = np.array(off, dtype=np.int64)
    return m.PackedTraces(shape, torch.cat(rows).contiguous(), torch.from_numpy(off).cuda(), off,
                          np.arange(packed.num_prompts, dtype=np.int64))


@pytest.mark.parametrize("policy", ["lru", "lfu"])
@pytest.mark.parametrize("ragged", [False, True])
@pytest.mark.parametrize("warmup", [0, 8])
def test_global_position_table_equals_shared(policy, ragged, warmup, monkeypatch):
    import paper_2508_17137_b200 as m
    from paper_2508_17137_b200 import _native as nat
    lib = m.load_library()
    L, E, k = 58, 256, 8
    shape = m.ModelShape(L, E, k)
    assert L * E > 8192
    # the workspace query covers the tables once the shape has more than 8192 keys
    assert lib.moeb_cache_sim_workspace_bytes_shape(2, 30, L, E) >= 2 * 30 * L * E * 2
    assert lib.moeb_cache_sim_workspace_bytes_shape(2, 30, 26, 64) == \
        (lib.moeb_cache_sim_workspace_bytes(2, 30) + 255) // 256 * 256
    packed = _packed(m, shape, 16, 32, 11, ragged)
    rows, W = packed.rows, shape.mask_words
    rng = np.random.default_rng(5)
    sparse = rng.integers(0, 2**63 - 1, (rows, W), dtype=np.int64)
    sparse &= rng.integers(0, 2**63 - 1, (rows, W), dtype=np.int64)
    sparse &= rng.integers(0, 2**63 - 1, (rows, W), dtype=np.int64)  # ~1/8 of the experts
    rand = torch.from_numpy(sparse).cuda()
    ones = torch.full((rows, W), -1, dtype=torch.int64, device="cuda")
    caps = [1, 5, 8, 9, 100, 742, 1484, 4000, L * E]
    streams = [(None, None, False), (rand, None, False), (ones, None, True)]
    monkeypatch.setenv("MOEB_K1_POS", "smem")
    want, want_pp, want_h = m.cache_replay(packed, streams, caps, warmup, k, policy,
                                           want_hits=True)
    monkeypatch.delenv("MOEB_K1_POS")
    got, got_pp, got_h = m.cache_replay(packed, streams, caps, warmup, k, policy, want_hits=True)
    got2, got2_pp, _ = m.cache_replay(packed, streams, caps, warmup, k, policy)
    torch.cuda.synchronize()
    assert torch.equal(got, want) and torch.equal(got_pp, want_pp) and torch.equal(got_h, want_h)
    assert torch.equal(got2, want) and torch.equal(got2_pp, want_pp)
    # and the C oracle (lru_only and the budgeted stream) at two capacities
    from oracle import oracle as orc
    truth = packed.truth.cpu().numpy().view(np.uint64)
    off = packed.row_off_host
    for si, pm in ((0, None), (1, sparse.view(np.uint64))):
        for ci in (4, 6):
            c, pp, _ = orc.cache_sim(truth, pm, off, L, E, warmup, caps[ci], k,
                                     policy=("lru", "lfu").index(policy))
            assert np.array_equal(got[si, ci].cpu().numpy(), c), (si, caps[ci])
            assert np.array_equal(got_pp[si, ci].cpu().numpy(), pp), (si, caps[ci])
    del nat
