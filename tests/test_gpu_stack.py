"""K1s (stack-distance replay, `k_stack_replay`) + the exact kernel over its
undecided prompts give exactly the exact kernel's counters and per-prompt
counters, with and without upstream (fused) access counts: every capacity
from 1 to all keys, predictions that are empty / learned / over the budget /
unbounded, ragged prompts, warm-up 0 and 8, several geometries."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _packed(m, shape, prompts, tokens, seed, ragged):
    packed = m.generate_packed(m.GeneratorConfig(prompts, tokens, shape, 8, 0.9, seed))
    if not ragged:
        return packed
    L = shape.num_layers
    truth_all = packed.truth.reshape(-1)
    rows, off = [], [0]
    for p in range(packed.num_prompts):
        T = 1 + (p * 7) % tokens
        r0 = int(packed.row_off_host[p])
        rows.append(truth_all[r0:r0 + T * L])
        off.append(off[-1] + T * L)
    off = np.array(off, dtype=np.int64)
    return m.PackedTraces(shape, torch.cat(rows).reshape(-1, 1).contiguous(),
                          torch.from_numpy(off).cuda(), off,
                          np.arange(packed.num_prompts, dtype=np.int64))


def _given(counters, L):
    c = counters[:, 0]
    return torch.cat([c[:, 0:1], c[:, 2:3], c[:, 4:4 + L], c[:, 4 + 2 * L:4 + 3 * L]], 1).contiguous()


@pytest.mark.parametrize("geom", [(26, 64, 6), (3, 64, 2), (5, 40, 4)])
@pytest.mark.parametrize("ragged", [False, True])
@pytest.mark.parametrize("warmup", [0, 8])
def test_stack_replay_equals_exact(geom, ragged, warmup, monkeypatch):
    import paper_2508_17137_b200 as m
    m.load_library()
    L, E, k = geom
    shape = m.ModelShape(L, E, k)
    packed = _packed(m, shape, 45, 60, 3 + L, ragged)
    rng = np.random.default_rng(L + E)
    w = rng.normal(0.0, 0.01, (E, L + E + 1))
    model = m.LinearModel(shape, m.LearnerConfig(epochs=0), w, trained=True)
    learned = m.make_predictor("learned_linear", shape, model=model).predict_masks(packed, k, warmup)
    rows = packed.rows
    wide = torch.from_numpy(rng.integers(0, 2**62, rows, dtype=np.int64)).cuda().reshape(-1, 1)
    wide &= (1 << E) - 1 if E < 64 else -1
    ones = torch.full((rows, 1), (1 << E) - 1 if E < 64 else -1, dtype=torch.int64, device="cuda")
    caps = sorted({1, 2, 5, 12, 20, max(1, L * E // 20), L * E // 10, L * E // 4, L * E // 2,
                   L * E})
    budget = k
    for masks, unbounded in ((learned, False), (None, False), (wide, False), (ones, True)):
        streams = [(masks, None, unbounded)]
        monkeypatch.setenv("MOEB_K1_STACK", "0")
        want, want_pp, _ = m.cache_replay(packed, streams, caps, warmup, budget)
        given = _given(want, L)
        monkeypatch.setenv("MOEB_K1_STACK", "1")
        got, _, _ = m.cache_replay(packed, streams, caps, warmup, budget, want_per_prompt=False,
                                   given_counts=given)
        got_pp, pp, _ = m.cache_replay(packed, streams, caps, warmup, budget)
        torch.cuda.synchronize()
        assert torch.equal(got, want), (masks is None, unbounded)
        assert torch.equal(got_pp, want) and torch.equal(pp, want_pp), (masks is None, unbounded)


@pytest.mark.parametrize("ragged", [False, True])
def test_stack_replay_equals_exact_headline_length(ragged, monkeypatch):
    """The bench's prompt length (C2: 363 decode tokens, 26 x 64 top-6,
    warm-up 8) at every C3 capacity: K1s's bounded look-back (previous-token
    formula, span unions, the per-warp row ring) across long prompts."""
    import paper_2508_17137_b200 as m
    m.load_library()
    shape = m.ModelShape(26, 64, 6)
    L = 26
    packed = _packed(m, shape, 40, 363, 7, ragged)
    w = np.random.default_rng(0).normal(0.0, 0.01, (64, 91))
    model = m.LinearModel(shape, m.LearnerConfig(epochs=0), w, trained=True)
    learned = m.make_predictor("learned_linear", shape, model=model).predict_masks(packed, 6, 8)
    caps = [m.CacheConfig(capacity_fraction=f).resolve_capacity(shape)
            for f in (0.05, 0.10, 0.15, 0.20, 0.25, 0.30, 0.40, 0.50)]
    for masks in (learned, None):
        streams = [(masks, None, False)]
        monkeypatch.setenv("MOEB_K1_STACK", "0")
        want, want_pp, _ = m.cache_replay(packed, streams, caps, 8, 6)
        monkeypatch.setenv("MOEB_K1_STACK", "1")
        got, pp, _ = m.cache_replay(packed, streams, caps, 8, 6)
        torch.cuda.synchronize()
        assert torch.equal(got, want) and torch.equal(pp, want_pp), masks is None
        assert int(want[0, 0, 0]) == sum(6 * L * (int(packed.row_off_host[p + 1] -
                                                   packed.row_off_host[p]) // L - 8)
                                          for p in range(40) if
                                          (packed.row_off_host[p + 1] -
                                           packed.row_off_host[p]) // L > 8)


def test_stack_replay_several_streams(monkeypatch):
    """Several prediction streams in one call (blockIdx.y): per-stream lists
    of undecided prompts and per-stream upstream counts."""
    import paper_2508_17137_b200 as m
    m.load_library()
    shape = m.ModelShape(26, 64, 6)
    L = 26
    packed = _packed(m, shape, 70, 50, 9, True)
    w = np.random.default_rng(4).normal(0.0, 0.01, (64, 91))
    model = m.LinearModel(shape, m.LearnerConfig(epochs=0), w, trained=True)
    learned = m.make_predictor("learned_linear", shape, model=model).predict_masks(packed, 6, 8)
    oracle = packed.truth.clone()
    rng = np.random.default_rng(5)
    noise = torch.from_numpy(rng.integers(0, 2**62, packed.rows, dtype=np.int64)).cuda()
    streams = [(learned, None, False), (oracle, None, False), (noise.reshape(-1, 1), None, False)]
    caps = [3, 83, 166, 400, 1000]
    monkeypatch.setenv("MOEB_K1_STACK", "0")
    want, want_pp, _ = m.cache_replay(packed, streams, caps, 8, 6)
    given = torch.stack([_given(want[i:i + 1], L)[0] for i in range(3)])
    monkeypatch.setenv("MOEB_K1_STACK", "1")
    got, _, _ = m.cache_replay(packed, streams, caps, 8, 6, want_per_prompt=False,
                               given_counts=given)
    got_pp, pp, _ = m.cache_replay(packed, streams, caps, 8, 6)
    torch.cuda.synchronize()
    assert torch.equal(got, want)
    assert torch.equal(got_pp, want) and torch.equal(pp, want_pp)


@pytest.mark.parametrize("geom", [(26, 64, 6), (3, 64, 2), (5, 40, 4)])
@pytest.mark.parametrize("ragged", [False, True])
@pytest.mark.parametrize("warmup", [0, 8])
@pytest.mark.parametrize("variant", ["default", "smem_u8", "nib"])
def test_stack_multi_equals_exact(geom, ragged, warmup, variant, monkeypatch):
    """K1m (every capacity above the prefetch budget in one stack-distance
    pass, moeb_cache_replay_stack) == the exact kernel: counters and
    per-prompt counters, learned / empty (lru_only) / over-budget random /
    unbounded all-ones predictions, several streams per call. Three layouts:
    last-access tables in the caller's global workspace (default), everything
    in shared memory, and 4-bit row counts (opt-in, budget + top-k <= 15)."""
    import paper_2508_17137_b200 as m
    if variant == "smem_u8":
        monkeypatch.setenv("MOEB_K1M_LR", "smem")
    if variant == "nib":  # 4-bit row counts (opt-in)
        monkeypatch.setenv("MOEB_K1M_NIB", "1")
    m.load_library()
    L, E, k = geom
    shape = m.ModelShape(L, E, k)
    packed = _packed(m, shape, 37, 70, 11 + L, ragged)
    rng = np.random.default_rng(L * E)
    w = rng.normal(0.0, 0.01, (E, L + E + 1))
    model = m.LinearModel(shape, m.LearnerConfig(epochs=0), w, trained=True)
    learned = m.make_predictor("learned_linear", shape, model=model).predict_masks(packed, k, warmup)
    rows = packed.rows
    wide = torch.from_numpy(rng.integers(0, 2**62, rows, dtype=np.int64)).cuda().reshape(-1, 1)
    wide &= (1 << E) - 1 if E < 64 else -1
    ones = torch.full((rows, 1), (1 << E) - 1 if E < 64 else -1, dtype=torch.int64, device="cuda")
    keys = L * E
    caps = sorted({k + 1, k + 3, 13, 20, max(k + 1, keys // 20), keys // 10, keys // 4,
                   keys // 2, keys})
    for streams in ([(learned, None, False), (None, None, False), (wide, None, False)],
                    [(ones, None, True)]):
        cs = [c for c in caps if c > (E if streams[0][2] else k)]
        monkeypatch.setenv("MOEB_K1M", "0")
        monkeypatch.setenv("MOEB_K1_STACK", "0")
        want, want_pp, _ = m.cache_replay(packed, streams, cs, warmup, k)
        monkeypatch.setenv("MOEB_K1M", "all")
        monkeypatch.delenv("MOEB_K1_STACK")
        got, got_pp, _ = m.cache_replay(packed, streams, cs, warmup, k)
        torch.cuda.synchronize()
        assert torch.equal(got, want), (len(streams), (got - want).abs().sum().item())
        assert torch.equal(got_pp, want_pp)


def test_stack_multi_headline_sweep(monkeypatch):
    """The C3 sweep's capacities on 363-token prompts: K1m for 15-50 %,
    K1s for 5 / 10 % (the default split) == the exact kernel everywhere."""
    import paper_2508_17137_b200 as m
    m.load_library()
    shape = m.ModelShape(26, 64, 6)
    packed = _packed(m, shape, 24, 363, 7, False)
    w = np.random.default_rng(0).normal(0.0, 0.01, (64, 91))
    model = m.LinearModel(shape, m.LearnerConfig(epochs=0), w, trained=True)
    learned = m.make_predictor("learned_linear", shape, model=model).predict_masks(packed, 6, 8)
    caps = [m.CacheConfig(capacity_fraction=f).resolve_capacity(shape)
            for f in (0.05, 0.10, 0.15, 0.20, 0.25, 0.30, 0.40, 0.50)]
    streams = [(learned, None, False), (None, None, False)]
    monkeypatch.setenv("MOEB_K1M", "0")
    monkeypatch.setenv("MOEB_K1_STACK", "0")
    want, want_pp, _ = m.cache_replay(packed, streams, caps, 8, 6)
    monkeypatch.delenv("MOEB_K1M")
    monkeypatch.delenv("MOEB_K1_STACK")
    got, got_pp, _ = m.cache_replay(packed, streams, caps, 8, 6)
    torch.cuda.synchronize()
    assert torch.equal(got, want) and torch.equal(got_pp, want_pp)
