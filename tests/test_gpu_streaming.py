"""StreamingReplay (double-buffered host batches) gives exactly the counters
and metrics of a direct replay of each batch."""
import math

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


def test_rank_decode_exhaustive_64_6():
    """Every one of the C(64, 6) = 74,974,368 ranks decodes (floating-point
    estimate + 5-entry window per level) and re-encodes to itself."""
    import paper_2508_17137_b200 as m
    m.load_library()
    n = math.comb(64, 6)
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    for lo in range(0, n, 1 << 25):
        rs = torch.arange(lo, min(n, lo + (1 << 25)), device="cuda", dtype=torch.int64)
        rs = rs.to(torch.int32)
        ms = torch.empty((rs.numel(), 1), dtype=torch.int64, device="cuda")
        m.ranks_to_masks(rs, 6, 64, ms, bad)
        assert torch.equal(m.masks_to_ranks(ms, 6, 64), rs)
    assert int(bad.item()) == 0


@pytest.mark.parametrize("geom", [(26, 64, 6), (3, 64, 2), (5, 40, 4), (4, 48, 7)])
def test_streaming_ranks_equals_masks(geom):
    """Host batches as u32 combinatorial ranks (4 B/row, decoded on device)
    give the counters and metrics of the mask batches; masks <-> ranks round
    trip (every k-subset of small E enumerated); out-of-range ranks and rows
    without exactly k experts are flagged."""
    import itertools
    import math

    import paper_2508_17137_b200 as m
    m.load_library()
    L, E, k = geom
    shape = m.ModelShape(L, E, k)
    b = m.generate_packed(m.GeneratorConfig(40, 30, shape, max(8, k), 0.9, 4))
    ranks = m.masks_to_ranks(b.truth, k, E)
    assert ranks.shape == (b.rows,) and ranks.dtype == torch.int32
    back = torch.empty_like(b.truth)
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    m.ranks_to_masks(ranks, k, E, back, bad)
    torch.cuda.synchronize()
    assert torch.equal(back, b.truth) and int(bad.item()) == 0
    # the combinatorial number system, restated: rank = sum_i C(c_i, i)
    t = b.truth.reshape(-1).cpu().numpy().view(np.uint64)[:500]
    r = ranks.cpu().numpy().view(np.uint32)[:500]
    for mask, rank in zip(t, r):
        ids = [e for e in range(E) if (int(mask) >> e) & 1]
        assert sum(math.comb(c, i + 1) for i, c in enumerate(ids)) == int(rank)
    if math.comb(E, k) <= 200000:  # every subset maps to 0 .. C(E, k) - 1 and back
        subs = list(itertools.combinations(range(E), k))
        mk = torch.tensor([sum(1 << e for e in s) - (1 << 64 if sum(1 << e for e in s) >= 1 << 63
                                                     else 0) for s in subs],
                          dtype=torch.int64, device="cuda")
        rk = m.masks_to_ranks(mk, k, E)
        assert sorted(rk.cpu().tolist()) == list(range(len(subs)))
    # every rank of a large random sample decodes and re-encodes to itself
    # (the decoder starts from a floating-point estimate per level)
    g = torch.Generator(device="cuda").manual_seed(L * E + k)
    rs = torch.randint(0, math.comb(E, k), (1 << 20,), device="cuda", generator=g,
                       dtype=torch.int64).to(torch.int32)
    ms = torch.empty((1 << 20, 1), dtype=torch.int64, device="cuda")
    m.ranks_to_masks(rs, k, E, ms, bad)
    assert torch.equal(m.masks_to_ranks(ms, k, E), rs) and int(bad.item()) == 0
    # the packed bit stream (rank_bits per row) decodes to the same masks
    bits = m.rank_bits(E, k)
    assert bits == (math.comb(E, k) - 1).bit_length()
    words = m.masks_to_ranks(b.truth, k, E, packed=True)
    assert words.numel() == m.packed_rank_words(b.rows, bits)
    back2 = torch.empty_like(b.truth)
    m.ranks_to_masks(words, k, E, back2, bad, rows=b.rows)
    torch.cuda.synchronize()
    assert torch.equal(back2, b.truth) and int(bad.item()) == 0
    wn = words.cpu().numpy().view(np.uint32).astype(np.uint64)
    for i in (0, 1, 7, b.rows - 1):  # the stream layout, restated
        bit = i * bits
        two = int(wn[bit // 32]) | (int(wn[bit // 32 + 1]) << 32)
        assert (two >> (bit % 32)) & ((1 << bits) - 1) == int(r[i]) if i < len(r) else True
    if L == 26:
        w = np.random.default_rng(2).normal(0.0, 0.01, (64, 91))
        model = m.LinearModel(shape, m.LearnerConfig(epochs=0), w, trained=True)
        pred = m.make_predictor("learned_linear", shape, model=model)
        sr = m.StreamingReplay(shape, b.row_off_host, b.prompt_ids)
        mask_host = b.truth.cpu().pin_memory()
        rank_host = ranks.cpu().pin_memory()
        r1 = sr.run(pred, [83, 166], 8, 6, [mask_host] * 3, metrics=True)
        r2 = sr.run(pred, [83, 166], 8, 6, [rank_host] * 3, metrics=True)
        r3 = sr.run(pred, [83, 166], 8, 6, [words.cpu().pin_memory()] * 3, metrics=True)
        torch.cuda.synchronize()
        assert int(sr.ids_bad.item()) == 0
        for (c1, v1), (c2, v2), (c3, v3) in zip(r1, r2, r3):
            assert torch.equal(c1, c2) and torch.equal(v1, v2)
            assert torch.equal(c1, c3) and torch.equal(v1, v3)
    over = ranks.clone()
    over[5] = math.comb(E, k)
    m.ranks_to_masks(over, k, E, back, bad)
    torch.cuda.synchronize()
    assert int(bad.item()) == 1
    wrong = b.truth.clone()
    wrong[7] = 1
    with pytest.raises(m.RangeError):
        m.masks_to_ranks(wrong, k, E)
    if k == 6:  # C(64, 8) >= 2^32: no 4-byte rank format
        with pytest.raises(m.ConfigError):
            m.masks_to_ranks(b.truth, 8, 64)


def _restate_row(fmt, v, k):
    """A row's ids from its bit field, as the format docs state it."""
    if fmt == "ids6":
        return [(v >> (6 * j)) & 63 for j in range(k)]
    ids = []
    for j in range(k // 2):
        pr = (v >> (11 * j)) & 2047
        b = max(q for q in range(1, 64) if q * (q - 1) // 2 <= pr)
        ids += [pr - b * (b - 1) // 2, b]
    if k % 2:
        ids.append((v >> (11 * (k // 2))) & 63)
    return ids


@pytest.mark.parametrize("fmt", ["ids6", "idpairs"])
@pytest.mark.parametrize("geom", [(26, 64, 6), (3, 64, 2), (5, 40, 4), (4, 48, 7), (2, 64, 8)])
def test_streaming_ids6_equals_masks(geom, fmt):
    """Host batches as packed 6-bit expert ids (4.5 B/row at k = 6, decoded
    with shifts) or packed sorted id pairs (11 bits per pair, 4.125 B/row,
    decoded by table lookups) give the counters, per-prompt counters and
    metrics of the mask batches; masks <-> stream round trip on a 1M-row
    random sample (ids 0 and 63 included); the stream layout restated; rows
    without exactly k distinct experts are flagged."""
    import paper_2508_17137_b200 as m
    m.load_library()
    L, E, k = geom
    shape = m.ModelShape(L, E, k)
    enc = m.masks_to_ids6 if fmt == "ids6" else m.masks_to_idpairs
    dec = m.ids6_to_masks if fmt == "ids6" else m.idpairs_to_masks
    bits = 6 * k if fmt == "ids6" else 11 * (k // 2) + 6 * (k % 2)
    b = m.generate_packed(m.GeneratorConfig(40, 30, shape, max(8, k), 0.9, 4))
    words = enc(b.truth, k)
    assert words.dtype == torch.int32 and words.numel() == (b.rows * bits + 31) // 32 + 2
    back = torch.empty_like(b.truth)
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    dec(words, k, b.rows, back, bad)
    torch.cuda.synchronize()
    assert torch.equal(back, b.truth) and int(bad.item()) == 0
    wn = words.cpu().numpy().view(np.uint32)
    stream = int.from_bytes(wn.tobytes(), "little")
    t = b.truth.reshape(-1).cpu().numpy().view(np.uint64)
    for i in (0, 1, 2, 7, b.rows // 2, b.rows - 1):  # the stream layout, restated
        v = (stream >> (bits * i)) & ((1 << bits) - 1)
        ids = [e for e in range(64) if (int(t[i]) >> e) & 1]
        assert _restate_row(fmt, v, k) == ids
    # random k-subsets of 64 experts (E = 64), 1M rows
    rng = np.random.default_rng(L + k)
    n = 1 << 20
    keys = rng.random((n, 64)).argsort(axis=1)[:, :k]
    keys[0] = np.arange(k)
    keys[1] = np.arange(64 - k, 64)
    ms_np = np.zeros(n, dtype=np.uint64)
    for j in range(k):
        ms_np |= np.uint64(1) << keys[:, j].astype(np.uint64)
    ms = torch.from_numpy(ms_np.view(np.int64)).cuda().reshape(-1, 1)
    w2 = enc(ms, k)
    out = torch.empty_like(ms)
    dec(w2, k, n, out, bad)
    torch.cuda.synchronize()
    assert torch.equal(out, ms) and int(bad.item()) == 0
    if L == 26:
        w = np.random.default_rng(2).normal(0.0, 0.01, (64, 91))
        model = m.LinearModel(shape, m.LearnerConfig(epochs=0), w, trained=True)
        pred = m.make_predictor("learned_linear", shape, model=model)
        sr = m.StreamingReplay(shape, b.row_off_host, b.prompt_ids)
        r1 = sr.run(pred, [83, 166], 8, 6, [b.truth.cpu().pin_memory()] * 3, metrics=True,
                    per_prompt=True)
        r2 = sr.run(pred, [83, 166], 8, 6, [words.cpu().pin_memory()] * 4, metrics=True,
                    per_prompt=True, wire=fmt)
        torch.cuda.synchronize()
        assert int(sr.ids_bad.item()) == 0
        for (c1, v1, p1), (c2, v2, p2) in zip(r1, r2):
            assert torch.equal(c1, c2) and torch.equal(v1, v2) and torch.equal(p1, p2)
    wrong = b.truth.clone()
    wrong[7] = 1
    with pytest.raises(m.RangeError):
        enc(wrong, k)
    dup = words.clone()  # all-ones fields: a repeated id 63 / a pair rank >= C(64, 2)
    dup[0] = -1
    dec(dup, k, b.rows, back, bad)
    torch.cuda.synchronize()
    assert int(bad.item()) == 1
