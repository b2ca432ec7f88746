"""Pin the CPU oracle (oracle/) against the reference's own outputs.

The fixtures in tests/golden/ were produced by tests/golden/make_golden.py from
the reference package itself; the known-answer tests below restate the
reference test suite's hand sequences (pkg/tests/test_cache.py,
test_engine.py, test_learner.py, test_metrics.py). CPU only.
"""
import numpy as np
import pytest


def _pred(case, kind):
    return case[f"pred_{kind}"]


def test_generator_bit_identical(golden, oracle):
    name, c = golden
    L, E, k = (int(x) for x in c["shape"])
    g = c["gen"]
    P, T = int(g[0]), int(g[1])
    spec = oracle.GenSpec(P, T, L, E, k, int(g[2]), float(g[3]), int(g[4]))
    truth, toks, row_off = oracle.generate_packed(spec, procs=1)
    assert np.array_equal(truth, c["truth"])
    assert np.array_equal(row_off, c["row_off"])
    assert np.array_equal(toks, c["token_ids"])


def test_generator_fanout_independent(oracle):
    spec = oracle.GenSpec(5, 9, 3, 8, 2, 3, 0.7, 2, first_prompt_id=40)
    a = oracle.generate_packed(spec, procs=1)
    b = oracle.generate_packed(spec, procs=3)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def _sim_args(c, kind):
    pred = _pred(c, kind)
    unbounded = kind == "next_layer_all"
    covered = c.get("covered") if kind == "external" else None
    return pred, unbounded, covered


def test_cache_sim_matches_reference(golden, oracle):
    name, c = golden
    L, E, _ = (int(x) for x in c["shape"])
    for kind in c["policies"]:
        kind = str(kind)
        pred, unbounded, covered = _sim_args(c, kind)
        if kind == "lru_only":
            assert not pred.any()
        for cap in c["capacities"]:
            counters, per_prompt, hits = oracle.cache_sim(
                c["truth"], pred, c["row_off"], L, E, int(c["warmup"]), int(cap),
                int(c["budget"]), unbounded=unbounded, covered=covered, want_hits=True)
            want = c[f"counters_{kind}_c{cap}"]
            assert np.array_equal(counters, want), (name, kind, cap)
            assert np.array_equal(per_prompt[:, :3], c[f"perprompt_{kind}_c{cap}"])
            assert np.array_equal(hits, c[f"hits_{kind}_c{cap}"]), (name, kind, cap)


def test_learned_linear_matches_reference(golden, oracle):
    name, c = golden
    L, E, _ = (int(x) for x in c["shape"])
    m = c["measured_rows"]
    for thr, kind in ((False, "learned_linear"), (True, "learned_linear_thr")):
        pred, logits = oracle.linear_predict(c["truth"], c["row_off"], L, E, c["weights"],
                                             float(c["decay"]), int(c["budget"]),
                                             threshold=thr, want_logits=True)
        assert np.array_equal(pred[m], _pred(c, kind)[m]), (name, kind)
        np.testing.assert_allclose(logits, c["logits_learned_linear"], rtol=0, atol=1e-14)


def test_eam_cosine_matches_reference(golden, oracle):
    name, c = golden
    if "eamidx" not in c:
        pytest.skip("no eam case")
    L, E, _ = (int(x) for x in c["shape"])
    pred, idx = oracle.eam_predict(c["truth"], c["row_off"], L, E, int(c["warmup"]),
                                   c["sketches"], int(c["budget"]))
    assert np.array_equal(idx, c["eamidx"])
    assert np.array_equal(pred, _pred(c, "eam_cosine"))


def test_trivial_predictors_match_reference(golden, oracle):
    name, c = golden
    L, E, _ = (int(x) for x in c["shape"])
    m = c["measured_rows"]
    budget = int(c["budget"])
    if "pred_oracle" in c:
        want = oracle.lowest_bits(c["truth"], budget, E)
        assert np.array_equal(want[m], c["pred_oracle"][m])
    if "pred_global_frequency" in c:
        _, order = oracle.global_frequency_order(c["train_truth"], c["train_row_off"], L, E)
        layers = oracle.row_layers(c["row_off"], L)
        sets = [frozenset(int(e) for e in order[l, :min(budget, E)]) for l in layers]
        want = oracle.sets_to_masks(sets, E)
        assert np.array_equal(want[m], c["pred_global_frequency"][m])
    if "pred_next_layer_all" in c:
        assert all(s == frozenset(range(E))
                   for s in oracle.masks_to_sets(c["pred_next_layer_all"][m], E))


def test_metrics_match_reference(golden, oracle):
    name, c = golden
    L, E, _ = (int(x) for x in c["shape"])
    for kind in c["policies"]:
        kind = str(kind)
        out = oracle.metrics(_pred(c, kind), c["truth"], c["row_off"], L, E, int(c["warmup"]))
        tp, fp, fn = out[:E], out[E:2 * E], out[2 * E:3 * E]
        n, exact, label = out[3 * E:]
        got = [oracle.f1_from_counts(tp, fp, fn), oracle.f1_from_counts(tp, fp, fn, True),
               exact / n, label / (n * E)]
        assert got == list(c[f"metrics_{kind}"]), (name, kind)


# ---- Known answers restated from the reference test suite --------------------

A, B, C = 0, 1, 2  # keys (0,0), (0,1), (0,2) of shape (4, 8, 2)


def _ops(oracle, seq, cap, L=4, E=8, policy=0):
    ops = [o for o, _ in seq]
    keys = [k for _, k in seq]
    return list(oracle.cache_ops(ops, keys, L, E, cap, policy))


def test_cache_kats(oracle):
    T, PF, BS = 1, 2, 0
    # test_cache.py:17-21
    assert _ops(oracle, [(T, A), (T, B), (T, A), (T, C), (T, B)], 2) == [0, 0, 1, 0, 0]
    assert _ops(oracle, [(T, A), (T, A)], 1) == [0, 1]  # :23-25
    assert _ops(oracle, [(T, A), (T, B), (T, A)], 1) == [0, 0, 0]  # :27-29
    # step pinning caps inserts (:52-56): prefetch A,B,C at cap 2 -> 2 inserted
    assert _ops(oracle, [(BS, 0), (PF, A), (PF, B), (PF, C)], 2)[1:] == [1, 1, 0]
    # resident refreshed not inserted (:58-65): A most recent -> C evicts B
    r = _ops(oracle, [(T, A), (T, B), (BS, 0), (PF, A), (T, C), (T, A), (T, B)], 2)
    assert r == [0, 0, 0, 0, 0, 1, 0]
    # pins survive touch eviction (:72-80)
    r = _ops(oracle, [(BS, 0), (PF, A), (T, B), (T, C), (T, A)], 2)
    assert r == [0, 1, 0, 0, 1]
    # pins released next step (:82-88): cap 1, prefetch A; next step prefetch B
    r = _ops(oracle, [(BS, 0), (PF, A), (BS, 0), (PF, B), (T, B), (T, A)], 1)
    assert r == [0, 1, 0, 1, 1, 0]


def test_cache_stack_property(oracle):
    # test_cache.py:111-123: LRU is a stack algorithm
    rng = np.random.default_rng(42)
    keys = [int(rng.integers(0, 4)) * 8 + int(rng.integers(0, 8)) for _ in range(600)]
    hits = [int(np.sum(oracle.cache_ops([1] * 600, keys, 4, 8, cap))) for cap in
            (1, 2, 4, 8, 16, 32)]
    assert hits == sorted(hits)


def test_engine_hand_micro_trace(oracle):
    # test_engine.py:33-43: shape (1,4,2), token0 {0,1} warm, token1 {0,2}
    truth = np.array([[0b0011], [0b0101]], dtype=np.uint64)
    counters, _, _ = oracle.cache_sim(truth, None, np.array([0, 2]), 1, 4, 1, 2, 2)
    assert counters[0] == 2 and counters[1] == 1 and counters[2] == 0


def test_topk_kats(oracle):
    # test_learner.py:144-152: ties -> lower id; threshold all negative -> empty
    m = oracle.mask_head(np.array([[2.0, -1.0, 0.5, 0.5]], dtype=np.float32), 2)
    assert oracle.masks_to_sets(m, 4) == [frozenset({0, 2})]
    m = oracle.mask_head(np.array([[-1.0, -2.0, -0.5]], dtype=np.float32), 2, threshold=True)
    assert oracle.masks_to_sets(m, 3) == [frozenset()]


def test_metrics_kat(oracle):
    # test_metrics.py:68-72 style: pred {0,1} vs truth {0,2}: F1(0)=1, F1(1)=F1(2)=0
    pred = oracle.sets_to_masks([{0, 1}], 4)
    truth = oracle.sets_to_masks([{0, 2}], 4)
    out = oracle.metrics(pred, truth, np.array([0, 1]), 1, 4, 0)
    E = 4
    assert oracle.f1_from_counts(out[:E], out[E:2 * E], out[2 * E:3 * E]) == pytest.approx(1 / 3)
    assert out[3 * E + 2] == 2  # label: 2 of 4 experts agree
