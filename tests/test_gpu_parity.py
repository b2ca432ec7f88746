"""CUDA path vs the reference (golden fixtures) and the pinned oracle.

Every test here calls through libmoeb.so (the C ABI) on the GPU. Integer and
mask results must be bit-exact; learned_linear logits within 1e-12 of the
reference's fp64 values (the kernel computes the same logits by an
equivalent fp64 recurrence, K3).
"""
import numpy as np
import pytest
import torch

from conftest import CASES, load_case

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(180)]


@pytest.fixture(scope="module")
def pkg():
    import paper_2508_17137_b200 as m
    m.load_library()
    return m


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()


def _host(t):
    return t.cpu().numpy().view(np.uint64)


def _shape(pkg, c):
    L, E, k = (int(x) for x in c["shape"])
    return pkg.ModelShape(L, E, k)


def _packed(pkg, c):
    shape = _shape(pkg, c)
    off = c["row_off"].astype(np.int64)
    return pkg.PackedTraces(shape, _dev(c["truth"]), torch.from_numpy(off).cuda(), off,
                            np.arange(len(off) - 1, dtype=np.int64))


@pytest.mark.parametrize("name", CASES)
def test_generator_bit_identical(pkg, name):
    c = load_case(name)
    shape = _shape(pkg, c)
    g = c["gen"]
    cfg = pkg.GeneratorConfig(int(g[0]), int(g[1]), shape, int(g[2]), float(g[3]), int(g[4]))
    packed = pkg.generate_packed(cfg)
    assert np.array_equal(_host(packed.truth), c["truth"])
    assert np.array_equal(packed.row_off_host, c["row_off"])
    assert np.array_equal(packed.token_ids.cpu().numpy(), c["token_ids"].reshape(-1))


@pytest.mark.parametrize("name", CASES)
def test_cache_sim_hit_sequences(pkg, name):
    """K1 reproduces the reference's per-touch hit/miss sequence, counters and
    per-prompt counters for every policy's prediction stream and capacity."""
    c = load_case(name)
    packed = _packed(pkg, c)
    kinds = [str(k) for k in c["policies"]]
    caps = [int(x) for x in c["capacities"]]
    streams = []
    for kind in kinds:
        cov = torch.from_numpy(c["covered"]).cuda() if kind == "external" else None
        streams.append((_dev(c[f"pred_{kind}"]), cov, kind == "next_layer_all"))
    counters, pp, hits = pkg.cache_replay(packed, streams, caps, int(c["warmup"]),
                                          int(c["budget"]), want_hits=True)
    counters, pp = counters.cpu().numpy(), pp.cpu().numpy()
    for i, kind in enumerate(kinds):
        for j, cap in enumerate(caps):
            assert np.array_equal(counters[i, j], c[f"counters_{kind}_c{cap}"]), (kind, cap)
            assert np.array_equal(pp[i, j, :, :3], c[f"perprompt_{kind}_c{cap}"]), (kind, cap)
            assert np.array_equal(_host(hits[i, j]), c[f"hits_{kind}_c{cap}"]), (kind, cap)


def test_cache_sim_null_stream_is_lru_only(pkg):
    c = load_case("v2lite_small")
    packed = _packed(pkg, c)
    counters, _, hits = pkg.cache_replay(packed, [(None, None, False)], [83, 166],
                                         int(c["warmup"]), int(c["budget"]), want_hits=True)
    for j, cap in enumerate([83, 166]):
        assert np.array_equal(counters[0, j].cpu().numpy(), c[f"counters_lru_only_c{cap}"])
        assert np.array_equal(_host(hits[0, j]), c[f"hits_lru_only_c{cap}"])


@pytest.mark.parametrize("kernel", ["warp", "thread"])
@pytest.mark.parametrize("name", CASES)
def test_lfu_matches_oracle(pkg, oracle, name, kernel, monkeypatch):
    """LFU (builder-defined) vs its C oracle restatement: the warp-per-
    simulation kernel (default) and the thread-per-simulation one."""
    monkeypatch.setenv("MOEB_LFU_KERNEL", kernel)
    c = load_case(name)
    packed = _packed(pkg, c)
    L, E, _ = (int(x) for x in c["shape"])
    kinds = [k for k in ("lru_only", "learned_linear", "next_layer_all") if f"pred_{k}" in c]
    caps = [int(x) for x in c["capacities"]]
    streams = [(_dev(c[f"pred_{k}"]), None, k == "next_layer_all") for k in kinds]
    counters, pp, hits = pkg.cache_replay(packed, streams, caps, int(c["warmup"]),
                                          int(c["budget"]), policy="lfu", want_hits=True)
    for i, kind in enumerate(kinds):
        for j, cap in enumerate(caps):
            want, wpp, whits = oracle.cache_sim(c["truth"], c[f"pred_{kind}"], c["row_off"], L,
                                                E, int(c["warmup"]), cap, int(c["budget"]),
                                                unbounded=kind == "next_layer_all", policy=1,
                                                want_hits=True)
            assert np.array_equal(counters[i, j].cpu().numpy(), want), (kind, cap)
            assert np.array_equal(_host(hits[i, j]), whits), (kind, cap)


def test_cache_ops_kats(pkg):
    """The reference test-suite hand sequences (test_cache.py:17-88) on device."""
    shape = pkg.ModelShape(4, 8, 2)
    A, B, C = (0, 0), (0, 1), (0, 2)
    cache = pkg.ExpertCache(2, shape)
    assert [cache.touch(k) for k in (A, B, A, C, B)] == [False, False, True, False, False]
    cache = pkg.ExpertCache(1, shape)
    assert [cache.touch(k) for k in (A, A)] == [False, True]
    cache = pkg.ExpertCache(2, shape)
    cache.begin_step()
    assert cache.prefetch([A, B, C]) == 2
    cache = pkg.ExpertCache(2, shape)
    cache.touch(A)
    cache.touch(B)
    cache.begin_step()
    assert cache.prefetch([A]) == 0
    cache.touch(C)
    assert cache.touch(A) is True  # A survived (refreshed), B was evicted
    cache = pkg.ExpertCache(8, shape)
    assert cache.prefetch([A, B, C], limit=2) == 2
    cache = pkg.ExpertCache(2, shape)
    cache.begin_step()
    cache.prefetch([A])
    cache.touch(B)
    cache.touch(C)
    assert cache.touch(A)
    with pytest.raises(pkg.RangeError):
        cache.touch((9, 0))


def test_cache_ops_random_vs_oracle(pkg, oracle):
    rng = np.random.default_rng(5)
    shape = pkg.ModelShape(3, 70, 2)  # 2 mask words per layer
    n = 3000
    ops = rng.choice([0, 1, 1, 2], size=n).astype(np.int32)
    keys = rng.integers(0, shape.total_experts, size=n).astype(np.int32)
    for cap in (1, 3, 17, 100, 210):
        for pol, code in (("lru", 0), ("lfu", 1)):
            got = pkg.cache_ops(ops, keys, shape, cap, pol)
            want = oracle.cache_ops(ops, keys, 3, 70, cap, code)
            assert np.array_equal(got, want), (cap, pol)


@pytest.mark.parametrize("name", CASES)
def test_learned_linear(pkg, oracle, name):
    c = load_case(name)
    L, E, _ = (int(x) for x in c["shape"])
    packed = _packed(pkg, c)  # E > 64 runs the wide kernel (moeb_linear_predict_wide)
    shape = packed.shape
    m = c["measured_rows"]
    model = pkg.LinearModel(shape, pkg.LearnerConfig(epochs=0, decay=float(c["decay"])),
                            c["weights"], trained=True)
    for thr, kind in ((False, "learned_linear"), (True, "learned_linear_thr")):
        pred = pkg.make_predictor("learned_linear", shape, model=model, threshold=thr)
        logits = torch.zeros((packed.rows, E), dtype=torch.float64, device="cuda")
        vec = torch.zeros(3 * E + 3, dtype=torch.int64, device="cuda")
        masks = pred.predict_masks(packed, int(c["budget"]), int(c["warmup"]), metrics=vec,
                                   logits=logits)
        assert np.array_equal(_host(masks)[m], c[f"pred_{kind}"][m]), kind
        np.testing.assert_allclose(logits.cpu().numpy(), c["logits_learned_linear"], rtol=0,
                                   atol=1e-12)
        want = oracle.metrics(c[f"pred_{kind}"], c["truth"], c["row_off"], L, E,
                              int(c["warmup"]))
        assert np.array_equal(vec.cpu().numpy(), want)


@pytest.mark.parametrize("name", CASES)
def test_metrics_kernel(pkg, name):
    c = load_case(name)
    packed = _packed(pkg, c)
    E = packed.shape.num_experts
    for kind in c["policies"]:
        kind = str(kind)
        vec = pkg.metrics.mask_metrics(_dev(c[f"pred_{kind}"]), packed.truth, packed.row_off,
                                       packed.shape.num_layers, E, int(c["warmup"]))
        mc = pkg.MetricCounts.from_vector(vec.cpu().numpy(), E)
        got = [mc.macro_f1(), mc.macro_f1(True), mc.position_accuracy, mc.label_accuracy]
        assert got == list(c[f"metrics_{kind}"]), kind


@pytest.mark.parametrize("name", CASES)
def test_rule_predictors(pkg, name):
    c = load_case(name)
    packed = _packed(pkg, c)
    shape = packed.shape
    m = c["measured_rows"]
    b = int(c["budget"])
    assert np.array_equal(_host(pkg.make_predictor("oracle", shape, traces=packed)
                                .predict_masks(packed, b))[m], c["pred_oracle"][m])
    assert np.array_equal(_host(pkg.make_predictor("next_layer_all", shape)
                                .predict_masks(packed, b))[m], c["pred_next_layer_all"][m])
    assert not _host(pkg.make_predictor("lru_only", shape).predict_masks(packed, b)).any()
    if "pred_global_frequency" in c:
        off = c["train_row_off"].astype(np.int64)
        train = pkg.PackedTraces(shape, _dev(c["train_truth"]), torch.from_numpy(off).cuda(),
                                 off, np.arange(len(off) - 1))
        gf = pkg.make_predictor("global_frequency", shape, train_traces=train)
        assert np.array_equal(_host(gf.predict_masks(packed, b))[m],
                              c["pred_global_frequency"][m])


@pytest.mark.parametrize("name", CASES)
def test_eam_cosine(pkg, name):
    c = load_case(name)
    packed = _packed(pkg, c)
    shape = packed.shape
    coll = pkg.SketchCollection(c["sketches"], pkg.EamcConfig(capacity=len(c["sketches"])),
                                shape)
    pred = pkg.make_predictor("eam_cosine", shape, eamc=coll)
    idx = torch.zeros(packed.rows, dtype=torch.int32, device="cuda")
    masks = pred.predict_masks(packed, int(c["budget"]), int(c["warmup"]), idx_out=idx)
    assert np.array_equal(idx.cpu().numpy(), c["eamidx"])
    assert np.array_equal(_host(masks), c["pred_eam_cosine"])


@pytest.mark.parametrize("name", CASES)
def test_replay_traces_api(pkg, name):
    """End to end through the drop-in API: make_predictor + replay_traces."""
    c = load_case(name)
    packed = _packed(pkg, c)
    shape = packed.shape
    model = pkg.LinearModel(shape, pkg.LearnerConfig(epochs=0, decay=float(c["decay"])),
                            c["weights"], trained=True)
    preds = {"lru_only": pkg.make_predictor("lru_only", shape),
             "oracle": pkg.make_predictor("oracle", shape, traces=packed),
             "next_layer_all": pkg.make_predictor("next_layer_all", shape)}
    preds["learned_linear"] = pkg.make_predictor("learned_linear", shape, model=model)
    for kind, pred in preds.items():
        for cap in c["capacities"]:
            cfg = pkg.ReplayConfig(shape, pkg.CacheConfig(capacity_entries=int(cap),
                                                          prefetch_budget=int(c["budget"])),
                                   warmup_tokens=int(c["warmup"]), history_decay=float(c["decay"]))
            rep = pkg.replay_traces(packed, pred, cfg)
            v = c[f"counters_{kind}_c{cap}"]
            assert (rep.measured_accesses, rep.cache_hits, rep.prediction_hits) == tuple(v[:3])


def test_mask_head_vs_oracle(pkg, oracle):
    rng = np.random.default_rng(3)
    for E in (8, 64, 100, 256):
        z = rng.normal(size=(500, E)).astype(np.float32)
        z[:50, :4] = 0.5  # ties -> lower id
        z[50:60] = -np.abs(z[50:60])
        z[60, 3] = -0.0
        zt = torch.from_numpy(z).cuda()
        for k, thr in ((6, False), (8, False), (1, False), (6, True)):
            W = (E + 63) // 64
            out = torch.zeros((500, W), dtype=torch.int64, device="cuda")
            from paper_2508_17137_b200 import _native as nat
            nat.call("moeb_mask_head", nat.ptr(zt), 500, E, k, int(thr), nat.ptr(out),
                     nat.stream_ptr())
            assert np.array_equal(_host(out), oracle.mask_head(z, k, thr)), (E, k, thr)


def test_c1_scale_vs_oracle(pkg, oracle):
    """BASELINE config C1 (16 x 128, 26x64x6, seed 7): device generator,
    learned_linear, LRU + LFU at 10% vs the C oracle, bit-exact."""
    shape = pkg.ModelShape(26, 64, 6)
    packed = pkg.generate_packed(pkg.GeneratorConfig(16, 128, shape, 8, 0.9, 7))
    spec = oracle.GenSpec(16, 128, 26, 64, 6, 8, 0.9, 7)
    truth, _, off = oracle.generate_packed(spec, procs=1)
    assert np.array_equal(_host(packed.truth), truth)
    w = np.random.default_rng(0).normal(0.0, 0.01, (64, 91))
    model = pkg.LinearModel(shape, pkg.LearnerConfig(epochs=0), w, trained=True)
    pred = pkg.make_predictor("learned_linear", shape, model=model)
    masks = pred.predict_masks(packed, 6, 8)
    want_pred, _ = oracle.linear_predict(truth, off, 26, 64, w, 0.9, 6)
    assert np.array_equal(_host(masks), want_pred)
    counters, _, _ = pkg.cache_replay(packed, [(None, None, False), (masks, None, False)], [166],
                                      8, 6)
    c = counters.cpu().numpy()
    # survey §6: lru 187,914 / 299,520 hits; learned_linear 27,769 hits, 27,698 pred hits
    assert c[0, 0, 0] == 299520 and c[0, 0, 1] == 187914
    assert c[1, 0, 1] == 27769 and c[1, 0, 2] == 27698
    for pol in (0, 1):
        for i, pm in enumerate((None, want_pred)):
            want, _, _ = oracle.cache_sim(truth, pm, off, 26, 64, 8, 166, 6, policy=pol)
            got, _, _ = pkg.cache_replay(packed, [(None if pm is None else masks, None, False)],
                                         [166], 8, 6, policy=("lru", "lfu")[pol])
            assert np.array_equal(got[0, 0].cpu().numpy(), want)


@pytest.mark.parametrize("chunks", [1, 3, 7])
def test_pipelined_replay_matches_single_call(pkg, chunks):
    """PipelinedReplay (predict || replay || H2D over prompt chunks) gives the
    same counters and fused metrics as one unchunked predict + K1 call."""
    shape = pkg.ModelShape(26, 64, 6)
    packed = pkg.generate_packed(pkg.GeneratorConfig(40, 96, shape, 8, 0.9, 7))
    w = np.random.default_rng(0).normal(0.0, 0.01, (64, 91))
    model = pkg.LinearModel(shape, pkg.LearnerConfig(epochs=0), w, trained=True)
    pred = pkg.make_predictor("learned_linear", shape, model=model)
    vec = pkg.metrics.metric_vector(64, packed.device)
    masks = pred.predict_masks(packed, 6, 8, metrics=vec)
    want, _, _ = pkg.cache_replay(packed, [(masks, None, False)], [40, 166], 8, 6,
                                  want_per_prompt=False)
    pipe = pkg.PipelinedReplay(packed, chunks)
    assert len(pipe.bounds) == chunks
    vec2 = pkg.metrics.metric_vector(64, packed.device)
    timing = []
    got = pipe.run(pred, [40, 166], 8, 6, metrics=vec2, timing=timing)
    assert torch.equal(got, want) and torch.equal(vec2, vec)
    assert len(timing) == 2 * chunks
    # from pinned host rows into a fresh device buffer
    host = packed.truth.cpu().pin_memory()
    dst = pkg.PackedTraces(shape, torch.zeros_like(packed.truth), torch.zeros_like(packed.row_off),
                           packed.row_off_host, packed.prompt_ids)
    pipe2 = pkg.PipelinedReplay(dst, chunks)
    got2 = pipe2.run(pred, [40, 166], 8, 6, host_truth=host)
    assert torch.equal(got2, want)
    # LRU-only (no predictor launches) and LFU
    lru = pkg.make_predictor("lru_only", shape)
    want3, _, _ = pkg.cache_replay(packed, [(None, None, False)], [166], 8, 6, policy="lfu",
                                   want_per_prompt=False)
    assert torch.equal(pipe.run(lru, [166], 8, 6, policy="lfu"), want3)
    # overlapped steps (step i+1's predictor beside step i's replay, two mask
    # buffers): every step's counters, metrics and per-prompt counters equal
    want_pp = pkg.cache_replay(packed, [(masks, None, False)], [40, 166], 8, 6)[1]
    pipe3 = pkg.PipelinedReplay(packed, chunks, overlap_steps=True)
    outs = []
    for _ in range(5):
        v = pkg.metrics.metric_vector(64, packed.device)
        outs.append((pipe3.run(pred, [40, 166], 8, 6, metrics=v, per_prompt=True), v,
                     pipe3.last_per_prompt))
    pipe3.join()
    for c, v, pp in outs:
        assert torch.equal(c, want) and torch.equal(v, vec) and torch.equal(pp, want_pp)


@pytest.mark.parametrize("L,E,budget,decay", [(5, 64, 6, 0.0), (3, 40, 5, 0.5), (4, 64, 1, 0.0),
                                             (2, 33, 8, 0.5), (3, 256, 8, 0.0), (2, 100, 6, 0.5),
                                             (2, 200, 1, 0.0)])
def test_learned_linear_exact_ties(pkg, oracle, L, E, budget, decay):
    """Dyadic weights make logits exact in both the oracle and the kernel and
    create many exact ties, so the kernel's key-based selection must fall
    back to the exact fp64 passes (ties to the lower id) on every tied cut."""
    rng = np.random.default_rng(L * 1000 + E)
    shape = pkg.ModelShape(L, E, 6)
    P, T = 24, 20
    rows = P * T * L
    W = (E + 63) // 64
    truth = np.zeros((rows, W), dtype=np.uint64)
    for r in range(rows):
        for e in rng.choice(E, 6, replace=False):
            truth[r, e >> 6] |= np.uint64(1) << np.uint64(e & 63)
    if W == 1:
        truth = truth.reshape(-1)
    off = np.arange(P + 1, dtype=np.int64) * T * L
    w = rng.integers(-2, 3, size=(E, L + E + 1)).astype(np.float64) * 0.25
    packed = pkg.PackedTraces(shape, _dev(truth), torch.from_numpy(off).cuda(), off,
                              np.arange(P, dtype=np.int64))
    model = pkg.LinearModel(shape, pkg.LearnerConfig(epochs=0, decay=decay), w, trained=True)
    for thr in (False, True):
        pred = pkg.make_predictor("learned_linear", shape, model=model, threshold=thr)
        masks = pred.predict_masks(packed, budget, 0)
        want, logits = oracle.linear_predict(truth, off, L, E, w, decay, budget, threshold=thr,
                                             want_logits=True)
        got = _host(masks).reshape(-1)
        want = want.reshape(-1)
        bad = np.nonzero(got != want)[0]
        assert bad.size == 0, (thr, bad[:5], got[bad[:3]], want[bad[:3]])
    # ties really occur at the top-k cut
    srt = -np.sort(-logits, axis=1)
    assert np.mean(srt[:, budget - 1] == srt[:, budget]) > 0.05


@pytest.mark.parametrize("G", ["16", "32", "8"])
def test_ragged_prompts(pkg, oracle, G, monkeypatch):
    """Prompts of different lengths share warps (K1 pads the shorter group
    with no-op rows): counters, per-prompt counters and hit masks vs the C
    oracle, for every lane-group width."""
    monkeypatch.setenv("MOEB_K1_G", G)
    shape = pkg.ModelShape(26, 64, 6)
    full = pkg.generate_packed(pkg.GeneratorConfig(37, 40, shape, 8, 0.9, 5))
    L = 26
    truth_all = full.truth.cpu().numpy().view(np.uint64).reshape(-1)
    rows, off = [], [0]
    for p in range(37):
        T = 9 + (p * 7) % 31
        r0 = int(full.row_off_host[p])
        rows.append(truth_all[r0:r0 + T * L])
        off.append(off[-1] + T * L)
    truth = np.concatenate(rows)
    off = np.array(off, dtype=np.int64)
    packed = pkg.PackedTraces(shape, _dev(truth), torch.from_numpy(off).cuda(), off,
                              np.arange(37, dtype=np.int64))
    w = np.random.default_rng(1).normal(0.0, 0.01, (64, 91))
    model = pkg.LinearModel(shape, pkg.LearnerConfig(epochs=0), w, trained=True)
    masks = pkg.make_predictor("learned_linear", shape, model=model).predict_masks(packed, 6, 8)
    caps = [3, 40, 166, 700]
    for pm in (masks, None):
        counters, pp, hits = pkg.cache_replay(packed, [(pm, None, False)], caps, 8, 6,
                                              want_hits=True)
        pred_h = np.zeros_like(truth) if pm is None else _host(pm).reshape(-1)
        for j, cap in enumerate(caps):
            want, wpp, whits = oracle.cache_sim(truth, pred_h, off, 26, 64, 8, cap, 6,
                                                want_hits=True)
            assert np.array_equal(counters[0, j].cpu().numpy(), want), (G, cap)
            assert np.array_equal(pp[0, j].cpu().numpy().reshape(-1), np.asarray(wpp).reshape(-1))
            assert np.array_equal(_host(hits[0, j]).reshape(-1), np.asarray(whits).reshape(-1))
