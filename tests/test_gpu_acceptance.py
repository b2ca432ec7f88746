"""The reference acceptance suite's criteria 2 and 3 and the headline C2
sample, reproduced through this package's public API on the GPU and compared
with counters the REFERENCE produced (tests/golden/make_acceptance_golden.py,
tests/golden/make_c2_golden.py; /root/reference/pkg/tests/test_acceptance.py
:98-165, pkg/test_output.txt:258-259, bench.py --impl reference's sample).

Everything upstream of the replay runs on device too: the trace generator,
learner.train (device SGD), the recent-mode EAMC, the JSONL writer/parser of
the external predictor's table."""
import hashlib
import json
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def m():
    import paper_2508_17137_b200 as m
    m.load_library()
    return m


@pytest.fixture(scope="module")
def acc():
    with open(os.path.join(GOLD, "acceptance.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="module")
def fixtures(m):
    """test_acceptance.py:48-78: test / train / learner-train prompts, the
    recent EAMC and the seed-7 learned model."""
    full = m.ModelShape(27, 64, 6)
    test = m.generate_packed(m.GeneratorConfig(50, 128, full, 8, 0.9, 7))
    train = m.generate_packed(m.GeneratorConfig(500, 128, full, 8, 0.9, 7, first_prompt_id=1000))
    eamc = m.build_eamc(train, m.EamcConfig(mode="recent", capacity=500))
    lt = m.generate_packed(m.GeneratorConfig(40, 48, full, 8, 0.9, 7, first_prompt_id=2000))
    model = m.train(lt, full, m.LearnerConfig(seed=7))
    return full, test, train, eamc, model


def _cfg(m, full, f):
    return m.ReplayConfig(full, m.CacheConfig(capacity_fraction=f, prefetch_budget=6),
                          warmup_tokens=8)


def test_criterion_02_hit_vectors(m, acc, fixtures):
    """Criterion 2 (test_acceptance.py:98-116): the cache-hit vectors over
    [0.05, 0.1, 0.25, 0.5, 1.0] for four predictors on test prompts 0..19,
    equal to the reference's integers."""
    full, test, train, eamc, model = fixtures
    replay_set = test.select(0, 20)
    factories = {
        "lru_only": lambda: m.make_predictor("lru_only", full),
        "global_frequency": lambda: m.make_predictor("global_frequency", full,
                                                     train_traces=train),
        "eam_cosine": lambda: m.make_predictor("eam_cosine", full, eamc=eamc),
        "learned_linear": lambda: m.make_predictor("learned_linear", full, model=model),
    }
    for kind, fac in factories.items():
        got = []
        for f in acc["capacities"]:
            r = m.replay_traces(replay_set, fac(), _cfg(m, full, f))
            got.append([r.measured_accesses, r.cache_hits, r.prediction_hits])
        assert got == acc["criterion2"][kind], kind
        hits = [g[1] for g in got]
        assert hits == sorted(hits)


def test_criterion_03_rates(m, acc, fixtures):
    """Criterion 3 (test_acceptance.py:119-165; pkg/test_output.txt:258-259:
    0.0000 / 0.1405 / 1.0000 at 0.05, 0.6253 / 0.1407 / 1.0000 at 0.1), the
    external table written to JSONL and parsed back on device."""
    full, test, _, eamc, _ = fixtures
    table = m.PredictionTable(full, *_truth_table(m, test))
    ext = m.parse_predictions(m.write_predictions_jsonl(table, full), full)
    printed = {"0.05": (0.0000, 0.1405, 1.0000), "0.1": (0.6253, 0.1407, 1.0000)}
    for f in (0.05, 0.1):
        cfg = _cfg(m, full, f)
        res = {}
        for kind, pred in (("lru_only", m.make_predictor("lru_only", full)),
                           ("eam_cosine", m.make_predictor("eam_cosine", full, eamc=eamc)),
                           ("external", m.make_predictor("external", full, predictions=ext))):
            r = m.replay_traces(test, pred, cfg)
            res[kind] = [r.measured_accesses, r.cache_hits, r.prediction_hits,
                         r.uncovered_queries]
        assert res == acc["criterion3"][str(f)], f
        rates = tuple(round(res[k][1] / res[k][0], 4)
                      for k in ("lru_only", "eam_cosine", "external"))
        assert rates == printed[str(f)]


def _truth_table(m, packed):
    """(prompt_id, token_index, layer_id, masks) device arrays of every row."""
    L = packed.shape.num_layers
    dev = packed.device
    pid, tok, lay = [], [], []
    for i in range(packed.num_prompts):
        n = int(packed.row_off_host[i + 1] - packed.row_off_host[i])
        r = np.arange(n)
        pid.append(np.full(n, packed.prompt_ids[i]))
        tok.append(r // L)
        lay.append(r % L)
    t = lambda a, dt: torch.from_numpy(np.concatenate(a)).to(dev, dt)  # noqa: E731
    return (t(pid, torch.int64), t(tok, torch.int64), t(lay, torch.int32),
            packed.truth.clone())


# ---------------------------------------------------------------------------
# The headline configuration (bench.py / BASELINE configs[1]): the reference
# arm's own 256-prompt x 363-token C2 sample, every C3 capacity.
# ---------------------------------------------------------------------------

@pytest.fixture(scope="module")
def c2(m):
    g = np.load(os.path.join(GOLD, "c2_sample256.npz"))
    shape = m.ModelShape(26, 64, 6)
    packed = m.generate_packed(m.GeneratorConfig(256, 363, shape, 8, 0.9, 7))
    sha = hashlib.sha256(packed.truth.cpu().numpy().tobytes()).digest()
    assert sha == g["truth_sha256"].tobytes(), "device generator != reference traces"
    w = np.random.default_rng(0).normal(0.0, 0.01, (64, 91))
    model = m.LinearModel(shape, m.LearnerConfig(epochs=0), w, trained=True)
    return g, shape, packed, model


def test_c2_headline_replay_traces(m, c2):
    """replay_traces (the drop-in call) at every C3 capacity: aggregate,
    per-layer and per-prompt counters equal the reference's SimReport, for
    learned_linear (K3 -> K1s + exact kernel) and lru_only (exact kernel)."""
    g, shape, packed, model = c2
    for kind in ("learned_linear", "lru_only"):
        for j, f in enumerate(g["fractions"]):
            pred = (m.make_predictor(kind, shape, model=model) if kind == "learned_linear"
                    else m.make_predictor(kind, shape))
            cfg = m.ReplayConfig(shape, m.CacheConfig(capacity_fraction=float(f),
                                                      prefetch_budget=6), warmup_tokens=8)
            assert cfg.cache.resolve_capacity(shape) == g["capacities"][j]
            r = m.replay_traces(packed, pred, cfg)
            vec = np.concatenate([[r.measured_accesses, r.cache_hits, r.prediction_hits,
                                   r.uncovered_queries], r.layer_accesses, r.layer_cache_hits,
                                  r.layer_prediction_hits])
            assert np.array_equal(vec, g[f"counters_{kind}"][j]), (kind, f)
            pp = np.array([[r.per_prompt[p].measured_accesses, r.per_prompt[p].cache_hits,
                            r.per_prompt[p].prediction_hits, 0] for p in range(256)])
            assert np.array_equal(pp, g[f"perprompt_{kind}"][j]), (kind, f)


def test_c2_headline_bench_pipeline(m, c2):
    """The bench's timed step (PipelinedReplay: K3 with fused replay counts,
    K1s + exact kernel, K7 on its own stream) and a multi-capacity sweep give
    the reference's counters, and the fused metric counters give the
    reference's integer metrics and its macro_f1 / accuracy floats."""
    g, shape, packed, model = c2
    pred = m.make_predictor("learned_linear", shape, model=model)
    caps = [int(c) for c in g["capacities"]]
    for chunks in (1, 3):
        pipe = m.PipelinedReplay(packed, chunks)
        vec = m.metrics.metric_vector(64, packed.device)
        counters = pipe.run(pred, caps, 8, 6, metrics=vec)
        torch.cuda.synchronize()
        assert np.array_equal(counters[0].cpu().numpy(), g["counters_learned_linear"])
        assert np.array_equal(vec.cpu().numpy(), g["metrics_ints"])
        mc = m.MetricCounts.from_vector(vec.cpu().numpy(), 64)
        got = [mc.macro_f1(), mc.macro_f1(include_all=True), mc.position_accuracy,
               mc.label_accuracy]
        assert got == list(g["metrics_floats"])
    pts = m.sweep(packed, lambda: m.make_predictor("lru_only", shape), "lru_only",
                  [float(f) for f in g["fractions"]], shape, 6, 8)
    for j, p in enumerate(pts):
        assert p.report.cache_hits == g["counters_lru_only"][j][1]
