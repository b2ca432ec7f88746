"""The drop-in API entry points end to end on the GPU, against the
reference's own results: sweep / replay_traces reports and CSV bytes
(tests/golden/report_csv.json, made by make_report_golden.py from the
reference on bit-identical generated traces), collect_prediction_sets and
prediction_metrics against the golden prediction streams."""
import json
import os

import numpy as np
import pytest

from conftest import load_case

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = json.load(open(os.path.join(ROOT, "tests", "golden", "report_csv.json")))
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def m():
    import paper_2508_17137_b200 as m
    m.load_library()
    return m


def _same(rep, d):
    v = d["v"]
    assert [rep.measured_accesses, rep.cache_hits, rep.prediction_opportunities,
            rep.prediction_hits, rep.uncovered_queries] == v
    assert rep.layer_accesses.tolist() == d["la"]
    assert rep.layer_cache_hits.tolist() == d["lc"]
    assert rep.layer_prediction_hits.tolist() == d["lp"]
    got = {str(k): [c.measured_accesses, c.cache_hits, c.prediction_opportunities,
                    c.prediction_hits] for k, c in rep.per_prompt.items()}
    assert got == d["pp"]


def test_sweep_and_replay_match_reference(m):
    from paper_2508_17137_b200 import engine as E
    shape = m.ModelShape(4, 8, 2)
    traces = m.generate_packed(m.GeneratorConfig(5, 12, shape, 3, 0.8, 3))
    cfg = m.ReplayConfig(shape, m.CacheConfig(capacity_fraction=0.25, prefetch_budget=2),
                         warmup_tokens=2)
    rep = m.replay_traces(traces, m.make_predictor("oracle", shape, traces=traces), cfg)
    _same(rep, G["report"])
    assert E.report_prompts_csv(rep).decode() == G["prompts"]
    assert E.report_layers_csv(rep).decode() == G["layers"]
    pts = m.sweep(traces, lambda: m.make_predictor("lru_only", shape), "lru_only",
                  [0.1, 0.25, 0.5], shape, 2, 2)
    for p, d in zip(pts, G["points"]):
        assert p.capacity_fraction == d["f"]
        _same(p.report, d["report"])
    assert E.sweep_csv(pts).decode() == G["sweep"]
    assert E.sweep_layers_csv(pts).decode() == G["sweep_layers"]
    # list-of-PromptTrace input (the reference's type) gives the same report
    rep2 = m.replay_traces(traces.unpack(), m.make_predictor("oracle", shape, traces=traces), cfg)
    _same(rep2, G["report"])


def test_collect_prediction_sets_and_metrics(m):
    c = load_case("v2lite_small")
    import torch
    shape = m.ModelShape(*(int(x) for x in c["shape"]))
    truth = c["truth"].astype(np.uint64)
    off = c["row_off"]
    packed = m.PackedTraces(shape, torch.from_numpy(truth.view(np.int64)).cuda(),
                            torch.from_numpy(off).cuda(), off, np.arange(len(off) - 1))
    model = m.LinearModel(shape, m.LearnerConfig(epochs=0, decay=float(c["decay"])),
                          c["weights"], trained=True)
    pred = m.make_predictor("learned_linear", shape, model=model)
    cfg = m.ReplayConfig(shape, m.CacheConfig(capacity_fraction=0.1,
                                              prefetch_budget=int(c["budget"])),
                         warmup_tokens=int(c["warmup"]), history_decay=float(c["decay"]))
    ps, ts, ls = m.collect_prediction_sets(packed, pred, cfg)
    want = c["pred_learned_linear"][c["measured_rows"]]
    assert len(ps) == len(want)
    for s, w in zip(ps, want):
        assert s == frozenset(e for e in range(64) if (int(w[0] if np.ndim(w) else w) >> e) & 1)
    mc = m.prediction_metrics(packed, pred, cfg)
    gm = c["metrics_learned_linear"]  # [macro_f1, macro_f1(all), position_acc, label_acc]
    assert mc.macro_f1() == gm[0]
    assert mc.macro_f1(include_all=True) == gm[1]
    assert mc.position_accuracy == gm[2]
    assert mc.label_accuracy == gm[3]
    assert m.macro_f1(ps, ts, 64) == gm[0]
