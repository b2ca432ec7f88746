"""The CSV report emitters reproduce the reference's bytes for the same
counters (tests/golden/report_csv.json: reference replay + sweep of small
generated traces, formatted by moesim.engine)."""
import json
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = json.load(open(os.path.join(ROOT, "tests", "golden", "report_csv.json")))


def _report(m, shape, d):
    v = d["v"]
    rep = m.SimReport(shape, v[0], v[1], v[2], v[3], v[4], np.array(d["la"], dtype=np.int64),
                      np.array(d["lc"], dtype=np.int64), np.array(d["lp"], dtype=np.int64))
    from paper_2508_17137_b200.engine import PromptCounters
    for k, c in d["pp"].items():
        rep.per_prompt[int(k)] = PromptCounters(*c)
    return rep


def test_report_csvs_match_reference():
    import paper_2508_17137_b200 as m
    from paper_2508_17137_b200 import engine as E
    shape = m.ModelShape(*G["shape"])
    rep = _report(m, shape, G["report"])
    assert E.report_summary_csv(rep, "oracle", 8).decode() == G["summary"]
    assert E.report_layers_csv(rep).decode() == G["layers"]
    assert E.report_prompts_csv(rep).decode() == G["prompts"]
    pts = [m.SweepPoint(p["f"], p["kind"], _report(m, shape, p["report"])) for p in G["points"]]
    assert E.sweep_csv(pts).decode() == G["sweep"]
    assert E.sweep_layers_csv(pts).decode() == G["sweep_layers"]
