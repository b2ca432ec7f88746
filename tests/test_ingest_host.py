"""CPU checks of the ingestion host logic: the per-line restatements
(traceio._csv_record / _prediction_record, used for error messages and for
lines outside the device grammar) reproduce the reference's exception for
every single-data-line golden case, and the device grammar's scope is what
the kernels assume."""
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = json.load(open(os.path.join(ROOT, "tests", "golden", "ingest_cases.json")))


def _single_line(kind):
    out = []
    for c in CASES:
        if c["kind"] != kind or "error" not in c["result"] or c["result"]["error"] != "ParseError":
            continue
        text = c["data"].encode("latin-1").decode("utf-8", errors="strict")
        lines = text.split("\n")
        if lines and lines[-1] == "":
            lines.pop()
        body = lines[1:] if kind == "csv" else lines
        if kind == "csv" and (not lines or lines[0] != "prompt_id,token_index,layer_id,"
                              "expert_ids,token_id,embedding"):
            continue
        line_no = c["result"]["line"]
        idx = line_no - (2 if kind == "csv" else 1)
        if 0 <= idx < len(body) and "duplicate" not in c["result"]["message"]:
            out.append((c, body[idx]))
    return out


@pytest.mark.parametrize("case_line", _single_line("csv"), ids=lambda x: x[0]["tag"])
def test_csv_line_restatement(case_line):
    import paper_2508_17137_b200 as m
    from paper_2508_17137_b200 import traceio
    c, line = case_line
    shape = m.ModelShape(*c["shape"])
    with pytest.raises(m.ParseError) as ei:
        _, verr = traceio._csv_record(line, c["result"]["line"], shape)
        if verr is not None:
            raise verr
    assert str(ei.value) == c["result"]["message"]
    assert ei.value.line == c["result"]["line"]


@pytest.mark.parametrize("case_line", _single_line("jsonl"), ids=lambda x: x[0]["tag"])
def test_jsonl_line_restatement(case_line):
    import paper_2508_17137_b200 as m
    from paper_2508_17137_b200 import traceio
    c, line = case_line
    with pytest.raises(m.ParseError) as ei:
        traceio._prediction_record(line, c["result"]["line"], m.ModelShape(*c["shape"]))
    assert str(ei.value) == c["result"]["message"]


def test_parse_error_is_value_error():
    import paper_2508_17137_b200 as m
    e = m.ParseError(7, "x")
    assert isinstance(e, ValueError) and e.line == 7 and str(e) == "line 7: x"
