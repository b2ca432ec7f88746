"""Golden cases for the trace/prediction file formats, produced by the
REFERENCE itself (moesim.traceio, read-only at /root/reference).

    python tests/golden/make_ingest_golden.py

Writes tests/golden/ingest_cases.json: a list of cases
  {"kind": "csv"|"jsonl", "shape": [L, E, k], "data": <latin-1 text of the
   file bytes>, "result": {"ok": <canonical output>} or
   {"error": <exception class name>, "message": str(exc), "line": exc.line?}}
where the canonical output is write_trace_csv(parse_trace_csv(data)) for CSV
(latin-1 text) and the sorted [[key..., experts...], ...] table for JSONL.
Cases: the reference test-suite inputs (tests/test_traceio.py) plus seeded
mutations of small valid files (field-level edits drawn from Python's
int()/float()/json edge cases, line swaps/duplications/deletions, blank and
CRLF lines, non-ASCII digits).
"""

from __future__ import annotations

import json
import os
import random
import sys

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

INT_EDGES = [" 5", "5 ", "+5", "-0", "1_0", "1__0", "_1", "1_", "007", "", " ", "+", "5\r",
             "\x0b5\x0c", "\x1c5", "x", "-1", "99999999999999999999", "٥", "0x10", "1.0",
             "9223372036854775807", "--1", "2", "0", "63", "64", "26", "25", "7"]
FLOAT_EDGES = ["1.", ".5", ".", "1e5", "1.e5", ".5e-3", "e5", "1e", "1e+", "1_0.5", "1_.5",
               "1._5", "1e1_0", "inf", "-Infinity", "nAn", "infin", "+inf ", "1.5_", "0x10",
               "1.5e5.5", " 1.5\x1c", "1.5", "1_000.000_1", ".e1", "1.5e_1", "in f",
               "-nan", "++1", "0.1", "2.5e-07", "", "1.5|2", "abc", "-0.0", "1E5"]


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import moesim
    from moesim import traceio
    return moesim, traceio


def _result_csv(traceio, moesim, data: bytes, shape):
    try:
        out = traceio.write_trace_csv(traceio.parse_trace_csv(data, shape))
        return {"ok": out.decode("latin-1")}
    except Exception as exc:  # noqa: BLE001
        r = {"error": type(exc).__name__, "message": str(exc)}
        if hasattr(exc, "line"):
            r["line"] = exc.line
        return r


def _result_jsonl(traceio, data: bytes, shape):
    try:
        t = traceio.parse_predictions(data, shape)
        return {"ok": sorted([list(k) + sorted(v) for k, v in t.items()])}
    except Exception as exc:  # noqa: BLE001
        r = {"error": type(exc).__name__, "message": str(exc)}
        if hasattr(exc, "line"):
            r["line"] = exc.line
        return r


def main():
    moesim, traceio = _ref()
    ModelShape = moesim.ModelShape
    H = traceio.TRACE_HEADER
    cases = []

    def add_csv(data, shape, tag):
        if isinstance(data, str):
            data = data.encode("utf-8")
        cases.append({"kind": "csv", "tag": tag, "shape": [shape.num_layers, shape.num_experts,
                                                          shape.top_k],
                      "data": data.decode("latin-1"),
                      "result": _result_csv(traceio, moesim, data, shape)})

    def add_jsonl(data, shape, tag):
        if isinstance(data, str):
            data = data.encode("utf-8")
        cases.append({"kind": "jsonl", "tag": tag, "shape": [shape.num_layers, shape.num_experts,
                                                            shape.top_k],
                      "data": data.decode("latin-1"),
                      "result": _result_jsonl(traceio, data, shape)})

    FULL, SMALL = ModelShape(27, 64, 6), ModelShape(2, 8, 2)

    def small_csv(rows):
        return H + "\n" + "\n".join(rows) + "\n"

    # --- the reference test suite's inputs (tests/test_traceio.py) ---
    rows = [f"0,0,{layer},1|5|9|12|33|60,482," for layer in range(27)]
    add_csv(small_csv(rows), FULL, "direct_field_mapping")
    r2 = list(rows)
    r2[3] = "0,0,3,1|5|9,482,"
    add_csv(small_csv(r2), FULL, "cardinality_error_line5")
    add_csv(small_csv([r for i, r in enumerate(rows) if i != 3]), FULL, "incomplete_coverage")
    add_csv("a,b,c\n", FULL, "bad_header")
    add_csv(small_csv(["0,0,0,1|2,5"]), SMALL, "wrong_column_count")
    add_csv(small_csv(["0,x,0,1|2,5,"]), SMALL, "non_integer")
    add_csv(small_csv(["0,0,0,1|2,5,", "0,0,1,1|2,5,", "0,0,0,3|4,5,"]), SMALL, "duplicate_key")
    add_csv(small_csv(["0,0,0,1|2,5,0.5|-1.25", "0,0,1,1|2,5,"]), SMALL, "embedding")
    add_csv(small_csv(["0,0,0,1|2,5,"]), ModelShape(1, 8, 2), "single_record")
    gen = traceio.write_trace_csv(traceio.generate_synthetic(
        traceio.GeneratorConfig(4, 6, SMALL, hot_set_size=3, skew=0.8, seed=9)))
    add_csv(gen, SMALL, "generated_round_trip")
    add_csv(small_csv(["0,1,0,1|2,5,", "0,0,1,1|2,5,", "0,1,1,1|2,5,", "0,0,0,1|2,5,"]), SMALL,
            "unsorted")
    add_csv(small_csv(["0,0,0,1|2,5,0.1|2.5e-07"]), ModelShape(1, 8, 2), "embedding_round_trip")
    add_csv(b"", SMALL, "empty_file")
    add_csv(H.encode(), SMALL, "header_only_no_newline")
    add_csv((H + "\n").encode(), SMALL, "header_only")
    add_csv(b"\n", SMALL, "blank_file")
    add_csv(small_csv(["0,0,0,1|2,5,", "0,0,1,1|2,5,"]).encode() + b"\xff\n", SMALL, "bad_utf8")

    # --- seeded mutations of small valid files ---
    rng = random.Random(1234)
    base_cfgs = [(ModelShape(3, 8, 2), 3, 4, 3), (ModelShape(2, 70, 3), 2, 3, 4),
                 (ModelShape(26, 64, 6), 2, 2, 8)]
    for shape, P, T, h in base_cfgs:
        blob = traceio.write_trace_csv(traceio.generate_synthetic(
            traceio.GeneratorConfig(P, T, shape, hot_set_size=h, skew=0.7, seed=5)))
        lines = blob.decode().rstrip("\n").split("\n")
        add_csv(blob, shape, f"gen_{shape.num_experts}")
        for it in range(60):
            ls = list(lines)
            op = rng.randrange(8)
            i = rng.randrange(1, len(ls))
            if op <= 2:  # field edit
                f = ls[i].split(",")
                c = rng.randrange(6)
                if c == 3:
                    parts = f[3].split("|")
                    parts[rng.randrange(len(parts))] = rng.choice(INT_EDGES)
                    if rng.random() < 0.2:
                        parts.append(rng.choice(parts))
                    f[3] = "|".join(parts)
                elif c == 5:
                    f[5] = "|".join(rng.choice(FLOAT_EDGES) for _ in range(rng.randint(1, 3)))
                else:
                    f[c] = rng.choice(INT_EDGES)
                ls[i] = ",".join(f)
            elif op == 3:  # swap two lines
                k = rng.randrange(1, len(ls))
                ls[i], ls[k] = ls[k], ls[i]
            elif op == 4:  # duplicate a line elsewhere
                ls.insert(rng.randrange(1, len(ls) + 1), ls[i])
            elif op == 5:  # delete a line
                del ls[i]
            elif op == 6:  # extra / missing columns, blank line
                ls[i] = rng.choice([ls[i] + ",", ls[i].rsplit(",", 1)[0], "", ls[i] + "\r"])
            else:  # shuffle all data lines (valid, unsorted)
                body = ls[1:]
                rng.shuffle(body)
                ls = ls[:1] + body
            text = "\n".join(ls) + ("\n" if rng.random() < 0.8 else "")
            add_csv(text, shape, f"mut_{shape.num_experts}_{it}")

    # --- predictions JSONL: reference tests + mutations ---
    add_jsonl(b'{"prompt_id":0,"token_index":4,"layer_id":2,"experts":[3,17,22,41,50,63]}\n',
              FULL, "direct_mapping")
    add_jsonl(b'{"prompt_id":0,"token_index":0,"layer_id":0,"experts":[1]}\n'
              b'{"prompt_id":0,"token_index":0,"layer_id":0,"experts":[2]}\n', FULL, "dup_key")
    add_jsonl(b'{"prompt_id":0,"token_index":0,"layer_id":0,"experts":[64]}\n', FULL,
              "expert_range")
    add_jsonl(b'{"prompt_id":0,"token_index":0,"layer_id":0,"experts":[1]}\n'
              b'{"prompt_id":0,\n', FULL, "malformed_line2")
    add_jsonl(traceio.write_predictions_jsonl({(0, 1, 2): frozenset({5, 3}),
                                               (1, 0, 0): frozenset({0})}), FULL, "round_trip")
    add_jsonl(b"", FULL, "empty")
    add_jsonl(b"\n\n  \n", FULL, "blank_lines")
    JEDGE = ['{"prompt_id": 1, "token_index": 2, "layer_id": 3, "experts": [4, 5]}',
             '{"experts":[1,2],"layer_id":0,"token_index":7,"prompt_id":3}',
             ' \t{"prompt_id":0,"token_index":0,"layer_id":0,"experts":[]}\r',
             '{"prompt_id":1.0,"token_index":0,"layer_id":0,"experts":[1]}',
             '{"prompt_id":"3","token_index":0,"layer_id":0,"experts":[1]}',
             '{"prompt_id":true,"token_index":0,"layer_id":0,"experts":[1]}',
             '{"prompt_id":0,"token_index":0,"layer_id":0,"experts":[1],"extra":{"a":[1,2]}}',
             '{"prompt_id":0,"token_index":0,"layer_id":0}',
             '{"prompt_id":0,"token_index":0,"layer_id":0,"experts":5}',
             '[1,2,3]', '{"prompt_id":0,"prompt_id":1,"token_index":0,"layer_id":0,"experts":[1]}',
             '{"\\u0070rompt_id":0,"token_index":0,"layer_id":0,"experts":[1]}',
             '{"prompt_id":0,"token_index":0,"layer_id":99,"experts":[1]}',
             '{"prompt_id":0,"token_index":0,"layer_id":-1,"experts":[1]}',
             '{"prompt_id":0,"token_index":0,"layer_id":0,"experts":[-1,99]}',
             '{"prompt_id":0,"token_index":0,"layer_id":0,"experts":[1,1,2]}',
             '{"prompt_id":01,"token_index":0,"layer_id":0,"experts":[1]}',
             '{"prompt_id":-5,"token_index":-2,"layer_id":0,"experts":[0]}',
             '{"prompt_id":0,"token_index":0,"layer_id":0,"experts":[1,]}',
             '{"prompt_id":0,"token_index":0,"layer_id":0,"experts":[1.5]}',
             '{"prompt_id":0,"token_index":0,"layer_id":0,"experts":[1e0]}',
             '\x1c', '\x0c  ', '{"prompt_id":99999999999999999999,"token_index":0,"layer_id":0,'
             '"experts":[1]}', 'null', '{}', '{"prompt_id":0 "token_index":0}',
             '{"prompt_id":٥,"token_index":0,"layer_id":0,"experts":[1]}',
             '{"prompt_id":0,"token_index":0,"layer_id":0,"experts":[2]} x']
    for it, shp in enumerate([FULL, ModelShape(4, 200, 3)]):
        table = {}
        for _ in range(25):
            key = (rng.randrange(5), rng.randrange(6), rng.randrange(shp.num_layers))
            table[key] = frozenset(rng.sample(range(shp.num_experts), rng.randint(0, 4)))
        base = traceio.write_predictions_jsonl(table).decode().rstrip("\n").split("\n")
        add_jsonl("\n".join(base) + "\n", shp, f"jgen_{it}")
        for k in range(60):
            ls = list(base)
            op = rng.randrange(5)
            i = rng.randrange(len(ls))
            if op <= 1:
                ls[i] = rng.choice(JEDGE)
            elif op == 2:
                ls.insert(rng.randrange(len(ls) + 1), ls[i])
            elif op == 3:
                rng.shuffle(ls)
            else:
                ls.insert(i, rng.choice(["", "   ", "\t"]))
            add_jsonl("\n".join(ls) + ("\n" if rng.random() < 0.7 else ""), shp, f"jmut_{it}_{k}")
    for k, line in enumerate(JEDGE):
        add_jsonl(line + "\n", FULL, f"jedge_{k}")

    path = os.path.join(HERE, "ingest_cases.json")
    with open(path, "w") as fh:
        json.dump(cases, fh)
    n_ok = sum("ok" in c["result"] for c in cases)
    print(f"wrote {path}: {len(cases)} cases ({n_ok} valid)")


if __name__ == "__main__":
    main()
