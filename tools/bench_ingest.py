"""Trace-ingestion benchmark: the C2 trace (6,994 prompts x
363 tokens x 26 layers, 66 M rows) as the reference's CSV, parsed on device,
against the reference's parse_trace_csv on a bounded sample on the host.

    python tools/bench_ingest.py [--prompts 6994] [--ref-prompts 8]

Prints one JSON line: device writer / parser throughput (rows/s, file GB/s),
per-kernel CUDA-event times with their HBM roofline fraction, end-to-end
parse from host bytes, and the reference's rows/s.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prompts", type=int, default=6994)
    ap.add_argument("--tokens", type=int, default=363)
    ap.add_argument("--ref-prompts", type=int, default=8)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_2508_17137_b200 as m
    from paper_2508_17137_b200 import _native as nat
    from paper_2508_17137_b200 import traceio as tio

    m.load_library()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm = float(peaks["hbm_gbs"])
    shape = m.ModelShape(26, 64, 6)
    packed = m.generate_packed(m.GeneratorConfig(args.prompts, args.tokens, shape, 8, 0.9, 7))
    rows = packed.rows
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    # device writer
    m.write_trace_csv(packed.select(0, min(8, packed.num_prompts)))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    blob = m.write_trace_csv(packed)
    w_s = time.perf_counter() - t0
    nbytes = len(blob)

    # device parser, end to end from host bytes (H2D inside)
    for _ in range(1):
        back = m.parse_trace_csv(blob, shape)
    torch.cuda.synchronize()
    e2e = []
    for _ in range(args.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        back = m.parse_trace_csv(blob, shape)
        torch.cuda.synchronize()
        e2e.append(time.perf_counter() - t0)
    assert torch.equal(back.truth, packed.truth), "round trip"

    # kernel timings (inputs resident)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    buf = tio._upload(blob, packed.device)
    torch.cuda.synchronize()
    upload_s = time.perf_counter() - t0
    a, b = ev(), ev()
    a.record()
    nl = tio._find_bytes(buf, nbytes, 10)
    b.record()
    torch.cuda.synchronize()
    scan_ms = a.elapsed_time(b)
    n_data = nl.numel() - 1
    W = 1
    dev = packed.device
    outs = dict(status=torch.empty(n_data, dtype=torch.uint8, device=dev),
                pid=torch.empty(n_data, dtype=torch.int64, device=dev),
                tok=torch.empty(n_data, dtype=torch.int64, device=dev),
                lay=torch.empty(n_data, dtype=torch.int32, device=dev),
                masks=torch.empty((n_data, W), dtype=torch.int64, device=dev),
                tid=torch.empty(n_data, dtype=torch.int64, device=dev),
                emb=torch.empty(n_data, dtype=torch.uint8, device=dev))
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    times = []
    for _ in range(args.reps + 1):
        a, b = ev(), ev()
        a.record()
        nat.call("moeb_parse_trace_csv", nat.ptr(buf), nbytes, nat.ptr(nl), nl.numel(), 1,
                 n_data, 26, 64, 6, *(nat.ptr(outs[k]) for k in
                                      ("status", "pid", "tok", "lay", "masks", "tid", "emb")),
                 nat.ptr(flags), nat.stream_ptr())
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    parse_ms = min(times[1:])
    out_bytes_per_row = 1 + 8 + 8 + 4 + 8 * W + 8 + 1
    parse_bytes = nbytes + n_data * out_bytes_per_row

    # reference on a bounded sample (host, single process: the reference parser is serial)
    ref = None
    sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
    try:
        from moesim import traceio as rtio
        sample = m.write_trace_csv(packed.select(0, args.ref_prompts))
        rshape = __import__("moesim").ModelShape(26, 64, 6)
        t0 = time.perf_counter()
        rtio.parse_trace_csv(sample, rshape)
        dt = time.perf_counter() - t0
        srows = int(packed.row_off_host[args.ref_prompts])
        ref = {"rows_per_s": srows / dt, "seconds": dt, "sample_rows": srows, "cores": 1,
               "sample": f"{args.ref_prompts} C2 prompts ({len(sample)} bytes), "
                         "moesim.traceio.parse_trace_csv"}
    except Exception as exc:  # noqa: BLE001
        ref = {"unavailable": str(exc)}

    print(json.dumps({
        "workload": f"C2 trace CSV: {args.prompts} prompts x {args.tokens} tokens x 26 layers",
        "rows": rows, "csv_bytes": nbytes,
        "write_s": w_s, "write_rows_per_s": rows / w_s,
        "parse_e2e_s": min(e2e), "parse_e2e_rows_per_s": rows / min(e2e),
        "parse_e2e_file_gbs": nbytes / min(e2e) / 1e9,
        "upload_s": upload_s, "upload_gbs": nbytes / upload_s / 1e9,
        "kernels": {
            "newline_scan": {"ms": scan_ms, "bytes": 2 * nbytes,
                             "gbs": 2 * nbytes / scan_ms / 1e6,
                             "frac_hbm": 2 * nbytes / scan_ms / 1e6 / hbm},
            "k_parse_trace_csv": {"ms": parse_ms, "bytes": parse_bytes,
                                  "gbs": parse_bytes / parse_ms / 1e6,
                                  "frac_hbm": parse_bytes / parse_ms / 1e6 / hbm,
                                  "algorithmic": f"file bytes + {out_bytes_per_row} B/row"}},
        "reference": ref,
        "speedup_e2e_vs_reference": (rows / min(e2e)) / ref["rows_per_s"] if "rows_per_s" in ref
        else None,
    }))


if __name__ == "__main__":
    main()
