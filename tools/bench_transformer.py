"""Transformer predictor throughput on a slice of the C2 workload (1 GPU).

    python tools/bench_transformer.py [--prompts 700] [--steps 3]

Prints per-stage CUDA-event times and achieved TFLOP/s (algorithmic FLOPs:
SURVEY §8(d), attention counted with the actual window lengths)."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2508_17137_b200 as m  # noqa: E402
from paper_2508_17137_b200 import _native as nat  # noqa: E402
from paper_2508_17137_b200 import transformer as T  # noqa: E402


def flops_per_pass(rows, win_lens, E):
    d, F, dh = 512, 2048, 256
    dense = rows * (4 * (2 * d * 3 * d + 2 * d * d + 4 * d * F) + 2 * d * dh + 2 * dh * E)
    attn = 4 * sum(4 * int(n) * int(n) * d for n in win_lens)  # 4 layers, QK^T + PV
    return dense, attn


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prompts", type=int, default=700)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--bf16", action="store_true")
    args = ap.parse_args()
    m.load_library()
    shape = m.ModelShape(26, 64, 6)
    packed = m.generate_packed(m.GeneratorConfig(args.prompts, 363, shape, 8, 0.9, 7))
    t0 = time.time()
    W = T.TransformerWeights.random(26, 64, seed=0, fp16=not args.bf16)
    torch.cuda.synchronize()
    init_s = time.time() - t0
    pred = m.make_predictor("transformer", shape, transformer=W)
    ws, wl = T.windows_of(packed.row_off_host)
    dense, attn = flops_per_pass(packed.rows, wl, 64)
    for _ in range(2):
        pred.forward_logits(packed)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(args.steps):
        pred.forward_logits(packed)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / args.steps
    timing = {}
    pred.forward_logits(packed, timing=timing)
    torch.cuda.synchronize()
    stages = {k: round(sum(a.elapsed_time(b) for a, b, _ in v), 3) for k, v in timing.items()}
    out = {"rows": packed.rows, "tokens": packed.rows // 26, "ms": ms, "stages_ms": stages,
           "trace_tok_per_s": packed.rows / 26 / (ms / 1e3),
           "tflops_total": (dense + attn) / (ms / 1e3) / 1e12,
           "dense_tflop": dense / 1e12, "attn_tflop": attn / 1e12, "init_s": init_s}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
