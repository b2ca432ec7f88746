"""Transformer predictor training step throughput (1 GPU): one step = forward
with saved activations, BCE loss, backward, clipping and AdamW, over a batch
of whole C2 prompts (synthetic traces, random-init weights).

    python tools/bench_train_transformer.py [--prompts 16] [--steps 5]
"""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2508_17137_b200 as m  # noqa: E402
from paper_2508_17137_b200 import transformer as T  # noqa: E402
from paper_2508_17137_b200 import transformer_train as TT  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prompts", type=int, default=16)
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    m.load_library()
    shape = m.ModelShape(26, 64, 6)
    packed = m.generate_packed(m.GeneratorConfig(args.prompts, 363, shape, 8, 0.9, 7))
    tr = TT.TransformerTrainer(T.init_state(26, 64, seed=0), 26, 64)
    for _ in range(2):
        tr.step(packed)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    s.record()
    losses = []
    for _ in range(args.steps):
        losses.append(tr.step(packed)["loss"])
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / args.steps
    print(json.dumps({"prompts": args.prompts, "rows": packed.rows, "ms_per_step": ms,
                      "trace_tok_per_s": packed.rows / 26 / (ms / 1e3),
                      "rows_per_s": packed.rows / (ms / 1e3), "losses": losses,
                      "wall_s": time.time() - t0}))


if __name__ == "__main__":
    main()
