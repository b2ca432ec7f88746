"""Where the end-to-end step goes: H2D copy of the C2 rank batch alone, its
device decode alone, and both on a copy stream beside K3 on another stream."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_17137_b200 as m  # noqa: E402


def timed(fn, stream=None, n=5):
    s = stream or torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(n):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def main():
    m.load_library()
    shape = m.ModelShape(26, 64, 6)
    packed = m.generate_packed(m.GeneratorConfig(6994, 363, shape, 8, 0.9, 7))
    ranks = m.masks_to_ranks(packed.truth, 6, 64)
    host = ranks.cpu().pin_memory()
    dev = torch.empty_like(ranks)
    out = torch.empty_like(packed.truth)
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    print("copy alone ms", round(timed(lambda: dev.copy_(host, non_blocking=True)), 3))
    print("decode alone ms", round(timed(lambda: m.ranks_to_masks(dev, 6, 64, out, bad)), 3))
    w = np.random.default_rng(0).normal(0.0, 0.01, (64, 91))
    model = m.LinearModel(shape, m.LearnerConfig(epochs=0), w, trained=True)
    pred = m.make_predictor("learned_linear", shape, model=model)
    cnt = torch.zeros(54, dtype=torch.int64, device="cuda")
    print("K3 alone ms", round(timed(lambda: pred.predict_masks(packed, 6, 8, counts=cnt)), 3))
    sc, sk = torch.cuda.Stream(), torch.cuda.Stream()

    def both():
        with torch.cuda.stream(sc):
            dev.copy_(host, non_blocking=True)
            m.ranks_to_masks(dev, 6, 64, out, bad)
        with torch.cuda.stream(sk):
            pred.predict_masks(packed, 6, 8, counts=cnt)
        torch.cuda.current_stream().wait_stream(sc)
        torch.cuda.current_stream().wait_stream(sk)

    print("copy+decode || K3 ms", round(timed(both), 3))

    def copy_k3():
        with torch.cuda.stream(sc):
            dev.copy_(host, non_blocking=True)
        with torch.cuda.stream(sk):
            pred.predict_masks(packed, 6, 8, counts=cnt)
        torch.cuda.current_stream().wait_stream(sc)
        torch.cuda.current_stream().wait_stream(sk)

    print("copy || K3 ms", round(timed(copy_k3), 3))
    for i in range(4):
        print("K3 alone again ms", round(timed(lambda: pred.predict_masks(packed, 6, 8, counts=cnt)), 3))
        print("copy || K3 again ms", round(timed(copy_k3), 3))
    ws = m._native.workspace(m._native.load_library().moeb_linear_workspace_bytes(packed.rows, 26, 64), "cuda")
    outm = torch.empty_like(packed.truth)
    from paper_2508_17137_b200 import _native as nat

    def raw():
        nat.call("moeb_linear_predict_counts", nat.ptr(packed.truth), nat.ptr(packed.row_off),
                 packed.num_prompts, 26, 64, nat.ptr(pred.weights_on(packed.device)), 0.9, 6, 0, 8, 6,
                 nat.ptr(outm), None, None, nat.ptr(cnt), packed.rows, nat.ptr(ws), ws.numel(),
                 nat.stream_ptr())
    for i in range(3):
        print("K3 raw (fixed workspace) ms", round(timed(raw), 3))


if __name__ == "__main__":
    main()
