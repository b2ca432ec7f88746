"""A small run of every replay/predict kernel for compute-sanitizer
(tools/sanitize.sh): K3t + refine + exact re-evaluation, the fp64 K3, K1s +
the exact LRU kernel (with and without prompts handed over), K1m, the LFU
kernel, K6 (EAM session), K7 (metrics), the rank wire formats (u32 and the
packed stream), the transformer forward (GEMMs, the persistent attention,
LayerNorm) and one training step (attention backward, optimiser)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_17137_b200 as m  # noqa: E402


def main():
    m.load_library()
    shape = m.ModelShape(26, 64, 6)
    packed = m.generate_packed(m.GeneratorConfig(24, 60, shape, 8, 0.9, 7))
    w = np.random.default_rng(0).normal(0.0, 0.01, (64, 91))
    model = m.LinearModel(shape, m.LearnerConfig(epochs=0), w, trained=True)
    lin = m.make_predictor("learned_linear", shape, model=model)
    cnt = torch.zeros(54, dtype=torch.int64, device="cuda")
    masks = lin.predict_masks(packed, 6, 8, counts=cnt)            # K3t
    os.environ["MOEB_K3"] = "fp64"
    masks64 = lin.predict_masks(packed, 6, 8, counts=cnt)          # fp64 K3
    os.environ.pop("MOEB_K3")
    assert torch.equal(masks, masks64)
    caps = [5, 83, 166, 416, 832]
    for stack in ("1", "0"):
        os.environ["MOEB_K1_STACK"] = stack
        m.cache_replay(packed, [(masks, None, False), (None, None, False)], caps, 8, 6)
    os.environ.pop("MOEB_K1_STACK")
    m.cache_replay(packed, [(masks, None, False)], caps, 8, 6, policy="lfu")
    train = m.generate_packed(m.GeneratorConfig(30, 40, shape, 8, 0.9, 7, first_prompt_id=1000))
    eamc = m.build_eamc(train, m.EamcConfig(mode="recent", capacity=30))
    m.make_predictor("eam_cosine", shape, eamc=eamc).predict_masks(packed, 6, 8)   # K6
    vec = m.metrics.metric_vector(64, packed.device)
    m.metrics.mask_metrics(masks, packed.truth, packed.row_off, 26, 64, 8, vec)  # K7
    os.environ["MOEB_K1M"] = "all"                                  # K1m
    m.cache_replay(packed, [(masks, None, False)], [83, 166, 249, 332, 416, 499, 665, 832], 8, 6)
    os.environ.pop("MOEB_K1M")
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    for packed_fmt in (False, True):
        ranks = m.masks_to_ranks(packed.truth, 6, 64, packed=packed_fmt)
        back = torch.empty_like(packed.truth)
        m.ranks_to_masks(ranks, 6, 64, back, bad, rows=packed.rows)
        torch.cuda.synchronize()
        assert torch.equal(back, packed.truth)
    # transformer forward and one training step on a few prompts
    from oracle import transformer_ref as R
    from paper_2508_17137_b200 import transformer as T
    from paper_2508_17137_b200 import transformer_train as TT
    small = m.generate_packed(m.GeneratorConfig(3, 30, shape, 8, 0.9, 7))
    ref = R.TransformerRef(R.TransformerSpec(26, 64, seed=0))
    W = T.TransformerWeights(R.export_weights(ref), 26, 64)
    m.make_predictor("transformer", shape, transformer=W).forward_logits(small)
    TT.TransformerTrainer(R.export_weights(ref), 26, 64).step(small)
    torch.cuda.synchronize()
    print("sanitize case done")


if __name__ == "__main__":
    main()
