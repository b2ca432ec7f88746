"""BASELINE C3 / C5 runs on one GPU (results into gpurun_out/, summarised in
profiles/).

  python tools/bench_sweep.py c3 [--prompts 6994]   capacity sweep 5-50 % x
      {LRU, LFU, MoE-Infinity eam_cosine (recent EAMC, S=100 from 100 disjoint
      prompts), learned_linear, transformer} on C2 traces
  python tools/bench_sweep.py c5 [--prompts 7000]   DeepSeek-V3 shape
      (58 x 256, top-8, hot 16), 128 tokens: transformer + LRU / LFU 10 %
All timings are CUDA-event device times; hit rates are exact counters.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_17137_b200 as m  # noqa: E402
from paper_2508_17137_b200 import sketches as SK  # noqa: E402
from paper_2508_17137_b200 import transformer as TR  # noqa: E402

CAPS = [0.05, 0.10, 0.15, 0.20, 0.25, 0.30, 0.40, 0.50]


def timed(fn):
    """CUDA-event time of one call, after one untimed warm-up call (lazy
    module loading, workspace allocation)."""
    fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1)


def c3(args):
    shape = m.ModelShape(26, 64, 6)
    packed = m.generate_packed(m.GeneratorConfig(args.prompts, 363, shape, 8, 0.9, 7))
    toks = packed.rows // 26
    caps = [m.CacheConfig(capacity_fraction=f).resolve_capacity(shape) for f in CAPS]
    eamc_tr = m.generate_packed(m.GeneratorConfig(100, 363, shape, 8, 0.9, 7,
                                                  first_prompt_id=10**6))
    coll = SK.build_eamc(eamc_tr, SK.EamcConfig(mode="recent", capacity=100))
    w = np.random.default_rng(0).normal(0.0, 0.01, (64, 91))
    model = m.LinearModel(shape, m.LearnerConfig(epochs=0), w, trained=True)
    preds = {
        "lru_only": m.make_predictor("lru_only", shape),
        "eam_cosine": m.make_predictor("eam_cosine", shape, eamc=coll),
        "learned_linear": m.make_predictor("learned_linear", shape, model=model),
    }
    if args.transformer:
        preds["transformer"] = m.make_predictor(
            "transformer", shape, transformer=TR.TransformerWeights.random(26, 64, seed=0))
    res = {"workload": f"C2 traces: {args.prompts} prompts x 363 tokens, 26x64 top-6",
           "capacities": CAPS, "capacity_entries": caps, "policies": {}}
    for kind, pred in preds.items():
        masks, pms = timed(lambda: pred.predict_masks(packed, 6, 8))
        policies = [("lru", kind)] + ([("lfu", "lfu")] if kind == "lru_only" else [])
        for pol, name in policies:
            stream = (None if kind == "lru_only" else masks, None, False)
            (cnt, _, _), sms = timed(lambda: m.cache_replay(packed, [stream], caps, 8, 6, pol,
                                                            want_per_prompt=False))
            c = cnt[0].cpu().numpy()
            res["policies"][name] = {
                "predict_ms": 0.0 if kind == "lru_only" else pms, "sim_ms_all_caps": sms,
                "trace_tok_per_s_all_caps": toks * len(caps) / ((pms + sms) / 1e3),
                "hit_rate": [int(c[j, 1]) / int(c[j, 0]) for j in range(len(caps))],
                "prediction_hit_rate": [int(c[j, 2]) / int(c[j, 0]) for j in range(len(caps))]}
            print(name, json.dumps(res["policies"][name]), flush=True)
    return res


def c5(args):
    shape = m.ModelShape(58, 256, 8)
    t0 = time.time()
    packed = m.generate_packed(m.GeneratorConfig(args.prompts, 128, shape, 16, 0.9, 7))
    gen_s = time.time() - t0
    toks = packed.rows // 58
    cap = m.CacheConfig(capacity_fraction=0.1).resolve_capacity(shape)
    res = {"workload": f"C5: {args.prompts} prompts x 128 tokens, 58x256 top-8, hot 16",
           "capacity_entries": cap, "generate_s": gen_s}
    for pol in ("lru", "lfu"):
        (cnt, _, _), sms = timed(lambda: m.cache_replay(packed, [(None, None, False)], [cap], 8,
                                                        8, pol, want_per_prompt=False))
        c = cnt[0, 0].cpu().numpy()
        res[f"{pol}_only"] = {"sim_ms": sms, "trace_tok_per_s": toks / (sms / 1e3),
                              "hit_rate": int(c[1]) / int(c[0])}
        print(pol, res[f"{pol}_only"], flush=True)
    # learned_linear on the V3 shape (wide K3, 256 experts) + LRU 10 %
    w = np.random.default_rng(0).normal(0.0, 0.01, (256, 58 + 256 + 1))
    lin = m.make_predictor("learned_linear", shape,
                           model=m.LinearModel(shape, m.LearnerConfig(epochs=0), w, trained=True))
    lin.predict_masks(packed.select(0, 8), 8, 8)
    masks, pms = timed(lambda: lin.predict_masks(packed, 8, 8))
    (cnt, _, _), sms = timed(lambda: m.cache_replay(packed, [(masks, None, False)], [cap], 8, 8,
                                                    want_per_prompt=False))
    c = cnt[0, 0].cpu().numpy()
    res["learned_linear"] = {"predict_ms": pms, "sim_ms": sms,
                             "trace_tok_per_s": toks / ((pms + sms) / 1e3),
                             "hit_rate": int(c[1]) / int(c[0]),
                             "prediction_hit_rate": int(c[2]) / int(c[0])}
    print("learned_linear", res["learned_linear"], flush=True)
    del masks
    if args.transformer:
        pred = m.make_predictor("transformer", shape,
                                transformer=TR.TransformerWeights.random(58, 256, seed=0))
        sub = packed.select(0, min(args.prompts, args.transformer_prompts))
        pred.predict_masks(sub, 8, 8)
        masks, pms = timed(lambda: pred.predict_masks(sub, 8, 8))
        (cnt, _, _), sms = timed(lambda: m.cache_replay(sub, [(masks, None, False)], [cap], 8, 8,
                                                        want_per_prompt=False))
        c = cnt[0, 0].cpu().numpy()
        res["transformer"] = {"prompts": sub.num_prompts, "predict_ms": pms, "sim_ms": sms,
                              "trace_tok_per_s": (sub.rows // 58) / ((pms + sms) / 1e3),
                              "hit_rate": int(c[1]) / int(c[0]),
                              "prediction_hit_rate": int(c[2]) / int(c[0])}
        print("transformer", res["transformer"], flush=True)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["c3", "c5"])
    ap.add_argument("--prompts", type=int, default=None)
    ap.add_argument("--no-transformer", dest="transformer", action="store_false")
    ap.add_argument("--transformer-prompts", type=int, default=700)
    args = ap.parse_args()
    m.load_library()
    if args.prompts is None:
        args.prompts = 6994 if args.which == "c3" else 7000
    out = (c3 if args.which == "c3" else c5)(args)
    os.makedirs("gpurun_out", exist_ok=True)
    with open(f"gpurun_out/{args.which}.json", "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
