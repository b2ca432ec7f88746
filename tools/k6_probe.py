"""K6 (EAM cosine session predictor) on the full C2 batch: the token-batched
kernel vs the row-by-row one (MOEB_K6=row); identical indices and masks."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_17137_b200 as m  # noqa: E402


def main():
    m.load_library()
    shape = m.ModelShape(26, 64, 6)
    P = int(sys.argv[1]) if len(sys.argv) > 1 else 6994
    packed = m.generate_packed(m.GeneratorConfig(P, 363, shape, 8, 0.9, 7))
    tr = m.generate_packed(m.GeneratorConfig(100, 363, shape, 8, 0.9, 7, first_prompt_id=10**6))
    eamc = m.build_eamc(tr, m.EamcConfig(mode="recent", capacity=100))
    pred = m.make_predictor("eam_cosine", shape, eamc=eamc)
    out = {}
    for mode in ("tok", "row"):
        if mode == "row":
            os.environ["MOEB_K6"] = "row"
        else:
            os.environ.pop("MOEB_K6", None)
        idx = torch.empty(packed.rows, dtype=torch.int32, device="cuda")
        masks = pred.predict_masks(packed, 6, 8, idx_out=idx)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            masks = pred.predict_masks(packed, 6, 8, idx_out=idx)
        e1.record()
        torch.cuda.synchronize()
        out[mode] = (masks.clone(), idx.clone())
        print(mode, "ms", round(e0.elapsed_time(e1) / 3, 3), flush=True)
    print("masks equal", torch.equal(out["tok"][0], out["row"][0]),
          "idx equal", torch.equal(out["tok"][1], out["row"][1]))


if __name__ == "__main__":
    main()
