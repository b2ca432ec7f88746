import os, sys, torch
sys.path.insert(0, "/root/repo")
import paper_2508_17137_b200 as m
m.load_library()
shape = m.ModelShape(26, 64, 6)
packed = m.generate_packed(m.GeneratorConfig(6994, 363, shape, 8, 0.9, 7))
for packed_fmt in (False, True):
    ranks = m.masks_to_ranks(packed.truth, 6, 64, packed=packed_fmt)
    out = torch.empty_like(packed.truth)
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    f = lambda: m.ranks_to_masks(ranks, 6, 64, out, bad, rows=packed.rows)
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): f()
    e1.record(); torch.cuda.synchronize()
    ok = torch.equal(out, packed.truth)
    print(os.environ.get("MOEB_RANK_DECODE", "seeded"), "packed" if packed_fmt else "u32", round(e0.elapsed_time(e1) / 20, 3), "ms", ok)
