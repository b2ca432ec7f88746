import os, sys, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2508_17137_b200 as m
m.load_library()
shape = m.ModelShape(26, 64, 6)
packed = m.generate_packed(m.GeneratorConfig(int(sys.argv[1]), 363, shape, 8, 0.9, 7))
caps = [m.CacheConfig(capacity_fraction=f).resolve_capacity(shape) for f in (0.15,0.2,0.25,0.3,0.4,0.5)]
os.environ["MOEB_K1M"] = "all"
for _ in range(2):
    m.cache_replay(packed, [(None, None, False)], caps, 8, 6, want_per_prompt=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); m.cache_replay(packed, [(None, None, False)], caps, 8, 6, want_per_prompt=False); e1.record(); torch.cuda.synchronize()
print("K1m ms", e0.elapsed_time(e1))
