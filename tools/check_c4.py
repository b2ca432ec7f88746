"""Full-scale C4 exactness check: tensor-core matcher vs the fp64 brute-force
scan (moeb_match_queries) on 100k sketches x 1920 layer-0 queries."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_17137_b200 as m  # noqa: E402
from paper_2508_17137_b200 import sketches as SK  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
shape = m.ModelShape(26, 64, 6)
lib = m.generate_packed(m.GeneratorConfig(S, 32, shape, 8, 0.9, 11, first_prompt_id=10**6))
coll = SK.build_eamc(lib, SK.EamcConfig(mode="recent", capacity=S))
q = SK.token_query_counts(m.generate_packed(m.GeneratorConfig(16, 128, shape, 8, 0.9, 7)), 8)
tc = SK.TensorCoreMatcher(coll)
idx, sim, nrr = tc.match_counts(q)
t0 = time.time()
bidx, bsim = coll.match_nearest_batch(q.to(torch.float64).cpu().numpy())
bt = time.time() - t0
got = idx.cpu().numpy()
bad = np.nonzero(got != bidx)[0]
print(f"S={S} queries={len(got)} mismatches={len(bad)} brute-force {bt:.1f}s "
      f"max|dsim|={np.abs(sim.cpu().numpy() - bsim).max():.2e} reranked/query={nrr.float().mean():.3f}")
for i in bad[:5]:
    print(i, got[i], bidx[i], sim[i].item(), bsim[i])
sys.exit(1 if len(bad) else 0)
