import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2508_17137_b200 as m
from paper_2508_17137_b200 import sketches as SK
m.load_library()
shape = m.ModelShape(26, 64, 6)
packed = m.generate_packed(m.GeneratorConfig(2000, 363, shape, 8, 0.9, 7))
eamc_tr = m.generate_packed(m.GeneratorConfig(100, 363, shape, 8, 0.9, 7, first_prompt_id=10**6))
coll = SK.build_eamc(eamc_tr, SK.EamcConfig(mode="recent", capacity=100))
pred = m.make_predictor("eam_cosine", shape, eamc=coll)
for _ in range(2):
    pred.predict_masks(packed, 6, 8)
torch.cuda.synchronize()
