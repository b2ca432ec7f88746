#!/bin/bash
# GPU box: transformer stages with 2-SM pair GEMM tiles (default) vs single-CTA tiles
for v in 1 0 1 0; do
  MOEB_GEMM_PAIR=$v timeout 300 python tools/bench_transformer.py --prompts 700 --steps 3 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('pair=$v', round(d['ms'],1), d['stages_ms'])"
done 2>&1 | tee gpurun_out/gemm_pair_probe.log
