#!/bin/bash
# GPU box: transformer leg of bench.py (700-prompt C2 slice), per-kernel times
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --eam-sketches 0 "$@" 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); t=d['transformer']
print('tok/s', round(t['trace_tok_per_s']), 'ms', round(t['ms_per_step'],1), 'TF', round(t['tflops_achieved'],1))
for k,v in t['kernels'].items(): print('  ', k, round(v['ms'],2), 'ms', round(v['tflops'],1), 'TF/s')
print('  hit', t['hit_rate_10pct'], t['prediction'])"
