#!/bin/bash
# GPU box: id-pair decode by square root: streaming tests, decode times, e2e A/B
mkdir -p gpurun_out
timeout 600 python -m pytest -q -x tests/test_gpu_streaming.py 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"to_masks" --csv \
  --log-file gpurun_out/wire_idpairs2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  --eam-sketches 0 --transformer-prompts 0 --e2e-format idpairs > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/wire_idpairs2.csv 2>&1 | head -3
for f in idpairs ids6 idpairs ids6 idpairs ids6; do
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --eam-sketches 0 --transformer-prompts 0 --e2e-format $f 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$f', round(d['value']/1e6,1), 'M dev', round(d['e2e']['value']/1e6,1), 'M e2e')"
done 2>&1 | tee gpurun_out/idpairs_probe.log
