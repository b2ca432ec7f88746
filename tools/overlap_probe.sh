#!/bin/bash
# GPU box: e2e leg (default wire format) with batch i+1's predictor beside
# batch i's replay (MOEB_STREAM_OVERLAP=1) vs one compute stream, interleaved
mkdir -p gpurun_out
for o in 1 0 1 0 1 0; do
  MOEB_STREAM_OVERLAP=$o timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --eam-sketches 0 --transformer-prompts 0 2>gpurun_out/overlap.err | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('stream_overlap=$o', round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,1), 'M dev', round(d['e2e']['value']/1e6,1), 'M e2e')"
done 2>&1 | tee gpurun_out/overlap_probe_ids6.log
python tools/h2d_probe.py 2>&1 | tail -3
