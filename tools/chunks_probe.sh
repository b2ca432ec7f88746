#!/bin/bash
# GPU box: the headline step with the C2 batch split into 1-4 prompt chunks
# pipelined across the predict / replay streams (K3t of chunk i+1 beside
# K1s of chunk i)
mkdir -p gpurun_out
for c in 1 2 3 4 1 2 3 4; do
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --eam-sketches 0 \
    --transformer-prompts 0 --chunks $c 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('chunks $c', round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,1), 'M dev', round(d['e2e']['value']/1e6,1), 'M e2e', d['kernels_ms'])"
done 2>&1 | tee gpurun_out/chunks_probe.log
