#!/bin/bash
# GPU box: e2e with the first 6-bit-id batch landing range by range (default)
# vs as one copy (MOEB_STREAM_SPLIT=0), interleaved
mkdir -p gpurun_out
timeout 600 python -m pytest -q -x tests/test_gpu_streaming.py 2>&1 | tail -1
for v in 1 0 1 0 1 0; do
  MOEB_STREAM_SPLIT=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --eam-sketches 0 --transformer-prompts 0 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('split=$v', round(d['value']/1e6,1), 'M dev', round(d['e2e']['value']/1e6,1), 'M e2e')"
done 2>&1 | tee gpurun_out/ids6_split_probe.log
