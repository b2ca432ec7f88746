#!/bin/bash
# GPU box: the e2e leg with packed 6-bit ids (4.5 B/row, shift decode) vs the
# 27-bit rank stream (3.375 B/row, digit-search decode), interleaved
mkdir -p gpurun_out
timeout 600 python -m pytest -q -x tests/test_gpu_streaming.py > gpurun_out/ids6_tests.log 2>&1
tail -1 gpurun_out/ids6_tests.log
for f in idpairs ids6 packed-ranks idpairs ids6 packed-ranks; do
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --eam-sketches 0 --transformer-prompts 0 --e2e-format $f 2>gpurun_out/ids6.err | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$f', round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,1), 'M dev', round(d['e2e']['value']/1e6,1), 'M e2e', d['e2e']['h2d_bytes_per_step'])"
done 2>&1 | tee gpurun_out/ids6_probe.log
tail -2 gpurun_out/ids6.err
