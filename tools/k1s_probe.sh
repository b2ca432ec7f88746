#!/bin/bash
# GPU box: K1s with its row loads one batch ahead: stack / parity tests, the
# headline bench twice, K1s launch times (ncu)
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_stack.py tests/test_gpu_parity.py > gpurun_out/k1s_tests.log 2>&1
tail -1 gpurun_out/k1s_tests.log
for i in 1 2; do
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --eam-sketches 0 --transformer-prompts 0 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,1), 'M dev', round(d['e2e']['value']/1e6,1), 'M e2e', round(d['pipelined_steps']['value']/1e6,1), 'M pipelined', d['kernels_ms']['k_cache_sim'], d['parity']['counters_equal'])"
done 2>&1 | tee gpurun_out/k1s_probe.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_stack_replay|k_metrics64" --csv \
  --log-file gpurun_out/k1s_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  --eam-sketches 0 --transformer-prompts 0 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/k1s_launches.csv 2>&1 | head -5
