#!/bin/bash
# GPU box: K7 (k_metrics64) with the 4-row carry-save adders: metric tests,
# the headline bench (device + e2e), and K7's launch times (ncu)
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_k3t.py > gpurun_out/k7_tests.log 2>&1
tail -2 gpurun_out/k7_tests.log
for i in 1 2; do
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --eam-sketches 0 --transformer-prompts 0 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,1), 'M dev', round(d['e2e']['value']/1e6,1), 'M e2e', d['kernels_ms'], d['parity']['counters_equal'], d['parity']['metric_counts_equal'])"
done 2>&1 | tee gpurun_out/k7_probe.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_metrics64|k_stack_replay" --csv \
  --log-file gpurun_out/k7_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  --eam-sketches 0 --transformer-prompts 0 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/k7_launches.csv 2>&1 | head -8
