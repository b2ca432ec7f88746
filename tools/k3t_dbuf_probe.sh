#!/bin/bash
# GPU box: K3t with two TMEM accumulators: K3t tests + parity, bench x2
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_k3t.py tests/test_gpu_parity.py > gpurun_out/k3t_dbuf_tests.log 2>&1
tail -1 gpurun_out/k3t_dbuf_tests.log
for i in 1 2 3; do
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --eam-sketches 0 --transformer-prompts 0 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,1), 'M dev', round(d['e2e']['value']/1e6,1), 'M e2e', round(d['pipelined_steps']['value']/1e6,1), 'M pipelined', d['kernels_ms']['k_linear_tc'], d['parity']['counters_equal'])"
done 2>&1 | tee gpurun_out/k3t_dbuf_probe.log
