#!/bin/bash
# GPU box: the wide K3 (E > 64) with REDUX-based top-k: parity tests + C5 times
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_acceptance.py -k "learned or wide or ties or acceptance or v3" > gpurun_out/k3w_tests.log 2>&1
tail -1 gpurun_out/k3w_tests.log
for i in 1 2; do
  timeout 600 python tools/bench_sweep.py c5 --no-transformer 2>&1 | grep -E "^(lru|learned)"
done 2>&1 | tee gpurun_out/k3w_probe.log
