#!/bin/bash
# GPU box: the V3 (58 x 256) exact LRU kernel with the key-position table in
# global memory (default) vs shared memory (MOEB_K1_POS=smem): tests + C5 times
mkdir -p gpurun_out
timeout 600 python -m pytest -q -x tests/test_gpu_pos_table.py > gpurun_out/pos_table_tests.log 2>&1
tail -2 gpurun_out/pos_table_tests.log
for v in global smem global; do
  if [ $v = smem ]; then export MOEB_K1_POS=smem; else unset MOEB_K1_POS; fi
  echo "== $v"
  timeout 600 python tools/bench_sweep.py c5 --no-transformer 2>&1 | grep -E "^(lru|lfu|learned)"
done 2>&1 | tee gpurun_out/pos_table_probe.log
