#!/bin/bash
# GPU box: K1m layouts -- last-access tables in global memory + 4-bit row
# counts (default), global + u8 (MOEB_K1M_NIB=0), all in shared memory
# (MOEB_K1M_LR=smem MOEB_K1M_NIB=0): stack tests + the C3 sweep
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_stack.py > gpurun_out/k1m_lr_tests.log 2>&1
tail -2 gpurun_out/k1m_lr_tests.log
for v in nib u8 smem nib u8 smem; do
  unset MOEB_K1M_LR MOEB_K1M_NIB
  [ $v = u8 ] && export MOEB_K1M_NIB=0
  [ $v = smem ] && export MOEB_K1M_NIB=0 MOEB_K1M_LR=smem
  echo "== $v"
  timeout 900 python tools/bench_sweep.py c3 --no-transformer 2>&1 | grep -E "^(lru_only|learned_linear)" | cut -c1-130
done 2>&1 | tee gpurun_out/k1m_lr_probe.log
