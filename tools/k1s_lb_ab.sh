#!/bin/bash
# GPU box: K1s with __launch_bounds__(128, 10) (in-tree) vs without (build_alt/libmoeb_base.so), interleaved
for v in new base new base new base new base; do
  if [ $v = base ]; then L=$PWD/build_alt/libmoeb_base.so; else L=""; fi
  MOEB_LIB=$L timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --eam-sketches 0 --transformer-prompts 0 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,1), 'M dev', round(d['e2e']['value']/1e6,1), 'M e2e', round(d['pipelined_steps']['value']/1e6,1), 'M pipelined', round(d['kernels_ms']['k_cache_sim'],3))"
done 2>&1 | tee gpurun_out/k1s_lb_ab.log
