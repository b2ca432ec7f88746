#!/bin/bash
# GPU box: one `ncu --set full` capture of kernel regex $1 from the headline bench -> gpurun_out/prof_$2.ncu-rep
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$1" -s ${3:-1} -c 1 \
  -o gpurun_out/prof_$2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --eam-sketches 0 \
  --transformer-prompts 0 > gpurun_out/ncu_$2.log 2>&1
tail -2 gpurun_out/ncu_$2.log
