#!/bin/bash
# GPU box: one ncu --set full capture of kernel regex $1 from the transformer leg
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$1" -s ${3:-2} -c 1 \
  -o gpurun_out/prof_$2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --eam-sketches 0 \
  --transformer-prompts 200 > gpurun_out/ncu_$2.log 2>&1
tail -2 gpurun_out/ncu_$2.log
