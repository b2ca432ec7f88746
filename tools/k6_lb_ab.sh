#!/bin/bash
# GPU box: K6 token-batched kernel with register caps (5 / 6 CTAs per SM) vs 4
for v in base eam5 eam6 base eam5 eam6; do
  if [ $v = base ]; then L=""; else L=$PWD/build_alt/libmoeb_$v.so; fi
  echo "== $v"; MOEB_LIB=$L timeout 300 python tools/k6_probe.py 2>&1 | tail -3
done 2>&1 | tee gpurun_out/k6_lb_ab.log
