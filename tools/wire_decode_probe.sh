#!/bin/bash
# GPU box: decode-kernel times of the e2e wire formats (ncu launch list)
mkdir -p gpurun_out
timeout 600 python -m pytest -q -x tests/test_gpu_streaming.py 2>&1 | tail -1
for f in idpairs ids6 packed-ranks; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"to_masks" --csv \
    --log-file gpurun_out/wire_$f.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    --eam-sketches 0 --transformer-prompts 0 --e2e-format $f > /dev/null 2>&1
  echo "== $f"; python tools/ncu_summary.py launches gpurun_out/wire_$f.csv 2>&1 | head -3
done 2>&1 | tee gpurun_out/wire_decode_probe.log
