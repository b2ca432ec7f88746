#!/bin/bash
# GPU box: the final round-2 evidence -- tests + smoke, the default bench
# line, the reference arm, the launch list of the bench command
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/tests_final.log 2>&1; tail -1 gpurun_out/tests_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
python -c "
import json; d=json.load(open('gpurun_out/bench_final.json'))
print(d['value'], d['e2e']['value'], d['pipelined_steps']['value'], d['ms_per_step'], d['roofline']['frac'], d['parity']['counters_equal'], d['clocks'])"
timeout 900 python bench.py --impl reference --steps 3 > gpurun_out/bench_ref_final.json 2>&1
tail -c 300 gpurun_out/bench_ref_final.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  --eam-sketches 0 --transformer-prompts 0 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/launches_final.csv > gpurun_out/launches_final.txt 2>&1
head -14 gpurun_out/launches_final.txt
