#!/bin/bash
# Run on the GPU box (under gpurun): parity tests, bench, ncu launch list and
# one `ncu --set full` capture per kernel regex. Outputs land in gpurun_out/.
#   tools/profile.sh TAG [kernel-regex ...]
TAG=${1:-run}; shift
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/tests_$TAG.log 2>&1; tail -3 gpurun_out/tests_$TAG.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_launches_$TAG.log 2>&1
for k in "$@"; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
    -o gpurun_out/prof_${TAG}_$k python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_${TAG}_$k.log 2>&1
done
ls gpurun_out
