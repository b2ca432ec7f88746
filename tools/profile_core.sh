#!/bin/bash
# GPU box: tests, the default bench line, the launch list and ncu captures of
# the headline kernels only (K1s, K1, K3) -> gpurun_out/ (stays under 64 MiB).
TAG=${1:-run}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/tests_$TAG.log 2>&1; tail -2 gpurun_out/tests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -c 300 gpurun_out/bench_$TAG.json; tail -2 gpurun_out/bench_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_launches_$TAG.log 2>&1
cap() {  # regex name skip
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:$1" -s $3 -c 1 -o gpurun_out/prof_${TAG}_$2 python bench.py --steps 1 --warmup 3 \
    --no-cpu-baseline --eam-sketches 0 --transformer-prompts 0 > gpurun_out/ncu_${TAG}_$2.log 2>&1
}
cap "k_stack_replay" k1s 1
cap "k_cache_sim_warp" k1 1
cap "k_linear_predict" k3 1
du -sh gpurun_out
