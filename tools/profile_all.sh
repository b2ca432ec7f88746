#!/bin/bash
# GPU box: full round evidence -- GPU tests, default bench line, ncu launch
# list, and one `ncu --set full` capture per hot kernel. TAG = $1.
TAG=${1:-run}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/tests_$TAG.log 2>&1; tail -2 gpurun_out/tests_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -c 600 gpurun_out/bench_$TAG.json; tail -2 gpurun_out/bench_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_launches_$TAG.log 2>&1
cap() {  # regex name skip
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:$1" -s $3 -c 1 -o gpurun_out/prof_${TAG}_$2 python bench.py --steps 1 --warmup 3 \
    --no-cpu-baseline --eam-sketches 0 --transformer-prompts 200 > gpurun_out/ncu_${TAG}_$2.log 2>&1
}
cap "k_cache_sim_warp" k1 1
cap "k_linear_predict" k3 1
cap "k_window_attention_fa" attn 2
cap "k_gemm<.int.256, .int.5, .int.2," gemm_ffn1 2
cap "k_gemm<.int.256, .int.4, .int.6," gemm_resid 2
cap "k_layernorm_rows" layernorm 2
ls gpurun_out | grep $TAG
