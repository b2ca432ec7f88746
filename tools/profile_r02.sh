#!/bin/bash
# GPU box: the round-2 evidence set -> gpurun_out/ (summarised into profiles/
# by tools/collect_r02.sh). Tests + smoke, the default bench line, the
# reference arm, the launch list, ncu captures of the headline kernels and
# the side workloads (C3 sweep, C5, transformer, training).
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/tests_$TAG.log 2>&1; tail -2 gpurun_out/tests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -c 400 gpurun_out/bench_$TAG.json; tail -2 gpurun_out/bench_$TAG.err
timeout 900 python bench.py --impl reference --steps 3 > gpurun_out/bench_ref_$TAG.json 2>&1
tail -c 300 gpurun_out/bench_ref_$TAG.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  --eam-sketches 0 --transformer-prompts 0 > gpurun_out/ncu_launches_$TAG.log 2>&1
cap() {  # regex name skip
  timeout 900 ncu --set full --clock-control none --import-source on \
    -k "regex:$1" -s $3 -c 1 -o gpurun_out/prof_${TAG}_$2 python bench.py --steps 1 --warmup 3 \
    --no-cpu-baseline --eam-sketches 0 --transformer-prompts 0 > gpurun_out/ncu_${TAG}_$2.log 2>&1
}
cap "^k_linear_tc$" k3t 1
cap "k_stack_replay" k1s 1
cap "k_ranks_to_masks" ranks 1
cap "k_metrics64" k7 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_eam_predict_tok -c 1 \
  -o gpurun_out/prof_${TAG}_k6 python tools/k6_probe.py 2000 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stack_multi -c 1 \
  -o gpurun_out/prof_${TAG}_k1m python tools/k1m_probe.py 2000 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_window_attention_fb -c 1 \
  -o gpurun_out/prof_${TAG}_attn python tools/bench_transformer.py > /dev/null 2>&1
timeout 600 python tools/rank_decode_probe.py > gpurun_out/rank_decode_$TAG.log 2>&1
timeout 600 python tools/bench_sweep.py c3 > gpurun_out/c3_$TAG.log 2>&1; tail -1 gpurun_out/c3_$TAG.log | cut -c1-200
timeout 600 python tools/bench_sweep.py c5 > gpurun_out/c5_$TAG.log 2>&1; tail -1 gpurun_out/c5_$TAG.log | cut -c1-200
timeout 600 python tools/bench_transformer.py > gpurun_out/transformer_$TAG.json 2>&1
timeout 600 python tools/bench_train_transformer.py > gpurun_out/train_transformer_$TAG.json 2>&1
timeout 600 python tools/k3_probe.py > gpurun_out/k3_probe_$TAG.log 2>&1
timeout 600 python tools/k6_probe.py > gpurun_out/k6_probe_$TAG.log 2>&1
# text summaries on the box (the captures themselves can exceed the merge limit)
for f in gpurun_out/prof_${TAG}_*.ncu-rep; do
  timeout 300 python tools/ncu_summary.py report $f > ${f%.ncu-rep}_ncu.txt 2>&1
  timeout 300 python tools/ncu_stalls.py $f 25 > ${f%.ncu-rep}_stalls.txt 2>&1
done
python tools/ncu_summary.py launches gpurun_out/launches_$TAG.csv > gpurun_out/launches_$TAG.txt 2>&1
for f in gpurun_out/prof_${TAG}_*.ncu-rep; do
  case $f in *k3t*) ;; *) rm -f $f ;; esac
done
du -sh gpurun_out
