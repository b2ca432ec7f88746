#!/bin/bash
# Here (after `gpurun -- bash tools/profile_all.sh TAG`): copy the bench line
# and summarise the launch list and ncu captures into profiles/TAG_*.
TAG=${1:?tag}
cp gpurun_out/bench_$TAG.json profiles/${TAG}_bench.json
python tools/ncu_summary.py launches gpurun_out/launches_$TAG.csv > profiles/${TAG}_launches.txt
for k in k1s k1 k3 attn gemm_ffn1 gemm_resid layernorm; do
  [ -f gpurun_out/prof_${TAG}_$k.ncu-rep ] && \
    timeout 300 python tools/ncu_summary.py report gpurun_out/prof_${TAG}_$k.ncu-rep > profiles/${TAG}_${k}_ncu.txt
done
grep -h "dram__bytes\|gpu__time_duration" profiles/${TAG}_k1_ncu.txt profiles/${TAG}_k3_ncu.txt
