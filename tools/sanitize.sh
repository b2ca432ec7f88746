#!/bin/bash
# GPU box: compute-sanitizer memcheck / racecheck / synccheck over
# tools/sanitize_case.py -> gpurun_out/sanitize_<tool>.log
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
    python tools/sanitize_case.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.log
done
