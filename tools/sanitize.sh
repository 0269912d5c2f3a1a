#!/bin/bash
# compute-sanitizer over one call of every kernel family (tools/sanitize_cases.py)
mkdir -p gpurun_out
T=${1:-r02}
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py \
      > gpurun_out/san_${T}_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_${T}_summary.txt
done
