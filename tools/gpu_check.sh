#!/bin/bash
mkdir -p gpurun_out
T=${1:-x}
for tool in memcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py > gpurun_out/san_${T}_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_${T}_summary.txt
done
bash tools/profile_round.sh r02 ncu1
