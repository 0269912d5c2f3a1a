#!/bin/bash
mkdir -p gpurun_out
T=${1:-x}
timeout 1500 compute-sanitizer --tool synccheck --print-limit 50 python tools/sanitize_cases.py > gpurun_out/san_${T}_synccheck.log 2>&1
echo "synccheck rc=$?" > gpurun_out/san_${T}_summary.txt
bash tools/sweep_tf32.sh fwd > gpurun_out/${T}_sweep_fwd.txt 2>&1
bash tools/sweep_tf32.sh deconv_w > gpurun_out/${T}_sweep_deconv.txt 2>&1
