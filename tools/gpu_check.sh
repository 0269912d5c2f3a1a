#!/bin/bash
mkdir -p gpurun_out
T=${1:-x}
timeout 900 python -m pytest tests/test_gpu_bench_step.py -q -x > gpurun_out/${T}_tests.log 2>&1
bash tools/profile_round.sh r02 ncu3
