#!/bin/bash
mkdir -p gpurun_out
T=${1:-x}
timeout 600 python -m pytest tests/test_gpu_allreduce.py -q -x > gpurun_out/${T}_ar.log 2>&1
