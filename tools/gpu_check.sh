#!/bin/bash
mkdir -p gpurun_out
T=${1:-x}
timeout 900 python -m pytest tests/test_gpu_3d.py -q -x > gpurun_out/${T}_3d.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/${T}_pytest.log 2>&1
