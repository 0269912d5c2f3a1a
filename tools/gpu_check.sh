#!/bin/bash
mkdir -p gpurun_out
T=${1:-x}
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/${T}_pytest.log 2>&1
timeout 900 python bench.py --layers > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
