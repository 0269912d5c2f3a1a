#!/bin/bash
mkdir -p gpurun_out
T=${1:-x}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "narrow" > gpurun_out/${T}_tests.log 2>&1
for dt in tf32 bf16; do
  echo "== $dt" >> gpurun_out/${T}_time.txt
  CKS_DTYPE=$dt python tools/time_op.py 2 wgrad stem 10 >> gpurun_out/${T}_time.txt 2>&1
  CKS_DTYPE=$dt timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:wgrad_row -c 1 python tools/prof_layer.py 2 stem wgrad 1 2>&1 | grep -E "dram|duration|hit" >> gpurun_out/${T}_time.txt
done
