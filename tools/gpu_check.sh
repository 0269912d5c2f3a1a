#!/bin/bash
mkdir -p gpurun_out
T=${1:-x}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_3d.py -q -x -k "row_tiles or 3d_layers or c1" > gpurun_out/${T}_tests.log 2>&1
export CKS_EXPERIMENTS=1
for dt in tf32 bf16; do
  for tc in 1 0 2; do
    echo "== $dt tc=$tc" >> gpurun_out/${T}_time.txt
    CKS_DTYPE=$dt CKS_WGRAD_TC=$tc python tools/time_op.py 2 wgrad l1_0 20 >> gpurun_out/${T}_time.txt 2>&1
    CKS_DTYPE=$dt CKS_WGRAD_TC=$tc timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:wgrad_kernel -c 1 python tools/prof_layer.py 2 l1_0 wgrad 1 2>&1 | grep -E "dram|duration" >> gpurun_out/${T}_time.txt
  done
done
