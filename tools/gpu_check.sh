#!/bin/bash
mkdir -p gpurun_out
T=${1:-x}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_3d.py tests/test_gpu_allreduce.py -q -x -k "row_tiles or c1 or 3d_layers or random or full_size or reduced_batch or allreduce" > gpurun_out/${T}_tests.log 2>&1
export CKS_EXPERIMENTS=1
for dt in tf32 bf16; do
  for pp in 1 0; do
    echo "== $dt pp=$pp" >> gpurun_out/${T}_time.txt
    CKS_DTYPE=$dt CKS_WGRAD_PP=$pp python tools/time_op.py 2 wgrad l1_0 20 >> gpurun_out/${T}_time.txt 2>&1
    CKS_DTYPE=$dt CKS_WGRAD_PP=$pp python tools/time_op.py 1 wgrad vgg32_64to64_s1 20 >> gpurun_out/${T}_time.txt 2>&1
  done
done
