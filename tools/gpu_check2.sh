#!/bin/bash
mkdir -p gpurun_out
T=${1:-x}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "row_tiles or full_size or reduced_batch" > gpurun_out/${T}_tests.log 2>&1
export CKS_EXPERIMENTS=1
for dt in tf32 bf16; do
  for m in 1 0; do
    echo "== $dt mt128=$m" >> gpurun_out/${T}_time.txt
    CKS_DTYPE=$dt CKS_WGRAD_MT128=$m python tools/time_op.py 2 wgrad l2_0 20 >> gpurun_out/${T}_time.txt 2>&1
  done
done
