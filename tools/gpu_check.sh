#!/bin/bash
mkdir -p gpurun_out
T=${1:-x}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "pair_tiles or full_size" > gpurun_out/${T}_tests.log 2>&1
export CKS_EXPERIMENTS=1
for op in fwd deconv; do
  for pt in 1 0; do
    echo "== $op pair_tf32=$pt" >> gpurun_out/${T}_time.txt
    CKS_DTYPE=tf32 CKS_PAIR_TF32=$pt python tools/time_op.py 2 $op l3a,l3_0,l3ds,l4a,l4_0 20 >> gpurun_out/${T}_time.txt 2>&1
  done
done
