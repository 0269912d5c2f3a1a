#!/bin/bash
mkdir -p gpurun_out
T=${1:-x}
export CKS_EXPERIMENTS=1
for op in fwd deconv_w; do
  for w in 1 0; do
    echo "== $op wide=$w" >> gpurun_out/${T}_time.txt
    CKS_DTYPE=tf32 CKS_TF32_WIDE=$w python tools/time_op.py 2 $op l1_0,l2_0,l2a,l3a,l4_0 20 >> gpurun_out/${T}_time.txt 2>&1
  done
done
