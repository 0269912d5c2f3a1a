#!/bin/bash
mkdir -p gpurun_out
T=${1:-x}
export CKS_EXPERIMENTS=1
for op in fwd deconv_w; do
  for w in 1 0; do
    echo "== bf16 $op wide=$w" >> gpurun_out/${T}_time.txt
    CKS_DTYPE=bf16 CKS_BF16_WIDE=$w python tools/time_op.py 2 $op l1_0,l2_0,l2a,l3a 20 >> gpurun_out/${T}_time.txt 2>&1
    CKS_DTYPE=bf16 CKS_BF16_WIDE=$w python tools/time_op.py 1 $op all 20 >> gpurun_out/${T}_time.txt 2>&1
  done
done
