#!/bin/bash
mkdir -p gpurun_out
T=${1:-x}
export CKS_EXPERIMENTS=1
for dt in tf32 bf16; do
  for h in 0 1; do
    echo "== $dt hwnc=$h" >> gpurun_out/${T}_time.txt
    if [ $h = 1 ]; then export CKS_HWNC_TEST=1; else unset CKS_HWNC_TEST; fi
    CKS_DTYPE=$dt python tools/time_op.py 2 fwd l1_0,l2a,l2_0,l3_0,l4_0 20 >> gpurun_out/${T}_time.txt 2>&1
  done
done
