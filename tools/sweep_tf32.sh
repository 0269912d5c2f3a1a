#!/bin/bash
export CKS_EXPERIMENTS=1  # environment knobs live only in the experiments build (libcks_exp.so)
# usage: tools/sweep_tf32.sh OP -- C3 3x3 layers in TF32 under forced igemm configs (BN,PBW,Z) x K-block bytes
OP=$1
export CKS_DTYPE=tf32
L=l1_0,l2a,l2_0,l3a,l3_0,l4a,l4_0
echo "== default"; python tools/time_op.py 2 $OP $L 20 2>&1 | awk '{print $1, $3}'
for kb in 128 64 32; do
  for cfg in "64,1,1" "64,2,1" "64,3,1" "64,4,1" "128,1,1" "128,2,1"; do
    echo "== $cfg kb=$kb"; CKS_IGEMM_KB=$kb CKS_IGEMM_CFG=$cfg python tools/time_op.py 2 $OP $L 20 2>&1 | awk '{print $1, $3}'
  done
done
