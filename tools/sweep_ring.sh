#!/bin/bash
export CKS_EXPERIMENTS=1  # environment knobs live only in the experiments build (libcks_exp.so)
# usage: tools/sweep_ring.sh CONFIG OP LAYERS -- A-slot granularity / B-ring depth
# (CKS_IGEMM_CFG="BN,PBW,Z,APOS,BST"; 0 = plan default)
for cfg in "0,0,0" "0,0,0,1,2" "0,0,0,1,3" "0,0,0,2,2" "0,0,0,2,3"; do
  echo "== $cfg"; CKS_IGEMM_CFG=$cfg python tools/time_op.py $1 $2 $3 20 2>&1 | awk '{print $1, $3}'
done
