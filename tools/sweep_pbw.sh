#!/bin/bash
export CKS_EXPERIMENTS=1  # environment knobs live only in the experiments build (libcks_exp.so)
# usage: tools/sweep_pbw.sh CONFIG OP -- every layer under forced pixel-block widths / BN (CKS_IGEMM_CFG="BN,PBW,Z")
echo "== default"; python tools/time_op.py $1 $2 all 20 2>&1 | awk '{print $1, $3}'
for cfg in "0,1,0" "0,2,0" "0,3,0" "0,4,0" "64,1,0" "64,2,0" "64,4,0"; do
  echo "== $cfg"; CKS_IGEMM_CFG=$cfg python tools/time_op.py $1 $2 all 20 2>&1 | awk '{print $1, $3}'
done
