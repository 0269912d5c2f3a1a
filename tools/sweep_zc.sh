#!/bin/bash
export CKS_EXPERIMENTS=1  # environment knobs live only in the experiments build (libcks_exp.so)
# usage: tools/sweep_zc.sh CONFIG OP -- every layer: default plan, legacy split-K off/on,
# and forced cluster split-K configs (CKS_IGEMM_CFG="BN,PBW,Z", 0 = default)
echo "== default"; python tools/time_op.py $1 $2 all 20 2>&1 | awk '{print $1, $3}'
echo "== legacy"; CKS_IGEMM_ZC=0 python tools/time_op.py $1 $2 all 20 2>&1 | awk '{print $1, $3}'
for cfg in "0,0,1" "64,1,2" "64,1,4" "64,1,8" "128,1,2" "128,1,4" "128,1,8" "128,2,4" "64,2,4"; do
  echo "== $cfg"; CKS_IGEMM_CFG=$cfg python tools/time_op.py $1 $2 all 20 2>&1 | awk '{print $1, $3}'
done
