#!/bin/bash
export CKS_EXPERIMENTS=1  # environment knobs live only in the experiments build (libcks_exp.so)
# usage: tools/sweep_z.sh CONFIG OP  -- time every layer of CONFIG with the default
# igemm tile choice and forced split-K Z = 1, 2, 4, 8 (CKS_IGEMM_CFG="BN,PBW,Z", 0 = default)
for cfg in "0,0,0" "0,0,1" "0,0,2" "0,0,4" "0,0,8" "64,1,4" "64,1,8"; do
  echo "== $cfg"; CKS_IGEMM_CFG=$cfg python tools/time_op.py $1 $2 all 20 2>&1 | awk '{print $1, $3}'
done
