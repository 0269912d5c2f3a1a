#!/bin/bash
export CKS_EXPERIMENTS=1  # environment knobs live only in the experiments build (libcks_exp.so)
# usage: tools/sweep_cfg.sh OP  -- time every C2 layer under several igemm configs
OP=$1
for cfg in "128,2,1" "128,1,1" "64,2,1" "64,1,1" "64,4,1" "128,1,2" "64,1,2" "128,2,2" "64,2,2"; do
  echo "== $cfg"; CKS_IGEMM_CFG=$cfg python tools/time_op.py 1 $OP all 20 2>&1 | awk '{print $1, $3}'
done
