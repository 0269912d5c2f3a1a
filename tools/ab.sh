#!/bin/bash
export CKS_EXPERIMENTS=1  # environment knobs live only in the experiments build (libcks_exp.so)
# usage: tools/ab.sh CONFIG OP LAYERS "ENV_A" "ENV_B" ... -- per-layer warm timing under env settings
cfg=$1; op=$2; lay=$3; shift 3
for e in "$@"; do
  echo "== $e"; env $e python tools/time_op.py $cfg $op $lay 20 2>&1 | awk '{print $1, $3}'
done
