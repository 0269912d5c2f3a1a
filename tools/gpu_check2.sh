#!/bin/bash
mkdir -p gpurun_out
T=${1:-x}
export CKS_EXPERIMENTS=1
for zc in 2 0 2 0; do
  CKS_WGRAD_ZC=$zc timeout 600 python bench.py --steps 30 --no-cpu-baseline --no-zins --no-e2e >> gpurun_out/${T}_c5_zc$zc.json 2>/dev/null
  CKS_WGRAD_ZC=$zc timeout 600 python bench.py --config 1 --steps 50 --no-cpu-baseline --no-zins --no-e2e --companion none >> gpurun_out/${T}_c2_zc$zc.json 2>/dev/null
done
