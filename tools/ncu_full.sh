#!/bin/bash
# usage: tools/ncu_full.sh TAG CONFIG LAYER OP KERNEL_REGEX   (env passes through, e.g. CKS_DEBUG_FLAGS)
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:$5 -s 1 -c 1 -o gpurun_out/prof_$1 -f \
    python tools/prof_layer.py $2 $3 $4 3 > gpurun_out/prof_$1.log 2>&1 || true
