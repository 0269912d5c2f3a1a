#!/bin/bash
mkdir -p gpurun_out
T=${1:-x}
timeout 900 python -m pytest tests/test_gpu_ks_mp.py tests/test_gpu_parity.py -q -x -k "multiphase or config_layers or narrow" > gpurun_out/${T}_tests.log 2>&1
export CKS_EXPERIMENTS=1
for dt in bf16 tf32; do
  for mp in 1 0; do
    echo "== $dt mp=$mp" >> gpurun_out/${T}_time.txt
    CKS_DTYPE=$dt CKS_KS_MP=$mp python tools/time_op.py 3 deconv_w G32to64 10 >> gpurun_out/${T}_time.txt 2>&1
  done
done
