#!/bin/bash
mkdir -p gpurun_out
T=${1:-x}
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/${T}_pytest.log 2>&1
for dt in tf32 bf16; do
  echo "== $dt" >> gpurun_out/${T}_time.txt
  CKS_DTYPE=$dt python tools/time_op.py 2 fwd stem,l1_0,l2_0 20 >> gpurun_out/${T}_time.txt 2>&1
done
timeout 900 python bench.py --layers > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
