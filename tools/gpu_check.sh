#!/bin/bash
mkdir -p gpurun_out
T=${1:-x}
for v in eager g1 g2; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_probe_$v.csv \
     python tools/ncu_graph_probe.py $v > gpurun_out/${T}_probe_$v.log 2>&1
done
timeout 300 ncu --graph-profiling graph --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_probe_g2graph.csv \
     python tools/ncu_graph_probe.py g2 > gpurun_out/${T}_probe_g2graph.log 2>&1
timeout 900 python -m pytest tests/test_gpu_grid.py -q -x > gpurun_out/${T}_pytest.log 2>&1
