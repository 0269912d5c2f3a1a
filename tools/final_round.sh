#!/bin/bash
# End-of-round measurement on one B200 (gpurun): GPU tests, smoke, bench lines (C5 headline incl.
# e2e + cpu_baseline, C2 / C4 / C6 with per-layer tables, C5 at 32 images / GPU, the oracle arm).
mkdir -p gpurun_out
T=${1:-fin}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py --layers > gpurun_out/${T}_c5.json 2> gpurun_out/${T}_c5_layers.txt
timeout 300 python bench.py --config 1 --steps 50 --no-cpu-baseline --layers > gpurun_out/${T}_c2.json 2> gpurun_out/${T}_c2_layers.txt
timeout 300 python bench.py --config 3 --steps 50 --no-cpu-baseline --layers > gpurun_out/${T}_c4.json 2> gpurun_out/${T}_c4_layers.txt
timeout 300 python bench.py --config 5 --steps 30 --no-cpu-baseline --no-e2e --layers > gpurun_out/${T}_c6.json 2> gpurun_out/${T}_c6_layers.txt
timeout 300 python bench.py --batch 32 --steps 30 --no-cpu-baseline --no-e2e --no-zins --layers > gpurun_out/${T}_c5_n32.json 2> gpurun_out/${T}_c5_n32_layers.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err
