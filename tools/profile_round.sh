#!/bin/bash
# Round-end measurement on one B200 (gpurun): bench lines, the ncu launch list
# and DRAM traffic of one bench step, and ncu --set full captures of the top
# kernels.  usage: tools/profile_round.sh TAG [bench|lists|ncu1|ncu2|ncu3]
# (gpurun copies back <= 64 MiB of gpurun_out/: captures are split in two calls)
TAG=${1:-r02}
PART=${2:-bench}
mkdir -p gpurun_out
if [ "$PART" = bench ]; then
  timeout 900 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
  timeout 300 python bench.py --config 1 --steps 50 --no-cpu-baseline --layers > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
  timeout 300 python bench.py --config 3 --steps 50 --no-cpu-baseline --layers > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
  timeout 300 python bench.py --config 5 --steps 30 --no-cpu-baseline --no-e2e --layers > gpurun_out/bench_c6.json 2> gpurun_out/bench_c6.err
  timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
  CKS_BENCH_DIST=1 timeout 600 python -m torch.distributed.run --nproc-per-node 1 --master-addr 127.0.0.1 \
      --master-port 29533 bench.py --allreduce fused --steps 20 --no-cpu-baseline --no-zins --no-e2e --companion none \
      > gpurun_out/bench_c5_fused1.json 2> gpurun_out/bench_c5_fused1.err
elif [ "$PART" = lists ]; then
  # ncu lists the eager warm-up pass (one full step, same kernels and arguments)
  # node by node; the step graphs are profiled whole (--graph-profiling graph):
  # node-level replay of the bench's graphs stops at the first igemm node with
  # LaunchFailed, which ends the profiled process.
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
      python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-zins --companion none > gpurun_out/ncu_launch.log 2>&1
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/traffic_$TAG.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-zins \
      --companion none > gpurun_out/ncu_traffic.log 2>&1
  timeout 600 ncu --graph-profiling graph --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/graphs_$TAG.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-zins \
      --companion none > gpurun_out/ncu_graph.log 2>&1
elif [ "$PART" = ncu1 ]; then
  CKS_DTYPE=tf32 bash tools/ncu_full.sh ${TAG}_tf32_fwd_l1 2 l1_0 fwd igemm
  CKS_DTYPE=tf32 bash tools/ncu_full.sh ${TAG}_tf32_wgrad_l1 2 l1_0 wgrad wgrad_kernel
elif [ "$PART" = ncu2 ]; then
  CKS_DTYPE=tf32 bash tools/ncu_full.sh ${TAG}_tf32_fwdrow_stem 2 stem fwd fwd_row
  CKS_DTYPE=tf32 bash tools/ncu_full.sh ${TAG}_tf32_wgradrow_stem 2 stem wgrad wgrad_row
else
  bash tools/ncu_full.sh ${TAG}_bf16_fwd_l3 2 l3_0 fwd igemm
  CKS_DTYPE=tf32 bash tools/ncu_full.sh ${TAG}_tf32_deconv_l1 2 l1_0 deconv_w igemm
fi
