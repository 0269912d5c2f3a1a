#!/bin/bash
# Round-end measurement on one B200 (gpurun): bench lines, the ncu launch list
# and DRAM traffic of one bench step, and ncu --set full captures of the top
# kernels.  usage: tools/profile_round.sh TAG [bench|lists|ncu1|ncu2]
# (gpurun copies back <= 64 MiB of gpurun_out/: captures are split in two calls)
TAG=${1:-r01}
PART=${2:-bench}
mkdir -p gpurun_out
if [ "$PART" = bench ]; then
  timeout 300 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
  timeout 300 python bench.py --config 2 --steps 20 --no-cpu-baseline --layers > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
  timeout 300 python bench.py --config 3 --steps 50 --no-cpu-baseline --layers > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
  timeout 300 python bench.py --config 5 --steps 30 --no-cpu-baseline --no-e2e --layers > gpurun_out/bench_c6.json 2> gpurun_out/bench_c6.err
  timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
  timeout 300 python bench.py --dtype tf32 --steps 30 --no-cpu-baseline > gpurun_out/bench_c2_tf32.json 2> gpurun_out/bench_c2_tf32.err
elif [ "$PART" = lists ]; then
  # ncu lists the eager warm-up pass (one full step, same kernels and arguments);
  # its replay of the bench's CUDA graph then stops at the first igemm node with
  # LaunchFailed (profiler-only: the graph runs clean outside ncu and under
  # compute-sanitizer), which ends the profiled process.
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
      python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-zins > gpurun_out/ncu_launch.log 2>&1
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/traffic_$TAG.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-zins \
      > gpurun_out/ncu_traffic.log 2>&1
elif [ "$PART" = ncu1 ]; then
  bash tools/ncu_full.sh ${TAG}_fwd_vgg16 1 vgg16_128to128_s1 fwd igemm
  bash tools/ncu_full.sh ${TAG}_deconv_vgg8 1 vgg8_256to256_s1 deconv_only igemm
  bash tools/ncu_full.sh ${TAG}_wgrad_vgg16 1 vgg16_128to128_s1 wgrad wgrad_kernel
  bash tools/ncu_full.sh ${TAG}_zc_vgg4 1 vgg4_512to512_s2 fwd igemm
else
  bash tools/ncu_full.sh ${TAG}_fwd_l3 2 l3_0 fwd igemm
  bash tools/ncu_full.sh ${TAG}_wgrad_l1 2 l1_0 wgrad wgrad_kernel
  bash tools/ncu_full.sh ${TAG}_fwdrow_stem 2 stem fwd fwd_row
  bash tools/ncu_full.sh ${TAG}_wgradrow_stem 2 stem wgrad wgrad_row
  bash tools/ncu_full.sh ${TAG}_pair_l3 2 l3_1 fwd igemm
fi
