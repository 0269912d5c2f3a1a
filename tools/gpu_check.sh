mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/g1_pytest.log 2>&1
timeout 300 python bench.py --config 2 --steps 20 --no-cpu-baseline --layers > gpurun_out/g1_c3.json 2> gpurun_out/g1_c3.err
timeout 300 python bench.py --config 2 --dtype tf32 --steps 10 --no-cpu-baseline --layers > gpurun_out/g1_c3tf32.json 2> gpurun_out/g1_c3tf32.err
timeout 300 python bench.py --steps 50 --no-cpu-baseline > gpurun_out/g1_c2.json 2> gpurun_out/g1_c2.err
