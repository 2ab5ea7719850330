#!/bin/bash
# round-2 re-entry: verify HEAD on the GPU (all -m gpu tests, bench, strong 1M, launch list, smoke)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2k_gpu.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/r2k_gpu.log 2>&1
echo "gpu rc=$?" >> gpurun_out/r2k_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2k_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r2k_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --strong --gaussians 1000000 > gpurun_out/r2k_strong1m.json 2> gpurun_out/r2k_strong1m.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2k_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
echo done
