#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r2l_gpu.log 2>&1; echo "gpu rc=$?" >> gpurun_out/r2l_gpu.log; tail -3 gpurun_out/r2l_gpu.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r2l_bench.json 2>gpurun_out/r2l_bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2l_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bwd_gauss_v|k_onesweep|k_used_keys|k_rank" -c 12 -o gpurun_out/r2l_full python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
echo done
