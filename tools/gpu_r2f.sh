#!/bin/bash
python -m pytest tests -x -q -m gpu --durations=5 > gpurun_out/r2f_gpu.log 2>&1
echo "gpu rc=$?" >> gpurun_out/r2f_gpu.log
python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
