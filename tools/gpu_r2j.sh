#!/bin/bash
python -m pytest tests -x -q -m gpu > gpurun_out/r2j_gpu.log 2>&1
echo "gpu rc=$?" >> gpurun_out/r2j_gpu.log
python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/r2j_bench.json 2> gpurun_out/r2j_bench.err
python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --strong --gaussians 1000000 > gpurun_out/r2j_strong1m.json 2> gpurun_out/r2j_strong1m.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2j_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
