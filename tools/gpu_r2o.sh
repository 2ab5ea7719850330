#!/bin/bash
mkdir -p gpurun_out
T=${TAG:-r2o}
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/${T}_gpu.log 2>&1; echo "gpu rc=$?" >> gpurun_out/${T}_gpu.log; tail -2 gpurun_out/${T}_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2>gpurun_out/${T}_bench.err; tail -2 gpurun_out/${T}_bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
RFS_NVTX=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_nvtx.json 2>&1
timeout 900 python tools/bench_density.py --iterations 600 > gpurun_out/${T}_density.json 2> gpurun_out/${T}_density.err; tail -2 gpurun_out/${T}_density.err
echo done
