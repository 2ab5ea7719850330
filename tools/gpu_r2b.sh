#!/bin/bash
# K6 parallel path: bitwise vs streaming, full gpu suite, bench + launch list
python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "k6_parallel or slow_path" > gpurun_out/r2b_k6.log 2>&1
echo "k6 rc=$?" >> gpurun_out/r2b_k6.log
python -m pytest tests -x -q -m gpu > gpurun_out/r2b_gpu.log 2>&1
echo "gpu rc=$?" >> gpurun_out/r2b_gpu.log
python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
