#!/bin/bash
python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "k6_parallel or slow_path or live_counts or forward_config1" > gpurun_out/r2e_k6.log 2>&1
echo "k6 rc=$?" >> gpurun_out/r2e_k6.log
python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2e_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_hits_cand|k_hits_walk" -c 4 \
    -o gpurun_out/r2e_full python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
