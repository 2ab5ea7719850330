#!/bin/bash
# round 2: new bench-path parity tests + full gpu suite + bench
nproc > gpurun_out/r2a_nproc.txt
python -m pytest tests/test_gpu_bench_path.py tests/test_toggles.py -x -q -m gpu --durations=10 > gpurun_out/r2a_newtests.log 2>&1
echo "newtests rc=$?" >> gpurun_out/r2a_newtests.log
python -m pytest tests -x -q -m gpu --deselect tests/test_gpu_bench_path.py > gpurun_out/r2a_gpu.log 2>&1
echo "gpu rc=$?" >> gpurun_out/r2a_gpu.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
