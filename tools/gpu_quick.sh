#!/bin/bash
# quick loop: parity subset + bench + launch list, tag $1
T=${1:-q}
python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_path.py tests/test_gpu_dp.py -x -q -m gpu -k "forward or backward or bench_step_config2_vs_oracle and 64 or straddling or dp_step" > gpurun_out/${T}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${T}_tests.log
python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
