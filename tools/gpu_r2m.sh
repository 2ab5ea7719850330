#!/bin/bash
mkdir -p gpurun_out
T=${TAG:-r2m}
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/${T}_gpu.log 2>&1; echo "gpu rc=$?" >> gpurun_out/${T}_gpu.log; tail -3 gpurun_out/${T}_gpu.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/${T}_bench.json 2>gpurun_out/${T}_bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
if [ -n "${NCU_K:-}" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K}" -c ${NCU_C:-1} -o gpurun_out/${T}_full python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
fi
echo done
