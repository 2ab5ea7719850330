#!/bin/bash
# tests + bench + launch list; then compute-sanitizer (memcheck/racecheck/synccheck) over the small driver
mkdir -p gpurun_out
T=${TAG:-r2n}
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/${T}_gpu.log 2>&1; echo "gpu rc=$?" >> gpurun_out/${T}_gpu.log; tail -3 gpurun_out/${T}_gpu.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/${T}_bench.json 2>gpurun_out/${T}_bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
if [ -n "${SANITIZE:-}" ]; then
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_step.py > gpurun_out/${T}_sanitize_$tool.txt 2>&1
  echo "exit=$?" >> gpurun_out/${T}_sanitize_$tool.txt
  tail -4 gpurun_out/${T}_sanitize_$tool.txt
done
fi
echo done
