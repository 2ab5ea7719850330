#!/bin/bash
# sanitizers over the small end-to-end driver + bench with the restated roofline + launch list
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_step.py > gpurun_out/r2i_sanitize_$tool.txt 2>&1
  echo "exit=$?" >> gpurun_out/r2i_sanitize_$tool.txt
done
python bench.py --steps 20 --warmup 5 > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2i_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
