#!/usr/bin/env bash
# Runs on the GPU box (via gpurun): bench line, launch list, ncu --set full of
# the top kernels.  Outputs land in gpurun_out/; tools/summarize_profiles.py
# turns them into the tracked summaries under profiles/.
set -u
TAG=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --sort cub > gpurun_out/${TAG}_bench_cub.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
# one steady-state step only (cudaProfilerStart/Stop in tools/ncu_step.py): ~30 kernels
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -o gpurun_out/${TAG}_full python tools/ncu_step.py > gpurun_out/${TAG}_ncu.log 2>&1
# config 5: one training iteration's launch list and the 400-iteration timing (captured iterations)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_c5_launches.csv python tools/bench_density.py --iterations 8 --eager > /dev/null 2>&1
python tools/launch_list.py gpurun_out/${TAG}_c5_launches.csv > gpurun_out/${TAG}_c5_launches.txt 2>&1
timeout 600 python tools/bench_density.py --iterations 600 > gpurun_out/${TAG}_density.json 2> gpurun_out/${TAG}_density.err
echo done
