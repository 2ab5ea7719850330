#!/bin/bash
# ncu --set full of kernels matching regex $2 (tag $1, count $3) on the bench step
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -c ${3:-4} \
    -o gpurun_out/$1_full python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/$1_ncu.log 2>&1
tail -3 gpurun_out/$1_ncu.log
