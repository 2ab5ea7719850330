#!/bin/bash
# ncu --set full of the SSIM kernels (source-level), config-2-sized batch
mkdir -p gpurun_out
TAG=${TAG:-lossq}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ssim -s 2 -c 2 \
    -o gpurun_out/${TAG}_full python tools/prof_loss.py > gpurun_out/${TAG}_ncu.log 2>&1
python tools/prof_loss.py
