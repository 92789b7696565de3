#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fft_low_shfl -c 1 -o gpurun_out/t39_shfl -f python tools/dev/fft_low_time.py > gpurun_out/t39_ncu.log 2>&1
