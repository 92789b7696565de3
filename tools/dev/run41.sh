#!/bin/bash
# k_bottom full capture with source correlation (c4b)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bottom -s 1 -c 1 -o gpurun_out/t41_bottom -f python tools/dev/prof_run.py c4b 2 > gpurun_out/t41_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fft2 -s 3 -c 1 -o gpurun_out/t41_fft -f python tools/dev/prof_run.py c4b 2 > gpurun_out/t41_ncu2.log 2>&1
