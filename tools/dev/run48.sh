#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fft2 -s 0 -c 1 -o gpurun_out/t48_psi -f python tools/dev/prof_run.py c4b 2 > gpurun_out/t48_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ipsi_bs -s 0 -c 1 -o gpurun_out/t48_mcomb -f python tools/dev/prof_run.py c4b 2 > gpurun_out/t48_ncu2.log 2>&1
