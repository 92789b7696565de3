#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_small_cluster.py tests/test_gpu_parity.py -q -x > gpurun_out/t19_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t19_tests.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_small -s 2 -c 1 -o gpurun_out/t19_small16 -f python tools/dev/prof_run.py c1 3 > gpurun_out/t19_ncu.log 2>&1
