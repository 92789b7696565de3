#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_small_cluster.py tests/test_gpu_parity.py -q -x > gpurun_out/t32_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t32_tests.log
timeout 600 python tools/dev/small_ab.py > gpurun_out/t32_ab_c1.log 2>&1
timeout 600 python tools/dev/small_ab.py 16384 4096 > gpurun_out/t32_ab_c2.log 2>&1
timeout 300 python tools/dev/small_trace.py 65536 16 > gpurun_out/t32_trace16.log 2>&1
