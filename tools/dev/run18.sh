#!/bin/bash
# k_small cluster shapes: parity, then c1 timing per shape
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_small_cluster.py tests/test_gpu_parity.py -q -x > gpurun_out/t18_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t18_tests.log
for cl in 4 8 16; do
  GF2X_SMALL_CL=$cl timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 10 > gpurun_out/t18_c1_$cl.log 2>&1
  GF2X_SMALL_CL=$cl timeout 300 python bench.py --config c1 --graph --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 10 > gpurun_out/t18_c1g_$cl.log 2>&1
done
