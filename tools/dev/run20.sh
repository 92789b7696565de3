#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_small_cluster.py -q -x > gpurun_out/t20_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t20_tests.log
for cl in 4 8 16; do
  GF2X_SMALL_CL=$cl timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 10 > gpurun_out/t20_c1_$cl.log 2>&1
  GF2X_SMALL_NO_KT=1 GF2X_SMALL_CL=$cl timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 10 > gpurun_out/t20_c1nokt_$cl.log 2>&1
done
GF2X_SMALL_BATCH=1 timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 10 > gpurun_out/t20_c2small.log 2>&1
GF2X_SMALL_BATCH=1 GF2X_SMALL_NO_KT=1 timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 10 > gpurun_out/t20_c2small_nokt.log 2>&1
