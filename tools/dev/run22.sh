#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_small_cluster.py tests/test_gpu_parity.py -q -x > gpurun_out/t22_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t22_tests.log
for cl in 4 8 16; do
  GF2X_SMALL_CL=$cl timeout 300 python bench.py --config c1 --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 10 > gpurun_out/t22_c1_$cl.log 2>&1
done
GF2X_SMALL_BATCH=1 timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 10 > gpurun_out/t22_c2small.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_small -s 2 -c 1 -o gpurun_out/t22_small16 -f python tools/dev/prof_run.py c1 3 > gpurun_out/t22_ncu.log 2>&1
