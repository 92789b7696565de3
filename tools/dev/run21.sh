#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_small_cluster.py -q -x > gpurun_out/t21_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t21_tests.log
for cl in 8 16; do
  GF2X_SMALL_CL=$cl timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 10 > gpurun_out/t21_c1_$cl.log 2>&1
  GF2X_SMALL_NO_SEGCVT=1 GF2X_SMALL_CL=$cl timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 10 > gpurun_out/t21_c1noseg_$cl.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_small -s 2 -c 1 -o gpurun_out/t21_small16 -f python tools/dev/prof_run.py c1 3 > gpurun_out/t21_ncu.log 2>&1
