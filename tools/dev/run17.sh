#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_tc_experiment.py -q -x > gpurun_out/t17_tc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t17_tc.log
for o in 1 2 3 4; do echo "occ $o" >> gpurun_out/t17_tctime.log; GF2X_TC_OCC=$o timeout 300 python tools/dev/tc_time.py >> gpurun_out/t17_tctime.log 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ipsi -c 1 -o gpurun_out/t17_ipsi_tc -f python tools/dev/tc_time.py > gpurun_out/t17_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ipsi_bs -c 1 -o gpurun_out/t17_ipsi_bs -f python tools/dev/tc_time.py >> gpurun_out/t17_ncu.log 2>&1
