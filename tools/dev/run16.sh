#!/bin/bash
# tensor-core psi^-1 experiment: parity, timing, then one ncu capture if both ran clean
mkdir -p gpurun_out
python -c "from paper_1708_09746_b200 import build; build.build()" > gpurun_out/t16_build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_tc_experiment.py -q -x > gpurun_out/t16_tc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t16_tc.log
timeout 300 python tools/dev/tc_time.py > gpurun_out/t16_tctime.log 2>&1; rc=$?; echo "tctime rc=$rc" >> gpurun_out/t16_tctime.log
if [ $rc = 0 ] && grep -q "0 0 correct" gpurun_out/t16_tctime.log; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ipsi -c 2 -o gpurun_out/t16_ipsi -f \
    python tools/dev/tc_time.py > gpurun_out/t16_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/t16_ncu.log
fi
