#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fft_low_experiment.py tests/test_gpu_graph.py -q -x > gpurun_out/t38_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t38_tests.log
timeout 300 python tools/dev/fft_low_time.py > gpurun_out/t38_time.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bottom|k_fft_low_shfl" -s 2 -c 2 -o gpurun_out/t38_fftlow -f python tools/dev/fft_low_time.py > gpurun_out/t38_ncu.log 2>&1
