#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_r28.py tests/test_gpu_parity.py tests/test_gpu_digests.py -m gpu -x -q > gpurun_out/t63_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t63_gpu.log
L=paper_1708_09746_b200/libgf2x_b200.so
python tools/dev/ab_bench.py c4b 10 $L paper_1708_09746_b200/libgf2x_b200_prev.so > gpurun_out/t63_c4b.txt 2>&1
