#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c3 or c4 or stage" > gpurun_out/t57_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t57_gpu.log
L=paper_1708_09746_b200/libgf2x_b200.so
python tools/dev/ab_bench.py c4b 10 $L paper_1708_09746_b200/libgf2x_b200_nob0.so > gpurun_out/t57_c4b.txt 2>&1
