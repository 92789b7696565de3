#!/bin/bash
mkdir -p gpurun_out
L=paper_1708_09746_b200/libgf2x_b200.so
GF2X_TOP_SEAM=1 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c3 or c4 or stage or sizes" > gpurun_out/t51_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t51_gpu.log
python tools/dev/ab_bench.py c4b 10 $L $L@GF2X_TOP_SEAM=1 > gpurun_out/t51_c4b.txt 2>&1
