#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_digests.py -m gpu -x -q -k "c3 or c4 or stage or cvt" > gpurun_out/t44_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t44_gpu.log
L=paper_1708_09746_b200/libgf2x_b200.so
python tools/dev/ab_bench.py c4b 10 $L $L@GF2X_NO_SEAM=1 > gpurun_out/t44_c4b.txt 2>&1
