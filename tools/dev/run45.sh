#!/bin/bash
# R28 (combine before the 64-bit iBasisCvt): full GPU suite + A/B
mkdir -p gpurun_out
L=paper_1708_09746_b200/libgf2x_b200.so
python tools/dev/ab_bench.py c4b 10 $L $L@GF2X_NO_MCOMB=1 > gpurun_out/t45_c4b.txt 2>&1
python tools/dev/ab_bench.py c2 10 $L $L@GF2X_NO_MCOMB=1 > gpurun_out/t45_c2.txt 2>&1
python tools/dev/ab_bench.py c3 10 $L $L@GF2X_NO_MCOMB=1 > gpurun_out/t45_c3.txt 2>&1
python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/t45_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t45_gpu.log
