#!/bin/bash
# seam kernel: parity + A/B vs the residue-sweep kernel
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_digests.py tests/test_gpu_sweep.py tests/test_gpu_cvt_variants.py tests/test_gpu_cvt_split.py -m gpu -x -q > gpurun_out/t43_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t43_gpu.log
L=paper_1708_09746_b200/libgf2x_b200.so
for c in c4b c3; do
python tools/dev/ab_bench.py $c 10 $L $L@GF2X_NO_SEAM=1 > gpurun_out/t43_$c.txt 2>&1
done
