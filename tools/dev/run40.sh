#!/bin/bash
# session-start check: quick parity + c4b bench with per-kernel breakdown
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_digests.py -m gpu -x -q > gpurun_out/t40_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t40_gpu.log
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/t40_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/t40_bench.log
