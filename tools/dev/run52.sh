#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_w128.py -m gpu -q > gpurun_out/t52_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t52_gpu.log
python bench.py --w 128 --steps 10 --warmup 3 --no-cpu-baseline --no-companion --e2e-steps 3 > gpurun_out/t52_w128.log 2>&1
GF2X_NO_MCOMB=1 python bench.py --w 128 --steps 10 --warmup 3 --no-cpu-baseline --no-companion --e2e-steps 3 > gpurun_out/t52_w128_old.log 2>&1
