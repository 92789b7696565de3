#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_trunc.py tests/test_gpu_r28.py tests/test_gpu_sweep.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/t64_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t64_gpu.log
python bench.py --bits 268435520 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/t64_trunc.log 2>&1
GF2X_NO_MCOMB=1 python bench.py --bits 268435520 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/t64_trunc_old.log 2>&1
