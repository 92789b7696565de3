#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_frob.py -q -x > gpurun_out/t37_frob.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t37_frob.log
timeout 600 python bench.py --alg frob --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/t37_frob_bench.log 2>&1
GF2X_BITCVT_NOREG=1 timeout 600 python bench.py --alg frob --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/t37_frob_bench_noreg.log 2>&1
