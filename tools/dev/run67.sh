#!/bin/bash
# A/B: k_fft2 thread stores (GF2X_FFT_ST=0) vs TMA tensor stores (1); parity with 1
mkdir -p gpurun_out
for rep in 1 2; do
for st in 0 1; do
GF2X_FFT_ST=$st python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 --no-companion > gpurun_out/t67_st${st}_$rep.json 2> gpurun_out/t67_st${st}_$rep.err
done; done
GF2X_FFT_ST=1 python bench.py --config c4a --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 --no-companion > gpurun_out/t67_c4a_st1.json 2>&1
GF2X_FFT_ST=1 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_digests.py tests/test_gpu_sweep.py tests/test_gpu_r28.py tests/test_gpu_trunc.py tests/test_gpu_graph.py tests/test_gpu_w128.py -m gpu -x -q > gpurun_out/t67_tests.log 2>&1; echo "rc=$?" >> gpurun_out/t67_tests.log
