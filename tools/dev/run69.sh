#!/bin/bash
# A/B: k_fft2 TMA tile loads (GF2X_FFT_LD=1) and TMA stores in the changeRepr pass (GF2X_FFT_ST=2)
mkdir -p gpurun_out
for rep in 1 2; do
GF2X_FFT_LD=0 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 --no-companion > gpurun_out/t69_base_$rep.json 2> gpurun_out/t69_base_$rep.err
GF2X_FFT_LD=1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 --no-companion > gpurun_out/t69_ld_$rep.json 2> gpurun_out/t69_ld_$rep.err
GF2X_FFT_ST=2 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 --no-companion > gpurun_out/t69_psist_$rep.json 2> gpurun_out/t69_psist_$rep.err
done
GF2X_FFT_LD=1 GF2X_FFT_ST=2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_digests.py tests/test_gpu_sweep.py tests/test_gpu_r28.py tests/test_gpu_trunc.py tests/test_gpu_graph.py -m gpu -x -q > gpurun_out/t69_tests.log 2>&1; echo "rc=$?" >> gpurun_out/t69_tests.log
