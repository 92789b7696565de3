#!/bin/bash
# A/B: k_cvt_rb_tma thread stores (0) vs TMA stores (1: next load at iteration start, 2: after the first phase)
mkdir -p gpurun_out
for rep in 1 2; do
for st in 0 1 2; do
GF2X_RB_ST=$st python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 --no-companion > gpurun_out/t66_st${st}_$rep.json 2> gpurun_out/t66_st${st}_$rep.err
done; done
for st in 1 2; do
GF2X_RB_ST=$st timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_digests.py tests/test_gpu_sweep.py tests/test_gpu_r28.py -m gpu -x -q > gpurun_out/t66_tests_st$st.log 2>&1; echo "rc=$?" >> gpurun_out/t66_tests_st$st.log
done
