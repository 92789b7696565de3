#!/bin/bash
# A/B: L2 prefetch of the next tile (GF2X_L2PF bit 0: k_bottom, bit 1: k_ipsi_bs R28 path)
mkdir -p gpurun_out
for rep in 1 2; do
for pf in 0 1 2 3; do
GF2X_L2PF=$pf python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 --no-companion > gpurun_out/t68_pf${pf}_$rep.json 2> gpurun_out/t68_pf${pf}_$rep.err
done; done
GF2X_L2PF=3 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_digests.py tests/test_gpu_sweep.py tests/test_gpu_r28.py tests/test_gpu_trunc.py -m gpu -x -q > gpurun_out/t68_tests.log 2>&1; echo "rc=$?" >> gpurun_out/t68_tests.log
