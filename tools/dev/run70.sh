#!/bin/bash
# c2 with the ψ-pass register prefetch for small tiles; c1/c3/c4a/c4b with the defaults of this tree; GPU tests
mkdir -p gpurun_out
for c in c2 c3 c1; do
python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 3 --no-companion > gpurun_out/t70_$c.json 2> gpurun_out/t70_$c.err
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sweep.py tests/test_gpu_digests.py -m gpu -x -q > gpurun_out/t70_tests.log 2>&1; echo "rc=$?" >> gpurun_out/t70_tests.log
