#!/bin/bash
# round-2 closing validation: full GPU suite, default bench, smoke
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/t56_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t56_gpu.log
python bench.py --steps 20 --warmup 5 > gpurun_out/t56_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/t56_bench.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t56_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/t56_smoke.log
