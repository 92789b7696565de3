#!/bin/bash
# round-2 session-3 validation on the current tree: full GPU suite, default bench, smoke, c4b launch list
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/t65_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t65_gpu.log
python bench.py --steps 20 --warmup 5 > gpurun_out/t65_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/t65_bench.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t65_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/t65_smoke.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/t65_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/t65_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/t65_ncu.log
