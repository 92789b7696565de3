#!/bin/bash
# round-2 final validation: GPU suite, benches, smoke, ncu evidence
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/t36_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t36_gpu.log
python bench.py --steps 20 --warmup 5 > gpurun_out/t36_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/t36_bench.log
for c in c1 c2 c3; do python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 10 > gpurun_out/t36_bench_$c.log 2>&1; done
python bench.py --config c1 --graph --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 10 > gpurun_out/t36_bench_c1g.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t36_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/t36_smoke.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 18 -c 18 --csv --log-file gpurun_out/t36_c4b_launches.csv python tools/dev/prof_run.py c4b 2 > gpurun_out/t36_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_small -s 2 -c 1 -o gpurun_out/t36_small16 -f python tools/dev/prof_run.py c1 3 > gpurun_out/t36_ncu3.log 2>&1
