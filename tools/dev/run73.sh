#!/bin/bash
# round-2 session-4 closing measurement of HEAD: full GPU suite, smoke, bench lines, c4b launch list
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/t73_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t73_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t73_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/t73_smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/t73_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/t73_bench.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 18 -c 18 --csv --log-file gpurun_out/t73_c4b_launches.csv python tools/dev/prof_run.py c4b 2 > gpurun_out/t73_ncu1.log 2>&1
python bench.py --config c4a --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 5 > gpurun_out/t73_bench_c4a.log 2>&1
for c in c1 c2 c3; do python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 10 > gpurun_out/t73_bench_$c.log 2>&1; done
python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/t73_bench_c5.log 2>&1
python bench.py --config c4b --graph --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 --no-companion > gpurun_out/t73_bench_c4b_graph.log 2>&1
python bench.py --w 128 --steps 10 --warmup 3 --no-cpu-baseline --no-companion --e2e-steps 3 > gpurun_out/t73_bench_w128.log 2>&1
python bench.py --alg frob --steps 5 --warmup 3 --no-cpu-baseline --no-companion --e2e-steps 2 > gpurun_out/t73_bench_frob.log 2>&1
python bench.py --bits 268435520 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/t73_bench_trunc.log 2>&1
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/t73_bench_ref.log 2>&1
