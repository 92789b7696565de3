python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/t9_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t9_gpu.log
python bench.py --steps 20 --warmup 5 > gpurun_out/t9_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/t9_bench.log
for c in c1 c2 c3 c5; do python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 10 > gpurun_out/t9_bench_$c.log 2>&1; done
python bench.py --config c4b --w 128 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 5 > gpurun_out/t9_bench_w128.log 2>&1
python bench.py --config c4b --alg frob --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/t9_bench_frob.log 2>&1
python bench.py --bits 268435520 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 5 > gpurun_out/t9_bench_trunc.log 2>&1
python tools/dev/prof_run.py c4b 2 > gpurun_out/t9_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 18 -c 18 --csv --log-file gpurun_out/t9_launches.csv python tools/dev/prof_run.py c4b 2 > gpurun_out/t9_ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -s 18 -c 18 -o gpurun_out/t9_full python tools/dev/prof_run.py c4b 2 > gpurun_out/t9_ncu2.log 2>&1
