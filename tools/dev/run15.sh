python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/t15_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t15_gpu.log
python bench.py --steps 20 --warmup 5 > gpurun_out/t15_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/t15_bench.log
for c in c1 c2 c3; do python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 10 > gpurun_out/t15_bench_$c.log 2>&1; done
python bench.py --config c1 --graph --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 10 > gpurun_out/t15_bench_c1g.log 2>&1
python tools/dev/gpu_shard_timing.py 536870912 > gpurun_out/t15_shard.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t15_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/t15_smoke.log
