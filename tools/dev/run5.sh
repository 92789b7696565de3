python -m pytest tests/test_gpu_parity.py tests/test_gpu_sweep.py tests/test_gpu_graph.py tests/test_gpu_w128.py -q -x > gpurun_out/t5_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t5_gpu.log
L=paper_1708_09746_b200
python tools/dev/ab_bench.py c1 20 $L/libgf2x_b200.so $L/libgf2x_b200.so@GF2X_NO_SMALL=1 > gpurun_out/t5_ab_c1.log 2>&1
python tools/dev/ab_bench.py c2 10 $L/libgf2x_b200.so $L/libgf2x_b200.so@GF2X_NO_SMALL=1 > gpurun_out/t5_ab_c2.log 2>&1
for c in c1 c2; do python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 10 > gpurun_out/t5_bench_$c.log 2>&1; done
python bench.py --config c1 --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 10 --graph > gpurun_out/t5_bench_c1g.log 2>&1
