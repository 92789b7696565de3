python -m pytest tests/test_gpu_parity.py tests/test_gpu_sweep.py tests/test_gpu_graph.py -q -x > gpurun_out/t8_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t8_gpu.log
L=paper_1708_09746_b200
python tools/dev/ab_bench.py c1 30 $L/libgf2x_b200.so > gpurun_out/t8_ab_c1.log 2>&1
python bench.py --config c1 --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 20 > gpurun_out/t8_bench_c1.log 2>&1
