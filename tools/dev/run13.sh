python -m pytest tests/test_gpu_parity.py tests/test_gpu_sweep.py tests/test_gpu_trunc.py tests/test_gpu_graph.py -q -x -k "not c5" > gpurun_out/t13_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t13_gpu.log
L=paper_1708_09746_b200
python tools/dev/ab_bench.py c2 10 $L/libgf2x_b200.so > gpurun_out/t13_ab.log 2>&1
python tools/dev/ab_bench.py c3 20 $L/libgf2x_b200.so >> gpurun_out/t13_ab.log 2>&1
python tools/dev/ab_bench.py c4b 10 $L/libgf2x_b200.so >> gpurun_out/t13_ab.log 2>&1
