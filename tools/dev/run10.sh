timeout 900 python -m pytest tests/test_gpu_shard_procs.py tests/test_gpu_comm.py -q -x > gpurun_out/t10_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t10_gpu.log
python -m pytest tests/test_gpu_parity.py -q -x -k "not c5" > gpurun_out/t10_par.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t10_par.log
L=paper_1708_09746_b200
python tools/dev/ab_bench.py c4b 10 $L/libgf2x_b200.so > gpurun_out/t10_ab.log 2>&1
