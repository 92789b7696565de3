python -m pytest tests/test_gpu_frob.py -q -x > gpurun_out/t14_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t14_gpu.log
python bench.py --config c4b --alg frob --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/t14_frob.log 2>&1
