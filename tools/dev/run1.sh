set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python tools/dev/ab_bench.py c4b 10 paper_1708_09746_b200/libgf2x_b200_r1.so paper_1708_09746_b200/libgf2x_b200.so paper_1708_09746_b200/libgf2x_b200_s8.so > gpurun_out/t1_ab.log 2>&1
python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/t1_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t1_gpu.log
python bench.py --steps 20 --warmup 5 > gpurun_out/t1_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/t1_bench.log
