python -m pytest tests/test_gpu_cvt_variants.py tests/test_gpu_parity.py -q -x -k "not c5" > gpurun_out/t6_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t6_gpu.log
L=paper_1708_09746_b200
python tools/dev/ab_bench.py c4b 10 $L/libgf2x_b200.so $L/libgf2x_b200.so@GF2X_RB_TMA=1 > gpurun_out/t6_ab.log 2>&1
python tools/dev/gpu_shard_timing.py 536870912 > gpurun_out/t6_shard.log 2>&1
python tools/dev/prof_run.py c1 3 > gpurun_out/t6_plain_c1.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_small -s 1 -c 1 -o gpurun_out/t6_small python tools/dev/prof_run.py c1 3 > gpurun_out/t6_ncu.log 2>&1
