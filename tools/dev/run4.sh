python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/t4_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t4_gpu.log
python bench.py --steps 20 --warmup 5 > gpurun_out/t4_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/t4_bench.log
python tools/dev/prof_run.py c4b 2 > gpurun_out/t4_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 14 -c 14 --csv --log-file gpurun_out/t4_launches.csv python tools/dev/prof_run.py c4b 2 > gpurun_out/t4_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -s 14 -c 14 -o gpurun_out/t4_full python tools/dev/prof_run.py c4b 2 > gpurun_out/t4_ncu2.log 2>&1
