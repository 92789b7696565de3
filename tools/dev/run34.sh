#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bottom|k_fft2" -s 0 -c 3 -o gpurun_out/t34_c2 -f python tools/dev/prof_run.py c2 3 > gpurun_out/t34_ncu.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/t34_c2_launches.csv python tools/dev/prof_run.py c2 2 > gpurun_out/t34_ncu2.log 2>&1
