#!/bin/bash
# full ncu capture of one warm c4b multiply; the raw page is exported on the box (the .ncu-rep with sources exceeds
# gpurun's 64 MiB return limit), the report itself returns only if small enough
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none -s 18 -c 18 -o gpurun_out/t75_c4b_full -f python tools/dev/prof_run.py c4b 2 > gpurun_out/t75_ncu2.log 2>&1; echo "ncu rc=$?" >> gpurun_out/t75_ncu2.log
ncu -i gpurun_out/t75_c4b_full.ncu-rep --page raw --csv > gpurun_out/t75_c4b_full_raw.csv 2>> gpurun_out/t75_ncu2.log
ls -la gpurun_out/ >> gpurun_out/t75_ncu2.log
sz=$(stat -c %s gpurun_out/t75_c4b_full.ncu-rep)
if [ "$sz" -gt 50000000 ]; then rm gpurun_out/t75_c4b_full.ncu-rep; fi
