#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/dev/small_ab.py > gpurun_out/t23_ab_c1.log 2>&1
timeout 600 python tools/dev/small_ab.py 16384 4096 > gpurun_out/t23_ab_c2.log 2>&1
timeout 600 python tools/dev/small_ab.py 40000 > gpurun_out/t23_ab_m11b.log 2>&1
