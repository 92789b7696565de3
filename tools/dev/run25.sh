#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/dev/small_trace.py 65536 16 > gpurun_out/t25_trace16.log 2>&1
timeout 300 python tools/dev/small_trace.py 65536 4 > gpurun_out/t25_trace4.log 2>&1
