#!/bin/bash
# A/B: bottom layer count 5 vs 6
mkdir -p gpurun_out
L=paper_1708_09746_b200/libgf2x_b200.so
for c in c4b c3 c2; do
python tools/dev/ab_bench.py $c 10 $L $L@GF2X_BOT_B=5 > gpurun_out/t42_$c.txt 2>&1
done
