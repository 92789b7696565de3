#!/bin/bash
# geometry re-check after the TMA tile I/O: bottom layers 5 vs 6, FFT column bits 5 vs 6, maxr; c4b and c4a
mkdir -p gpurun_out
run() { tag=$1; shift; env "$@" python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 > gpurun_out/t71_$tag.json 2> gpurun_out/t71_$tag.err; }
run base X=0
run bot5 GF2X_BOT_B=5
run fftc5 GF2X_FFT_C=5
run maxr6 GF2X_MAXR=6
run base2 X=0
