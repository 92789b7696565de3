#!/bin/bash
# round-2 session-4: full ncu capture of one warm c4b multiply on HEAD (TMA tile loads/stores in k_fft2 / k_cvt_rb_tma)
mkdir -p gpurun_out
python tools/dev/prof_run.py c4b 2 > gpurun_out/t74_plain.log 2>&1; echo "plain rc=$?" >> gpurun_out/t74_plain.log
timeout 1500 ncu --set full --clock-control none --import-source on -s 18 -c 18 -o gpurun_out/t74_c4b_full -f python tools/dev/prof_run.py c4b 2 > gpurun_out/t74_ncu2.log 2>&1; echo "ncu rc=$?" >> gpurun_out/t74_ncu2.log
ls -la gpurun_out/ >> gpurun_out/t74_ncu2.log
