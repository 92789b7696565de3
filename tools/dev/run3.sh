L=paper_1708_09746_b200
python tools/dev/ab_bench.py c4b 10 $L/libgf2x_b200.so $L/libgf2x_b200.so@GF2X_CVT_SLAB=1 $L/libgf2x_b200_slab1.so@GF2X_CVT_SLAB=1 $L/libgf2x_b200.so@GF2X_CVT_SLAB=1,GF2X_SLAB_CLUSTER=4 $L/libgf2x_b200.so@GF2X_NO_CVT_TOP=1 > gpurun_out/t3_ab.log 2>&1
python tools/dev/ab_bench.py c2 10 $L/libgf2x_b200.so > gpurun_out/t3_ab_c2.log 2>&1
python tools/dev/ab_bench.py c1 20 $L/libgf2x_b200.so > gpurun_out/t3_ab_c1.log 2>&1
python tools/dev/ab_bench.py c3 20 $L/libgf2x_b200.so $L/libgf2x_b200_r1.so > gpurun_out/t3_ab_c3.log 2>&1
